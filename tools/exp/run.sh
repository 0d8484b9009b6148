cd $GRAFT_REPO_ROOT
cp paper_2308_05199_b200/libgzccl.so /tmp/orig.so
for v in NOLOOKBACK NOSLOW BOTH; do
  cp tools/exp/libgzccl_$v.so paper_2308_05199_b200/libgzccl.so
  echo "== $v"; timeout 120 python tools/bench_codec.py 16777216 1e-4 compress 2>&1 | grep compress | head -1
done
cp /tmp/orig.so paper_2308_05199_b200/libgzccl.so
echo "== base"; timeout 120 python tools/bench_codec.py 16777216 1e-4 compress 2>&1 | grep compress | head -1
