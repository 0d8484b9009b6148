cd $GRAFT_REPO_ROOT
cp paper_2308_05199_b200/libgzccl.so /tmp/orig.so
cp tools/exp/libgzccl_NOLOOKBACK.so paper_2308_05199_b200/libgzccl.so
echo "== NOLOOKBACK"; timeout 120 python tools/bench_codec.py 16777216 1e-4 compress 2>&1 | grep compress | head -1
timeout 120 python tools/bench_codec.py 134217728 1e-4 compress 2>&1 | grep compress | head -1
python tools/prof_codec.py > gpurun_out/plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_nolb python tools/prof_codec.py > gpurun_out/ncu_nolb.log 2>&1
cp /tmp/orig.so paper_2308_05199_b200/libgzccl.so
