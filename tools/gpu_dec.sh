# codec change check: codec gpu tests, then old vs new library (small sizes graph-timed, large bench_all)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -m gpu -x -q 2>&1 | tail -2
for lib in build_cmp/old.so paper_2308_05199_b200/libgzccl.so; do
  echo "== $lib"
  GZ_LIB=$PWD/$lib timeout 300 python tools/exp/small.py 12 16 18 20 22
  GZ_LIB=$PWD/$lib timeout 300 python tools/bench_all.py 24 27
done
