# decoder change check: codec gpu tests, then old vs new library on smooth and noise data
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -m gpu -x -q 2>&1 | tail -2
for lib in build_cmp/old.so paper_2308_05199_b200/libgzccl.so; do
  echo "== $lib"
  GZ_LIB=$PWD/$lib timeout 300 python tools/bench_all.py 24 27
  GZ_LIB=$PWD/$lib GZ_DATA=noise GZ_EB=1e-7 timeout 300 python tools/bench_all.py 24
  GZ_LIB=$PWD/$lib GZ_DATA=noise GZ_EB=2e-6 timeout 300 python tools/bench_all.py 24
done
