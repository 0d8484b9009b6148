# comm tests on 4 GPUs + ncu of the small (2^16) step / gather kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_comm_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 30 -c 1 -o gpurun_out/small_step -f python tools/exp/small.py 16 > gpurun_out/ncu_small1.log 2>&1; echo "ncu1 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_gather -s 30 -c 1 -o gpurun_out/small_gather -f python tools/exp/small.py 16 > gpurun_out/ncu_small2.log 2>&1; echo "ncu2 rc=$?"
