# round 2: comparators + errors on 2 GPUs, cost-model calibration, decode A/B vs round 1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2g_comm.txt 2>&1; echo "comm pytest rc=$?"; tail -3 gpurun_out/r2g_comm.txt; grep -h "mgpu ranks\|failures:" gpurun_out/r2g_comm.txt | head
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/calibrate_costmodel.py gpurun_out/b200_cost_params.json > gpurun_out/r2g_calib.log 2>&1; echo "calib rc=$?"; grep -v Warning gpurun_out/r2g_calib.log | tail -45
python tools/exp/ab_codec.py paper_2308_05199_b200/libgzccl.so tools/exp/_old/libgzccl_r1.so
