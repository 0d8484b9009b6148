# round 2: 2-GPU comm tests, cost-model calibration, compute-sanitizer runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2f_comm.txt 2>&1; echo "comm pytest rc=$?"; tail -3 gpurun_out/r2f_comm.txt; grep -h "mgpu ranks" gpurun_out/r2f_comm.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/calibrate_costmodel.py gpurun_out/b200_cost_params.json > gpurun_out/r2f_calib.log 2>&1; echo "calib rc=$?"; tail -40 gpurun_out/r2f_calib.log
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_codec.py > gpurun_out/r2f_sanitize_$T.log 2>&1; echo "$T rc=$?"; tail -4 gpurun_out/r2f_sanitize_$T.log
done
