# round 2: 4-GPU run: comm tests (2..4 ranks), bench N=1/2/4 + reference arms, peer-step ncu with NVLink counters, calibration at N=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --query-metrics 2>/dev/null | grep -i "nvl" | head -20 > gpurun_out/r2j_nvl_metrics.txt
timeout 2400 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2j_comm.txt 2>&1; echo "comm pytest rc=$?"; tail -3 gpurun_out/r2j_comm.txt; grep -h "mgpu ranks\|failures:" gpurun_out/r2j_comm.txt | head
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2j_bench_n1.json 2>gpurun_out/r2j_bench_n1.err; echo "n1 rc=$?"; tail -c 900 gpurun_out/r2j_bench_n1.json
for N in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2j_bench_n$N.json 2>gpurun_out/r2j_bench_n$N.err; echo "n$N rc=$?"; tail -1 gpurun_out/r2j_bench_n$N.json | cut -c1-1500
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/r2j_ref_n$N.json 2>gpurun_out/r2j_ref_n$N.err; echo "ref n$N rc=$?"; tail -1 gpurun_out/r2j_ref_n$N.json | cut -c1-300
done
python tools/prof_peer_step.py 33554432 5
M=$(grep -io "nvl[a-z_]*__bytes[a-z_.]*" gpurun_out/r2j_nvl_metrics.txt | sort -u | tr '\n' ',' | sed 's/,$//')
echo "nvl metrics: $M"
timeout 900 ncu --set full --import-source on --clock-control none ${M:+--metrics $M} -k regex:k_tile_encode -s 1 -c 1 -o gpurun_out/r2j_peer_step python tools/prof_peer_step.py 33554432 2 > gpurun_out/r2j_peer_ncu.log 2>&1; echo "peer ncu rc=$?"; tail -3 gpurun_out/r2j_peer_ncu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29576 tools/calibrate_costmodel.py gpurun_out/b200_cost_params.json > gpurun_out/r2j_calib.log 2>&1; echo "calib rc=$?"; grep -A3 '"checks"' gpurun_out/r2j_calib.log | head; grep ratio gpurun_out/r2j_calib.log
