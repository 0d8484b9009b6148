# round 2: fixes check: rd NaN at 3 ranks (oversubscribed), comm tests N=2, peer step NVLink counters
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29591 tools/exp/rd_nan_debug.py 2>&1 | grep "rank [0-9]" | head
timeout 1500 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2l_comm.txt 2>&1; echo "comm pytest rc=$?"; tail -2 gpurun_out/r2l_comm.txt; grep -h "mgpu ranks\|failures:" gpurun_out/r2l_comm.txt | sort | uniq | head
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,lts__t_bytes.sum --clock-control none -k regex:k_tile_encode -c 4 --csv python tools/prof_peer_step.py 33554432 3 > gpurun_out/r2l_peer_nvl.csv 2>&1; echo "peer nvl rc=$?"; grep -E "k_tile_encode|==ERR" gpurun_out/r2l_peer_nvl.csv | cut -c1-300 | head -30
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 1 -c 1 -o gpurun_out/r2l_peer_step python tools/prof_peer_step.py 33554432 2 > gpurun_out/r2l_peer_full.log 2>&1; echo "peer full rc=$?"; tail -2 gpurun_out/r2l_peer_full.log
