# round 2: ncu of the fused reduce-scatter step reading a PEER GPU's slots (2 GPUs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_peer_step.py 33554432 3 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 1 -c 1 -o gpurun_out/r2_step_peer -f python tools/prof_peer_step.py 33554432 2 > gpurun_out/r2_ncu_step_peer.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,lts__t_bytes.sum --clock-control none -k regex:k_tile_encode -c 4 --csv python tools/prof_peer_step.py 33554432 3 > gpurun_out/r2_step_peer_nvl.csv 2>&1
tail -n 3 gpurun_out/r2_ncu_step_peer.log
