# the allgather's peer decode (slots over NVLink) with TMA bulk staging: timing + ncu counters
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_peer_decode.py 67108864 5 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:k_tile_decode -c 4 --csv python tools/prof_peer_decode.py 67108864 2 > gpurun_out/r2s2_agdec_nvl.csv 2>&1; echo "ncu rc=$?"
grep -E "gpu__time_duration|nvlrx|dram__bytes_read|issue_active" gpurun_out/r2s2_agdec_nvl.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head -16
