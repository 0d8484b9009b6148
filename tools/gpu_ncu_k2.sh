cd $GRAFT_REPO_ROOT
python tools/prof_codec.py 134217728 compress || exit 1
ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_gather -s 2 -c 1 -o gpurun_out/prof_k2big -f python tools/prof_codec.py 134217728 compress > gpurun_out/ncu_k2big.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --cache-control none -k regex:"k_gather|k_tile_encode" python tools/prof_codec.py 134217728 compress 2>&1 | grep -E "k_gather|k_tile|duration|bytes|hit" | tail -10
