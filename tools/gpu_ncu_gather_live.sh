# k_gather with warm caches, application replay (no memory save/restore between passes):
# is the encoder's scratch still in L2 when the gather reads it?
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,lts__t_sector_hit_rate.pct,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct -k regex:"k_gather|k_tile_encode" -s 4 -c 2 python tools/prof_codec.py 16777216 compress > gpurun_out/gl_ncu.txt 2>&1
grep -E "k_gather|k_tile_encode|duration|hit_rate|dram__bytes|passes" gpurun_out/gl_ncu.txt | head -40
