cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/bench_codec.py 16777216 1e-4 compress 2>&1 | tail -1
timeout 300 python tools/bench_codec.py 134217728 1e-4 compress 2>&1 | tail -1
for n in 16777216 134217728; do
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"k_tile_encode|k_gather" -c 2 python tools/prof_codec.py $n compress 2>&1 | grep -E "k_tile|k_gather|duration|inst_exec|warps_active" | tail -8
done
