# index (idx_emit) change: GPU tests, N=1 bench, launch list of the bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/i_bench_n1.json 2>gpurun_out/i_bench_n1.err; echo "n1 rc=$?"; tail -1 gpurun_out/i_bench_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i_launches_n1.csv python bench.py --steps 5 --warmup 3 > gpurun_out/i_ncu.log 2>&1; echo "ncu rc=$?"
