# round 2, first GPU check (1 GPU): all gpu tests, smoke, bench N=1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/r2a_pytest.txt 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2a_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench_n1.json 2>gpurun_out/r2a_bench_n1.err; echo "bench rc=$?"; cat gpurun_out/r2a_bench_n1.json; tail -5 gpurun_out/r2a_bench_n1.err
