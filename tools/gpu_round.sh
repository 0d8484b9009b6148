# full round-end style run: gpu tests, bench N=1 (ours + reference), ncu launch list + full capture
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_n1.json 2>&1; echo "ref rc=$?"; cat gpurun_out/bench_ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 3 -c 1 -o gpurun_out/prof_bench_enc -f python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gather -s 3 -c 1 -o gpurun_out/prof_bench_gather -f python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 3 -c 1 -o gpurun_out/prof_bench_dec -f python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_full3.log 2>&1; echo "ncu full3 rc=$?"
