# final refresh: all gpu tests (4 GPUs), smoke, bench N=1/2/4, N=1 ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/f_bench_n1.json 2>gpurun_out/f_bench_n1.err; echo "n1 rc=$?"; cat gpurun_out/f_bench_n1.json
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/f_bench_n$N.json 2>gpurun_out/f_bench_n$N.err; echo "n$N rc=$?"; tail -1 gpurun_out/f_bench_n$N.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref_n1.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/f_ref_n1.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_n1.csv python bench.py --steps 5 --warmup 3 > gpurun_out/f_ncu.log 2>&1; echo "ncu rc=$?"
