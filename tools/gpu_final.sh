# round-end validation: all GPU tests on 4 GPUs, bench lines at N=1 (ours + reference) and N=2,3,4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_n1.json 2>/dev/null; tail -1 gpurun_out/final_n1.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1
for N in 2 3 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 10 --warmup 3 2>/dev/null | tail -1
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --impl reference --gpus $N --steps 1 --warmup 0 2>/dev/null | tail -1
done
