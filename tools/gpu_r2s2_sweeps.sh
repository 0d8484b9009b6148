# cfg4 sweeps at N = 2 and (on a 4-GPU box) N = 4 with the final build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for N in 2 4; do
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29750 + N)) bench.py --gpus $N --sweep --sweep-max-mib 2048 > gpurun_out/r2s2_sweep_n$N.jsonl 2> gpurun_out/r2s2_sweep_n$N.err; echo "sweep N=$N rc=$?"
done
