# N=8 rehearsal on a 4-GPU box: 8 ranks, two per GPU (gloo object plumbing, CUDA-IPC data
# path), every multi-GPU parity check of tests/mgpu_worker.py incl. the reference's N=8
# golden cases; then N=5..7 the same way
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for N in ${REHEARSE_NS:-8 6 5}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2971$N tests/mgpu_worker.py > gpurun_out/n${N}_rehearsal.log 2>&1
  echo "N=$N rc=$?"; grep -E "mgpu ranks|failures:" gpurun_out/n${N}_rehearsal.log | head -5
done
# the bench's N>1 path at N=8 (timings meaningless with two ranks per GPU)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29788 bench.py --gpus 8 --steps 2 --warmup 3 > gpurun_out/n8_bench.json 2>gpurun_out/n8_bench.err
echo "bench N=8 rc=$?"; tail -1 gpurun_out/n8_bench.json; tail -3 gpurun_out/n8_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29789 bench.py --impl reference --gpus 8 --steps 1 --warmup 0 2>/dev/null | tail -1
