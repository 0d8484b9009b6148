# bench.py N=$N alternating between builds (REPS=2, N=4)
cd $GRAFT_REPO_ROOT
N=${N:-4}
for r in $(seq 1 ${REPS:-2}); do for so in "$@"; do
  cp $so paper_2308_05199_b200/libgzccl.so
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29720 + r)) bench.py --gpus $N --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$so', d['value'], 'step_us', d['roofline']['avg_step_us'], 'parity', d['parity'])"
done; done
