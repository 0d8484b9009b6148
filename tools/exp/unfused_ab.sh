# allreduce last step fused vs decode-reduce + compress (GZ_UNFUSED_LAST), bench.py N=$N
cd $GRAFT_REPO_ROOT
N=${N:-2}
for r in 1 2; do for u in 0 1; do
  GZ_UNFUSED_LAST=$u timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29730 + r)) bench.py --gpus $N --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('unfused=$u', d['value'], 'step_us', d['roofline']['avg_step_us'], 'parity', d['parity'])"
done; done
