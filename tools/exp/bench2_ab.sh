# bench.py N=2 alternating between builds: tools/exp/bench2_ab.sh a.so b.so ... (REPS=2)
cd $GRAFT_REPO_ROOT
for r in $(seq 1 ${REPS:-2}); do for so in "$@"; do
  cp $so paper_2308_05199_b200/libgzccl.so
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700 + r)) bench.py --gpus 2 --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$so', d['value'], 'step_us', d['roofline']['avg_step_us'], 'e2e', d['e2e']['value'], 'parity', d['parity'])"
done; done
