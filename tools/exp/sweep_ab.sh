# small-message sweep (N=$N, up to $MAX MiB) alternating between builds
cd $GRAFT_REPO_ROOT
N=${N:-2}; MAX=${MAX:-16}
for so in "$@"; do
  cp $so paper_2308_05199_b200/libgzccl.so
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29790 bench.py --gpus $N --sweep --sweep-max-mib $MAX 2>/dev/null | python -c "
import json,sys
out=[]
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); c=d['config']
    if c['eb']==1e-4: out.append('%d:%.1fus' % (c['bytes_per_rank']>>20, d['ms_per_step']*1e3))
print('$so', ' '.join(out))"
done
