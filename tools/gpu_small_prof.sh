# small-message allreduce: stamps timeline at N=2 and the size sweep vs NCCL
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-sp}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/prof_ring_stamps.py 1 4 16 64 > gpurun_out/${TAG}_stamps.txt 2>&1; echo stamps rc=$?
grep "MiB rank" gpurun_out/${TAG}_stamps.txt
GZ_NO_STAMPS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/prof_ring_stamps.py 1 4 16 64 > gpurun_out/${TAG}_nostamps.txt 2>&1
grep "MiB rank" gpurun_out/${TAG}_nostamps.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --sweep --sweep-max-mib 256 > gpurun_out/${TAG}_sweep_n2.jsonl 2>gpurun_out/${TAG}_sweep_n2.err; echo "sweep rc=$?"; python -c "
import json
for l in open('gpurun_out/${TAG}_sweep_n2.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); c=d['config']; e=d['detail']
    print(c['bytes_per_rank']>>20, c['eb'], d['value'], e['nccl_allreduce_gbs'], e['ratio_vs_nccl'], d['ms_per_step'])"
