# slotted allgather: comm tests + bench N=2 (+ ag_mode A/B)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2n_comm.txt 2>&1; echo "comm pytest rc=$?"; tail -2 gpurun_out/r2n_comm.txt; grep -h "mgpu ranks\|failures:" gpurun_out/r2n_comm.txt | sort | uniq | head
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2n_bench_n2.json 2>gpurun_out/r2n_bench_n2.err; echo "n2 rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/r2n_bench_n2.json').read().strip().splitlines()[-1]); print(d['value'], d['detail'], d['e2e']['value'], d['parity'], d['roofline']['avg_step_us'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29583 bench.py --gpus 2 --sweep --sweep-max-mib 512 > gpurun_out/r2n_sweep_n2.jsonl 2>gpurun_out/r2n_sweep_n2.err; echo "sweep rc=$?"; python -c "
import json
for l in open('gpurun_out/r2n_sweep_n2.jsonl'):
    if not l.startswith('{'): continue
    d=json.loads(l); c=d['config']; e=d['detail']
    print(c['bytes_per_rank']>>20, c['eb'], d['value'], e['nccl_allreduce_gbs'], e['ratio_vs_nccl'], d['ms_per_step'])"
