# cfg4: the full allreduce message-size sweep (1 MiB .. 2 GiB per rank x eb 1e-2/1e-3/1e-4) at N = $1,
# plus the N-GPU bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${1:-4}
T=r2s2
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus $N --sweep --sweep-max-mib 2048 > gpurun_out/${T}_sweep_n$N.jsonl 2> gpurun_out/${T}_sweep_n$N.err; echo "sweep rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29642 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/${T}_bench_n$N.json 2> gpurun_out/${T}_bench_n$N.err; echo "bench rc=$?"
python - <<PY
import json
for l in open("gpurun_out/${T}_sweep_n$N.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l); c = d["config"]; e = d["detail"]
    print(c["bytes_per_rank"] >> 20, c["eb"], d["value"], e.get("nccl_allreduce_gbs"), e.get("ratio_vs_nccl"), e.get("compression_ratio"), d["ms_per_step"])
d = json.loads(open("gpurun_out/${T}_bench_n$N.json").read().strip().splitlines()[-1])
print("bench", d["value"], d["detail"], d["e2e"]["value"], d["roofline"]["frac"], d["parity"])
PY
