# cfg4 sweep at N=2 (1 MiB .. 2 GiB x 3 eb) and the reference arm at N=1 and N=2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r2s2
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 --sweep --sweep-max-mib 2048 > gpurun_out/${T}_sweep_n2.jsonl 2> gpurun_out/${T}_sweep_n2.err; echo "sweep rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref_n1.json 2> gpurun_out/${T}_ref_n1.err; echo "ref n1 rc=$?"; tail -1 gpurun_out/${T}_ref_n1.json | cut -c1-400
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/${T}_ref_n2.json 2> gpurun_out/${T}_ref_n2.err; echo "ref n2 rc=$?"; tail -1 gpurun_out/${T}_ref_n2.json | cut -c1-400
python - <<PY
import json
for l in open("gpurun_out/${T}_sweep_n2.jsonl"):
    if not l.startswith("{"): continue
    d = json.loads(l); c = d["config"]; e = d["detail"]
    print(c["bytes_per_rank"] >> 20, c["eb"], d["value"], e.get("nccl_allreduce_gbs"), e.get("ratio_vs_nccl"), e.get("compression_ratio"), d["ms_per_step"])
PY
