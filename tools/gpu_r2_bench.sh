# bench lines at N = 1 and N = $1 (default 2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${1:-2}
TAG=${2:-r2b}
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_n1.json 2> gpurun_out/${TAG}_bench_n1.err; echo "n1 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err; echo "n$N rc=$?"
python - <<PY
import json
for f in ["gpurun_out/${TAG}_bench_n1.json", "gpurun_out/${TAG}_bench_n$N.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["unit"], "e2e", d["e2e"]["value"], "roofline", d["roofline"].get("frac"), d["roofline"].get("achieved"), "parity", d.get("parity"))
    print("  detail", {k: v for k, v in d.get("detail", {}).items() if not isinstance(v, (dict, list))})
PY
