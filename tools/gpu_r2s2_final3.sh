# end-of-session validation on 4 GPUs: full GPU suite, bench N=1/2/4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r2s2z
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${T}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; echo "n1 rc=$?"
for N in 2 4; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29680 + N)) bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/${T}_bench_n$N.json 2> gpurun_out/${T}_bench_n$N.err; echo "n$N rc=$?"
done
python - <<PY
import json
for N in (1, 2, 4):
    f = "gpurun_out/${T}_bench_n%d.json" % N
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], {k: v for k, v in d["detail"].items() if not isinstance(v, (dict, list))}, d["parity"])
PY
