# end-of-session validation: full GPU suite (2 GPUs), bench N=1 and N=2, decoder ncu with the TMA store
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r2s2f
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/${T}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; echo "n1 rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/${T}_bench_n2.json 2> gpurun_out/${T}_bench_n2.err; echo "n2 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 1 -c 1 -o gpurun_out/${T}_dec -f python tools/prof_codec.py 16777216 both > gpurun_out/${T}_ncu_dec.log 2>&1; echo "dec ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_n1.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1; echo "launch list rc=$?"
python - <<PY
import json
for f in ["gpurun_out/${T}_bench_n1.json", "gpurun_out/${T}_bench_n2.json"]:
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], {k: v for k, v in d["detail"].items() if not isinstance(v, (dict, list))})
PY
