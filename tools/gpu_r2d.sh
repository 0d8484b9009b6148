# round 2: single-kernel compressor check: codec/collective GPU tests, smoke, bench N=1, ncu launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py tests/test_bench_sizes_gpu.py tests/test_transport_gpu.py -q -x -p no:cacheprovider > gpurun_out/r2d_pytest.txt 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2d_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench_n1.json 2>gpurun_out/r2d_bench_n1.err; echo "n1 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r2d_bench_n1.json')); print(d['value'], d['detail']['compress_us'], d['detail']['decompress_us'], d['roofline']['frac'], d['detail']['codec_2p27'], d['e2e']['value'])"; tail -3 gpurun_out/r2d_bench_n1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r2d_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r2d_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open('gpurun_out/r2d_launches.csv')))
hdr = None; agg = collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            agg[d['Kernel Name'][:60]].append(float(d['Metric Value'].replace(',', '')))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):3d} mean={sum(v)/len(v):9.2f} min={min(v):9.2f}")
PY
