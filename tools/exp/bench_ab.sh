# bench.py N=1 alternating between builds: tools/exp/bench_ab.sh a.so b.so ... (REPS=2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in $(seq 1 ${REPS:-2}); do
for so in "$@"; do
  cp $so paper_2308_05199_b200/libgzccl.so
  python bench.py --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['detail']
print('$so', 'value', d['value'], 'compress_us', e['compress_us'], 'decompress_us', e['decompress_us'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'], '2p27', e['codec_2p27']['compress_us'], e['codec_2p27']['decompress_us'])"
done; done
