mkdir -p gpurun_out
{
echo "== TG on"; timeout 300 python tools/exp/pair_encode/pair_ab.py
echo "== TG off"; GZ_TRAILING_GATHER=0 timeout 300 python tools/exp/pair_encode/pair_ab.py
echo "== TG on again"; timeout 300 python tools/exp/pair_encode/pair_ab.py
} > gpurun_out/tg_ab.log 2>&1
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_bench_sizes_gpu.py -x -q > gpurun_out/tg_tests.log 2>&1
echo "rc $?" >> gpurun_out/tg_tests.log
cat gpurun_out/tg_ab.log; tail -5 gpurun_out/tg_tests.log
