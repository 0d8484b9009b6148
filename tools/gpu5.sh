cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/bench_codec.py 16777216 1e-4 2>&1 | tail -3
timeout 300 python tools/bench_codec.py 134217728 1e-4 2>&1 | tail -3
python tools/prof_codec.py > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_ -s 4 -c 2 -o gpurun_out/prof3 python tools/prof_codec.py > gpurun_out/ncu3.log 2>&1
tail -1 gpurun_out/ncu3.log
