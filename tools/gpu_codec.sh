cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python tools/bench_codec.py 16777216 1e-4 2>&1 | tail -2
timeout 300 python tools/bench_codec.py 134217728 1e-4 2>&1 | tail -2
