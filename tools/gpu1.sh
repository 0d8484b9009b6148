set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 300 python __graft_entry__.py 2>&1 | tail -5
timeout 300 python tools/bench_codec.py 16777216 1e-4 2>&1 | tail -5
timeout 300 python tools/bench_codec.py 134217728 1e-4 2>&1 | tail -5
