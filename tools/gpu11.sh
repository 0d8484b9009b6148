cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -3
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -2
