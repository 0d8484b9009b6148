cd $GRAFT_REPO_ROOT
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 tests/mgpu_worker.py 2>&1 | grep -v "^\s*$" | grep -v "^  File \"/opt\|^    " | head -40
