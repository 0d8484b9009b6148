cd $GRAFT_REPO_ROOT
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 tools/prof_allreduce.py 512 2>&1 | grep rank
