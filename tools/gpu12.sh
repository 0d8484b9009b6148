cd $GRAFT_REPO_ROOT
nvidia-smi topo -m 2>&1 | head -5
timeout 900 python -m pytest tests/test_comm_gpu.py -x -q -s 2>&1 | tail -15
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 2>&1 | grep -v Warning | tail -3
