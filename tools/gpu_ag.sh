# allgather variants at 512 MiB: N=4 and N=2, device time of graph replays
cd $GRAFT_REPO_ROOT
for N in 4 2; do
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N tools/prof_ring_stamps.py"
for m in auto bulk multi; do
  echo "== N=$N ag_mode=$m"; GZ_AG_MODE=$m GZ_NO_STAMPS=1 $T 16 64 512 2>&1 | grep "rank0"
done; done
GZ_AG_MODE=bulk timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 tools/prof_ring_stamps.py 512 2>&1 | grep "MiB rank0"
