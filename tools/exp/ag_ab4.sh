# A/B of library builds on the N=4 ring allreduce timeline (512 MiB) and N=2
cd $GRAFT_REPO_ROOT
for r in 1 2; do for L in $*; do echo "== $L"; GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29595 tools/prof_ring_stamps.py 512 2>&1 | grep "MiB rank0"; GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593 tools/prof_ring_stamps.py 512 2>&1 | grep "MiB rank0"; done; done
