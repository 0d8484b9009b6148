# A/B: fused step with / without the L2 prefetch of the next tile (peer slots, 2 GPUs)
cd $GRAFT_REPO_ROOT
for r in 1 2; do for L in ahead0 ahead24 ahead48; do echo "== $L"; GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python tools/prof_peer_step.py 33554432 7; GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python tools/prof_peer_step.py 67108864 5; done; done
