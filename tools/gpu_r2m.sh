# A/B of the fused step (peer slots) and codec, base vs step-wait build
cd $GRAFT_REPO_ROOT
for L in base stepwait; do echo "== $L"; for r in 1 2; do GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python tools/prof_peer_step.py 33554432 7; GZCCL_LIB=tools/exp/_old/libgzccl_$L.so python tools/prof_peer_step.py 67108864 5; done; done
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
