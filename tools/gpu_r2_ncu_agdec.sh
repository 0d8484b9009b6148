# allgather decode of a peer's slots: live times (peer vs local) + ncu of the peer decode (2 GPUs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_peer_decode.py 67108864 5 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -c 1 -o gpurun_out/r2_agdec_peer -f python tools/prof_peer_decode.py 67108864 1 > gpurun_out/r2_ncu_agdec.log 2>&1
tail -n 2 gpurun_out/r2_ncu_agdec.log
