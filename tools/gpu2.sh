cd $GRAFT_REPO_ROOT
python tools/prof_codec.py > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_enc python tools/prof_codec.py > gpurun_out/ncu_enc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_decode -s 2 -c 1 -o gpurun_out/prof_dec python tools/prof_codec.py > gpurun_out/ncu_dec.log 2>&1
tail -3 gpurun_out/ncu_enc.log gpurun_out/ncu_dec.log
