cd $GRAFT_REPO_ROOT
python tools/prof_codec.py 16777216 compress > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof7 python tools/prof_codec.py 16777216 compress > gpurun_out/ncu7.log 2>&1
tail -1 gpurun_out/ncu7.log
