cd $GRAFT_REPO_ROOT
python tools/prof_codec.py 134217728 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_ -s 4 -c 2 -o gpurun_out/prof5 python tools/prof_codec.py 134217728 > gpurun_out/ncu5.log 2>&1
tail -1 gpurun_out/ncu5.log
