cd $GRAFT_REPO_ROOT
python tools/prof_codec.py 16777216 compress || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_gather -s 2 -c 1 -o gpurun_out/prof_gather -f python tools/prof_codec.py 16777216 compress > gpurun_out/ncu_gather.log 2>&1
ncu --set full --import-source on --clock-control none --cache-control none -k regex:k_gather -s 2 -c 1 -o gpurun_out/prof_gather_warm -f python tools/prof_codec.py 16777216 compress > gpurun_out/ncu_gather.log 2>&1
tail -n 2 gpurun_out/ncu_gather.log
