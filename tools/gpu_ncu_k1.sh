cd $GRAFT_REPO_ROOT
python tools/prof_codec.py 16777216 compress || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_k1 -f python tools/prof_codec.py 16777216 compress > gpurun_out/ncu_k1.log 2>&1
tail -n 1 gpurun_out/ncu_k1.log
