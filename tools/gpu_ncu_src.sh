cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_codec.py 16777216 step || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_step -f python tools/prof_codec.py 16777216 step > gpurun_out/ncu_step.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_enc9 -f python tools/prof_codec.py 16777216 compress > gpurun_out/ncu_enc9.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 1 -c 1 -o gpurun_out/prof_dec9 -f python tools/prof_codec.py 16777216 both > gpurun_out/ncu_dec9.log 2>&1
tail -2 gpurun_out/ncu_*9.log gpurun_out/ncu_step.log
