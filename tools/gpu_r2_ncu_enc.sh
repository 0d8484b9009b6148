# round 2: ncu full capture (source counters) of the encoder and gather at cfg1, and of the decoder
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/prof_codec.py 16777216 compress || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/r2_enc -f python tools/prof_codec.py 16777216 compress > gpurun_out/r2_ncu_enc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather -s 2 -c 1 -o gpurun_out/r2_gather -f python tools/prof_codec.py 16777216 compress > gpurun_out/r2_ncu_gather.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 1 -c 1 -o gpurun_out/r2_dec -f python tools/prof_codec.py 16777216 both > gpurun_out/r2_ncu_dec.log 2>&1
tail -2 gpurun_out/r2_ncu_*.log
