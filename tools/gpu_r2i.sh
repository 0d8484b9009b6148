cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/r2i_enc python tools/prof_codec.py 16777216 compress > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 2 -c 1 -o gpurun_out/r2i_dec python tools/prof_codec.py 16777216 both > gpurun_out/r2i_ncu2.log 2>&1; echo "ncu rc=$?"
