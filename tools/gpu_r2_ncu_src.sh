# ncu source-level captures of the encoder, gather and decoder at cfg1 + PCIe bound
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/exp/pcie_bw.py > gpurun_out/s_pcie.txt 2>&1
python tools/prof_codec.py 16777216 both || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/s_enc -f python tools/prof_codec.py 16777216 compress > gpurun_out/s_ncu_enc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gather -s 2 -c 1 -o gpurun_out/s_gather -f python tools/prof_codec.py 16777216 compress > gpurun_out/s_ncu_gather.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 1 -c 1 -o gpurun_out/s_dec -f python tools/prof_codec.py 16777216 both > gpurun_out/s_ncu_dec.log 2>&1
tail -2 gpurun_out/s_ncu_*.log; cat gpurun_out/s_pcie.txt
