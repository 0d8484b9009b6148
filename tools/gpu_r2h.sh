cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/exp/ab_codec.py paper_2308_05199_b200/libgzccl.so tools/exp/_old/libgzccl_r1.so
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 3 -c 1 -o gpurun_out/r2h_step python tools/prof_codec.py 33554432 step > gpurun_out/r2h_ncu.log 2>&1; echo "ncu rc=$?"
