cd $GRAFT_REPO_ROOT
cp paper_2308_05199_b200/libgzccl.so /tmp/orig.so
cp tools/exp/libgzccl_NOLOOKBACK.so paper_2308_05199_b200/libgzccl.so
python tools/prof_codec.py 16777216 compress > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/prof_nolb python tools/prof_codec.py 16777216 compress > gpurun_out/ncu_nolb.log 2>&1
tail -1 gpurun_out/ncu_nolb.log
cp /tmp/orig.so paper_2308_05199_b200/libgzccl.so
