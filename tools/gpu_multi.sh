# one GPU call: the encoder ncu capture of the in-tree build, then an A/B of abso/ builds
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-m}
if [ -n "$NCU" ]; then
python tools/prof_codec.py 16777216 compress > /dev/null || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/${TAG}_enc -f python tools/prof_codec.py 16777216 compress > gpurun_out/${TAG}_ncu_enc.log 2>&1
echo ncu rc=$?
fi
timeout 900 python tools/exp/ab_codec2.py "$@" 2>&1 | grep -v -i warn | tee gpurun_out/${TAG}_multi.txt
