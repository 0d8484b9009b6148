# ncu source capture of the in-tree encoder at cfg1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-e}
python tools/prof_codec.py 16777216 compress || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_tile_encode -s 2 -c 1 -o gpurun_out/${TAG}_enc -f python tools/prof_codec.py 16777216 compress > gpurun_out/${TAG}_ncu_enc.log 2>&1
echo ncu rc=$?
