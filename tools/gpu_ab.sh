# A/B of candidate builds under abso/ (first = base) + the codec parity tests on the in-tree build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 900 python -m pytest tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.txt
timeout 900 python tools/exp/ab_codec2.py "$@" > gpurun_out/${TAG}_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/${TAG}_ab.txt | grep -v Warning | tail -40
