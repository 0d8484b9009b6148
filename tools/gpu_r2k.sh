cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_codec_gpu.py -q -p no:cacheprovider -k "nonfinite" 2>&1 | tail -15
python tools/exp/e2e_lanes.py
