# round 2: boundary tests (transports in the reference's algorithms, run_collective) + virtual collectives
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_transport_gpu.py tests/test_collectives_virtual_gpu.py tests/test_codec_gpu.py -q -p no:cacheprovider -x > gpurun_out/r2b_pytest.txt 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2b_pytest.txt
