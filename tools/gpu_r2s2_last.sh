# last validation: full GPU suite on 4 GPUs, then the cfg4 sweeps at N = 2 and 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s2_last_pytest.txt 2>&1; echo "pytest rc=$?"; tail -n 1 gpurun_out/r2s2_last_pytest.txt
bash tools/gpu_r2s2_sweeps.sh
