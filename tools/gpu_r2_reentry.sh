# re-entry validation: full GPU suite on 2 GPUs, then bench lines N=1 and N=2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/re_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/re_pytest.txt 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/re_pytest.txt
bash tools/gpu_r2_bench.sh 2 re
