# full GPU suite (multi-GPU tests use the GPUs the box has)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_check_pytest.txt 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r2_check_pytest.txt
grep -h "mgpu ranks\|FAIL\|Error" gpurun_out/r2_check_pytest.txt | sort | uniq -c | head
