# full GPU suite on a 4-GPU box (multi-GPU tests at 2, 3, 4 ranks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2s2_check4.txt 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r2s2_check4.txt
grep -h "mgpu ranks\|FAILED\|Error" gpurun_out/r2s2_check4.txt | sort | uniq -c | head
