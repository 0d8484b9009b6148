# small-message ring allreduce: correctness (4 GPUs) + device timelines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_comm_gpu.py tests/test_codec_gpu.py tests/test_collectives_virtual_gpu.py -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
T="timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/prof_ring_stamps.py"
echo "== auto (no stamps)"; GZ_NO_STAMPS=1 $T 1 4 16 64 256 512 2>&1 | grep "rank0"
echo "== auto, stamps"; $T 1 2>&1 | grep "MiB rank"
