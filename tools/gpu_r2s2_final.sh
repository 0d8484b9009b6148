# round 2 (second session) evidence: bench N=1 + launch list, the peer fused step at the
# N=2 chunk (2^26) with NVLink counters, bench N=2; concurrent PCIe duplex per GPU
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=r2s2
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_n1.json 2> gpurun_out/${T}_bench_n1.err; echo "n1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches_n1.csv python bench.py --steps 2 --warmup 1 > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tile_decode -s 1 -c 1 -o gpurun_out/${T}_dec -f python tools/prof_codec.py 16777216 both > gpurun_out/${T}_ncu_dec.log 2>&1; echo "dec ncu rc=$?"
python tools/prof_peer_step.py 67108864 3 > /dev/null 2>&1 || echo "peer step failed"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_tile_encode -c 4 --csv python tools/prof_peer_step.py 67108864 3 > gpurun_out/${T}_step26_peer_nvl.csv 2>&1; echo "step nvl rc=$?"
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/${T}_bench_n2.json 2> gpurun_out/${T}_bench_n2.err; echo "n2 rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 tools/exp/pcie_ranks.py > gpurun_out/${T}_pcie_ranks.txt 2>&1; echo "pcie rc=$?"; cat gpurun_out/${T}_pcie_ranks.txt | grep rank
