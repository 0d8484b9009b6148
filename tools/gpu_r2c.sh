# round 2: multi-GPU checks on N GPUs: comm tests (errors, graph replay), bench N=1 and N=$1, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=${1:-2}
nvidia-smi --query-gpu=name --format=csv,noheader | head -1
timeout 1500 python -m pytest tests/test_comm_gpu.py -q -p no:cacheprovider > gpurun_out/r2c_comm_n$N.txt 2>&1; echo "comm pytest rc=$?"; tail -15 gpurun_out/r2c_comm_n$N.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench_n1.json 2>gpurun_out/r2c_bench_n1.err; echo "n1 rc=$?"; cat gpurun_out/r2c_bench_n1.json; tail -3 gpurun_out/r2c_bench_n1.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/r2c_bench_n$N.json 2>gpurun_out/r2c_bench_n$N.err; echo "n$N rc=$?"; tail -1 gpurun_out/r2c_bench_n$N.json; tail -5 gpurun_out/r2c_bench_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29562 bench.py --impl reference --gpus $N --steps 3 --warmup 1 > gpurun_out/r2c_ref_n$N.json 2>gpurun_out/r2c_ref_n$N.err; echo "ref n$N rc=$?"; tail -1 gpurun_out/r2c_ref_n$N.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29563 bench.py --gpus $N --sweep --sweep-max-mib 256 > gpurun_out/r2c_sweep_n$N.jsonl 2>gpurun_out/r2c_sweep_n$N.err; echo "sweep rc=$?"; cut -c1-400 gpurun_out/r2c_sweep_n$N.jsonl | tail -4
