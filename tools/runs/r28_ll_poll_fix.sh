# after the LL poll fix: LL-SGD + LL-mean latency, multicast probe (N = visible GPUs)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
timeout 300 ./tools/mc_probe $N 20000 > gpurun_out/e2_mc_probe_n$N.jsonl 2>&1; echo mc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "latency_path or mixed_call" > gpurun_out/e2_pytest_vr.log 2>&1; echo vr=$?
timeout 900 python -m pytest tests/test_multigpu.py tests/test_multigpu_faults.py -q -x > gpurun_out/e2_pytest_mp_n$N.log 2>&1; echo mp=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29531 tools/sweep_sgd.py --graph --max-log2 24 > gpurun_out/e2_sweep_sgd_n${N}_graph.jsonl 2> gpurun_out/e2_sweep.err; echo sweep=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29532 tools/sweep.py --graph --max-log2 24 > gpurun_out/e2_sweep_mean_n${N}_graph.jsonl 2>> gpurun_out/e2_sweep.err; echo sweepm=$?
