# N = 4: LL-SGD crossover, multicast probe, TMA end-game/rotation variants, multi-process
# tests, benches (r50, c1)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e3_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/tune tools/tune.cu
timeout 300 ./tools/mc_probe $N 20000 > gpurun_out/e3_mc_probe_n$N.jsonl 2>&1; echo mc=$?
timeout 300 ./tools/mc_probe 2 20000 >> gpurun_out/e3_mc_probe_n$N.jsonl 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/e3_pytest_mp_n$N.log 2>&1; echo mp=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 tools/sweep_sgd.py --graph --max-log2 24 > gpurun_out/e3_sweep_sgd_n${N}_graph.jsonl 2> gpurun_out/e3_sweep.err; echo sweep=$?
timeout 600 ./tools/tune $N 25557032 f32 sgd 100 tail > gpurun_out/e3_tail_n$N.jsonl 2> gpurun_out/e3_tail.err; echo tail=$?
for c in r50 c1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus $N --config $c > gpurun_out/e3_bench_n${N}_$c.json 2> gpurun_out/e3_bench_$c.err; echo bench_$c=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --config c1 > gpurun_out/e3_bench_n2_c1.json 2> gpurun_out/e3_bench_n2c1.err; echo bench_n2c1=$?
