# LL-SGD parity + crossover sweep + TMA end-game variants (N=2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e1_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "latency_path or mixed_call or sgd_step" > gpurun_out/e1_pytest_vr.log 2>&1; echo vr=$?
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/e1_pytest_mp.log 2>&1; echo mp=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 tools/sweep_sgd.py --graph --max-log2 25 > gpurun_out/e1_sweep_sgd_n2_graph.jsonl 2> gpurun_out/e1_sweep.err; echo sweep=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 tools/sweep_sgd.py --max-log2 25 > gpurun_out/e1_sweep_sgd_n2_eager.jsonl 2>> gpurun_out/e1_sweep.err; echo sweep2=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/tune tools/tune.cu
timeout 600 ./tools/tune 2 25557032 f32 sgd 100 tail > gpurun_out/e1_tail_n2.jsonl 2> gpurun_out/e1_tail.err; echo tail=$?
timeout 600 ./tools/tune 2 44549160 f32 sgd 100 tail > gpurun_out/e1_tail_n2_r101.jsonl 2>> gpurun_out/e1_tail.err; echo tail2=$?
tail -3 gpurun_out/e1_pytest_vr.log gpurun_out/e1_pytest_mp.log
