# config-5 sweep refresh (LL mean with back-off) at N=2 and 4, graph + eager; the
# multi-process test suite at world 3 (odd N: the division is not a power of two)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c5_build.log 2>&1
for N in 2 4; do
  for mode in graph eager; do
    flag=""; if [ $mode = graph ]; then flag="--graph"; fi
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N tools/sweep.py $flag > gpurun_out/c5_sweep_n${N}_$mode.jsonl 2> gpurun_out/c5_sweep_n${N}_$mode.err; echo sweep_n${N}_$mode=$?
  done
done
CUDA_VISIBLE_DEVICES=0,1,2 timeout 1500 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/c5_mp_world3.log 2>&1; echo world3=$?
CUDA_VISIBLE_DEVICES=0,1,2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29620 bench.py --gpus 3 > gpurun_out/c5_bench_n3.json 2> gpurun_out/c5_bench_n3.err; echo bench3=$?
tail -2 gpurun_out/c5_mp_world3.log
