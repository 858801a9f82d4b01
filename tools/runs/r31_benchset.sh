# Full bench set: every config at N = 1, 2, 4 (run on a 4-GPU box) + fair multicast probe
# + the GPU test suite at world 4.  Output: gpurun_out/bs_*.json
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bs_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
timeout 300 ./tools/mc_probe 4 20000 > gpurun_out/bs_mc_probe_n4.jsonl 2>&1
timeout 300 ./tools/mc_probe 2 20000 >> gpurun_out/bs_mc_probe_n4.jsonl 2>&1
port=29600
for N in 1 2 4; do
  for c in r50 r101 r50bf16 r50bf16mp c1; do
    port=$((port+1))
    extra="--no-cpu-baseline"
    if [ $N = 1 ] && [ $c = r50 ]; then extra=""; fi
    if [ $N = 1 ]; then
      timeout 600 python bench.py --config $c $extra > gpurun_out/bs_n${N}_$c.json 2> gpurun_out/bs_n${N}_$c.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --config $c $extra > gpurun_out/bs_n${N}_$c.json 2> gpurun_out/bs_n${N}_$c.err
    fi
    echo "bench N=$N $c rc=$?"
  done
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/bs_pytest_n4.log 2>&1; echo pytest=$?
tail -2 gpurun_out/bs_pytest_n4.log
