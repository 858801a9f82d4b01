# final-code bench set, graph-timed: every config at N=1,2,4 (r50 at N=1..4 is r41)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1
for c in r101 r50bf16 r50bf16mp c1; do
  timeout 600 python bench.py --config $c > gpurun_out/b_bench_n1_$c.json 2> gpurun_out/b_bench_n1_$c.err; echo n1_$c=$?
  for N in 2 4; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2994$N bench.py --gpus $N --config $c > gpurun_out/b_bench_n${N}_$c.json 2> gpurun_out/b_bench_n${N}_$c.err; echo n${N}_$c=$?
  done
done
