# NVLink counter calibration v2 (field return codes + GPM rates); bench timing as a CUDA
# graph replay vs the eager loop at config 1 (launch-bound) and R50, N=1 and N=2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/q_build.log 2>&1
timeout 300 python tools/nvlink_counters.py > gpurun_out/q_calib.jsonl 2> gpurun_out/q_calib.err; echo calib=$?
for c in c1 r50; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/q_bench_n1_${c}_eager.json 2> gpurun_out/q_bench_n1_${c}_eager.err; echo n1_${c}_eager=$?
  timeout 600 python bench.py --config $c --no-cpu-baseline --graph > gpurun_out/q_bench_n1_${c}_graph.json 2> gpurun_out/q_bench_n1_${c}_graph.err; echo n1_${c}_graph=$?
  for m in "" "--graph"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 --config $c $m > gpurun_out/q_bench_n2_${c}${m/--/_}.json 2> gpurun_out/q_bench_n2_${c}${m/--/_}.err; echo n2_${c}${m}=$?
  done
done
cat gpurun_out/q_calib.jsonl; tail -3 gpurun_out/q_calib.err
