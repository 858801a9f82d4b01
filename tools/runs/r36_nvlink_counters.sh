# NVML NVLink counter calibration (known peer copy), then N=2 and N=4 benches carrying
# roofline.nvlink_traffic (measured NVLink bytes per launch vs algorithmic)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/n_build.log 2>&1
timeout 300 python tools/nvlink_counters.py > gpurun_out/n_calib.jsonl 2> gpurun_out/n_calib.err; echo calib=$?
for N in 2 4; do
  for c in r50 r101 r50bf16mp; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2970$N bench.py --gpus $N --config $c > gpurun_out/n_bench_n${N}_$c.json 2> gpurun_out/n_bench_n${N}_$c.err; echo bench${N}_$c=$?
  done
done
cat gpurun_out/n_calib.jsonl
