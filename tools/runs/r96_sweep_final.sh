# round 2, call 35 (4 GPUs): config 5 on the final tree -- allreduce_mean fp32 1 KiB - 1 GiB
# vs NCCL all_reduce(AVG), CUDA-graph replay, N = 2 and 4.
set -x; mkdir -p gpurun_out
P=30400
for N in 2 4; do
  P=$((P+1))
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    tools/sweep.py --graph --max-log2 30 > gpurun_out/s5_sweep_mean_n${N}.jsonl 2> gpurun_out/s5_sweep_mean_n${N}.err
  echo sweep N=$N rc=$?
done
