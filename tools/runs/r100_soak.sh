# round 2, call 38 (4 GPUs): soak test -- random call sequences for minutes, every call
# checked bit for bit (integer family), at N = 4 and N = 2.
set -x; mkdir -p gpurun_out
P=30500
for N in 4 2; do
  P=$((P+1))
  GDRAA_TIMEOUT_MS=30000 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
    tools/soak.py --seconds 240 > gpurun_out/soak_n$N.json 2> gpurun_out/soak_n$N.err
  echo soak N=$N rc=$?
  cut -c1-600 gpurun_out/soak_n$N.json
done
