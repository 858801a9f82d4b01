# round 2, call 40 (4 GPUs): soak test with sizes up to ResNet-50's (26 M elements), N = 4.
set -x; mkdir -p gpurun_out
GDRAA_TIMEOUT_MS=30000 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30601 \
  tools/soak.py --seconds 240 --max-elems 26000000 --seed 7 > gpurun_out/soak_large_n4.json 2> gpurun_out/soak_large_n4.err
echo soak rc=$?
cut -c1-400 gpurun_out/soak_large_n4.json
