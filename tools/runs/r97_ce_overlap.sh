# round 2, call 36 (2 GPUs): copy-engine vs SM data path beside a compute-bound backward.
set -x; mkdir -p gpurun_out
for K in 4 8; do
  timeout 600 tools/ce_overlap 25557032 $K 0 20 >> gpurun_out/ceo.jsonl 2>> gpurun_out/ceo.err; echo K=$K rc=$?
done
cat gpurun_out/ceo.jsonl
