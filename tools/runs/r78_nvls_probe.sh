# round 2, call 17 (4 GPUs): NVLS in-switch reduction probe -- bits (determinism, order
# vs the oracle's rank-ordered fold) and rate of ld_reduce-based allreduce data movement.
set -x; mkdir -p gpurun_out
nvidia-smi -L
for n in 2 3 4; do
  timeout 300 tools/nvls_probe $n 25557032 50 > gpurun_out/v_nvls_n$n.jsonl 2> gpurun_out/v_nvls_n$n.err; echo n=$n rc=$?
  cat gpurun_out/v_nvls_n$n.jsonl; tail -3 gpurun_out/v_nvls_n$n.err
done
