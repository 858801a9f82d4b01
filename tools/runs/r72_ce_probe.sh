# round 2, call 11 (2 GPUs): copy-engine pipeline bound (tools/ce_probe.cu) at R50 / R101 /
# 4 M elements, N = 2, no cross-device synchronisation modelled (a lower bound).
set -x; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ce_probe tools/ce_probe.cu; echo nvcc=$?
{ ./tools/ce_probe 25557032 20; ./tools/ce_probe 44549160 20; ./tools/ce_probe 4194304 50; } > gpurun_out/k_ce_probe.jsonl 2> gpurun_out/k_ce_probe.err; echo probe=$?
cat gpurun_out/k_ce_probe.jsonl
