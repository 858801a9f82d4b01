# LL128 premise probe: are 128-byte lines written by 8 lanes of one warp store seen whole
# over NVLink (flag in the last 8 bytes => payload present)?  2 GPUs, bounded spins.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ll128_probe tools/ll128_probe.cu > gpurun_out/l_build.log 2>&1; echo build=$?
timeout 120 tools/ll128_probe 262144 200 | tee gpurun_out/l_probe.jsonl; echo big=$?
timeout 120 tools/ll128_probe 1048576 100 | tee -a gpurun_out/l_probe.jsonl; echo huge=$?
timeout 120 tools/ll128_probe 4096 20000 | tee -a gpurun_out/l_probe.jsonl; echo small=$?
timeout 120 tools/ll128_probe 32768 5000 | tee -a gpurun_out/l_probe.jsonl; echo mid=$?
