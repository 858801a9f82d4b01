# LL128 probe negative control (flag stored before the payload: torn lines expected) and
# the positive case again, 2 GPUs
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ll128_probe tools/ll128_probe.cu > gpurun_out/l2_build.log 2>&1; echo build=$?
timeout 120 tools/ll128_probe 32768 2000 1 | tee gpurun_out/l2_probe.jsonl; echo control=$?
timeout 120 tools/ll128_probe 4096 5000 1 | tee -a gpurun_out/l2_probe.jsonl; echo control_small=$?
timeout 120 tools/ll128_probe 32768 5000 0 | tee -a gpurun_out/l2_probe.jsonl; echo positive=$?
