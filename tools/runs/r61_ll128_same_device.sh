# larger same-device sample after r60 ran through
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ll128_probe tools/ll128_probe.cu || exit 1
for cfg in "4096 200000" "65536 20000" "1048576 2000" "16384 50000"; do
  CUDA_MODULE_LOADING=EAGER timeout 120 /tmp/ll128_probe $cfg 0 1 >> gpurun_out/r61_ll128_same.jsonl; echo rc=$?
done
CUDA_MODULE_LOADING=EAGER timeout 120 /tmp/ll128_probe 65536 200 1 1 >> gpurun_out/r61_ll128_same.jsonl; echo control_rc=$?
cat gpurun_out/r61_ll128_same.jsonl
