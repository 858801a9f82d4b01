# r59 stalled: lazy module loading serialised the second grid; kernels now loaded up front (and EAGER)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ll128_probe tools/ll128_probe.cu || exit 1
for cfg in "4096 5000" "65536 1000" "1048576 100"; do
  CUDA_MODULE_LOADING=EAGER timeout 120 /tmp/ll128_probe $cfg 0 1 >> gpurun_out/r60_ll128_same.jsonl; echo rc=$?
done
CUDA_MODULE_LOADING=EAGER timeout 120 /tmp/ll128_probe 65536 200 1 1 >> gpurun_out/r60_ll128_same.jsonl; echo control_rc=$?
cat gpurun_out/r60_ll128_same.jsonl
