# r58 stalled (both grids gave up): sender now on its own non-blocking stream, the last
# acknowledged epoch reported
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ll128_probe tools/ll128_probe.cu || exit 1
for cfg in "4096 5000" "65536 1000" "1048576 100"; do
  timeout 120 /tmp/ll128_probe $cfg 0 1 >> gpurun_out/r59_ll128_same.jsonl; echo rc=$?
done
timeout 120 /tmp/ll128_probe 65536 200 1 1 >> gpurun_out/r59_ll128_same.jsonl; echo control_rc=$?
cat gpurun_out/r59_ll128_same.jsonl
