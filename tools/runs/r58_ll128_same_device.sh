# LL128 premise on one GPU: do 128-byte lines written by one 8-lane store arrive whole when
# writer and reader share a device (the virtual-rank case where the r53-r56 SGD tear was seen)?
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ll128_probe tools/ll128_probe.cu || exit 1
for cfg in "4096 20000" "65536 2000" "1048576 200"; do
  timeout 120 /tmp/ll128_probe $cfg 0 1 >> gpurun_out/r58_ll128_same.jsonl; echo rc=$?
done
timeout 120 /tmp/ll128_probe 65536 500 1 1 >> gpurun_out/r58_ll128_same.jsonl; echo control_rc=$?
cat gpurun_out/r58_ll128_same.jsonl
