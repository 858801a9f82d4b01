# reproduce the r51 LL128 SGD failure (r53: as committed; r54: with __syncwarp before every
# LL128 line store and load): the vr SGD latency-path test at f32 with the size
# rule on, five times per N (1 GPU)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r_build.log 2>&1
for i in 1 2 3 4 5; do
  GDRAA_LL128=auto timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "test_vr_sgd_latency_path and False-f32" > gpurun_out/r_auto_$i.log 2>&1; echo auto_$i=$?; tail -1 gpurun_out/r_auto_$i.log
done
for i in 1 2; do
  GDRAA_LL128=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "test_vr_sgd_latency_path and False-f32" > gpurun_out/r_forced_$i.log 2>&1; echo forced_$i=$?; tail -1 gpurun_out/r_forced_$i.log
done
grep -h "AssertionError: " gpurun_out/r_*.log | head -10
