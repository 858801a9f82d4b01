# round 2, call 2 (4 GPUs): (1) tools/tune phase breakdowns incl. the mixed-precision step
# and "solo" rank-0-alone runs; (2) bench.py at every config, N = 2 and 4, with the per-CTA
# exit fence now the default; (3) NVLink counters via nvidia-smi; (4) ncu: the solo N=2
# TMA kernel (NVLink rx/tx bytes per launch) and a virtual-rank N=4 R50 call (HBM, stalls).
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b_build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu; echo nvcc=$?
L50=25557032
{
./tools/tune 2 $L50 f32 sgd 50 lib
./tools/tune 2 $L50 f32 sgd 50 solo
./tools/tune 4 $L50 f32 sgd 50 lib
./tools/tune 4 $L50 f32 sgd 50 solo
./tools/tune 2 $L50 bf16 mp 50 lib
./tools/tune 2 $L50 bf16 mp 50 tma
./tools/tune 4 $L50 bf16 mp 50 lib
./tools/tune 4 $L50 bf16 mp 50 tma
./tools/tune 4 $L50 bf16 mp 50 solo
} > gpurun_out/b_tune.jsonl 2> gpurun_out/b_tune.err; echo tune=$?
nvidia-smi nvlink -gt d -i 0 > gpurun_out/b_nvlink_before.txt 2>&1; echo nvsmi_nvlink=$?
for N in 2 4; do
  for cfg in r50 r101 r50bf16 r50bf16mp c1; do
    timeout 600 python3 bench.py --gpus $N --config $cfg --e2e-steps 10 > gpurun_out/b_bench_n${N}_${cfg}.json 2> gpurun_out/b_bench_n${N}_${cfg}.err
    echo bench N=$N $cfg rc=$?
  done
done
nvidia-smi nvlink -gt d -i 0 > gpurun_out/b_nvlink_after.txt 2>&1
timeout 600 python bench.py > gpurun_out/b_bench_n1_r50.json 2> gpurun_out/b_bench_n1_r50.err; echo bench1=$?
# ncu (each command first ran plainly with exit 0 directly before)
./tools/tune 2 $L50 f32 sgd 10 solo > gpurun_out/b_plain_solo.log 2>&1 && \
ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
    --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 5 -c 1 \
    -o gpurun_out/b_solo_n2_tma ./tools/tune 2 $L50 f32 sgd 10 solo > gpurun_out/b_ncu_solo.log 2>&1; echo ncu_solo=$?
python tools/vr_profile.py 4 r50 3 > gpurun_out/b_plain_vr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 2 -c 1 \
    -o gpurun_out/b_vr_n4_r50 python tools/vr_profile.py 4 r50 3 > gpurun_out/b_ncu_vr.log 2>&1; echo ncu_vr=$?
