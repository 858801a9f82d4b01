# round 2, call 3 (4 GPUs): (1) N=1 A/B of the current build vs b48b841 (the r62 build) on
# one box; (2) tune: 4 vs 8 elements per consumer thread for bf16 broadcasts, NVLS
# multicast all-gather / barriers at N=2/4; (3) ncu: solo rank-0 captures at N=4 (fp32
# sgd, bf16 mixed-precision) with NVLink counters; launch list of bench N=1.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c_pytest_n4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/c_pytest_n4.log
for N in 2 4; do
  timeout 600 python3 bench.py --gpus $N --config r50bf16mp --e2e-steps 3 --no-nccl > gpurun_out/c_bench_n${N}_r50bf16mp.json 2> gpurun_out/c_bench_n${N}_mp.err; echo benchmp$N=$?
done
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/c_ab_now_$rep.json 2> gpurun_out/c_ab_now_$rep.err; echo now=$?
  GDRAA_LIB_PATH=$PWD/paper_1802_02326_b200/lib_ab/libgdraa_b48b841.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/c_ab_old_$rep.json 2> gpurun_out/c_ab_old_$rep.err; echo old=$?
done
L50=25557032
{
./tools/tune 2 $L50 bf16 mp 50 ve
./tools/tune 4 $L50 bf16 mp 50 ve
./tools/tune 2 $L50 f32 sgd 50 mc
./tools/tune 4 $L50 f32 sgd 50 mc
./tools/tune 4 $L50 bf16 mp 50 mc
./tools/tune 2 $L50 bf16 mp 50 mc
} > gpurun_out/c_tune.jsonl 2> gpurun_out/c_tune.err; echo tune=$?
./tools/tune 4 $L50 f32 sgd 10 solo > gpurun_out/c_plain_solo4.log 2>&1 && \
ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
    --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 5 -c 1 \
    -o gpurun_out/c_solo_n4_tma ./tools/tune 4 $L50 f32 sgd 10 solo > gpurun_out/c_ncu_solo4.log 2>&1; echo ncu_solo4=$?
./tools/tune 4 $L50 bf16 mp 10 solo > gpurun_out/c_plain_solo4mp.log 2>&1 && \
ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum \
    --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 5 -c 1 \
    -o gpurun_out/c_solo_n4_mp_tma ./tools/tune 4 $L50 bf16 mp 10 solo > gpurun_out/c_ncu_solo4mp.log 2>&1; echo ncu_solo4mp=$?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c_plain_bench1.json 2> gpurun_out/c_plain_bench1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_launches_n1.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/c_ncu_launches.log 2>&1; echo ncu_launches=$?
