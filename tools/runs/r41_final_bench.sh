# after the bench fix: N=1 bench + reference arm + ncu launch list + full capture,
# N=2/3/4 benches, then config 5 NCCL algorithm/protocol logs and the Ring comparator
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f_build.log 2>&1
timeout 600 python bench.py > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err; echo bench1=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_ref_n1.json 2> gpurun_out/f_ref_n1.err; echo ref1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/f_launches_n1.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gdraa_kernel -s 5 -c 1 -o gpurun_out/f_n1_r50 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu2.log 2>&1; echo ncu2=$?
for N in 2 3 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N bench.py --gpus $N > gpurun_out/f_bench_n$N.json 2> gpurun_out/f_bench_n$N.err; echo bench$N=$?
done
bash tools/runs/r40_nccl_algos.sh
