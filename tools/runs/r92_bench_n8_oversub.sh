# round 2, call 31 (1 GPU): functional check of bench.py's N = 8 path (eight ranks
# time-sliced on one GPU, gloo plumbing): the JSON line an 8-GPU driver run would print.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/o_build.log 2>&1; echo build=$?
GDRAA_BENCH_OVERSUBSCRIBE=1 timeout 1200 python3 bench.py --gpus 8 --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/o_bench_n8.json 2> gpurun_out/o_bench_n8.err; echo bench8=$?
GDRAA_BENCH_OVERSUBSCRIBE=1 timeout 900 python3 bench.py --gpus 8 --config r50bf16mp --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/o_bench_n8_mp.json 2> gpurun_out/o_bench_n8_mp.err; echo bench8mp=$?
tail -c 1500 gpurun_out/o_bench_n8.json; tail -5 gpurun_out/o_bench_n8.err
