# round 2, call 10 (4 GPUs): validation of the final tree (RB reverted): smoke, GPU suite at
# world 4, the opt-in world-8 test, bench N = 1, 2, 4 (R50 fp32) in the driver's form; then
# solo rank-0 ncu captures (NVLink + DRAM counters) for the remaining N >= 2 configs,
# reduced to CSV on the box.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/j_smoke.log 2>&1; echo smoke=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/j_pytest_n4.log 2>&1; echo pytest=$?
tail -2 gpurun_out/j_pytest_n4.log
GDRAA_TEST_OVERSUBSCRIBE=1 timeout 900 python -m pytest tests/test_multigpu.py -q -k world8 > gpurun_out/j_pytest_world8.log 2>&1; echo world8=$?
timeout 600 python3 bench.py > gpurun_out/j_bench_n1.json 2> gpurun_out/j_bench_n1.err; echo bench1=$?
for N in 2 4; do
  timeout 600 python3 bench.py --gpus $N > gpurun_out/j_bench_n$N.json 2> gpurun_out/j_bench_n$N.err; echo bench$N=$?
done
NVL=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum
L50=25557032; L101=44549160
for spec in "2 $L101 f32 sgd r101_n2" "4 $L101 f32 sgd r101_n4" "2 $L50 bf16 sgd r50bf16_n2" "4 $L50 bf16 sgd r50bf16_n4" "2 $L50 bf16 mp r50bf16mp_n2"; do
  set -- $spec
  ./tools/tune $1 $2 $3 $4 10 solo > gpurun_out/j_plain_$5.log 2>&1 && \
  ncu --set full --metrics $NVL --clock-control none -k regex:gdraa_tma_kernel -s 5 -c 1 \
      -o gpurun_out/j_solo_$5 ./tools/tune $1 $2 $3 $4 10 solo > gpurun_out/j_ncu_$5.log 2>&1; echo ncu $5=$?
  ncu -i gpurun_out/j_solo_$5.ncu-rep --page raw --csv > gpurun_out/j_solo_$5.raw.csv 2>&1; rm -f gpurun_out/j_solo_$5.ncu-rep
done
du -sh gpurun_out
set +x
echo "=== summary"
tail -2 gpurun_out/j_pytest_n4.log; tail -2 gpurun_out/j_pytest_world8.log; tail -1 gpurun_out/j_smoke.log
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/j_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["n_gpus"], d["config"]["path"], round(d["ms_per_step"] * 1e3, 2), round(d["value"], 1), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
PY
