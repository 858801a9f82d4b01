# round 2, call 23 (4 GPUs): the tree after bucket sets / streamed sets / the shared
# consumer code -- smoke, GPU suite at world 4, bench lines at N = 2 and 4.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/z_pytest_n4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/z_pytest_n4.log
for N in 4 2; do
  for cfg in r50 r101 r50bf16 r50bf16mp c1; do
    timeout 600 python3 bench.py --gpus $N --config $cfg --e2e-steps 10 > gpurun_out/z_bench_n${N}_${cfg}.json 2> gpurun_out/z_bench_n${N}_${cfg}.err
    echo bench N=$N $cfg rc=$?
  done
done
set +x
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/z_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["config"]["path"], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
PY
