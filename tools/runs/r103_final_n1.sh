# round 2, call 42 (1 GPU, the driver's configuration): the final tree -- build, smoke,
# GPU suite, bench.py default line and the reference arm, exactly as the driver runs them.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests/ -q -m gpu --durations=15 > gpurun_out/fin_pytest_n1.log 2>&1; echo pytest=$?
timeout 600 python3 bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref_n1.json 2> gpurun_out/fin_ref_n1.err; echo ref=$?
timeout 600 python3 bench.py > gpurun_out/fin_bench_n1.json 2> gpurun_out/fin_bench_n1.err; echo bench=$?
set +x
tail -2 gpurun_out/fin_pytest_n1.log; tail -1 gpurun_out/fin_smoke.log
python - <<'PY'
import json
for f in ("gpurun_out/fin_bench_n1.json", "gpurun_out/fin_ref_n1.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d.get("impl", "ours"), round(d["ms_per_step"], 4), round(d["value"], 1), d.get("roofline", {}).get("frac"), d.get("e2e", {}).get("value"), d.get("clocks"))
PY
