# round 2, call 7 (4 GPUs): GPU suite at world 4 with the final kernel choice (TMA for all
# N >= 2) and N = 1 shape; the opt-in world-8 test (2 ranks per GPU, time-sliced); the
# bench set at N = 2, 4 for every config; NEXT-3 overlap re-measured with the CTA fence.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g_pytest_n4.log 2>&1; echo pytest=$?
tail -2 gpurun_out/g_pytest_n4.log
GDRAA_TEST_OVERSUBSCRIBE=1 timeout 900 python -m pytest tests/test_multigpu.py -q -k world8 > gpurun_out/g_pytest_world8.log 2>&1; echo world8=$?
tail -3 gpurun_out/g_pytest_world8.log
for N in 2 4; do
  for cfg in r50 r101 r50bf16 r50bf16mp c1; do
    timeout 600 python3 bench.py --gpus $N --config $cfg --e2e-steps 10 > gpurun_out/g_bench_n${N}_${cfg}.json 2> gpurun_out/g_bench_n${N}_${cfg}.err
    echo bench N=$N $cfg rc=$?
  done
done
P=29800
for b in 2 4 8; do
  for cap in 0 32; do
    P=$((P+1))
    GDRAA_MAX_CTAS=$cap timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
      tools/overlap.py --buckets $b > gpurun_out/g_overlap_n2_b${b}_c${cap}.json 2> gpurun_out/g_overlap_n2_b${b}_c${cap}.err
    echo overlap b=$b cap=$cap rc=$?
  done
done
du -sh gpurun_out
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/g_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        n = d.get("nccl_reference") or {}
        print(f.split("/")[-1], d["config"]["path"], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4), round(n.get("ms", 0) * 1e3, 1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
for f in sorted(glob.glob("gpurun_out/g_overlap_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], {k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items() if k in ("buckets", "max_ctas", "bwd_us", "comm_us", "comm_bucketed_us", "serial_us", "overlap_us", "speedup")})
    except Exception as e:
        print(f, "ERR", e)
PY
