# round 2, call 9 (2 GPUs): the receive-buffer (RB) kernel -- the paper's push design with
# per-CTA-pair flags -- first parity (vr RB tests, the whole GPU suite at world 2), then
# graph-timed sweeps at N = 2: sgd_step on the LL / RB / two-shot paths, allreduce_mean
# with and without RB, and the bench configs the RB limit now covers.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rb_path" > gpurun_out/i_pytest_rb.log 2>&1; echo pytest_rb=$?
tail -3 gpurun_out/i_pytest_rb.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/i_pytest_n2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/i_pytest_n2.log
P=30000
for path in rb two_shot ll; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
    tools/sweep_sgd.py --path $path --graph --max-log2 26 > gpurun_out/i_sweep_sgd_n2_$path.jsonl 2> gpurun_out/i_sweep_sgd_n2_$path.err
  echo sweep_sgd $path rc=$?
done
for rb in default 0; do
  P=$((P+1))
  if [ $rb = 0 ]; then export GDRAA_RB_MAX_BYTES=0; else unset GDRAA_RB_MAX_BYTES; fi
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
    tools/sweep.py --graph --min-log2 20 --max-log2 28 > gpurun_out/i_sweep_mean_n2_rb$rb.jsonl 2> gpurun_out/i_sweep_mean_n2_rb$rb.err
  echo sweep_mean rb=$rb rc=$?
done
unset GDRAA_RB_MAX_BYTES
for cfg in r50bf16 r50bf16mp; do
  for rb in default 0; do
    if [ $rb = 0 ]; then export GDRAA_RB_MAX_BYTES=0; else unset GDRAA_RB_MAX_BYTES; fi
    timeout 600 python3 bench.py --gpus 2 --config $cfg --e2e-steps 3 --no-nccl > gpurun_out/i_bench_n2_${cfg}_rb$rb.json 2> gpurun_out/i_bench_n2_${cfg}_rb$rb.err
    echo bench $cfg rb=$rb rc=$?
  done
done
unset GDRAA_RB_MAX_BYTES
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/i_sweep_*.jsonl")):
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    print(f.split("/")[-1], [(r.get("bytes", r.get("g_bytes")), round(r.get("gdraa_us", r.get("us", 0)), 1)) for r in rows])
for f in sorted(glob.glob("gpurun_out/i_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], d["config"]["path"], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4))
    except Exception as e:
        print(f, "ERR", e)
PY
