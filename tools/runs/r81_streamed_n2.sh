# round 2, call 20 (2 GPUs): streamed bucket sets across processes -- GPU suite at world 2,
# then NEXT-3 overlap: per-call buckets / bucket set / streamed set, interleaved; and the
# bench R50 line at N = 2 (the per-call kernel after the consumer refactor).
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo smoke=$?
GDRAA_TIMEOUT_MS=20000 timeout 600 python -m pytest tests/test_multigpu.py -m gpu -x -q -k "bucketed" > gpurun_out/u_pytest_bucketed.log 2>&1; echo pytest_bucketed=$?
tail -3 gpurun_out/u_pytest_bucketed.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/u_pytest_n2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/u_pytest_n2.log
timeout 600 python3 bench.py --gpus 2 --e2e-steps 10 > gpurun_out/u_bench_n2_r50.json 2> gpurun_out/u_bench_n2_r50.err; echo bench=$?
P=29950
for rep in 1 2; do
for b in 4 8; do
  for cap in 0 32; do
    for mode in plain set st32 st148; do
      P=$((P+1))
      case $mode in plain) arg="";; set) arg="--set";; st32) arg="--streamed 32";; st148) arg="--streamed 148";; esac
      tag=b${b}_c${cap}_${mode}_$rep
      GDRAA_TIMEOUT_MS=20000 GDRAA_MAX_CTAS=$cap timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
        tools/overlap.py --buckets $b $arg > gpurun_out/u_overlap_n2_$tag.json 2> gpurun_out/u_overlap_n2_$tag.err
      echo overlap $tag rc=$?
    done
  done
done
done
set +x
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/u_overlap_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1][12:], {k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items() if k in ("bwd_us", "comm_us", "comm_bucketed_us", "serial_us", "overlap_us", "speedup")})
    except Exception as e:
        print(f, "ERR", e)
d = json.loads(open("gpurun_out/u_bench_n2_r50.json").read().strip().splitlines()[-1])
print("bench n2", d["ms_per_step"] * 1e3, d["roofline"]["frac"])
PY
