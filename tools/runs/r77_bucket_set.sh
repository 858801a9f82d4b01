# round 2, call 16 (2 GPUs): bucket sets (deferred exit barrier, gdraa_bucket_set_*):
# the GPU suite at world 2, then NEXT-3 overlap with and without sets, interleaved.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/s_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "bucket_set or forced_kernel or bucketed" > gpurun_out/s_pytest_set.log 2>&1; echo pytest_set=$?
tail -3 gpurun_out/s_pytest_set.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s_pytest_n2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/s_pytest_n2.log
P=29900
for rep in 1 2; do
for b in 2 4 8; do
  for cap in 0 32; do
    for set in "" "--set"; do
      P=$((P+1))
      tag=b${b}_c${cap}${set:+_set}_$rep
      GDRAA_MAX_CTAS=$cap timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
        tools/overlap.py --buckets $b $set > gpurun_out/s_overlap_n2_$tag.json 2> gpurun_out/s_overlap_n2_$tag.err
      echo overlap $tag rc=$?
    done
  done
done
done
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/s_overlap_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], {k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items() if k in ("buckets", "max_ctas", "bucket_set", "bwd_us", "comm_us", "comm_bucketed_us", "serial_us", "overlap_us", "speedup")})
    except Exception as e:
        print(f, "ERR", e)
PY
