# round 2, call 8 (2 GPUs): where the two-shot kernel's per-call constant goes at small and
# mid sizes: tools/tune phase stamps at N = 2 for 64 Ki .. 4 Mi elements, and the
# graph-timed two-shot sgd sweep with and without the per-call IterDone store into the
# host-mapped job-server page (GDRAA_NO_DONE=1).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
{
for L in 65536 262144 1048576 4194304; do
  ./tools/tune 2 $L f32 sgd 200 lib
done
} > gpurun_out/h_tune_small.jsonl 2> gpurun_out/h_tune_small.err; echo tune=$?
P=29900
for rep in 1 2; do
for nd in 0 1; do
  P=$((P+1))
  GDRAA_NO_DONE=$nd timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
    tools/sweep_sgd.py --path two_shot --graph --max-log2 24 > gpurun_out/h_sweep_sgd_nodone${nd}_$rep.jsonl 2> gpurun_out/h_sweep_nodone${nd}_$rep.err
  echo sweep nodone=$nd rc=$?
done
done
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for l in open("gpurun_out/h_tune_small.jsonl"):
    d = json.loads(l); print(d["L"], d["kernel"], d["grid"], d["us"], d["phase_us"])
for f in sorted(glob.glob("gpurun_out/h_sweep_sgd_*.jsonl")):
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    print(f.split("/")[-1], [(r["g_bytes"], round(r["us"], 2)) for r in rows])
PY
