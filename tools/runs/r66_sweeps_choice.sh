# round 2, call 5 (4 GPUs): with the per-CTA exit fence the two-shot kernel's constant
# dropped, so (1) the small-message crossovers (mean and sgd_step, LL vs two-shot) and
# (2) the LSU/TMA kernel choice for bf16 at N <= 2 are re-measured; (3) config 5 (mean
# 1 KiB - 1 GiB vs NCCL) re-run at N = 2 and 4.  All CUDA-graph timed.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/e_pytest_n4.log 2>&1; echo pytest=$?
tail -2 gpurun_out/e_pytest_n4.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/e_ab_now_$rep.json 2> gpurun_out/e_ab_now_$rep.err; echo now=$?
  GDRAA_LIB_PATH=$PWD/paper_1802_02326_b200/lib_ab/libgdraa_b48b841.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/e_ab_old_$rep.json 2> gpurun_out/e_ab_old_$rep.err; echo old=$?
done
L50=25557032
{
./tools/tune 1 $L50 f32 sgd 100 lsu
./tools/tune 1 $L50 bf16 sgd 100 lsu
for N in 2 4; do
  ./tools/tune $N $L50 bf16 sgd 50 lib
  ./tools/tune $N $L50 bf16 mean 50 lib
  ./tools/tune $N $L50 bf16 mp 50 lib
done
} > gpurun_out/e_tune_choice.jsonl 2> gpurun_out/e_tune_choice.err; echo tune=$?
P=29700
for N in 2 4; do
  for path in ll two_shot; do
    P=$((P+1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      tools/sweep_sgd.py --path $path --graph --max-log2 25 > gpurun_out/e_sweep_sgd_n${N}_${path}.jsonl 2> gpurun_out/e_sweep_sgd_n${N}_${path}.err
    echo sweep_sgd N=$N $path rc=$?
  done
  for ll in default 0; do
    P=$((P+1))
    if [ $ll = 0 ]; then export GDRAA_LL_MAX_BYTES=0; else unset GDRAA_LL_MAX_BYTES; fi
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      tools/sweep.py --graph --max-log2 30 > gpurun_out/e_sweep_mean_n${N}_ll${ll}.jsonl 2> gpurun_out/e_sweep_mean_n${N}_ll${ll}.err
    echo sweep_mean N=$N ll=$ll rc=$?
  done
  unset GDRAA_LL_MAX_BYTES
done
du -sh gpurun_out
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/e_ab_*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f.split("/")[-1], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
for l in open("gpurun_out/e_tune_choice.jsonl"):
    d = json.loads(l); print(d["world"], d["dtype"], d["mode"], d["kernel"], d["shape"][:24], d["grid"], d["us"])
for f in sorted(glob.glob("gpurun_out/e_sweep_*.jsonl")):
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    print(f.split("/")[-1], [(r.get("bytes", r.get("g_bytes")), round(r.get("gdraa_us", r.get("us", 0)), 1), round(r.get("nccl_us", 0), 1)) for r in rows][:30])
PY
