# round 2, call 4 (4 GPUs; r64 ran the same A/Bs but its gpurun_out exceeded 64 MiB and
# was lost -- ncu reports are now reduced to CSV on the box and deleted):
# (1) GPU suite (incl. the distributed-exit variant); (2) N=1 A/B current vs b48b841;
# (3) tune: 8-wide bf16 consumer, NVLS multicast AG/barrier, distributed exit at N=2/4;
# (4) ncu: solo rank-0 N=4 captures (fp32, bf16 mp) with NVLink counters; N=1 launch list.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1; echo build=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/d_pytest_n4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/d_pytest_n4.log
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/d_ab_now_$rep.json 2> gpurun_out/d_ab_now_$rep.err; echo now=$?
  GDRAA_LIB_PATH=$PWD/paper_1802_02326_b200/lib_ab/libgdraa_b48b841.so timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/d_ab_old_$rep.json 2> gpurun_out/d_ab_old_$rep.err; echo old=$?
done
L50=25557032
{
./tools/tune 2 $L50 bf16 mp 50 ve
./tools/tune 4 $L50 bf16 mp 50 ve
./tools/tune 2 $L50 f32 sgd 50 mc
./tools/tune 4 $L50 f32 sgd 50 mc
./tools/tune 4 $L50 bf16 mp 50 mc
for rep in 1 2; do
  for N in 2 4; do
    ./tools/tune $N $L50 f32 sgd 50 lib
    GDRAA_DIST_EXIT=1 ./tools/tune $N $L50 f32 sgd 50 lib
    ./tools/tune $N $L50 bf16 mp 50 lib
    GDRAA_DIST_EXIT=1 ./tools/tune $N $L50 bf16 mp 50 lib
  done
done
} > gpurun_out/d_tune.jsonl 2> gpurun_out/d_tune.err; echo tune=$?
for N in 2 4; do
  for cfg in r50 r50bf16mp; do
    for d in 0 1; do
      GDRAA_DIST_EXIT=$d timeout 600 python3 bench.py --gpus $N --config $cfg --e2e-steps 3 --no-nccl > gpurun_out/d_bench_dist${d}_n${N}_${cfg}.json 2> gpurun_out/d_bench_dist${d}_n${N}_${cfg}.err
      echo bench dist=$d N=$N $cfg rc=$?
    done
  done
done
NVL=nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum
./tools/tune 4 $L50 f32 sgd 10 solo > gpurun_out/d_plain_solo4.log 2>&1 && \
ncu --set full --metrics $NVL --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 5 -c 1 \
    -o gpurun_out/d_solo_n4_tma ./tools/tune 4 $L50 f32 sgd 10 solo > gpurun_out/d_ncu_solo4.log 2>&1; echo ncu_solo4=$?
./tools/tune 4 $L50 bf16 mp 10 solo > gpurun_out/d_plain_solo4mp.log 2>&1 && \
ncu --set full --metrics $NVL --clock-control none --import-source on -k regex:gdraa_tma_kernel -s 5 -c 1 \
    -o gpurun_out/d_solo_n4_mp_tma ./tools/tune 4 $L50 bf16 mp 10 solo > gpurun_out/d_ncu_solo4mp.log 2>&1; echo ncu_solo4mp=$?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/d_plain_bench1.json 2> gpurun_out/d_plain_bench1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/d_launches_n1.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/d_ncu_launches.log 2>&1; echo ncu_launches=$?
# keep gpurun_out small: raw CSV pages instead of the reports
for r in gpurun_out/d_solo_n4_tma gpurun_out/d_solo_n4_mp_tma; do
  ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>&1; ncu -i $r.ncu-rep --page details --csv > $r.details.csv 2>&1; rm -f $r.ncu-rep
done
du -sh gpurun_out
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/d_ab_*.json")) + sorted(glob.glob("gpurun_out/d_bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
for l in open("gpurun_out/d_tune.jsonl"):
    d = json.loads(l)
    print(d["world"], d["dtype"], d["mode"], d["kernel"], d["shape"][-22:], d["us"])
PY
