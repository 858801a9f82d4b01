# round 2, call 6 (1 GPU, the driver's configuration): GPU suite + smoke; N=1 launch-shape
# A/B in bench.py (default U4 x 512 x 1/SM vs three other shapes vs b48b841), the default
# bench line, then ncu of the N=1 kernel (full set, and the launch list).
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_n1.log 2>&1; echo pytest=$?
tail -2 gpurun_out/f_pytest_n1.log
AB=$PWD/paper_1802_02326_b200/lib_ab
for rep in 1 2 3; do
  for v in default n1_u1_t512_m3 n1_u2_t1024_m1 n1_u4_t256_m2 b48b841; do
    if [ $v = default ]; then unset GDRAA_LIB_PATH; else export GDRAA_LIB_PATH=$AB/libgdraa_$v.so; fi
    timeout 300 python bench.py --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ab_${v}_$rep.json 2> gpurun_out/f_ab_${v}_$rep.err; echo $v=$?
  done
done
unset GDRAA_LIB_PATH
timeout 600 python bench.py > gpurun_out/f_bench_n1_r50.json 2> gpurun_out/f_bench_n1_r50.err; echo bench1=$?
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_plain_bench1.json 2> gpurun_out/f_plain_bench1.err && \
ncu --set full --clock-control none --import-source on -k regex:gdraa_kernel -s 5 -c 1 -o gpurun_out/f_n1_r50 \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu_full.log 2>&1; echo ncu_full=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_n1.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu_launches.log 2>&1; echo ncu_launches=$?
ncu -i gpurun_out/f_n1_r50.ncu-rep --page raw --csv > gpurun_out/f_n1_r50.raw.csv 2>&1; rm -f gpurun_out/f_n1_r50.ncu-rep
du -sh gpurun_out
set +x
echo "=== summary"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/f_ab_*.json")) + ["gpurun_out/f_bench_n1_r50.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split("/")[-1], round(d["ms_per_step"] * 1e3, 2), round(d["roofline"]["frac"], 4), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    except Exception as e:
        print(f, "ERR", e)
PY
