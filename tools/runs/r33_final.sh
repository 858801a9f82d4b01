# final round check on a 4-GPU box: GPU suite, N=1 bench + ncu launch list + full capture,
# LL-SGD kernel capture (virtual ranks), N=2/N=4 benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest_n4.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/f_bench_n1.json 2> gpurun_out/f_bench_n1.err; echo bench1=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 5 -c 40 --csv --log-file gpurun_out/f_launches_n1.csv python bench.py --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gdraa_kernel -s 5 -c 1 -o gpurun_out/f_n1_r50 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/f_ncu2.log 2>&1; echo ncu2=$?
cat > /tmp/ll_vr.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_1802_02326_b200 import gdraa
N, L = 2, 1 << 20
g = [torch.randn(L, device="cuda") * 1e-3 for _ in range(N)]
w0 = torch.randn(L, device="cuda")
w = [w0.clone() for _ in range(N)]
v = [torch.zeros(L, device="cuda") for _ in range(N)]
for _ in range(8):
    gdraa.gdraa_vr_sgd_step(w, g, v, 0.1, 0.9)
torch.cuda.synchronize()
print("ok")
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gdraa_ll_sgd_kernel -s 3 -c 1 -o gpurun_out/f_ll_sgd_vr2 python /tmp/ll_vr.py > gpurun_out/f_ncu3.log 2>&1; echo ncu3=$?
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N bench.py --gpus $N > gpurun_out/f_bench_n$N.json 2> gpurun_out/f_bench_n$N.err; echo bench$N=$?
done
tail -2 gpurun_out/f_pytest_n4.log
