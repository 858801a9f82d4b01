# LL128 served by size (n*s*(N-1) >= 512 KiB) by default: smoke, full GPU suite at world 4
# (vr parity now crosses both LL formats; the forced-LL128 worker interleaves SGD steps),
# config-5 sweeps (graph) at N=2,4, N=2 bench at config 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/u_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/u_pytest_n4.log 2>&1; echo pytest=$?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2997$N tools/sweep.py --graph > gpurun_out/u_sweep_n${N}_graph.jsonl 2> gpurun_out/u_sweep_n${N}_graph.err; echo sweep_n$N=$?
done
tail -3 gpurun_out/u_pytest_n4.log; tail -1 gpurun_out/u_smoke.log
