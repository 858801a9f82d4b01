# LL128 form of the small-message SGD step (fp32): forced-LL128 worker (mean + sgd +
# mixed sequences), full GPU suite at world 4, smoke, benches at config 1 (N=2, 4) and
# R50 N=2, sweep_sgd at N=2 (graph)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k ll128 > gpurun_out/v_vr.log 2>&1; echo vr=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest_n4.log 2>&1; echo pytest=$?
for N in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2998$N bench.py --gpus $N --config c1 > gpurun_out/v_bench_n${N}_c1.json 2> gpurun_out/v_bench_n${N}_c1.err; echo bench_c1_n$N=$?
done
for f in 0 1; do
  GDRAA_LL128=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29990 tools/sweep_sgd.py --graph --path ll --min-log2 10 --max-log2 22 > gpurun_out/v_sweep_sgd_n2_ll128_$f.jsonl 2> gpurun_out/v_sweep_sgd_n2_ll128_$f.err; echo sweep_sgd_$f=$?
done
tail -3 gpurun_out/v_vr.log; tail -3 gpurun_out/v_pytest_n4.log; tail -1 gpurun_out/v_smoke.log
