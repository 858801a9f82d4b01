# final check with LL128 off by default: smoke, GPU suite at world 4, default bench N=1 +
# reference arm, benches c1 N=2 and r50 N=2/4, and (informational) the LL128 worker
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/y_pytest_n4.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/y_bench_n1.json 2> gpurun_out/y_bench_n1.err; echo bench1=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/y_ref_n1.json 2> gpurun_out/y_ref_n1.err; echo ref1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29971 bench.py --gpus 2 --config c1 > gpurun_out/y_bench_n2_c1.json 2> gpurun_out/y_bench_n2_c1.err; echo bench2_c1=$?
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2997$N bench.py --gpus $N > gpurun_out/y_bench_n$N.json 2> gpurun_out/y_bench_n$N.err; echo bench$N=$?
done
for i in 1 2 3; do GDRAA_TEST_LL128=1 timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k ll128 > gpurun_out/y_ll128_$i.log 2>&1; echo ll128_worker_$i=$?; done
tail -3 gpurun_out/y_pytest_n4.log; tail -1 gpurun_out/y_smoke.log
