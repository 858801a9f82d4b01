# final check of the round's last code (LL128 SGD from n*4*(N-1) >= 3 MiB): smoke, GPU
# suite at world 4, default bench N=1 + reference arm, benches c1 at N=2 and r50 at N=2/4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/z_pytest_n4.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/z_bench_n1.json 2> gpurun_out/z_bench_n1.err; echo bench1=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/z_ref_n1.json 2> gpurun_out/z_ref_n1.err; echo ref1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29981 bench.py --gpus 2 --config c1 > gpurun_out/z_bench_n2_c1.json 2> gpurun_out/z_bench_n2_c1.err; echo bench2_c1=$?
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2998$N bench.py --gpus $N > gpurun_out/z_bench_n$N.json 2> gpurun_out/z_bench_n$N.err; echo bench$N=$?
done
tail -3 gpurun_out/z_pytest_n4.log; tail -1 gpurun_out/z_smoke.log
