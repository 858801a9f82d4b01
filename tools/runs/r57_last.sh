# last check of the round's final tree: smoke, GPU suite at world 4, default bench N=1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/k_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/k_pytest_n4.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/k_bench_n1.json 2> gpurun_out/k_bench_n1.err; echo bench1=$?
tail -2 gpurun_out/k_pytest_n4.log; tail -1 gpurun_out/k_smoke.log; cat gpurun_out/k_bench_n1.json | head -c 400
