set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/v_bench_n1.json 2> gpurun_out/v_bench_n1.err; echo bench1=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/v_bench_n2.json 2> gpurun_out/v_bench_n2.err; echo bench2=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_ref_n1.json 2> gpurun_out/v_ref.err; echo ref=$?
tail -3 gpurun_out/v_pytest.log
