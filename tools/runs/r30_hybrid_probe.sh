# N=2: hybrid SM+copy-engine NVLink probe; LL-mean latency with back-off; full GPU tests
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e6_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/nvlink_probe tools/nvlink_probe.cu
timeout 600 ./tools/nvlink_probe 256 > gpurun_out/e6_nvlink_probe_n2.jsonl 2> gpurun_out/e6_probe.err; echo probe=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/sweep.py --graph --max-log2 24 > gpurun_out/e6_sweep_mean_n2_graph.jsonl 2> gpurun_out/e6_sweep.err; echo sweepm=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e6_pytest_n2.log 2>&1; echo pytest=$?
tail -2 gpurun_out/e6_pytest_n2.log
