# N=2: LL-SGD with rotating buffer sets, poll back-off variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e5_build.log 2>&1
for sl in 0 256 1024; do
GDRAA_LL_SLEEP_NS=$sl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2956$sl tools/ll_debug.py > gpurun_out/e5_lldbg_sleep$sl.jsonl 2> gpurun_out/e5_lldbg_$sl.err; echo lldbg$sl=$?
done
for sl in 0 256; do
GDRAA_LL_SLEEP_NS=$sl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --config c1 --no-nccl --steps 200 > gpurun_out/e5_c1_sleep$sl.json 2> gpurun_out/e5_c1_$sl.err; echo c1_$sl=$?
GDRAA_LL_SLEEP_NS=$sl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572 tools/sweep_sgd.py --graph --max-log2 22 > gpurun_out/e5_sweep_sgd_graph_sleep$sl.jsonl 2> gpurun_out/e5_sweep_$sl.err; echo sweep_$sl=$?
done
