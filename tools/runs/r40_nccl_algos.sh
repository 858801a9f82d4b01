# config 5: NCCL's algorithm/protocol choice per size (NCCL_DEBUG=INFO, TUNING) at N=2,4,
# and a non-NVLS comparator sweep with NCCL_ALGO=Ring (graph replay)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/a_build.log 2>&1
for N in 2 4; do
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,NVLS timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N tools/sweep.py --min-log2 10 --max-log2 30 > gpurun_out/a_sweep_n${N}_debug.jsonl 2> gpurun_out/a_sweep_n${N}_debug.err; echo debug_n$N=$?
  python tools/nccl_algos.py gpurun_out/a_sweep_n${N}_debug.err > gpurun_out/a_nccl_algos_n$N.json; echo parse_n$N=$?
  NCCL_ALGO=Ring timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2991$N tools/sweep.py --graph > gpurun_out/a_sweep_n${N}_graph_ring.jsonl 2> gpurun_out/a_sweep_n${N}_graph_ring.err; echo ring_n$N=$?
done
head -c 3000 gpurun_out/a_nccl_algos_n2.json
