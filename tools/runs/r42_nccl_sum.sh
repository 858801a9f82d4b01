# config 5 with NCCL timed on SUM (NVLS in-switch reduction is eligible; AVG picked Ring
# everywhere in r41) at N=2,4, graph replay, plus the NCCL tuner log for SUM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s_build.log 2>&1
for N in 2 4; do
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING,NVLS timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2992$N tools/sweep.py --graph --nccl-op sum > gpurun_out/s_sweep_n${N}_graph_sum.jsonl 2> gpurun_out/s_sweep_n${N}_graph_sum.err; echo sum_n$N=$?
  python tools/nccl_algos.py gpurun_out/s_sweep_n${N}_graph_sum.err > gpurun_out/s_nccl_algos_sum_n$N.json; echo parse_n$N=$?
done
