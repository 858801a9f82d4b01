# A/B: grid sized by small (end-game) chunks vs big chunks, mid sizes, N=2 and N=4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g_build.log 2>&1
for N in 2 4; do
  for gs in 0 1; do
    GDRAA_GRID_SMALL=$gs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N tools/sweep.py --graph --min-log2 20 --max-log2 27 > gpurun_out/g_mean_n${N}_gs$gs.jsonl 2> gpurun_out/g_mean_n${N}_gs$gs.err; echo mean_n${N}_gs$gs=$?
    GDRAA_GRID_SMALL=$gs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2964$N tools/sweep_sgd.py --graph --path two_shot --min-log2 16 --max-log2 26 > gpurun_out/g_sgd_n${N}_gs$gs.jsonl 2> gpurun_out/g_sgd_n${N}_gs$gs.err; echo sgd_n${N}_gs$gs=$?
  done
done
