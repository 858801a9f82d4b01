# LL128 line format for the small-message mean (opt-in GDRAA_LL128=1): vr parity, the
# multi-process suite with it on (world 4), and config-5 sweeps LL vs LL128 at N=2,4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k ll128 > gpurun_out/m_vr.log 2>&1; echo vr=$?
GDRAA_LL128=1 timeout 1200 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/m_mp.log 2>&1; echo mp=$?
for N in 2 4; do
  for f in 0 1; do
    GDRAA_LL128=$f timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2996$N tools/sweep.py --graph --max-log2 23 > gpurun_out/m_sweep_n${N}_ll128_$f.jsonl 2> gpurun_out/m_sweep_n${N}_ll128_$f.err; echo sweep_n${N}_$f=$?
  done
done
tail -3 gpurun_out/m_vr.log; tail -3 gpurun_out/m_mp.log
