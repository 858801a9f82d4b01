# after fixing the thresholds at init: multi-process + fault tests, the two sweeps
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e9_build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_multigpu_faults.py -q -x > gpurun_out/e9_mp_n$N.log 2>&1; echo mp=$?
for p in ll two_shot; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 tools/sweep_sgd.py --graph --path $p --max-log2 25 > gpurun_out/e9_sweep_sgd_n${N}_$p.jsonl 2> gpurun_out/e9_sweep_$p.err; echo sweep_$p=$?
done
tail -3 gpurun_out/e9_mp_n$N.log
