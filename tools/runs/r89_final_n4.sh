# round 2, call 28 (4 GPUs): the final tree at world 4 -- smoke (with the streamed set),
# GPU suite, bench R50 at N = 4 / 2, and NEXT-3 overlap vs an NCCL+torch reference.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo smoke=$?
tail -1 gpurun_out/q_smoke.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/q_pytest_n4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/q_pytest_n4.log
for N in 4 2; do
  timeout 600 python3 bench.py --gpus $N --e2e-steps 10 > gpurun_out/q_bench_n${N}_r50.json 2> gpurun_out/q_bench_n${N}_r50.err; echo bench N=$N rc=$?
done
P=30300
for N in 2 4; do
for bg in "4 3072" "8 2304"; do
  set -- $bg; b=$1; gm=$2
  for mode in plain0 st64 nccl; do
    P=$((P+1))
    case $mode in plain0) arg="";; st64) arg="--streamed 64";; nccl) arg="--nccl";; esac
    tag=n${N}_b${b}_${mode}
    GDRAA_TIMEOUT_MS=20000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P \
      tools/overlap.py --buckets $b --gemm $gm $arg > gpurun_out/q_overlap_$tag.json 2> gpurun_out/q_overlap_$tag.err
    echo overlap $tag rc=$?
  done
done
done
