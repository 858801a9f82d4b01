# round 2, first GPU call (4 GPUs): smoke, full GPU suite at world 4 (incl. the new
# vr range / done-flag / gated tests), bench N=1 and the self-launched N=2/4 form the
# driver uses, and the exit-fence A/B (per thread vs per CTA) at N=2/4, r50 and r50bf16mp.
set -x; mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/a_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/a_pytest_n4.log 2>&1; echo pytest=$?
tail -5 gpurun_out/a_pytest_n4.log
timeout 600 python bench.py > gpurun_out/a_bench_n1.json 2> gpurun_out/a_bench_n1.err; echo bench1=$?
for N in 2 4; do
  timeout 600 python3 bench.py --gpus $N > gpurun_out/a_bench_n$N.json 2> gpurun_out/a_bench_n$N.err; echo bench$N=$?
done
for rep in 1 2; do
for N in 2 4; do
  for cfg in r50 r50bf16mp; do
    for f in thread cta; do
      GDRAA_EXIT_FENCE=$f timeout 600 python bench.py --gpus $N --config $cfg --no-nccl --e2e-steps 3 \
        > gpurun_out/a_fence_${f}_n${N}_${cfg}_${rep}.json 2> gpurun_out/a_fence_${f}_n${N}_${cfg}_${rep}.err
      echo fence $f N=$N $cfg rep=$rep rc=$?
    done
  done
done
done
