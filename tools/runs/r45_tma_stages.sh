# OUTCOME (r45): all variants within +-0.8%; the GDRAA_TMA_STAGES / GDRAA_TMA_PER_SM knobs
# existed only for this A/B (commit 51c0220) and were removed afterwards.
# A/B: TMA ring depth 4 (default, 128 KB smem: one CTA per SM) vs 3 stages (96 KB), the
# latter with the grid at 2 CTAs/SM or capped at 1/SM so the next call's CTAs (PDL) fit
# beside the running ones; N=2 and N=4, R50 and R101 fp32, graph-timed bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p_build.log 2>&1
run() {  # tag N config env...
  tag=$1; N=$2; c=$3; shift 3
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2995$N bench.py --gpus $N --config $c --no-cpu-baseline --no-nccl --e2e-steps 3 > gpurun_out/p_${tag}_n${N}_$c.json 2> gpurun_out/p_${tag}_n${N}_$c.err; echo ${tag}_n${N}_$c=$?
}
for N in 2 4; do
  for c in r50 r101; do
    run st4 $N $c GDRAA_TMA_STAGES=4
    run st3 $N $c GDRAA_TMA_STAGES=3
    run st3pm1 $N $c GDRAA_TMA_STAGES=3 GDRAA_TMA_PER_SM=1
    run st3pm1pdl0 $N $c GDRAA_TMA_STAGES=3 GDRAA_TMA_PER_SM=1 GDRAA_PDL=0
    run st4pdl0 $N $c GDRAA_TMA_STAGES=4 GDRAA_PDL=0
  done
done
