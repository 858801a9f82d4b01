# round 2, call 21 (2 GPUs): streamed sets whose kernel starts only when the first bucket
# is final; overlap at 32 CTAs (per-call, set, streamed 16/32/64) and comm-only at 148.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1; echo build=$?
GDRAA_TIMEOUT_MS=20000 timeout 900 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -m gpu -x -q -k "bucket" > gpurun_out/x_pytest_bucket.log 2>&1; echo pytest_bucket=$?
tail -3 gpurun_out/x_pytest_bucket.log
P=30050
for rep in 1 2; do
for b in 4 8; do
  for mode in plain32 set32 st16 st32 st64 co_plain co_st148; do
    P=$((P+1))
    cap=0
    case $mode in plain32) arg=""; cap=32;; set32) arg="--set"; cap=32;; st16) arg="--streamed 16";; st32) arg="--streamed 32";; st64) arg="--streamed 64";; co_plain) arg="--comm-only";; co_st148) arg="--comm-only --streamed 148";; esac
    tag=b${b}_${mode}_$rep
    GDRAA_TIMEOUT_MS=20000 GDRAA_MAX_CTAS=$cap timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
      tools/overlap.py --buckets $b $arg > gpurun_out/x_overlap_n2_$tag.json 2> gpurun_out/x_overlap_n2_$tag.err
    echo overlap $tag rc=$?
  done
done
done
