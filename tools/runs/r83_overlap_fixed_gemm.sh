# round 2, call 22 (2 GPUs): NEXT-3 overlap with a FIXED backward (same GEMMs for every
# mode), per-call buckets (full grid / 32 CTAs), bucket set (32), streamed (32/48/64/96).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/y_build.log 2>&1; echo build=$?
P=30150
for rep in 1 2; do
for bg in "4 3072" "8 2304"; do
  set -- $bg; b=$1; gm=$2
  for mode in plain0 plain32 set32 st32 st48 st64 st96; do
    P=$((P+1))
    cap=0
    case $mode in plain0) arg="";; plain32) arg=""; cap=32;; set32) arg="--set"; cap=32;; st32) arg="--streamed 32";; st48) arg="--streamed 48";; st64) arg="--streamed 64";; st96) arg="--streamed 96";; esac
    tag=b${b}_${mode}_$rep
    GDRAA_TIMEOUT_MS=20000 GDRAA_MAX_CTAS=$cap timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P \
      tools/overlap.py --buckets $b --gemm $gm $arg > gpurun_out/y_overlap_n2_$tag.json 2> gpurun_out/y_overlap_n2_$tag.err
    echo overlap $tag rc=$?
  done
done
done
