# compute-sanitizer over every kernel (single GPU, virtual ranks) + fault tests (N=2)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for k in lsu tma; do
  for ll in default off; do
    if [ $ll = off ]; then export GDRAA_LL_MAX_BYTES=0; else unset GDRAA_LL_MAX_BYTES; fi
    GDRAA_KERNEL=$k timeout 900 $CS --tool memcheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_memcheck_${k}_ll$ll.log 2>&1; echo memcheck_${k}_ll$ll=$?
  done
done
unset GDRAA_LL_MAX_BYTES
GDRAA_KERNEL=tma GDRAA_LL_MAX_BYTES=0 timeout 900 $CS --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_racecheck_tma.log 2>&1; echo racecheck_tma=$?
GDRAA_KERNEL=tma GDRAA_LL_MAX_BYTES=0 timeout 900 $CS --tool synccheck --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/san_synccheck_tma.log 2>&1; echo synccheck_tma=$?
timeout 900 python -m pytest tests/test_multigpu_faults.py -q > gpurun_out/san_faults.log 2>&1; echo faults=$?
tail -3 gpurun_out/san_*.log
