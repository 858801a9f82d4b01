# round 2, call 18 (1 GPU): the multi-process tests on one GPU with the bucket-set
# finalize test and config 4 at world 8 (full size, eight time-sliced processes).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1; echo build=$?
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_multigpu_faults.py -m gpu -v --durations=0 > gpurun_out/m_mp1b.log 2>&1; echo mp=$?
tail -40 gpurun_out/m_mp1b.log
