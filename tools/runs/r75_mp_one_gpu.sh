# round 2, call 14 (1 GPU): the multi-process tests with world 2 time-sliced on one GPU
# (tests.conftest.mp_world), as the driver's one-GPU round-end run will now execute them.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_multigpu_faults.py -m gpu -v --durations=0 > gpurun_out/m_mp1.log 2>&1; echo mp=$?
tail -40 gpurun_out/m_mp1.log
