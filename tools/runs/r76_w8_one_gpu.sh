# round 2, call 15 (1 GPU): world 8 on ONE GPU (eight processes / contexts, time-sliced):
# how long the opt-in oversubscribed test takes there, to decide whether the driver's
# one-GPU run can afford it by default.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/m_build.log 2>&1; echo build=$?
GDRAA_TEST_OVERSUBSCRIBE=1 timeout 900 python -m pytest tests/test_multigpu.py -k world8 -m gpu -v --durations=0 > gpurun_out/m_w8_1gpu.log 2>&1; echo w8=$?
tail -15 gpurun_out/m_w8_1gpu.log
