# round 2, call 26 (1 GPU): config-5 sizes through the multi-process path (time-sliced
# world 2) and the bucketed test with the one-launch-per-streamed-set assertion.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c_build.log 2>&1; echo build=$?
GDRAA_TIMEOUT_MS=30000 timeout 1200 python -m pytest tests/test_multigpu.py -m gpu -q -k "config5 or bucketed" --durations=5 > gpurun_out/c_pytest.log 2>&1; echo pytest=$?
tail -12 gpurun_out/c_pytest.log
