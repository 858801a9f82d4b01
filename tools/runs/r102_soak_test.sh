# round 2, call 41 (1 GPU): the short soak test with time-sliced ranks on one GPU.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sk_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -v -k soak > gpurun_out/sk_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/sk_pytest.log
