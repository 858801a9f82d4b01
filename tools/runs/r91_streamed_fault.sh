# round 2, call 30 (1 GPU): the persistent bucket-set kernel's timeout path.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_multigpu_faults.py -m gpu -v > gpurun_out/h_pytest.log 2>&1; echo pytest=$?
tail -12 gpurun_out/h_pytest.log
