# round 2, call 27 (1 GPU): the C-ABI programs (virtual ranks; job server + 2 forked ranks).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/k_build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_c_abi.py -m gpu -v > gpurun_out/k_pytest.log 2>&1; echo pytest=$?
tail -12 gpurun_out/k_pytest.log
