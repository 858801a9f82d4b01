# round 2, call 37 (2 GPUs): the final tree's GPU suite at world 2.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/y2_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/y2_pytest_n2.log 2>&1; echo pytest=$?
tail -3 gpurun_out/y2_pytest_n2.log
