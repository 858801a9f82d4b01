# GPU suite after the init-release refactor and the bench contract tests (4 GPUs), smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/t_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest_n4.log 2>&1; echo pytest=$?
tail -3 gpurun_out/t_pytest_n4.log; tail -1 gpurun_out/t_smoke.log
