# full-size multi-process parity (sampled windows) at N = visible GPUs
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e7_build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -x -k full_size > gpurun_out/e7_full_n$N.log 2>&1; echo full=$?
tail -3 gpurun_out/e7_full_n$N.log
