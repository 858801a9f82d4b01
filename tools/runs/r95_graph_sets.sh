# round 2, call 34 (1 GPU): bucket sets captured into a CUDA graph; streamed sets refuse.
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/j_build.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -v -k "graph_capture" > gpurun_out/j_pytest.log 2>&1; echo pytest=$?
tail -8 gpurun_out/j_pytest.log
