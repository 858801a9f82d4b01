# round 2, call 19 (1 GPU): streamed bucket sets over virtual ranks (first run).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1; echo build=$?
GDRAA_TIMEOUT_MS=20000 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamed" > gpurun_out/t_streamed_vr.log 2>&1; echo streamed=$?
tail -30 gpurun_out/t_streamed_vr.log
