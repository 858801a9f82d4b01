# round 2, call 25 (1 GPU): bucket sets with calls on two streams (vr).
set -x; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/w_build.log 2>&1; echo build=$?
GDRAA_TIMEOUT_MS=20000 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "bucket_set" > gpurun_out/w_pytest_sets.log 2>&1; echo pytest=$?
tail -5 gpurun_out/w_pytest_sets.log
