# LL128 diagnosis with the failing test's exact call sequence (vr N=4, 8), and the
# pytest case itself once more for comparison
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e_build.log 2>&1
GDRAA_LL128=auto timeout 300 python tools/ll128_diag.py 4 5 --full > gpurun_out/e_n4.jsonl 2> gpurun_out/e_n4.err; echo n4=$?
GDRAA_LL128=auto timeout 300 python tools/ll128_diag.py 8 3 --full > gpurun_out/e_n8.jsonl 2> gpurun_out/e_n8.err; echo n8=$?
GDRAA_LL128=auto timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "test_vr_sgd_latency_path and False-f32" > gpurun_out/e_pytest.log 2>&1; echo pytest=$?
grep '"r[0-9]' gpurun_out/e_n4.jsonl gpurun_out/e_n8.jsonl | head -6; tail -3 gpurun_out/e_n4.err
