# locate the LL128 SGD transition fault: vr N=4 and N=8, LL steps then LL128 steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/d_build.log 2>&1
GDRAA_LL128=auto timeout 300 python tools/ll128_diag.py 4 5 > gpurun_out/d_n4.jsonl 2> gpurun_out/d_n4.err; echo n4=$?
GDRAA_LL128=auto timeout 300 python tools/ll128_diag.py 8 3 > gpurun_out/d_n8.jsonl 2> gpurun_out/d_n8.err; echo n8=$?
grep -c '"r0"' gpurun_out/d_n4.jsonl; grep '"r' gpurun_out/d_n4.jsonl | head -5; tail -3 gpurun_out/d_n4.err
