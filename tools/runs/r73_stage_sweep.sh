# round 2, call 12 (4 GPUs): TMA ring geometry re-swept with the per-CTA fence: stage
# budget (chunk size) x depth for fp32 sgd at N = 2 and 4 and bf16 _mp at N = 2 and 4.
set -x; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -I include -o tools/tune tools/tune.cu -lcuda; echo nvcc=$?
L50=25557032
{
./tools/tune 2 $L50 f32 sgd 50 stage
./tools/tune 4 $L50 f32 sgd 50 stage
./tools/tune 2 $L50 bf16 mp 50 stage
./tools/tune 4 $L50 bf16 mp 50 stage
} > gpurun_out/l_tune_stage.jsonl 2> gpurun_out/l_tune_stage.err; echo tune=$?
set +x
python - <<'PY'
import json
for l in open("gpurun_out/l_tune_stage.jsonl"):
    d = json.loads(l); print(d["world"], d["dtype"], d["mode"], d["shape"], d["us"], d["phase_us"]["data_first_cta"], d["phase_us"]["cta_spread"])
PY
