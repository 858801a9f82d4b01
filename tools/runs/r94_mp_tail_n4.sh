# round 2, call 33 (4 GPUs): end-game (tail chunk / tail prefetch depth) variants of the
# TMA kernel for the mixed-precision step and bf16 step at N = 4 (the kernel furthest
# below its roofline), twice interleaved.
set -x; mkdir -p gpurun_out
timeout 600 tools/tune 4 25557032 bf16 mp 100 tail > gpurun_out/t_tail_n4_mp.jsonl 2> gpurun_out/t_tail_n4_mp.err; echo mp=$?
timeout 600 tools/tune 4 25557032 f32 sgd 100 tail > gpurun_out/t_tail_n4_sgd.jsonl 2> gpurun_out/t_tail_n4_sgd.err; echo sgd=$?
cut -c1-330 gpurun_out/t_tail_n4_mp.jsonl
