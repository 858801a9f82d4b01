# round 2, call 29 (2 GPUs): per-phase breakdown of the two-shot mean / sgd at mid sizes
# (1-64 MiB), where the alpha-beta fit's constant (19 us) exceeds the barrier constant.
set -x; mkdir -p gpurun_out
for L in 262144 1048576 2097152 4194304 16777216; do
  for mode in mean sgd; do
    GDRAA_LL_MAX_BYTES=0 GDRAA_LL_SGD_MAX_BYTES=0 timeout 120 tools/tune 2 $L f32 $mode 200 lib >> gpurun_out/p_phases_n2.jsonl 2>> gpurun_out/p_phases_n2.err
    echo L=$L $mode rc=$?
  done
done
cut -c1-400 gpurun_out/p_phases_n2.jsonl
