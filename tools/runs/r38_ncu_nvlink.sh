# OUTCOME (r38): NVML field values return NOT_SUPPORTED and GPM sampling fails on this
# pool; ncu on rank 0 of the 2-process bench (via a torchrun --no-python wrapper that ran
# ncu only when RANK=0, since removed) profiled no kernel and hung until the 1800 s limit.
# NVLink bytes per launch for N >= 2 therefore stay algorithmic only.
# NVLink (and DRAM) bytes per launch of the fused step at N=2 from ncu on rank 0 only,
# single-pass metric sets; the calibration tool again (fields + GPM, non-fatal)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1
timeout 300 python tools/nvlink_counters.py > gpurun_out/x_calib.jsonl 2> gpurun_out/x_calib.err; echo calib=$?
export GDRAA_TIMEOUT_MS=60000
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum
for c in r50 r50bf16mp; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29713 --no-python tools/ncu_rank0.sh --metrics $M --clock-control none -k regex:gdraa -s 25 -c 3 --csv --log-file gpurun_out/x_ncu_nvl_n2_$c.csv -- python bench.py --gpus 2 --config $c --steps 30 --warmup 20 --e2e-steps 3 --no-cpu-baseline --no-nccl --no-nvlink-counters > gpurun_out/x_ncu_nvl_n2_$c.log 2>&1; echo ncu_nvl_$c=$?
done
M2=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29714 --no-python tools/ncu_rank0.sh --metrics $M2 --clock-control none -k regex:gdraa -s 25 -c 3 --csv --log-file gpurun_out/x_ncu_dram_n2_r50.csv -- python bench.py --gpus 2 --config r50 --steps 30 --warmup 20 --e2e-steps 3 --no-cpu-baseline --no-nccl --no-nvlink-counters > gpurun_out/x_ncu_dram_n2_r50.log 2>&1; echo ncu_dram=$?
cat gpurun_out/x_calib.jsonl; grep -v "^==PROF==" gpurun_out/x_ncu_nvl_n2_r50.csv | head -30; tail -5 gpurun_out/x_ncu_nvl_n2_r50.log
