# N=2: why is the c1 bench slow through the LL-SGD path? + fair multicast probe
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e4_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mc_probe tools/mc_probe.cu -lcuda
timeout 300 ./tools/mc_probe 2 20000 > gpurun_out/e4_mc_probe_n2.jsonl 2>&1
run() { # name "ENV=.." "extra bench args"
  env $2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --config c1 --no-nccl --steps 200 $3 > gpurun_out/e4_c1_$1.json 2> gpurun_out/e4_c1_$1.err; echo $1=$?
}
run default "GDRAA_X=1" ""
run sets1 "GDRAA_X=1" "--sets 1"
run pdl0 "GDRAA_PDL=0" ""
run twoshot "GDRAA_LL_SGD_MAX_BYTES=0" ""
run ll1m "GDRAA_LL_SGD_MAX_BYTES=1048576" ""
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/sweep_sgd.py --min-log2 18 --max-log2 22 > gpurun_out/e4_sweep_sgd_eager.jsonl 2> gpurun_out/e4_sweep.err; echo sweep=$?
