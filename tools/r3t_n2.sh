# the N=2 bench path (view split, LoD broadcast, LPT training, fusion all-gather) with two ranks sharing the one GPU (gloo)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CS_BENCH_SHARED_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r3t_bench_n2_shared_gpu.log 2>&1; echo rc=$?
tail -1 gpurun_out/r3t_bench_n2_shared_gpu.log | cut -c1-600
CS_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r3t_bench_ref_n2.log 2>&1; echo rc=$?
tail -1 gpurun_out/r3t_bench_ref_n2.log | cut -c1-300
