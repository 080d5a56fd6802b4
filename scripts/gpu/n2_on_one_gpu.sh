# N = 2 code path of bench.py on one GPU (gloo collectives, both ranks on GPU 0): exercises
# the weak-scaling rows, basis broadcast, max-over-ranks timing, e2e barriers, the reference arm.
export LPD_BENCH_ONE_GPU_TEST=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --rows 65536 > gpurun_out/n2.json 2> gpurun_out/n2.err; echo rc=$?; tail -3 gpurun_out/n2.err; cat gpurun_out/n2.json | cut -c1-600
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --rows 8192 > gpurun_out/n2ref.json 2> gpurun_out/n2ref.err; echo rc=$?; tail -3 gpurun_out/n2ref.err; cat gpurun_out/n2ref.json | cut -c1-300
