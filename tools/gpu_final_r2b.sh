# final tree: GPU suite, smoke, the driver's bench command, and the torchrun launch path (1 rank)
mkdir -p gpurun_out/final2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final2/smoke.log
timeout 900 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; echo "bench rc=$?" >> gpurun_out/final2/bench.err
NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/final2/bench_torchrun.json 2> gpurun_out/final2/bench_torchrun.err; echo "torchrun rc=$?" >> gpurun_out/final2/bench_torchrun.err
tail -3 gpurun_out/final2/pytest_gpu.log; tail -2 gpurun_out/final2/smoke.log; tail -1 gpurun_out/final2/bench.err; tail -1 gpurun_out/final2/bench_torchrun.err
