cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests/test_gpu_abi_r2.py tests/test_gpu_multirank.py -x -q > gpurun_out/r2c_tests.log 2>&1; echo "tests rc=$?"
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29531 bench.py --gpus 2 --steps 2 --warmup 3 --workload C4-float --no-cpu-baseline --no-e2e --no-clocks > gpurun_out/r2c_bench2.json 2> gpurun_out/r2c_bench2.err; echo "bench2 rc=$?"
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29532 bench.py --gpus 2 --steps 2 --warmup 3 --workload C4-float --no-cpu-baseline --no-e2e --no-clocks --weak > gpurun_out/r2c_bench2w.json 2> gpurun_out/r2c_bench2w.err; echo "bench2 weak rc=$?"
