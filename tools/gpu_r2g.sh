cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py tests/test_gpu_hnodes.py tests/test_gpu_fixups.py -x -q > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2g_tests.log
timeout 1200 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
