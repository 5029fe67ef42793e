cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_hnodes.py tests/test_gpu_parity.py tests/test_gpu_abi_r2.py tests/test_gpu_bvh.py -x -q > gpurun_out/r2h_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/r2h_tests.log
UVD_TRACE_HOST=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/trace_bench2.json 2> gpurun_out/trace_host2.log; echo "trace rc=$?"
for i in 1 2 3; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r2h_b$i.json 2>&1; echo "b$i rc=$?"; done
