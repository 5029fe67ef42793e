cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fluence_multi.py tests/test_gpu_multirank.py tests/test_abi.py -x -q -rs > gpurun_out/r2i_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2i_tests.log
for i in 1 2; do timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/r2i_b$i.json 2>&1; echo "b$i rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gemv --csv --log-file gpurun_out/r2i_gemv.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
