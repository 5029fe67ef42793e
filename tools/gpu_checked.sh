cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export UVD_LIB=$PWD/paper_2103_14137_b200/libuvd_checked.so
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fixups.py tests/test_gpu_hnodes.py tests/test_gpu_order.py tests/test_gpu_area.py tests/test_gpu_abi_r2.py -x -q > gpurun_out/checked_tests.log 2>&1; echo "checked tests rc=$?"; tail -2 gpurun_out/checked_tests.log
timeout 900 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/checked_c5.json 2>&1; echo "checked C5 bench rc=$?"; tail -c 300 gpurun_out/checked_c5.json
timeout 900 python bench.py --workload C4-tower --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/checked_c4t.json 2>&1; echo "checked C4-tower bench rc=$?"
