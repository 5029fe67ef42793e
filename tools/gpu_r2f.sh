cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_abi_r2.py tests/test_gpu_parity.py tests/test_gpu_hnodes.py -x -q > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2f_tests.log
timeout 1500 python tools/parity_sample.py gpurun_out/parity_r02_final.json > gpurun_out/r2f_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/r2f_parity.log | cut -c1-400
