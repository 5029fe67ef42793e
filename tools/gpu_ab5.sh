cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py tests/test_gpu_fixups.py tests/test_gpu_vantage_pins.py -x -q > gpurun_out/ab5_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for f in 1 0 1 0; do UVD_FREE=$f timeout 600 $B > gpurun_out/ab5_c5_f$f.$RANDOM.json 2>&1; echo "f$f rc=$?"; done
for f in 1 0; do UVD_FREE=$f timeout 600 $B --workload C4-float > gpurun_out/ab5_c4_f$f.json 2>&1; echo "c4 f$f rc=$?"; done
for f in 1 0; do UVD_FREE=$f timeout 600 $B --workload C4-tower > gpurun_out/ab5_c4t_f$f.json 2>&1; echo "c4t f$f rc=$?"; done
