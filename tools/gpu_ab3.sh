cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_order.py -x -q > gpurun_out/ab4_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for g in 0 128 512 0 128 512; do UVD_ASM_GROUP=$g timeout 600 $B > gpurun_out/ab4_c5_g$g.$RANDOM.json 2>&1; echo "g$g rc=$?"; done
for g in 0 128; do UVD_ASM_GROUP=$g timeout 600 $B --workload C4-float > gpurun_out/ab4_c4_g$g.json 2>&1; echo "c4 g$g rc=$?"; done
