cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
L=$PWD/paper_2103_14137_b200
for v in prev lean w20 w24 prev lean w20; do
  case $v in prev) export UVD_LIB=$L/libuvd_prev.so;; lean) unset UVD_LIB;; w20) export UVD_LIB=$L/libuvd_w20.so;; w24) export UVD_LIB=$L/libuvd_w24.so;; esac
  timeout 600 $B > gpurun_out/ab10_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
for v in prev w20; do
  case $v in prev) export UVD_LIB=$L/libuvd_prev.so;; w20) export UVD_LIB=$L/libuvd_w20.so;; esac
  timeout 600 $B --workload C4-float > gpurun_out/ab10_c4_$v.json 2>&1; echo "c4 $v rc=$?"
done
unset UVD_LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py tests/test_gpu_area.py -x -q > gpurun_out/ab10_tests.log 2>&1; echo "tests rc=$?"
