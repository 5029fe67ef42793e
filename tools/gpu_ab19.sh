cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_abi_r2.py tests/test_gpu_hnodes.py -x -q > gpurun_out/ab19_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab19_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in pack head pack head pack head; do
  unset UVD_LIB
  case $v in head) export UVD_LIB=$L/libuvd_head.so;; esac
  timeout 600 $B > gpurun_out/ab19_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
