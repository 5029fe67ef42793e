cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
timeout 900 python -m pytest tests/test_gpu_hnodes.py tests/test_gpu_parity.py -x -q > gpurun_out/ab14_tests.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/ab14_tests.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in new head new head d8 d5; do
  unset UVD_LIB UVD_HDEPTH
  case $v in head) export UVD_LIB=$L/libuvd_head.so;; d8) export UVD_HDEPTH=8;; d5) export UVD_HDEPTH=5;; esac
  timeout 600 $B > gpurun_out/ab14_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
