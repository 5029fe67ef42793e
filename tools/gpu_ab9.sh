cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in new prev new prev; do
  if [ $v = prev ]; then export UVD_LIB=$PWD/paper_2103_14137_b200/libuvd_prev.so; else unset UVD_LIB; fi
  timeout 600 $B > gpurun_out/ab9_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
unset UVD_LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py tests/test_gpu_fixups.py -x -q > gpurun_out/ab9_tests.log 2>&1; echo "tests rc=$?"
