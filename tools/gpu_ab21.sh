cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
timeout 1200 python -m pytest tests/test_gpu_fixups.py tests/test_gpu_parity.py tests/test_gpu_area.py -x -q > gpurun_out/ab21_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab21_tests.log
for v in new head; do
  unset UVD_LIB; [ $v = head ] && export UVD_LIB=$L/libuvd_head.so
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fixup_run --csv --log-file gpurun_out/ab21_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > /dev/null 2>&1; echo "$v rc=$?"
done
