cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
for v in 12 8 6 4; do
  unset UVD_LIB; [ $v != 12 ] && export UVD_LIB=$L/libuvd_fix$v.so
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fixup_run --csv --log-file gpurun_out/ab22_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > /dev/null 2>&1; echo "$v rc=$?"
done
