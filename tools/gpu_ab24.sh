cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
for v in 128 64 256; do
  unset UVD_LIB; [ $v != 128 ] && export UVD_LIB=$L/libuvd_ft$v.so
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_front_radius|k_fixup_collect|k_sah_split|k_lamp_radius" --csv --log-file gpurun_out/ab24_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > /dev/null 2>&1; echo "$v rc=$?"
done
