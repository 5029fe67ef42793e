cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
L=$PWD/paper_2103_14137_b200
for v in base probe base probe; do
  case $v in base) unset UVD_LIB;; probe) export UVD_LIB=$L/libuvd_probe.so;; esac
  timeout 600 $B > gpurun_out/ab11_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
