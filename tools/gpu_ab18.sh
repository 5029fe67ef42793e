cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in na head na head na head; do
  unset UVD_LIB
  case $v in head) export UVD_LIB=$L/libuvd_head.so;; esac
  timeout 600 $B > gpurun_out/ab18_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
