cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in base ends base ends; do
  unset UVD_LIB; [ $v = ends ] && export UVD_LIB=$L/libuvd_ends.so
  timeout 600 $B > gpurun_out/ab27_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
