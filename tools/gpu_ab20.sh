cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for v in pairs base pairs base; do
  case $v in pairs) export UVD_PAIRS=1;; base) export UVD_PAIRS=0;; esac
  timeout 600 $B > gpurun_out/ab20_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
