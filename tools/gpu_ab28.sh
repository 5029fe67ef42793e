cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in 2 4 1 2 4 8; do
  export UVD_LAMP_CAP=$v
  timeout 600 $B > gpurun_out/ab28_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
