cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
run() { timeout 600 $B > gpurun_out/sw3_$1.$RANDOM.json 2>&1; echo "$1 rc=$?"; }
for i in 1 2 3; do
run base
UVD_ASM_SUPER=11 run s11
UVD_ASM_SUPER=12 run s12
UVD_ASM_SUPER=13 run s13
done
