cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
run() { timeout 600 $B > gpurun_out/sw2_$1.$RANDOM.json 2>&1; echo "$1 rc=$?"; }
run base
UVD_ASM_SUPER=8 run super8
UVD_ASM_SUPER=10 run super10
UVD_ASM_SUPER=11 run super11
UVD_FREE_CAP=0.05 run cap005
UVD_FREE_CAP=0.2 run cap02
UVD_BVH=ploc run ploc
UVD_LIB=$L/libuvd_uvd_leaf_max1.so run leaf1
UVD_LIB=$L/libuvd_uvd_leaf_max3.so run leaf3
UVD_LIB=$L/libuvd_uvd_leaf_max4.so run leaf4
run base
