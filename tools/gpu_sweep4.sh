cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=$PWD/paper_2103_14137_b200
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
run() { timeout 600 $B > gpurun_out/sw4_$1.$RANDOM.json 2>&1; echo "$1 rc=$?"; }
for i in 1 2; do
run base
UVD_HDEPTH=5 run h5
UVD_HDEPTH=7 run h7
UVD_HDEPTH=8 run h8
UVD_LIB=$L/libuvd_bins64.so run bins64
UVD_FREE_CAP=0.15 run cap015
done
