cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for c in 0.1 0.25 0.5 1.0; do UVD_FREE_CAP=$c timeout 600 $B > gpurun_out/ab7_c5_cap$c.json 2>&1; echo "cap$c rc=$?"; done
