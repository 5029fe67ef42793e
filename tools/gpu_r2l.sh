cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in C4-float C4-tower; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/r2l_$w.json 2> gpurun_out/r2l_$w.err; echo "$w rc=$?"
done
