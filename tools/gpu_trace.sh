cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
UVD_TRACE_HOST=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/trace_bench.json 2> gpurun_out/trace_host.log; echo "rc=$?"
