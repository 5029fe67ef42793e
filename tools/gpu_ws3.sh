cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/walkstats.py C5 600 > gpurun_out/ws7_c5.json 2> gpurun_out/ws7_c5.err; echo "c5 rc=$?"
timeout 900 python tools/walkstats.py C4-float 600 > gpurun_out/ws7_c4.json 2> gpurun_out/ws7_c4.err; echo "c4 rc=$?"
