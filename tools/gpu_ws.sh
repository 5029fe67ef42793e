cd $GRAFT_REPO_ROOT
python tools/walkstats.py C5 3000 > gpurun_out/ws_c5.json 2> gpurun_out/ws_c5.err; echo "c5 rc=$?"
python tools/walkstats.py C4-float 3000 > gpurun_out/ws_c4.json 2> gpurun_out/ws_c4.err; echo "c4 rc=$?"
