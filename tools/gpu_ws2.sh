cd $GRAFT_REPO_ROOT
WALKSTATS_DEFS="-DMARCH=0" python tools/walkstats.py C5 1000 > gpurun_out/ws4_c5.json 2> gpurun_out/ws4_c5.err; echo "rc=$?"
