cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_assemble_lane -c 1 -o gpurun_out/r02_k_assemble_free python tools/profile_assemble.py C5 512 1 > gpurun_out/prof_full.log 2>&1; echo "full rc=$?"
timeout 1500 ncu --nvtx --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_nvtx.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > gpurun_out/prof_nvtx.log 2>&1; echo "nvtx rc=$?"
