cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2j_all_tests.log 2>&1; echo "all tests rc=$?"
tail -3 gpurun_out/r2j_all_tests.log
timeout 1200 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/r2j_bench.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_assemble_lane -c 1 -o gpurun_out/r02_k_assemble_v5 python tools/profile_assemble.py C5 512 1 > gpurun_out/r2j_prof_full.log 2>&1; echo "full rc=$?"
timeout 1500 ncu --nvtx --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-clocks > gpurun_out/r2j_prof_nvtx.log 2>&1; echo "nvtx rc=$?"
