cd $GRAFT_REPO_ROOT
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for c in 0.05 0.15; do UVD_FREE_CAP=$c timeout 600 $B > gpurun_out/ab8_c5_cap$c.json 2>&1; echo "cap$c rc=$?"; done
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/ab8_all_tests.log 2>&1; echo "all tests rc=$?"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/ab8_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/ab8_bench.json 2> gpurun_out/ab8_bench.err; echo "bench rc=$?"
