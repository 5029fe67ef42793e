cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q -s -k "fixup or abi_r2 or vantage_pins or static" > gpurun_out/r2a_new_tests.log 2>&1; echo "new tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_all_tests.log 2>&1; echo "all tests rc=$?"
