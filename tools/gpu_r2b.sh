cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2000 python -m pytest tests -m gpu -q -s -k "fixup or abi_r2 or vantage_pins or static or multirank" > gpurun_out/r2b_new_tests.log 2>&1; echo "new tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo "bench rc=$?"
timeout 1800 python tools/parity_sample.py gpurun_out/r2b_parity.json > gpurun_out/r2b_parity.log 2>&1; echo "parity rc=$?"
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/r2b_all_tests.log 2>&1; echo "all tests rc=$?"
