cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2m_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2m_all_tests.log 2>&1; echo "all tests rc=$?"
tail -2 gpurun_out/r2m_all_tests.log
timeout 1200 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo "bench rc=$?"
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in noh base noh base; do
  unset UVD_HNODES; [ $v = noh ] && export UVD_HNODES=0
  timeout 600 $B > gpurun_out/r2m_ab_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
