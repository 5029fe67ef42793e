cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hnodes.py -x -q > gpurun_out/ab17_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/ab17_tests.log
timeout 900 python tools/hnode_check.py UVD_BEAM > gpurun_out/ab17_check.log 2>&1; echo "check rc=$?"
tail -3 gpurun_out/ab17_check.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in beam base beam base; do
  case $v in beam) export UVD_BEAM=1;; base) export UVD_BEAM=0;; esac
  timeout 600 $B > gpurun_out/ab17_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
