cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hnodes.py -x -q > gpurun_out/ab13_tests.log 2>&1; echo "node tests rc=$?"
tail -3 gpurun_out/ab13_tests.log
timeout 900 python tools/hnode_check.py UVD_QNODES > gpurun_out/ab13_check.log 2>&1; echo "check rc=$?"
tail -5 gpurun_out/ab13_check.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in q oct q oct; do
  case $v in q) export UVD_QNODES=1;; oct) export UVD_QNODES=0;; esac
  timeout 600 $B > gpurun_out/ab13_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
unset UVD_QNODES
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py tests/test_gpu_fixups.py tests/test_gpu_area.py tests/test_gpu_abi_r2.py -x -q > gpurun_out/ab13_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/ab13_parity.log
