cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_hnodes.py -x -q > gpurun_out/ab12_tests.log 2>&1; echo "hnode tests rc=$?"
tail -3 gpurun_out/ab12_tests.log
timeout 900 python tools/hnode_check.py > gpurun_out/ab12_check.log 2>&1; echo "check rc=$?"
cat gpurun_out/ab12_check.log | tail -5
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity"
for v in on off on off d4 d8 d10; do
  unset UVD_HDEPTH; export UVD_HNODES=1
  case $v in off) export UVD_HNODES=0;; d4) export UVD_HDEPTH=4;; d8) export UVD_HDEPTH=8;; d10) export UVD_HDEPTH=10;; esac
  timeout 600 $B > gpurun_out/ab12_c5_$v.$RANDOM.json 2>&1; echo "$v rc=$?"
done
unset UVD_HNODES UVD_HDEPTH
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py tests/test_gpu_fixups.py tests/test_gpu_area.py tests/test_gpu_abi_r2.py -x -q > gpurun_out/ab12_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/ab12_parity.log
