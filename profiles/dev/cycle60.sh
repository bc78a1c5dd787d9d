# Register-resident cluster engine (cluster_reg.cuh): bitwise tests, then C1 rates
# with the engine on (WB_CLUSTER=1), off (two-step launches), and the old smem engine
out=gpurun_out
timeout 600 python -m pytest tests/test_two_step_gpu.py -q -k cluster -x > $out/c60_tests.log 2>&1; echo "tests rc $?"; tail -5 $out/c60_tests.log
for mode in "WB_CLUSTER=1" "WB_CLUSTER=0" "WB_CLUSTER=1 WB_CLUSTER_ENGINE=smem" "WB_CLUSTER=1"; do
  echo "== $mode"; env $mode timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep C1
done
