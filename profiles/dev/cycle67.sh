# cluster_reg: per-warp mbarrier dataflow instead of the per-step CTA barrier
# then ncu of one fp32 cluster sweep launch
out=gpurun_out
timeout 600 python -m pytest tests/test_two_step_gpu.py -q -k "cluster or graph" > $out/c67_tests.log 2>&1; echo "tests rc $?"; tail -3 $out/c67_tests.log
for mode in "WB_CLUSTER=1" "WB_CLUSTER=1 WB_CR_PC=1" "WB_CLUSTER=0"; do
  echo "== $mode"; env $mode timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep C1
done
WB_CLUSTER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster_reg -s 2 -c 1 -o /tmp/c67 python profiles/dev/c1_rate.py > $out/c67_ncu.log 2>&1; echo "ncu rc $?"
python profiles/analyze_ncu.py /tmp/c67.ncu-rep > $out/c67_ncu_summary.txt 2>&1; cat $out/c67_ncu_summary.txt
ncu -i /tmp/c67.ncu-rep --page raw --csv > $out/c67_ncu_raw.csv 2>/dev/null
ncu -i /tmp/c67.ncu-rep --page source --csv --print-source sass > $out/c67_ncu_sass.csv 2>/dev/null
