# two-step kernel feature levels (T2_BASE / T2_CHAIN / T2_FULL): GPU suite, 2D rates, 256^3 bench
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c30_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c30_tests.log
for i in 1 2; do
  echo "== r1"; (cd r1tree && timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell)
  echo "== r2"; timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
done
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256', round(d['value'],1), d['clocks']['sm_mhz'])"; done
