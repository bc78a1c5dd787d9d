# 2D: chained single-layer passes + staged cost sum; r1 vs current (64-bit) vs 32-bit offsets vs chain off
for i in 1 2; do
  echo "== r1"; (cd r1tree && timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell)
  echo "== r2"; timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
  echo "== r2 off32"; WAVEB200_LIB=paper_2509_15744_b200/_lib/off32.so timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
  echo "== r2 chain off"; WB_T2_CHAIN=0 timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
done
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_two_step_gpu.py tests/test_reference_loops_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
