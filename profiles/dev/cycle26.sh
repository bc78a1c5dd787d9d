# 2D C1: round-1 build vs current (64-bit offsets) vs current with 32-bit offsets
for i in 1 2; do
  echo "== r1"; (cd r1tree && timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell)
  echo "== r2"; timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
  echo "== r2 off32"; WAVEB200_LIB=paper_2509_15744_b200/_lib/off32.so timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
done
WAVEB200_LIB=paper_2509_15744_b200/_lib/off32.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:step2 --launch-skip 9700 -c 60 --csv python profiles/dev/c1_once.py > gpurun_out/c26_off32.csv 2>&1
