# 2D C1 / C3-2D: round-1 build (r1tree) vs current, same box
for i in 1 2; do
  echo "== r1"; (cd r1tree && timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell)
  echo "== r2"; timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
