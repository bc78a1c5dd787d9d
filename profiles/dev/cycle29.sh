# 2D: r1 vs current vs 32-bit offsets vs lean (32-bit, no chain / peer-store code); 3D 256^3 current vs 32-bit
L=paper_2509_15744_b200/_lib
for i in 1 2; do
  echo "== r1"; (cd r1tree && timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell)
  echo "== r2"; timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
  echo "== off32"; WAVEB200_LIB=$L/off32.so timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
  echo "== lean"; WAVEB200_LIB=$L/lean.so timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell
done
for lib in libwaveb200.so off32.so libwaveb200.so off32.so; do WAVEB200_LIB=$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256', '$lib', round(d['value'],1), d['clocks']['sm_mhz'])"; done
