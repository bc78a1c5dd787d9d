# chained-pass flag poll back-off: 32 / 128 (default) / 512 ns
L=paper_2509_15744_b200/_lib
for i in 1 2 3; do for lib in libwaveb200.so p32.so p512.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
for lib in libwaveb200.so p32.so p512.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --grid 192 --n-steps 600 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('192 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --grid 512 --n-steps 256 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('512 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done
