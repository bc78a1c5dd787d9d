# L2 prefetch knobs under chained passes: next-block prefetch off (np0), prefetch distance 1 / 3 (default 2)
L=paper_2509_15744_b200/_lib
for i in 1 2 3; do for lib in libwaveb200.so np0.so pf1.so pf3.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
for lib in libwaveb200.so np0.so pf1.so pf3.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --grid 512 --n-steps 128 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('512 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done
