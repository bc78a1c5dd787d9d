# next-block L2 prefetch off (np0) vs default, more repetitions; 256^3, 512^3, 1024^3, C5 slab
L=paper_2509_15744_b200/_lib
for i in 1 2 3; do for lib in libwaveb200.so np0.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
for i in 1 2; do for lib in libwaveb200.so np0.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --grid 512 --n-steps 256 --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('512 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
for lib in libwaveb200.so np0.so libwaveb200.so np0.so; do
  WAVEB200_LIB=$L/$lib timeout 600 python bench.py --grid 1024 --n-steps 32 --steps 2 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('1024 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done
for lib in libwaveb200.so np0.so; do
  WAVEB200_LIB=$L/$lib timeout 600 python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('c5 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done
