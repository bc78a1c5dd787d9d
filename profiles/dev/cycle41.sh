# Gcell-upd/s vs N at 256^3 (data-dependent speed? subnormal tail), packed vs scalar fp32
L=paper_2509_15744_b200/_lib
for n in 256 1024 2048 256 1024 2048; do for lib in libwaveb200.so pk0.so; do
  WAVEB200_LIB=$L/$lib timeout 300 python bench.py --n-steps $n --steps 3 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('N $n $lib', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
