# two-step chunk count sweep at 192^3 (bench FWI grid, N = 600) with chained passes
for nz in 0 6 8 10 12 16 24 0; do
  WB_T2_NZ=$nz timeout 300 python bench.py --grid 192 --n-steps 600 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('192 nz $nz', round(d['value'],1), d['clocks']['sm_mhz'])"
done
for nz in 0 8 12 16 0; do
  WB_T2_NZ=$nz timeout 300 python bench.py --grid 256 --n-steps 256 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256 nz $nz', round(d['value'],1), d['clocks']['sm_mhz'])"
done
