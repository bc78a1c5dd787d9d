# layer dispatch order: default vs always top-first (WB_T2_ZREV=2): TATO 192^3 phases, C3 3D, 256^3 bench
for i in 1 2; do for z in 0 2; do
  echo "== zrev $z"; WB_T2_ZREV=$z python profiles/dev/tato_phases.py | tail -3
  WB_T2_ZREV=$z timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256', round(d['value'],1), d['clocks']['sm_mhz'])"
done; done
