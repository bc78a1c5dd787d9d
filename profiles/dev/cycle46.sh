# L2 prefetch of the adjoint forces two planes ahead (WB_T2_FORCE_PREFETCH) A/B
L=paper_2509_15744_b200/_lib
timeout 1200 python -m pytest tests/test_two_step_gpu.py tests/test_parity_gpu.py tests/test_reference_loops_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do for lib in libwaveb200.so fp0.so; do
  echo "== $lib"; WAVEB200_LIB=$L/$lib python profiles/dev/tato_phases.py | tail -3
  WAVEB200_LIB=$L/$lib timeout 600 python profiles/configs.py --only "C3" 2>&1 | grep gcell | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['config'], d['precision'], round(d['gcell_upd_s'],1))"
done; done
for lib in libwaveb200.so fp0.so libwaveb200.so fp0.so; do WAVEB200_LIB=$L/$lib timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256 $lib', round(d['value'],1), d['clocks']['sm_mhz'])"; done
