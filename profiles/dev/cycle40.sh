# support bounding-box early-out A/B (bbox.so) vs sup_fc only (libwaveb200.so)
L=paper_2509_15744_b200/_lib
for i in 1 2; do for lib in libwaveb200.so bbox.so; do
  echo "== $lib"; WAVEB200_LIB=$L/$lib python profiles/dev/tato_phases.py | tail -3
  WAVEB200_LIB=$L/$lib timeout 600 python profiles/configs.py --only "C3" 2>&1 | grep gcell | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print(d['config'], d['precision'], round(d['gcell_upd_s'],1))"
done; done
