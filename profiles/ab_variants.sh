#!/bin/bash
# A/B of kernel build variants on the GPU box (dev): the default library runs
# the parity tests; every variant library runs a short bench.
#   profiles/ab_variants.sh <tag> var1.so var2.so ...
tag=$1; shift
out=gpurun_out
timeout 900 python -m pytest tests -q -m gpu --maxfail=5 > $out/${tag}_tests.log 2>&1; echo "tests rc $?"; tail -3 $out/${tag}_tests.log
for lib in default "$@"; do
  if [ "$lib" = default ]; then env_lib=""; else env_lib="paper_2509_15744_b200/_lib/$lib"; fi
  WAVEB200_LIB=$env_lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $out/${tag}_${lib}.json 2> $out/${tag}_${lib}.err
  python - "$out/${tag}_${lib}.json" "$lib" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(f"{sys.argv[2]:>12}: value {d['value']:.1f}  launch {d['roofline']['mean_launch_ms']*1e3:.1f} us  e2e {d['e2e']['value']:.1f}")
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
