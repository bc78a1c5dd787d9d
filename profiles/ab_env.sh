#!/bin/bash
# A/B of runtime tuning knobs (dev): short bench per environment setting.
#   profiles/ab_env.sh <tag> "VAR=a" "VAR=b" ...
tag=$1; shift
out=gpurun_out
for setting in "" "$@"; do
  name=${setting:-default}
  env $setting timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > $out/${tag}_${name}.json 2> $out/${tag}_${name}.err
  python - "$out/${tag}_${name}.json" "$name" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[1]))
    print(f"{sys.argv[2]:>14}: value {d['value']:.1f}  launch {d['roofline']['mean_launch_ms']*1e3:.1f} us  e2e {d['e2e']['value']:.1f}")
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
