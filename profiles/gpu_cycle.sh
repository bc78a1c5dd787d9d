#!/bin/bash
# One build-measure cycle on the GPU box (run under gpurun from the repo root):
#   parity tests, a short bench, then ncu on the fused step kernel (summarised
#   on the box; the .ncu-rep is dropped to stay under gpurun's 64 MiB return).
#   profiles/gpu_cycle.sh <tag> [bench args...]
tag=${1:-cycle}; shift
out=gpurun_out
timeout 900 python -m pytest tests -q -m gpu --maxfail=10 ${TESTS:-} > $out/${tag}_tests.log 2>&1; echo "tests rc $?"; tail -15 $out/${tag}_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-sample-steps 4 "$@" > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench rc $?"
python profiles/profile_step.py > $out/${tag}_prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-step2?_kernel} -s 10 -c 1 \
      -o /tmp/${tag}_step python profiles/profile_step.py > $out/${tag}_ncu.log 2>&1; echo "ncu rc $?"
if [ -f /tmp/${tag}_step.ncu-rep ]; then
  python profiles/analyze_ncu.py /tmp/${tag}_step.ncu-rep > $out/${tag}_ncu_summary.txt 2>&1
  ncu -i /tmp/${tag}_step.ncu-rep --page raw --csv > $out/${tag}_ncu_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_step.ncu-rep --page source --csv --print-source sass > $out/${tag}_ncu_sass.csv 2>/dev/null
  ncu -i /tmp/${tag}_step.ncu-rep --page source --csv --print-source cuda > $out/${tag}_ncu_src.csv 2>$out/${tag}_ncu_src.err
  cat $out/${tag}_ncu_summary.txt
fi
