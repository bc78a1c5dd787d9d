#!/bin/bash
# A/B of the two-step z-chunk count at a larger grid (dev):
#   profiles/dev/ab_nz_grid.sh <grid> <n_steps> nz1 nz2 ...   (0 = the model's choice)
grid=$1; nsteps=$2; shift 2
for nz in "$@"; do
  if [ "$nz" = 0 ]; then envs=""; else envs="WB_T2_NZ=$nz"; fi
  env $envs timeout 600 python bench.py --grid $grid --n-steps $nsteps --steps 3 --warmup 3 --no-cpu \
      > gpurun_out/nz_${grid}_${nz}.json 2> gpurun_out/nz_${grid}_${nz}.err
  python -c "
import json,sys
d=json.load(open('gpurun_out/nz_${grid}_${nz}.json'))
print('grid $grid nz $nz: value %.1f launch %.1f us clocks %s' % (d['value'], d['roofline']['mean_launch_ms']*1e3, d['clocks']['sm_mhz']))" || tail -3 gpurun_out/nz_${grid}_${nz}.err
done
