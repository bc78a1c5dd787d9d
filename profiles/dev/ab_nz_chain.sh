# A/B of the two-step chunk count with dataflow chaining (256^3 and 512^3 bench)
for g in 256 512; do
  for nz in 0 4 5 6 7 8 10 13 16; do
    WB_T2_NZ=$nz timeout 300 python bench.py --grid $g --steps 4 --warmup 3 --no-cpu --n-steps 256 > gpurun_out/nz_${g}_${nz}.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/nz_${g}_${nz}.json'));print('grid',$g,'nz',$nz,round(d['value'],1),d['clocks']['sm_mhz'])" 2>/dev/null || echo "grid $g nz $nz failed"
  done
done
