# z-layer model min_work 2.2 -> 1.9 waves: 192^3 C3 TATO (fp32 model=12 vs old 16 layers, fp64 model=8 vs old 12)
for i in 1 2; do
  for nz in 0 16; do WB_T2_NZ=$nz timeout 600 python profiles/configs.py --only "C3 TATO 3D" 2>&1 | grep '"single"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp32 nz=$nz', round(d['gcell_upd_s'],1))"; done
  for nz in 0 12; do WB_T2_NZ=$nz timeout 600 python profiles/configs.py --only "C3 TATO 3D" 2>&1 | grep '"double"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fp64 nz=$nz', round(d['gcell_upd_s'],1))"; done
done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv
