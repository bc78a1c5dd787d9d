# Final commit check: full GPU suite, smoke, C1 configs
out=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $out/r2q_tests.log 2>&1; echo "tests rc $?"; tail -2 $out/r2q_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/r2q_smoke.log 2>&1; tail -1 $out/r2q_smoke.log
for i in 1 2; do timeout 600 python profiles/configs.py --only C1 --out $out/r2q_configs_c1_$i.json > $out/r2q_configs_$i.log 2>&1; grep '"C1 2D FWI 256^2, N=3200", "precision"' $out/r2q_configs_$i.log; done
