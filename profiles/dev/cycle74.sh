# cluster_reg inline injections, default for fp32 and fp64: full GPU suite, smoke, C1 configs
out=gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > $out/c74_tests.log 2>&1; echo "tests rc $?"; tail -4 $out/c74_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/c74_smoke.log 2>&1; tail -1 $out/c74_smoke.log
timeout 600 python profiles/configs.py --only C1 --out $out/c74_configs_c1.json > $out/c74_configs.log 2>&1; echo "configs rc $?"; tail -6 $out/c74_configs.log
