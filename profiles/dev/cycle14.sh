timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --timeout-method thread -p no:cacheprovider > gpurun_out/c14_tests.log 2>&1; echo "tests rc $?"; tail -8 gpurun_out/c14_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c14_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/c14_smoke.log
timeout 1500 python profiles/configs.py --out gpurun_out/configs_r2d.json > gpurun_out/c14_configs.log 2>&1; echo "configs rc $?"; cut -c1-170 gpurun_out/c14_configs.log
