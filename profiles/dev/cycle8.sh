timeout 900 python -m pytest tests -q -m gpu -k "reference or slabs" --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/c8_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c8_tests.log
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c8_c5.json 2> gpurun_out/c8_c5.err; echo "c5 rc $?"; cat gpurun_out/c8_c5.json; tail -3 gpurun_out/c8_c5.err
timeout 1500 python profiles/configs.py --out gpurun_out/configs_r2a.json > gpurun_out/c8_configs.log 2>&1; echo "configs rc $?"; cat gpurun_out/c8_configs.log
timeout 1500 bash profiles/dev/ab_nz_chain.sh > gpurun_out/c8_nz.log 2>&1; echo "nz rc $?"; cat gpurun_out/c8_nz.log
