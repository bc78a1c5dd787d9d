timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --timeout-method thread -p no:cacheprovider > gpurun_out/c13_tests.log 2>&1; echo "tests rc $?"; tail -4 gpurun_out/c13_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c13_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/c13_smoke.log
timeout 900 python bench.py > gpurun_out/c13_bench.json 2> gpurun_out/c13_bench.err; echo "bench rc $?"; cat gpurun_out/c13_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/c13_ref.json 2> gpurun_out/c13_ref.err; echo "ref rc $?"; cat gpurun_out/c13_ref.json
timeout 1500 python profiles/configs.py --out gpurun_out/configs_r2c.json > gpurun_out/c13_configs.log 2>&1; echo "configs rc $?"; cut -c1-160 gpurun_out/c13_configs.log
timeout 1200 bash profiles/capture_round.sh r2c > gpurun_out/c13_capture.log 2>&1; echo "capture rc $?"; cat gpurun_out/launches_bench_r2c.txt | head -6; cat gpurun_out/r2c_ncu_summary.txt | head -14
