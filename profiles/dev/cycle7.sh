# full GPU suite, default bench (with the CPU reference), C5 bench, round capture
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 --timeout-method thread -p no:cacheprovider > gpurun_out/c7_tests.log 2>&1; echo "tests rc $?"; tail -6 gpurun_out/c7_tests.log
timeout 900 python bench.py > gpurun_out/c7_bench.json 2> gpurun_out/c7_bench.err; echo "bench rc $?"; cat gpurun_out/c7_bench.json
timeout 900 python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/c7_c5.json 2> gpurun_out/c7_c5.err; echo "c5 rc $?"; cat gpurun_out/c7_c5.json; tail -3 gpurun_out/c7_c5.err
timeout 1200 bash profiles/capture_round.sh r2a > gpurun_out/c7_capture.log 2>&1; echo "capture rc $?"; tail -20 gpurun_out/c7_capture.log
