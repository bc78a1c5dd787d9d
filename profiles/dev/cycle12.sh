for g in 256 512; do for t in 1 2 1 2; do timeout 300 python profiles/dev/f64_rate.py --grid $g --n-steps 256 --two-step $t 2>/dev/null | tail -1; done; done
timeout 300 python profiles/dev/f64_rate.py --grid 1024 --n-steps 64 --two-step 1 --reps 1 2>/dev/null | tail -1
timeout 300 python profiles/dev/f64_rate.py --grid 1024 --n-steps 64 --two-step 2 --reps 1 2>/dev/null | tail -1
timeout 900 python -m pytest tests/test_two_step_gpu.py tests/test_full_size_gpu.py -q -m gpu -x -k "double or f64 or bench_grid" --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/c12_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c12_tests.log
