timeout 900 python -m pytest tests/test_two_step_gpu.py tests/test_parity_gpu.py tests/test_reference_loops_gpu.py tests/test_device_loop_gpu.py -q -m gpu -x --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/c15_tests.log 2>&1; echo "tests rc $?"; tail -15 gpurun_out/c15_tests.log
timeout 600 python profiles/configs.py --only C1,C3 > gpurun_out/c15_tile.log 2>&1; echo "tile rc $?"; cut -c1-200 gpurun_out/c15_tile.log
WB_TILE2D=0 timeout 600 python profiles/configs.py --only C1,C3 > gpurun_out/c15_notile.log 2>&1; echo "notile rc $?"; cut -c1-200 gpurun_out/c15_notile.log
