timeout 600 python -m pytest tests/test_two_step_gpu.py -q -m gpu -x -k "cluster" --timeout 300 --timeout-method thread -p no:cacheprovider > gpurun_out/c11_tests.log 2>&1; echo "cluster tests rc $?"; tail -3 gpurun_out/c11_tests.log
WB_CLUSTER=1 timeout 600 python profiles/configs.py --only C1 > gpurun_out/c11_cl.log 2>&1; echo "cl rc $?"; cut -c1-150 gpurun_out/c11_cl.log
timeout 900 python profiles/dev/slab_timing.py --grid 1024 --n-steps 64 --parts 2 --reps 2 > gpurun_out/c11_slab1024.json 2>&1; echo "slab1024 rc $?"; cat gpurun_out/c11_slab1024.json | tail -2
timeout 900 python profiles/dev/slab_timing.py --grid 512 --n-steps 64 --parts 2 > gpurun_out/c11_slab512.json 2>&1; echo "slab512 rc $?"; cat gpurun_out/c11_slab512.json | tail -2
timeout 900 python profiles/dev/slab_timing.py --grid 256 --n-steps 128 --parts 4 > gpurun_out/c11_slab256.json 2>&1; echo "slab256 rc $?"; cat gpurun_out/c11_slab256.json | tail -2
