timeout 900 python -m pytest tests/test_slabs_mp_gpu.py -v -m gpu --timeout 400 --timeout-method thread -p no:cacheprovider > gpurun_out/c19_mp.log 2>&1; echo "mp rc $?"; grep -E "PASSED|FAILED|ERROR|Error|assert" gpurun_out/c19_mp.log | head -20
nvidia-smi --query-gpu=index,memory.used,utilization.gpu --format=csv
