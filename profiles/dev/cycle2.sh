set -x
timeout 120 python profiles/dev/slab_debug.py 40 16 128 4 21 40 > gpurun_out/dbg_nopdl.log 2>&1; echo "dbg1 rc $?"
WB_P2P_PDL=1 timeout 120 python profiles/dev/slab_debug.py 40 16 128 4 21 40 > gpurun_out/dbg_pdl.log 2>&1; echo "dbg2 rc $?"
tail -5 gpurun_out/dbg_nopdl.log gpurun_out/dbg_pdl.log
timeout 900 python -m pytest tests/test_slabs_gpu.py tests/test_ipc_gpu.py -v -m gpu --timeout 150 --timeout-method thread -p no:cacheprovider > gpurun_out/c2_slabs.log 2>&1; echo "slabs rc $?"
grep -E "PASSED|FAILED|ERROR|Timeout" gpurun_out/c2_slabs.log | tail -40
timeout 1500 python -m pytest tests/test_reference_loops_gpu.py tests/test_full_size_gpu.py "tests/test_parity_gpu.py::test_buffer_counter_reports_device_fields" -v -m gpu --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/c2_new.log 2>&1; echo "new rc $?"
grep -E "PASSED|FAILED|ERROR|Timeout|SKIPPED" gpurun_out/c2_new.log | tail -50
