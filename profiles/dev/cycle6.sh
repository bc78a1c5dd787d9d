run() { tag=$1; shift; timeout 90 env "$@" > gpurun_out/dbg6_$tag.log 2>&1; echo "$tag rc $?"; tail -3 gpurun_out/dbg6_$tag.log; }
run b_3slab_n64 python profiles/dev/slab_debug.py 30 16 64 3 16 40
run d_3slab_n128_src5 WHOLE=1 python profiles/dev/slab_debug.py 30 16 128 3 5 40
timeout 900 python -m pytest tests/test_slabs_gpu.py tests/test_ipc_gpu.py -q -m gpu --timeout 150 --timeout-method thread -p no:cacheprovider > gpurun_out/c6_slabs.log 2>&1; echo "slabs rc $?"; tail -15 gpurun_out/c6_slabs.log
