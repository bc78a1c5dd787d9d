# stability of the peer-store slab protocol: repeat the multi-process and in-process slab suites
for i in 1 2 3 4 5; do timeout 600 python -m pytest tests/test_slabs_mp_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/mp run $i: /"; done
for i in 1 2 3; do timeout 900 python -m pytest tests/test_slabs_gpu.py tests/test_ipc_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1 | sed "s/^/slab run $i: /"; done
