set -x
timeout 100 python profiles/dev/slab_debug.py 40 16 128 4 21 40 > gpurun_out/dbg3_default.log 2>&1; echo "dbg default rc $?"
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 100 python profiles/dev/slab_debug.py 40 16 128 4 21 40 > gpurun_out/dbg3_conn32.log 2>&1; echo "dbg conn32 rc $?"
timeout 100 python profiles/dev/slab_debug.py 30 16 128 3 16 40 > gpurun_out/dbg3_3slabs.log 2>&1; echo "dbg 3slabs rc $?"
for f in gpurun_out/dbg3_*.log; do echo "== $f"; tail -12 $f; done
timeout 600 python -m pytest tests/test_reference_loops_gpu.py -k optimize_design -q -m gpu --timeout 300 --timeout-method thread -p no:cacheprovider > gpurun_out/c3_design.log 2>&1; echo "design rc $?"; tail -5 gpurun_out/c3_design.log
timeout 900 python -m pytest tests/test_two_step_gpu.py tests/test_full_size_gpu.py -q -m gpu -x --timeout 300 --timeout-method thread -p no:cacheprovider -k "not big_grids" > gpurun_out/c3_two_step.log 2>&1; echo "two-step tests rc $?"; tail -5 gpurun_out/c3_two_step.log
for c in 0 1 0 1; do WB_T2_CHAIN=$c timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/c3_bench_chain$c.json 2>gpurun_out/c3_bench_chain$c.err; echo "chain $c rc $?"; python -c "import json;d=json.load(open('gpurun_out/c3_bench_chain$c.json'));print('chain',$c,d['value'],d['e2e']['value'],d['roofline']['frac'],d['clocks'])"; done
