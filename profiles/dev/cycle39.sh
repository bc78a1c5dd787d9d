# hoisted adjoint-force loads + support bounding box: GPU suite, TATO phases, C3 rates, 256^3 bench
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c39_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c39_tests.log
python profiles/dev/tato_phases.py
timeout 600 python profiles/configs.py --only "C3" 2>&1 | grep gcell | cut -c1-200
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('256', round(d['value'],1), d['clocks']['sm_mhz'])"; done
