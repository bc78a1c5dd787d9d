# packed ring-cell pairs (WB_T2_RING_PAIRS) A/B + two-step parity tests
L=paper_2509_15744_b200/_lib
timeout 1200 python -m pytest tests/test_two_step_gpu.py tests/test_parity_gpu.py tests/test_full_size_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for g in "256 1024" "512 128" "192 600"; do set -- $g; for lib in libwaveb200.so rp0.so libwaveb200.so rp0.so; do WAVEB200_LIB=$L/$lib timeout 300 python bench.py --grid $1 --n-steps $2 --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$1', '$lib', round(d['value'],1), d['clocks']['sm_mhz'])"; done; done
for lib in libwaveb200.so rp0.so; do WAVEB200_LIB=$L/$lib timeout 300 python profiles/dev/c1_rate.py 2>&1 | grep Gcell | sed "s/^/$lib /"; done
