set -x
(nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp) > gpurun_out/box.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x --maxfail=5 > gpurun_out/c1_tests.log 2>&1; echo "tests rc $?"
tail -30 gpurun_out/c1_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-sample-steps 4 > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err; echo "bench rc $?"
cat gpurun_out/c1_bench.json
