free -g | head -2
timeout 1500 python bench.py --workload c5 --scaling strong --steps 3 --warmup 3 > gpurun_out/c21_2048.json 2> gpurun_out/c21_2048.err; echo "2048^3 rc $?"; cat gpurun_out/c21_2048.json | cut -c1-2500; tail -5 gpurun_out/c21_2048.err
