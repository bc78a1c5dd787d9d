# final-build evidence: launch list + ncu full capture of the two-step kernel, all configs, default bench
bash profiles/capture_round.sh r2f
timeout 1500 python profiles/configs.py --out gpurun_out/configs_r2f.json > gpurun_out/configs_r2f.log 2>&1; echo "configs rc $?"
timeout 900 python bench.py > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err; echo "bench rc $?"; cut -c1-300 gpurun_out/bench_r2f.json
