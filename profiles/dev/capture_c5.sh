# C5 one-GPU evidence: plain run, ncu launch list of the timed step, ncu full of one two-step pass
out=gpurun_out
CMD="python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu"
timeout 600 $CMD > $out/c5_plain.json 2> $out/c5_plain.err; echo "plain rc $?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 2000 --csv \
    --log-file $out/launches_bench_c5.csv $CMD > $out/c5_ncu_launch.log 2>&1; echo "launches rc $?"
python profiles/launch_shares.py $out/launches_bench_c5.csv "--profile-from-start off -c 2000 $CMD" $out/launch_share_c5.json > $out/launches_bench_c5.txt
timeout 1500 ncu --set full --clock-control none --profile-from-start off -k regex:step2_kernel -s 4 -c 1 \
    -o /tmp/c5_step $CMD > $out/c5_ncu_full.log 2>&1; echo "full rc $?"
python profiles/analyze_ncu.py /tmp/c5_step.ncu-rep 1073741824 > $out/c5_ncu_summary.txt 2>&1
ncu -i /tmp/c5_step.ncu-rep --page raw --csv > $out/c5_ncu_raw.csv 2>/dev/null
head -8 $out/launches_bench_c5.txt; head -14 $out/c5_ncu_summary.txt
# fp64 two-step pass at 256^3 (the fp64 validation build's hot kernel)
timeout 900 ncu --set full --clock-control none -k regex:step2_kernel -s 10 -c 1 -o /tmp/f64_step \
    python profiles/profile_step.py --precision double > $out/f64_ncu.log 2>&1; echo "f64 rc $?"
python profiles/analyze_ncu.py /tmp/f64_step.ncu-rep > $out/f64_ncu_summary.txt 2>&1
ncu -i /tmp/f64_step.ncu-rep --page raw --csv > $out/f64_ncu_raw.csv 2>/dev/null
head -14 $out/f64_ncu_summary.txt
