# 2D C1 pass duration under ncu: round-1 build vs current
for t in r1tree .; do
  (cd $t && timeout 600 ncu --metrics gpu__time_duration.sum,launch__registers_per_thread,smsp__inst_executed.sum --clock-control none -k regex:step2 --launch-skip 9700 -c 60 --csv python profiles/dev/c1_once.py > /root/repo/gpurun_out/c25_$([ $t = . ] && echo r2 || echo r1).csv 2>&1); echo "$t rc $?"
done
