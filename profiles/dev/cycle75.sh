# ncu of the final cluster sweep (fp32 and fp64 C1 sweeps)
out=gpurun_out
for prec in single double; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:cluster_reg -s 2 -c 1 -o /tmp/c75_$prec python profiles/dev/c1_one.py $prec > $out/c75_ncu_$prec.log 2>&1; echo "ncu $prec rc $?"
  python profiles/analyze_ncu.py /tmp/c75_$prec.ncu-rep > $out/c75_ncu_summary_$prec.txt 2>&1; cat $out/c75_ncu_summary_$prec.txt | head -12
done
