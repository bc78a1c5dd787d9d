# every kernel of one C1 fp32 gradient: round-1 build vs current (32- and 64-bit offsets)
run() { timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 8000 --csv python profiles/dev/c1_once.py > $1 2>&1; echo "$1 rc $?"; }
(cd r1tree && run /root/repo/gpurun_out/c27_r1.csv)
run gpurun_out/c27_r2.csv
WAVEB200_LIB=paper_2509_15744_b200/_lib/off32.so run gpurun_out/c27_off32.csv
