#!/bin/bash
# Round-end evidence on one GPU (run under gpurun from the repo root):
#   a plain bench run, the ncu launch list of the same command, then
#   gpu_cycle.sh's `ncu --set full` capture of the two-step kernel.
#   profiles/capture_round.sh <tag>
tag=${1:-round}
out=gpurun_out
mkdir -p $out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu"   # one whole timed step
NCU_RANGE="--profile-from-start off"   # bench.py brackets its timed region
timeout 300 $CMD > $out/${tag}_plain.json 2>$out/${tag}_plain.err; echo "plain rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none $NCU_RANGE -c 2000 --csv \
    --log-file $out/launches_bench_${tag}.csv $CMD > $out/${tag}_ncu_launch.log 2>&1; echo "launches rc $?"
python profiles/launch_shares.py $out/launches_bench_${tag}.csv "$NCU_RANGE -c 2000 $CMD" $out/launch_share_${tag}.json > $out/launches_bench_${tag}.txt
[ -n "$NO_FULL" ] || TESTS="-k no_test_selected_zzz" profiles/gpu_cycle.sh ${tag} > $out/${tag}_cycle.log 2>&1; echo "cycle rc $?"
