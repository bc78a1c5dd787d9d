# final evidence on the final build (next-block prefetch off): GPU suite, smoke, launch list + ncu capture, configs, default bench, reference arm
o=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/r2j_tests_full.log 2>&1; echo "tests rc $?"; tail -2 $o/r2j_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/r2j_smoke.log 2>&1; echo "smoke rc $?"; tail -1 $o/r2j_smoke.log
NO_TESTS=1 bash profiles/capture_round.sh r2j
timeout 1500 python profiles/configs.py --out $o/configs_r2j.json > $o/configs_r2j.log 2>&1; echo "configs rc $?"
timeout 900 python bench.py > $o/bench_r2j.json 2> $o/bench_r2j.err; echo "bench rc $?"; cut -c1-200 $o/bench_r2j.json
timeout 900 python bench.py --impl reference > $o/bench_r2j_ref.json 2> $o/bench_r2j_ref.err; echo "ref rc $?"; cut -c1-200 $o/bench_r2j_ref.json
