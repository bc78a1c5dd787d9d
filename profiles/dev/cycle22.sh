# Round-end evidence: 2048^3 C5 strong rerun, full GPU suite, smoke, default bench + reference arm.
o=gpurun_out
timeout 1500 python bench.py --workload c5 --scaling strong --steps 3 --warmup 3 > $o/c22_2048.json 2> $o/c22_2048.err; echo "2048^3 rc $?"; cut -c1-400 $o/c22_2048.json
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $o/c22_tests.log 2>&1; echo "tests rc $?"; tail -3 $o/c22_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $o/c22_smoke.log 2>&1; echo "smoke rc $?"; tail -2 $o/c22_smoke.log
timeout 600 python bench.py > $o/c22_bench.json 2> $o/c22_bench.err; echo "bench rc $?"; cut -c1-300 $o/c22_bench.json
timeout 900 python bench.py --impl reference > $o/c22_ref.json 2> $o/c22_ref.err; echo "ref rc $?"; cut -c1-300 $o/c22_ref.json
