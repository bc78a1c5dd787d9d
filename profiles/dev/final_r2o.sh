# Final round-2 evidence on the committed build (one B200)
out=gpurun_out
mkdir -p $out
timeout 1200 python -m pytest tests -q -m gpu > $out/r2o_tests.log 2>&1; echo "tests rc $?"; tail -2 $out/r2o_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/r2o_smoke.log 2>&1; tail -1 $out/r2o_smoke.log
timeout 600 python bench.py > $out/r2o_bench.json 2> $out/r2o_bench.err; echo "bench rc $?"; cat $out/r2o_bench.json
NO_FULL= bash profiles/capture_round.sh r2o > $out/r2o_capture.log 2>&1; echo "capture rc $?"; tail -3 $out/r2o_capture.log
timeout 900 python profiles/configs.py --out $out/r2o_configs.json > $out/r2o_configs.log 2>&1; echo "configs rc $?"; tail -12 $out/r2o_configs.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/r2o_reference_arm.json 2> $out/r2o_reference_arm.err; echo "ref arm rc $?"; cat $out/r2o_reference_arm.json
