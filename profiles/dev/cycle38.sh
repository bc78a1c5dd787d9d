# precomputed support force coefficients (sup_fc): GPU suite, TATO 192^3 phases, C3 rates
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c38_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c38_tests.log
python profiles/dev/tato_phases.py
timeout 600 python profiles/configs.py --only "C3" 2>&1 | grep gcell | cut -c1-200
