# after removing the superseded 256-thread TMA engine: full GPU suite
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c33_tests.log 2>&1; echo "tests rc $?"; tail -3 gpurun_out/c33_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
