timeout 900 python -m pytest tests -q -m gpu -x -k "cluster or desk or tato or device_loop or reference or two_step or odd_shapes or calibrate" --timeout 600 --timeout-method thread -p no:cacheprovider > gpurun_out/c10_tests.log 2>&1; echo "tests rc $?"; tail -15 gpurun_out/c10_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c10_smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/c10_smoke.log
timeout 600 python profiles/configs.py --only C1,C3 > gpurun_out/c10_configs.log 2>&1; echo "configs rc $?"; cut -c1-220 gpurun_out/c10_configs.log
WB_CLUSTER=0 timeout 600 python profiles/configs.py --only C1 > gpurun_out/c10_configs_nocl.log 2>&1; echo "configs nocl rc $?"; cut -c1-220 gpurun_out/c10_configs_nocl.log
