# usage: bash tools/gpu_checks.sh — the GPU suite and the sanitize driver against the -DBQ_CHECKS build
cd $GRAFT_REPO_ROOT
export BQ_LIB=$GRAFT_REPO_ROOT/paper_1604_06697_b200/variants/libbq_checks.so
timeout 300 python tools/sanitize_driver.py > gpurun_out/checks_driver.log 2>&1; echo DRIVER $?; grep -c ok gpurun_out/checks_driver.log; grep -E "BQ_CHECK|MISMATCH|FAILS|Error" gpurun_out/checks_driver.log | head
BQ_HOST_LOOP=1 timeout 300 python tools/sanitize_driver.py > gpurun_out/checks_driver_host.log 2>&1; echo DRIVER_HOST $?; grep -E "BQ_CHECK|MISMATCH|FAILS|Error" gpurun_out/checks_driver_host.log | head
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/checks_tests.log 2>&1; echo TESTS $?; tail -5 gpurun_out/checks_tests.log; grep -m5 "BQ_CHECK" gpurun_out/checks_tests.log
