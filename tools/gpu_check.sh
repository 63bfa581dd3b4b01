# usage: bash tools/gpu_check.sh [pytest-args...]  — GPU tests + timing of one c2 sort/pass
cd $GRAFT_REPO_ROOT
python -m pytest tests -x -q -m gpu "$@" > gpurun_out/gpu_tests.log 2>&1; echo TESTS $?; tail -15 gpurun_out/gpu_tests.log
python tools/time_pass.py 2>&1 | tail -3
