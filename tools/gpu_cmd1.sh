# usage: bash tools/gpu_cmd1.sh — GPU tests, all-config timing, launch list of one c2 sort,
# ncu --set full of the largest int32 leaf class
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo TESTS $?; tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/time_configs.py > gpurun_out/configs.jsonl 2>&1; echo CFG $?; cut -c1-200 gpurun_out/configs.jsonl
python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu1.log 2>&1; echo NCU1 $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_leaf.*KI32.*1024' -s 2 -c 1 -o gpurun_out/prof_leaf python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu3.log 2>&1; echo NCU3 $?
