# usage: bash tools/gpu_cmd2.sh — leaf debug sorts, all-config timing, launch list of one c2 sort
cd $GRAFT_REPO_ROOT
python tools/dbg_leaf.py 2>&1 | tail -8
timeout 300 python tools/time_configs.py > gpurun_out/configs.jsonl 2>&1; echo CFG $?; cut -c1-160 gpurun_out/configs.jsonl
python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu1.log 2>&1; echo NCU1 $?
