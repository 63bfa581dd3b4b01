cd $GRAFT_REPO_ROOT
python tools/prof_pass.py --passes 0 --sort 1 --fast 1 --ways 8 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_mw8_ -c 3 -o gpurun_out/prof_mw python tools/prof_pass.py --passes 0 --sort 1 --fast 1 --ways 8 > gpurun_out/ncu_mw.log 2>&1; echo NCU $?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_mw.csv python tools/prof_pass.py --passes 0 --sort 1 --fast 1 --ways 8 > gpurun_out/ncu1.log 2>&1; echo NCU1 $?
