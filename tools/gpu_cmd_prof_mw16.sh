cd $GRAFT_REPO_ROOT
python tools/prof_pass.py --passes 0 --sort 1 --fast 1 --ways 16 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_mw_(count|scatter)" -c 2 -o gpurun_out/prof_mw16 python tools/prof_pass.py --passes 0 --sort 1 --fast 1 --ways 16 > gpurun_out/ncu_mw.log 2>&1; echo NCU $?
