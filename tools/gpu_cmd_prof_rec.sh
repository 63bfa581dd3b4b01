cd $GRAFT_REPO_ROOT
python tools/prof_pass.py --kind rec --n 67108864 --passes 0 --sort 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_part_fast -c 1 -o gpurun_out/prof_rec python tools/prof_pass.py --kind rec --n 67108864 --passes 0 --sort 1 > gpurun_out/ncu_rec.log 2>&1; echo NCU $?
