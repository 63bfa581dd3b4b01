# usage: bash tools/gpu_prof_r02.sh — ncu --set full captures for profiles/r02 (host-driven loop: same kernels)
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:k_part_fast -s 0 -c 1 -o gpurun_out/r02_part python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/n1.log 2>&1; echo PART $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_leaf.*KI32.*1024' -s 3 -c 1 -o gpurun_out/r02_leaf python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/n2.log 2>&1; echo LEAF $?
python tools/prof_pass.py --kind f64 --n 134217728 --passes 0 --sort 1 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8_(count|scatter)' -s 0 -c 2 -o gpurun_out/r02_mw8 python tools/prof_pass.py --kind f64 --n 134217728 --passes 0 --sort 1 > gpurun_out/n3.log 2>&1; echo MW8 $?
