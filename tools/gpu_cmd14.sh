# usage: bash tools/gpu_cmd14.sh — ncu --set full of the f64 8-way scatter (levels 0 and 3) and count (level 3)
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
python tools/prof_pass.py --kind f64 --n 134217728 --passes 0 --sort 1 > gpurun_out/p2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8_scatter' -s 0 -c 1 -o gpurun_out/r02_mw8s0 python tools/prof_pass.py --kind f64 --n 134217728 --passes 0 --sort 1 > gpurun_out/n3.log 2>&1; echo S0 $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8_(scatter|count)' -s 6 -c 2 -o gpurun_out/r02_mw8s3 python tools/prof_pass.py --kind f64 --n 134217728 --passes 0 --sort 1 > gpurun_out/n4.log 2>&1; echo S3 $?
