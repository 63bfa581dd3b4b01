# usage: bash tools/gpu_cmd3.sh REGEX SKIP — ncu --set full of one launch of the kernel matching REGEX in one c2 sort
cd $GRAFT_REPO_ROOT
BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$1" -s ${2:-2} -c 1 -o gpurun_out/prof_k env BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/ncu3.log 2>&1; echo NCU3 $?
