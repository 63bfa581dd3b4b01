# usage: bash tools/gpu_cmd5.sh KIND N REGEX SKIP — ncu --set full of one launch of REGEX in one sort of KIND
cd $GRAFT_REPO_ROOT
python tools/prof_pass.py --kind $1 --n $2 --passes 0 --sort 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$3" -s ${4:-0} -c 1 -o gpurun_out/prof_$5 python tools/prof_pass.py --kind $1 --n $2 --passes 0 --sort 1 > gpurun_out/ncu5.log 2>&1; echo NCU5 $?
