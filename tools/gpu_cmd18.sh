# usage: bash tools/gpu_cmd18.sh — ncu --set full of the warp-tile 8-way scatter and count (f64 c3 level 0, int32 c2 ways 8 level 0)
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8w_(scatter|count)' -s 0 -c 2 -o gpurun_out/r02_mw8w_f64 python tools/one_sort.py c3 > gpurun_out/n5.log 2>&1; echo F64 $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_mw8w_(scatter|count)' -s 0 -c 2 -o gpurun_out/r02_mw8w_i32 python tools/one_sort.py c2 --ways 8 > gpurun_out/n6.log 2>&1; echo I32 $?
