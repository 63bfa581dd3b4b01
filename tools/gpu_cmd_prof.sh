# profiling pass: launch list of one c2 sort (+2 single passes), ncu --set full of
# the fast partition pass and of the largest leaf class
cd $GRAFT_REPO_ROOT
python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu1.log 2>&1; echo NCU1 $?
ncu --set full --clock-control none --import-source on -k regex:k_part_fast -s 1 -c 1 -o gpurun_out/prof_part python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu2.log 2>&1; echo NCU2 $?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'k_leaf.*KI32.*13' -s 3 -c 1 -o gpurun_out/prof_leaf python tools/prof_pass.py --passes 2 --sort 1 --fast 1 > gpurun_out/ncu3.log 2>&1; echo NCU3 $?
