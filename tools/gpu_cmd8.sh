# usage: bash tools/gpu_cmd8.sh — bench (short) + ncu DRAM launch list of one c2 sort (host-driven loop)
cd $GRAFT_REPO_ROOT
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH $?; tail -c 3000 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/plain8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dram.csv env BQ_HOST_LOOP=1 python tools/prof_pass.py --passes 0 --sort 1 --fast 1 > gpurun_out/ncu8.log 2>&1; echo NCU8 $?
