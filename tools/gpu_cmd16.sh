# usage: bash tools/gpu_cmd16.sh — launch lists of one c3 sort and one c2 sort with ways=8 (host-driven loop)
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
python tools/one_sort.py c3 > gpurun_out/os_c3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/one_sort.py c3 > gpurun_out/osn_c3.log 2>&1; echo $?
python tools/one_sort.py c2 --ways 8 > gpurun_out/os_c2w8.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2w8.csv python tools/one_sort.py c2 --ways 8 > gpurun_out/osn_c2w8.log 2>&1; echo $?
