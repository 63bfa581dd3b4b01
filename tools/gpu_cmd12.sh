# usage: bash tools/gpu_cmd12.sh — launch lists of one c3 and one c5 sort (host-driven loop: same kernels)
cd $GRAFT_REPO_ROOT
export BQ_HOST_LOOP=1
for c in c5 c1; do
python tools/one_sort.py $c > gpurun_out/os_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python tools/one_sort.py $c > gpurun_out/osn_$c.log 2>&1; echo $c $?
done
