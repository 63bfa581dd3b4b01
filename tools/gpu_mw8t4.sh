# usage: bash tools/gpu_mw8t4.sh — 8-way parity, ways sweep, ncu of level-0 count (int32 c2, f64 c3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multiway or keyidx or full" 2>&1 | tail -2
timeout 300 python tools/time_configs.py --configs c3,c5 2>&1 | sed "s/^/w0 /" | cut -c1-110
SWEEP_LOGS=16,18,20,22,24,26,28 timeout 600 python tools/ways_sweep.py 2>&1 | tail -20
export BQ_HOST_LOOP=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mw8w_count" -c 1 -o gpurun_out/mw8c_c2 python tools/one_sort.py c2 --ways 8 > gpurun_out/ncu_mw8t.log 2>&1; tail -1 gpurun_out/ncu_mw8t.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mw8w_count" -c 1 -o gpurun_out/mw8c_c3 python tools/one_sort.py c3 > gpurun_out/ncu_mw8t3.log 2>&1; tail -1 gpurun_out/ncu_mw8t3.log
