# usage: bash tools/gpu_mw8t3.sh — 8-way parity, config timing by ways, ncu of level-0 count + scatter (int32 c2, f64 c3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multiway or keyidx or full" 2>&1 | tail -2
for w in 2 8; do timeout 300 python tools/time_configs.py --configs c1,c2 --ways $w 2>&1 | sed "s/^/w$w /" | cut -c1-110; done
timeout 300 python tools/time_configs.py --configs c3,c5 2>&1 | sed "s/^/w0 /" | cut -c1-110
export BQ_HOST_LOOP=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mw8t_scatter|k_mw8w_count" -c 2 -o gpurun_out/mw8t_c2c python tools/one_sort.py c2 --ways 8 > gpurun_out/ncu_mw8t.log 2>&1; tail -1 gpurun_out/ncu_mw8t.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mw8t_scatter|k_mw8w_count" -c 2 -o gpurun_out/mw8t_c3c python tools/one_sort.py c3 > gpurun_out/ncu_mw8t3.log 2>&1; tail -1 gpurun_out/ncu_mw8t3.log
