# usage: bash tools/gpu_mw8t2.sh — 8-way parity, config timing by ways, ncu of the int32 level-0 count + scatter
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "multiway or keyidx or full" 2>&1 | tail -3
for w in 2 8; do timeout 300 python tools/time_configs.py --configs c1,c2 --ways $w 2>&1 | sed "s/^/w$w /" | cut -c1-150; done
timeout 300 python tools/time_configs.py --configs c3,c5 2>&1 | sed "s/^/w0 /" | cut -c1-150
export BQ_HOST_LOOP=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mw8t_scatter|k_mw8w_count" -c 2 -o gpurun_out/mw8t_c2b python tools/one_sort.py c2 --ways 8 > gpurun_out/ncu_mw8t.log 2>&1; tail -1 gpurun_out/ncu_mw8t.log
