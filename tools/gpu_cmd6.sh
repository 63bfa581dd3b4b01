# usage: bash tools/gpu_cmd6.sh CONFIGS — time_configs in graph mode and in host-loop mode
cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_configs.py --configs $1 2>&1 | sed 's/^/graph /' | cut -c1-140
BQ_HOST_LOOP=1 timeout 300 python tools/time_configs.py --configs $1 2>&1 | sed 's/^/host /' | cut -c1-140
