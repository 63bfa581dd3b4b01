# usage: bash tools/gpu_cmd11.sh — full GPU suite + timing of every config
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 600 python tools/time_configs.py 2>&1 | cut -c1-170
