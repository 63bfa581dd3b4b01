# usage: bash tools/gpu_cmd10.sh — multiway correctness (parity subset) + timing of c1/c2(8-way)/c3/c5
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keyidx.py -q -m gpu -x -k "multiway or mw or ways or keyidx or pair or depth_cap or pattern" 2>&1 | tail -3
timeout 300 python tools/time_configs.py --configs c1,c3,c5 2>&1 | grep -v "ascending\|descending\|swapped" | cut -c1-150
timeout 300 python tools/time_configs.py --configs c2 --ways 8 2>&1 | cut -c1-150
