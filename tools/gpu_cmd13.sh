# usage: bash tools/gpu_cmd13.sh — multiway/pair/f64 parity subset, then c3/c5 timing main vs variants
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_keyidx.py tests/test_gpu_full.py -q -m gpu -x -k "multiway or mw or ways or keyidx or pair or nan or f64 or c3 or c5 or records" 2>&1 | tail -3
bash tools/time_variants_cfg.sh c3,c5 main old main old
