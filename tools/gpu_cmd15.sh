# usage: bash tools/gpu_cmd15.sh — parity suite, then c1/c2/c4a/c4b timing main vs variants
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
bash tools/time_variants_cfg.sh c1,c2,c4a,c4b main old pc1 pc8 main old
