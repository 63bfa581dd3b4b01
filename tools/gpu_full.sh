# usage: bash tools/gpu_full.sh — whole GPU suite, then the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -c 1500 gpurun_out/bench.json
