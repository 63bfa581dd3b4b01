# usage: bash tools/gpu_sanitize.sh TOOL [--small] — one compute-sanitizer tool over the small-n driver
# (host-driven level loop: the same kernels as the graph; the driver also runs once plainly first)
cd $GRAFT_REPO_ROOT
BQ_HOST_LOOP=1 timeout 300 python tools/sanitize_driver.py $2 > gpurun_out/san_plain.log 2>&1; echo PLAIN $?; tail -2 gpurun_out/san_plain.log
BQ_HOST_LOOP=1 timeout 2400 compute-sanitizer --tool $1 --print-limit 50 --error-exitcode 9 python tools/sanitize_driver.py $2 > gpurun_out/san_$1.log 2>&1; echo SAN $1 $?
tail -30 gpurun_out/san_$1.log
