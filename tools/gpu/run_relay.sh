cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 30 tools/lat_bench > gpurun_out/lat_bench.log 2>&1
( timeout -s KILL 30 python tools/relay_debug.py 0 0 0; echo "relay rc=$?" ) > gpurun_out/relay_debug.log 2>&1
cat gpurun_out/lat_bench.log; cat gpurun_out/relay_debug.log | tail -6
