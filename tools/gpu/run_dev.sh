# dev GPU session: each step bounded by its own timeout; outputs in gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout -s KILL 30 tools/decide_bench > gpurun_out/decide_bench.log 2>&1
( timeout -s KILL 40 python tools/relay_debug.py 0 0 0; echo "relay rc=$?" ) > gpurun_out/relay_debug.log 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1; echo "small rc=$?" >> gpurun_out/smallslice.log
timeout -s KILL 120 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1; echo "lat rc=$?" >> gpurun_out/latency_c.log
timeout -s KILL 600 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for f in decide_bench relay_debug smallslice latency_c; do echo "=== $f"; tail -n 14 gpurun_out/$f.log; done
echo "=== tests"; grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -n 15
