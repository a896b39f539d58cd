cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
timeout -s KILL 60 python tools/latency_stages.py > gpurun_out/latency_stages.log 2>&1
timeout -s KILL 120 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -n 4 gpurun_out/smallslice.log; tail -n 14 gpurun_out/latency_stages.log gpurun_out/latency_c.log
echo "=== tests"; grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -n 15
