cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for nb in 67108864 268435456 1073741824; do
  ( NBYTES=$nb timeout -s KILL 45 python tools/relay_fault_debug.py ) > gpurun_out/relay_fault_$nb.log 2>&1
done
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err
timeout -s KILL 300 python -m pytest tests/test_gpu_staged.py tests/test_gpu_integration.py tests/test_gpu_parity.py -q -x --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -n 8 gpurun_out/relay_fault_*.log gpurun_out/smallslice.log
echo "=== bench"; tail -c 3000 gpurun_out/bench_dev.json; tail -5 gpurun_out/bench_dev.err
echo "=== tests"; grep -E "passed|failed|FAILED|Error|staged" gpurun_out/gpu_tests.log | tail -n 15
