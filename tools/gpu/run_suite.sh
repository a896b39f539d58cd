cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider -rs > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|FAILED|Error|rc=|assert" gpurun_out/gpu_tests.log | tail -n 30
