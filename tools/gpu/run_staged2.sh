cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 300 python tools/staged_synth_bench.py --reps 5 > gpurun_out/staged_synth.log 2>&1; echo "staged rc=$?"
timeout -s KILL 400 python -m pytest tests/test_gpu_staged.py tests/test_gpu_relay.py -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_staged.log 2>&1; echo "tests rc=$?"
cat gpurun_out/staged_synth.log | tail -5; tail -5 gpurun_out/gpu_tests_staged.log
