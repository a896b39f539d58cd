cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 300 python tools/scenarios.py > gpurun_out/scenarios.log 2>&1; echo "rc=$?"
cat gpurun_out/scenarios.log | tail -20
