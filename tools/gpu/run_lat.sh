cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 60 python tools/latency_stages.py 4k > gpurun_out/latency_stages_4k.log 2>&1
cat gpurun_out/latency_stages_4k.log
