cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 60 python tools/latency_stages.py 4k > gpurun_out/latency_stages_4k.log 2>&1
timeout -s KILL 200 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "import json; d=json.load(open('gpurun_out/latency_stages_4k.log')); print(d['round_us_median'], d['stage_deltas_us']); print(d['state_deltas_us'])"
cat gpurun_out/latency_c.log
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -3
