cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
for m in 4k kv; do
  timeout -s KILL 60 python tools/latency_stages.py $m > gpurun_out/latency_stages_$m.log 2>&1
  LAT_B200='{"worker_fence": "gpu"}' timeout -s KILL 60 python tools/latency_stages.py $m > gpurun_out/latency_stages_${m}_gpu.log 2>&1
done
timeout -s KILL 120 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1
LAT_B200='{"worker_fence": "gpu"}' timeout -s KILL 120 python tools/latency_c.py > gpurun_out/latency_c_gpu.log 2>&1
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -n 4 gpurun_out/smallslice.log
for f in gpurun_out/latency_stages_*.log; do echo "== $f"; python -c "import json,sys; d=json.load(open('$f')); print(d['round_us_median'], d['stage_deltas_us'], d['worker_deltas_us'])"; done
tail -n 4 gpurun_out/latency_c.log gpurun_out/latency_c_gpu.log
echo "=== tests"; grep -E "passed|failed|FAILED|Error|rc=" gpurun_out/gpu_tests.log | tail -n 25
