cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 1000 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
for k in '{}' '{"copy": "ldg"}'; do
  echo "== $k"
  SPRAY_BENCH_B200="$k" timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --lat-batches 300 > gpurun_out/bench_k.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['batch_latency']['small_batches_cpp'], d.get('small_slices'))"
done
timeout -s KILL 120 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1
echo "=== tests"; grep -E "passed|failed|FAILED|Error|rc=" gpurun_out/gpu_tests.log | tail -n 25
tail -n 4 gpurun_out/smallslice.log | cut -c1-400; cat gpurun_out/latency_c.log
