cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"bulk_stages": 6}' '{"bulk_stages": 7}' '{"bulk_stages": 2}'; do
  echo "== $k"
  LAT_B200="$k" timeout -s KILL 120 python tools/latency_c.py 2>&1 | tail -3
  SPRAY_BENCH_B200="$k" timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --lat-batches 100 > gpurun_out/bench_k.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print('C3', d['value'], d['ms_per_step'], d['e2e']['value'], d['small_slices']['rails_1']['gbs'], d['small_slices']['rails_2']['gbs'])"
done
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
echo "=== tests"; grep -E "passed|failed|FAILED|Error|rc=" gpurun_out/gpu_tests.log | tail -n 25
