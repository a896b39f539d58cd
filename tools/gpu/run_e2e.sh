cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for i in 1 2; do
  timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-congestion --no-small --lat-batches 200 > gpurun_out/bench_k.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print('C3', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['batch_latency']['kv_batch_8192_intents'], d['batch_latency']['small_batches_cpp']['intent_4k_hbm_to_host']['p90_us'])"
done
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|FAILED" gpurun_out/gpu_tests.log | tail -3
