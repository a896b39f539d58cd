cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 60 tools/lat_bench > gpurun_out/lat_bench.log 2>&1
for k in '{}' '{"fence": "release"}' '{"fence": "release", "worker_fence": "gpu"}'; do
  echo "== $k"
  LAT_B200="$k" timeout -s KILL 120 python tools/latency_c.py 2>&1 | tail -3
  LAT_B200="$k" timeout -s KILL 60 python tools/latency_stages.py 4k 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['round_us_median'], d['stage_deltas_us'], d['worker_deltas_us'])"
  SPRAY_BENCH_B200="$k" timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --no-small --lat-batches 100 > gpurun_out/bench_k.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print('C3', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
LAT_B200='{}' timeout -s KILL 60 python tools/latency_stages.py kv > gpurun_out/latency_stages_kv.log 2>&1
cat gpurun_out/lat_bench.log
python -c "import json; d=json.load(open('gpurun_out/latency_stages_kv.log')); print(d['round_us_median'], d.get('round_us_hist'), d.get('round_us_edges')); print(d.get('fast_rounds')); print(d.get('slow_rounds'))"
