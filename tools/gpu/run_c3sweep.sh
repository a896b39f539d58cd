cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"fence_batch": 3}' '{"fence_batch": 4}' '{"grid": 41}' '{"grid": 57}' '{"grid": 65}' '{"worker_fence": "gpu", "fence_batch": 3}' '{"chunk_bytes": 65536, "fence_batch": 1}'; do
  SPRAY_BENCH_B200="$k" timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --no-small --lat-batches 10 > gpurun_out/bench_k.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_k.json').read()); print(sys.argv[1], 'C3', d['value'], d['ms_per_step'], d['e2e']['value'])" "$k"
done
