# C3 knob sweep: fence batching and posting window on the bench's KV batch (no side phases)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"fence_batch": 1}' '{"post_window": 4096}' '{"fence_batch": 1, "post_window": 4096}' '{"fence_batch": 2, "post_window": 4096}'; do
  echo "== $k"
  SPRAY_BENCH_B200="$k" timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --no-small --lat-batches 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
timeout -s KILL 60 python tools/latency_stages.py > gpurun_out/latency_stages.log 2>&1; tail -14 gpurun_out/latency_stages.log
