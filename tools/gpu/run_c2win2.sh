cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"post_window": 1048576}'; do
  echo "== $k"
  NV_B200="$k" timeout -s KILL 200 python tools/nvlink_bench.py c2 --reps 5 2>&1 | tail -1 | cut -c1-200
done
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
tail -3 gpurun_out/smallslice.log | cut -c1-120
timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --lat-batches 100 > gpurun_out/bench_k.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print('C3', d['value'], d['e2e']['value'])"
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_n2.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/gpu_tests_n2.log
