cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
LAT_KV_REVERSED=1 timeout -s KILL 200 python tools/latency_c.py > gpurun_out/latency_c.log 2>&1
timeout -s KILL 60 python tools/latency_stages.py 4k > gpurun_out/latency_stages_4k.log 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
timeout -s KILL 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc=$?"
timeout -s KILL 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err; echo "ref rc=$?"
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests.log | tail -5
cat gpurun_out/latency_c.log
python -c "import json; d=json.load(open('gpurun_out/latency_stages_4k.log')); print(d['round_us_median'], d['worker_deltas_us'])"
tail -n 3 gpurun_out/smallslice.log | cut -c1-200
python -c "import json; d=json.loads(open('gpurun_out/bench_r02.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','ms_per_step','e2e','gpu_launches','clocks')}); print(d['roofline']); print(d['batch_latency']['small_batches_cpp']); print(d.get('small_slices'))"
tail -c 600 gpurun_out/bench_ref_r02.json; cat gpurun_out/smoke.log | tail -3
