cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
timeout -s KILL 60 python tools/latency_stages.py 4k > gpurun_out/latency_stages_4k.log 2>&1
timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --lat-batches 100 > gpurun_out/bench_k.json 2>/dev/null
timeout -s KILL 1000 python -m pytest tests -m gpu -q --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python -c "
import json; d=json.load(open('gpurun_out/smallslice.json'))
for k,v in d.items(): print(k, v['gbs'], v['ms'], v.get('fb_split'), v['dec_split']['loop_cyc_per_dec'])"
python -c "import json; d=json.load(open('gpurun_out/latency_stages_4k.log')); print(d['round_us_median'], d['stage_deltas_us'])"
python -c "import json; d=json.loads(open('gpurun_out/bench_k.json').read()); print('C3', d['value'], d['e2e']['value'], d['small_slices']['rails_1']['gbs'], d['small_slices']['rails_2']['gbs'])"
echo "=== tests"; grep -E "passed|failed|FAILED|Error|rc=" gpurun_out/gpu_tests.log | tail -n 5
