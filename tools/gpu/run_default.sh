cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
t0=$(date +%s); python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? wall $(( $(date +%s) - t0 )) s"
t0=$(date +%s); python bench.py --impl reference > gpurun_out/bench_default_ref.json 2> gpurun_out/bench_default_ref.err; echo "ref rc=$? wall $(( $(date +%s) - t0 )) s"
python -c "import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['steps'], d['warmup'], d['cpu_baseline']['value'], d['gpu_launches'])"
tail -c 300 gpurun_out/bench_default_ref.json
