# final-build profiling: clean bench line, ncu launch list of the bench, full capture of the C3 engine launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; echo "bench rc=$?"
timeout 120 python tools/ncu_engine.py --runs 4 > gpurun_out/ncu_engine_clean.log 2>&1 || { echo "engine driver failed"; exit 1; }
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-congestion \
  --no-small --lat-batches 4 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --replay-mode application \
  -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/engine_r02c -f \
  python tools/ncu_engine.py --runs 4 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/*.ncu-rep
python -c "import json; d=json.loads(open('gpurun_out/bench_r02c.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('value','ms_per_step','e2e','gpu_launches','clocks')})"
