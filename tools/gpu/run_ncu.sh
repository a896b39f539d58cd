# worker-fence sweep on C3, then ncu: launch list, full capture of the C3 engine launch and
# of the small-slice (2-rail HBM->HBM) launch. Each program runs clean first (exit 0) without ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"worker_fence": "gpu"}' '{"worker_fence": "gpu", "fence_batch": 1}'; do
  echo "== $k"
  SPRAY_BENCH_B200="$k" timeout -s KILL 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-congestion --no-small --lat-batches 300 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['batch_latency']['small_batches_cpp'])"
done
timeout 120 python tools/ncu_engine.py --runs 4 > gpurun_out/ncu_engine_clean.log 2>&1 || { echo "engine driver failed"; exit 1; }
timeout 120 python tools/ncu_small.py --runs 4 --rails 2 > gpurun_out/ncu_small_clean.log 2>&1 || { echo "small driver failed"; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-congestion \
  --no-small --lat-batches 4 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --replay-mode application \
  -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/engine_r02 -f \
  python tools/ncu_engine.py --runs 4 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --replay-mode application \
  -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/small_r02 -f \
  python tools/ncu_small.py --runs 4 --rails 2 > gpurun_out/ncu_small.log 2>&1; echo "small rc=$?"
ls -la gpurun_out/*.ncu-rep
