# GPU suite, bench line, launch list and one full capture of spray_engine_kernel (1 x B200).
mkdir -p gpurun_out
timeout 200 python -m pytest tests -m gpu -x -q > gpurun_out/hold_gpu_tests.log 2>&1; tail -1 gpurun_out/hold_gpu_tests.log
timeout 200 python bench.py --steps 5 --warmup 3 > gpurun_out/pre_ncu_bench.json 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-congestion \
  --lat-batches 4 > gpurun_out/ncu_list.log 2>&1
echo "list rc=$?"
timeout 420 ncu --set full --clock-control none --import-source on --replay-mode application \
  -k regex:spray_engine_kernel --launch-skip 3 -c 1 -o gpurun_out/engine_final -f \
  python tools/ncu_engine.py --runs 4 > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
