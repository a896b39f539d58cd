cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{"diag": true}' '{"diag": true, "copy": "ldg"}'; do
  echo "== $k"
  ST_B200="$k" timeout -s KILL 120 python tools/staged_synth_bench.py --reps 2 --mib 256 1024 2>&1 | grep -v what
done
timeout -s KILL 400 python -m pytest tests/test_gpu_staged.py tests/test_gpu_relay.py -q --timeout 150 -p no:cacheprovider 2>&1 | tail -3
