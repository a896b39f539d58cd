cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{}' '{"post_window": 1048576}' '{"fence_batch": 1}' '{"copy": "ldg", "post_window": 1048576}'; do
  echo "== $k"
  NV_B200="$k" timeout -s KILL 200 python tools/nvlink_bench.py c2 --reps 5 2>&1 | tail -1 | cut -c1-260
done
