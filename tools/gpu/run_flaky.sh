cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for i in 1 2 3; do
  timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_rep$i.log 2>&1; echo "rep $i rc=$?"
  grep -E "passed|failed|FAILED" gpurun_out/gpu_tests_rep$i.log | tail -3
done
timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
