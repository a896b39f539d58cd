cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
for k in '{"diag": true, "chunk_bytes": 65536}' '{"diag": true, "chunk_bytes": 16384}' '{}'; do
  echo "== $k"
  ST_B200="$k" timeout -s KILL 120 python tools/staged_synth_bench.py --reps 3 --mib 64 256 1024 2>&1 | grep -v what
done
cp gpurun_out/staged_synth.json gpurun_out/staged_synth_default.json
