# 2-GPU session: GPU suite (relay / multi-process / staged peers), NVLink C2 bulk vs ldg,
# real-contention congestion, N=2 bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/topo_n2.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_n2.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_n2.log
for k in '{}' '{"copy": "ldg"}'; do
  NV_B200="$k" timeout -s KILL 200 python tools/nvlink_bench.py c2 --reps 5 > gpurun_out/nv_c2_$(echo $k | tr -dc a-z).log 2>&1
  NV_B200="$k" timeout -s KILL 200 python tools/nvlink_bench.py c2 --reps 5 --size 4294967296 > gpurun_out/nv_c2_4g_$(echo $k | tr -dc a-z).log 2>&1
done
timeout -s KILL 300 python tools/congestion_real.py > gpurun_out/congestion_real.log 2>&1
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests_n2.log | tail -8
for f in gpurun_out/nv_c2_*.log; do echo "== $f"; tail -c 600 $f; done
tail -30 gpurun_out/congestion_real.log
tail -c 1500 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
