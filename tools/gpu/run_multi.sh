# 2-GPU session: multi-GPU tests, real-contention congestion, N=2 bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/topo_n2.txt 2>&1
timeout -s KILL 500 python -m pytest tests/test_gpu_relay.py tests/test_gpu_multiproc.py tests/test_gpu_staged.py -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_n2.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_n2.log
timeout -s KILL 300 python tools/congestion_real.py > gpurun_out/congestion_real.log 2>&1
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
grep -E "passed|failed|FAILED" gpurun_out/gpu_tests_n2.log | tail -5
tail -30 gpurun_out/congestion_real.log
tail -c 2500 gpurun_out/bench_n2.json; tail -3 gpurun_out/bench_n2.err
