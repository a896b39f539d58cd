# 4-GPU session: GPU suite, bench lines at N = 2 and 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/topo_n4.txt 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q --timeout 150 -p no:cacheprovider > gpurun_out/gpu_tests_n4.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests_n4.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
grep -E "passed|failed|FAILED|rc=" gpurun_out/gpu_tests_n4.log | tail -5
for f in gpurun_out/bench_n4.json gpurun_out/bench_n2.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['e2e']['value'], json.dumps(d.get('nvlink', {}))[:900])"; done
tail -3 gpurun_out/bench_n4.err
