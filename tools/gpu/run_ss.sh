cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import torch; torch.zeros(1, device='cuda')" > /dev/null 2>&1
timeout -s KILL 120 python tools/smallslice.py > gpurun_out/smallslice.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/smallslice.json'))
for k,v in d.items(): print(k, v['gbs'], v['ms'], v['decide_ms'], v['p1_ms'], v.get('dec_extra_cyc_per_blk'), v['dec_split'])"
