"""Box probe: GPU count, topology, PCIe pinned-host and HBM copy bandwidth (CUDA events)."""
import json, subprocess, torch, time
out = {}
out["n_gpus"] = torch.cuda.device_count()
out["name"] = torch.cuda.get_device_name(0)
out["sm_count"] = torch.cuda.get_device_properties(0).multi_processor_count
try:
    out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
except Exception as e:
    out["topo"] = str(e)
out["numa"] = subprocess.run(["bash", "-c", "lscpu | grep -E 'NUMA|Model name|^CPU\\(s\\)'"], capture_output=True, text=True).stdout
def bw(fn, nbytes, iters=10):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    for _ in range(3): fn()
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return nbytes * iters / (s.elapsed_time(e) * 1e-3) / 1e9
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
out["h2d_gbs"] = bw(lambda: d.copy_(h, non_blocking=True), n)
out["d2h_gbs"] = bw(lambda: h.copy_(d, non_blocking=True), n)
out["d2d_gbs_delivered"] = bw(lambda: d2.copy_(d), n)
print(json.dumps(out, indent=1))
