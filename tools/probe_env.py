"""Probe the GPU box: host cores/RAM/NUMA, L2 size, pinned H2D/D2H bandwidth."""
import json, os, subprocess, time
import torch

def sh(c):
    try:
        return subprocess.run(c, shell=True, capture_output=True, text=True, timeout=60).stdout
    except Exception as e:
        return str(e)

out = {}
out["nproc"] = sh("nproc").strip()
out["lscpu"] = sh("lscpu | head -30")
out["free_g"] = sh("free -g")
out["numactl"] = sh("numactl -H 2>&1 | head -20")
out["smi"] = sh("nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max --format=csv")
out["topo"] = sh("nvidia-smi topo -m 2>&1 | head -20")
p = torch.cuda.get_device_properties(0)
out["l2_bytes"] = getattr(p, "L2_cache_size", None)
out["sms"] = p.multi_processor_count
out["total_mem"] = p.total_memory
res = {}
for mb in (64, 1024):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); reps = 5
        for _ in range(reps): fn()
        e.record(); torch.cuda.synchronize()
        res[f"{name}_{mb}MB_GBs"] = n * reps / (s.elapsed_time(e) * 1e-3) / 1e9
    # duplex
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    res[f"duplex_{mb}MB_GBs_each"] = n * 5 / dt / 1e9
out["pinned"] = res
# host memory bandwidth (single thread numpy add) rough
import numpy as np
a = np.ones(1 << 27, dtype=np.float32); b = np.ones(1 << 27, dtype=np.float32)
t0 = time.perf_counter(); a += b; dt = time.perf_counter() - t0
out["host_add_GBs_1thread"] = 3 * a.nbytes / dt / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_env.json", "w"), indent=1)
print(json.dumps(out, indent=1))
