"""Timeline of the end-to-end loop (bench.py's e2e: H2D of G on a side stream, double
buffered, zf_step with offload) on Llama-2-7B: per step the H2D span, the zf_step stream
span, the library's D2H span (profile phase 4 / 5) and how long the host thread spent inside
zf_step -- to see which of the host link's two directions, the kernels or a host-side wait
sets the pace.  usage (GPU box): python tools/e2e_timeline.py [devacc 0|1] [host_stages] [steps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_12242_b200 import _build  # noqa: E402

_build.build()
from paper_2505_12242_b200 import zf  # noqa: E402
from synth import gpu  # noqa: E402

devacc = len(sys.argv) > 1 and sys.argv[1] == "1"
hst = int(sys.argv[2]) if len(sys.argv) > 2 else 8
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
shapes = [(n, m) for _, n, m in synth.MODELS["llama2-7b"]()]
tot = sum(n * m for n, m in shapes)
g = [torch.empty(tot, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
p = torch.empty(tot, dtype=torch.bfloat16, device="cuda")


def views(b):
    out, off = [], 0
    for n, m in shapes:
        out.append(b[off:off + n * m].view(n, m))
        off += n * m
    return out


G0, P = views(g[0]), views(p)
for li, (n, m) in enumerate(shapes):
    gpu.fill_grad(G0[li], li, 0, gpu.ColScale(m, li))
    gpu.fill_param(P[li], li)
host_g = torch.empty(tot, dtype=torch.bfloat16, pin_memory=True)
host_g.copy_(g[0])
Gv = [views(g[0]), views(g[1])]
ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=100000, refresh_interval=4,
                 accum_interval=4, adam=zf.adam_params(lr=1e-5), offload=True, host_accumulate=True,
                 device_accumulate=devacc, host_stages=0 if devacc else hst)
stream = torch.cuda.current_stream()
h2d = torch.cuda.Stream()
base = torch.cuda.Event(enable_timing=True)
ev = {k: [torch.cuda.Event(enable_timing=True) for _ in range(steps)] for k in ("h0", "h1", "s0", "s1")}
up = [torch.cuda.Event(), torch.cuda.Event()]
used = [torch.cuda.Event(), torch.cuda.Event()]
host_in = []
torch.cuda.synchronize()
base.record(stream)
with torch.cuda.stream(h2d):
    ev["h0"][0].record(h2d)
    g[0].copy_(host_g, non_blocking=True)
    ev["h1"][0].record(h2d)
    up[0].record(h2d)
ctx.profile(True)
d2h = []
t0 = time.perf_counter()
for t in range(steps):
    b = t % 2
    stream.wait_event(up[b])
    ev["s0"][t].record(stream)
    a = time.perf_counter()
    ctx.step(t, Gv[b], P)
    host_in.append((a - t0, time.perf_counter() - a))
    ev["s1"][t].record(stream)
    used[b].record(stream)
    if t + 1 < steps:
        nb = (t + 1) % 2
        with torch.cuda.stream(h2d):
            h2d.wait_event(used[nb])
            ev["h0"][t + 1].record(h2d)
            g[nb].copy_(host_g, non_blocking=True)
            ev["h1"][t + 1].record(h2d)
            up[nb].record(h2d)
ctx.sync()
wall = time.perf_counter() - t0
pr = ctx.profile_read()
torch.cuda.synchronize()
rows = []
for t in range(steps):
    rows.append({k: round(base.elapsed_time(ev[k][t]), 1) for k in ev} | {"host_call_at": round(host_in[t][0] * 1e3, 1),
                                                                       "host_in_step_ms": round(host_in[t][1] * 1e3, 1)})
print(json.dumps({"devacc": devacc, "host_stages": hst, "wall_ms_per_step": wall * 1e3 / steps,
                  "d2h_step_ms": pr["d2h_step"], "d2h_window_ms": pr["d2h_window"],
                  "h1": ctx.host_stats(), "rows": rows}))
ctx.close()
