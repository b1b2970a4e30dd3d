"""Small zf_step runs for compute-sanitizer (memcheck / racecheck): ragged bf16 layers with
offload, host accumulation, f1, K7, warm-up and Zen-auto, plus the stateless primitives."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2505_12242_b200 import zf  # noqa: E402
from synth import gpu  # noqa: E402

shapes = [(37, 1001), (64, 512), (5, 2000), (130, 257)]
for kw in ({}, {"cpu_update": True}, {"device_accumulate": True}, {"warmup_steps": 2, "auto_gamma": 0.2}):
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=100000, refresh_interval=2,
                     accum_interval=2, offload=True, host_accumulate=True, **kw)
    Gs = [torch.empty(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    Ps = [torch.zeros(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    scs = [gpu.ColScale(m, i) for i, (n, m) in enumerate(shapes)]
    for t in range(5):
        for i, (G, sc) in enumerate(zip(Gs, scs)):
            sc.advance_to(t)
            gpu.fill_grad(G, i, t, sc)
        ctx.step(t, Gs, Ps)
    ctx.sync()
    ctx.close()
G = Gs[0]
norms = torch.empty(G.shape[1], device="cuda")
zf.zf_column_norms(G, norms)
idx = torch.empty(zf.k_for(G.shape[1], 100000), dtype=torch.int32, device="cuda")
zf.zf_topk_columns(norms, idx.numel(), idx)
out = torch.empty(G.shape[0] * (G.shape[1] - idx.numel()), dtype=torch.bfloat16, device="cuda")
zf.zf_compact_unselected(G, idx, out)
torch.cuda.synchronize()
print("sanitize run ok")
