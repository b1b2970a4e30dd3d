"""Small zf_step runs for compute-sanitizer (memcheck / racecheck): ragged bf16 layers with
offload, host accumulation, f1, K7, warm-up and Zen-auto, host staging slots, lagged
selection, grouped refresh, a one-rank NCCL communicator, state swap-out, overlapped f1,
p tiles on steady steps (no parameter subset), alternating gradient buffers and many X1
chunks, plus the stateless primitives."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2505_12242_b200 import zf  # noqa: E402
from synth import gpu  # noqa: E402

shapes = [(37, 1001), (64, 512), (5, 2000), (130, 257)]
os.environ["ZF_X1_CHUNK_KB"] = "16"   # several X1 chunks even at these sizes
for kw in ({}, {"cpu_update": True}, {"device_accumulate": True}, {"warmup_steps": 2, "auto_gamma": 0.2},
           {"host_stages": 8, "cpu_update": True}, {"lagged_selection": True},
           {"refresh_group_mb": 1}, {"nccl_id": zf.zf_nccl_unique_id()}, {"state_offload": True},
           {"cpu_update": True, "cpu_update_async": True}, {"param_subset": False}):
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=100000, refresh_interval=2,
                     accum_interval=2, offload=True, host_accumulate=True, **kw)
    # two gradient buffers, alternated as a training loop would (launch tables patched by k_patch)
    Gb = [[torch.empty(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes] for _ in range(2)]
    Ps = [torch.zeros(n, m, dtype=torch.bfloat16, device="cuda") for n, m in shapes]
    scs = [gpu.ColScale(m, i) for i, (n, m) in enumerate(shapes)]
    for t in range(7):
        Gs = Gb[t % 2]
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
M = torch.zeros(G.shape[0], idx.numel(), device="cuda")
V = torch.zeros_like(M)
st = torch.zeros(idx.numel(), dtype=torch.int32, device="cuda")
zf.zf_selective_adam(Ps[0], G, idx, M, V, st, zf.adam_params())
torch.cuda.synchronize()
print("sanitize run ok")
