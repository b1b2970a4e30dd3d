"""Per-step K3 time (refresh vs steady steps) on full Llama-2-7B for a set of context
options -- the A/B harness for K3 changes.  usage: python tools/k3_steps.py [ppm] [lr] [steps]
prints one JSON line per option set: K3 ms of every step, refresh mean, steady mean."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2505_12242_b200 import _build  # noqa: E402

_build.build()
from paper_2505_12242_b200 import zf  # noqa: E402
from synth import gpu  # noqa: E402

ppm = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
lr = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-5
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
model = os.environ.get("ZF_MODEL", "llama2-7b")
shapes = [(n, m) for _, n, m in synth.MODELS[model]()]
tot = sum(n * m for n, m in shapes)
bufs = [torch.empty(tot, dtype=torch.bfloat16, device="cuda") for _ in range(3)]


def views(b):
    out, off = [], 0
    for n, m in shapes:
        out.append(b[off:off + n * m].view(n, m))
        off += n * m
    return out


G0, G1, P = views(bufs[0]), views(bufs[1]), views(bufs[2])
for li, (n, m) in enumerate(shapes):
    sc = gpu.ColScale(m, li)
    gpu.fill_grad(G0[li], li, 0, sc)
    sc.advance_to(1)
    gpu.fill_grad(G1[li], li, 1, sc)
    gpu.fill_param(P[li], li)
torch.cuda.synchronize()
opts = [dict(param_subset=True), dict(param_subset=False)]
if os.environ.get("ZF_OPTS"):
    opts = [json.loads(x) for x in os.environ["ZF_OPTS"].split(";")]
for o in opts:
    ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=ppm, refresh_interval=4,
                     accum_interval=4, adam=zf.adam_params(lr=lr), **o)
    ks, ka, kb = [], [], []
    for t in range(steps):
        ctx.profile(True)
        ctx.step(t, G0 if t % 2 == 0 else G1, P)
        pr = ctx.profile_read()
        ks.append(round(pr["k3_update"][0] + pr["k3b_adam"][0], 3))
        ka.append(round(pr["k3_update"][0], 3))
        kb.append(round(pr["k3b_adam"][0], 3))
    ctx.sync()
    ctx.close()
    ref = [x for t, x in enumerate(ks) if t % 4 == 0 and t >= 4]
    st = [x for t, x in enumerate(ks) if t % 4 != 0 and t >= 4]
    print(json.dumps({"opts": o, "ppm": ppm, "lr": lr, "k3_ms": ks, "k3a_ms": ka, "k3b_ms": kb, "refresh": sum(ref) / len(ref),
                      "steady": sum(st) / len(st), "avg": (sum(ref) / len(ref) + 3 * sum(st) / len(st)) / 4}),
          flush=True)
