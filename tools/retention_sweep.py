"""f4 workload: retention-rate sweep of the channel selection on the synthetic gradients
("Temporal Locality ... the retention rate -- the fraction of previously
selected channels that continue to contain top-k gradients across 100 steps"; SPEC
S:122-130).

Runs the product kernels (K1 zf_column_norms, K2 zf_topk_columns through the C-ABI) on
the seeded column-concentrated generator for the 7 linears of one
Llama-2-7B decoder block, T steps, and reports for each top-k ratio:
  * consecutive retention |S_t & S_{t-1}| / k, averaged over t and matrices;
  * retention against step 0, |S_0 & S_t| / k, at t = 1, 4, 16, 64, T-1;
  * retention across one refresh period N = 4, |S_t & S_{t+4}| / k.
  * P:328's retention rate (fig. ratention_rate): the fraction of step t's top-1% gradient
    ELEMENTS (by magnitude) that lie in the fixed top-k% channel set chosen at step 0, at
    t = 1, 4, 16, 64, T-1 (the paper: > 95% over 100 iterations at 10%, > 90% at 5%).
It measures the generator's temporal locality (its calibrated per-step column redraw)
against the paper's numbers; it is not a benchmark.

usage (GPU box): python tools/retention_sweep.py [--steps 100] [--out profiles/r02_retention.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_retention.json"))
    args = ap.parse_args()
    import torch

    import synth
    from paper_2505_12242_b200 import _build
    _build.build()
    from paper_2505_12242_b200 import zf
    from synth import gpu

    shapes = [(n, m) for _, n, m in synth.llama2_7b_linears()[:7]]
    ratios = [10000, 30000, 50000, 100000]
    T = args.steps
    sels = {r: [[] for _ in shapes] for r in ratios}
    elem = {r: {} for r in ratios}          # P:328 element retention per probe step
    probes = [t for t in (1, 4, 16, 64, T - 1) if 0 < t < T]
    for li, (n, m) in enumerate(shapes):
        G = torch.empty(n, m, dtype=torch.bfloat16, device="cuda")
        norms = torch.empty(m, dtype=torch.float32, device="cuda")
        sc = gpu.ColScale(m, li)
        idx = {r: torch.empty(zf.k_for(m, r), dtype=torch.int32, device="cuda") for r in ratios}
        fixed_masks = globals().setdefault("_fixed", {})
        for t in range(T):
            sc.advance_to(t)
            gpu.fill_grad(G, li, t, sc)
            zf.zf_column_norms(G, norms)
            for r in ratios:
                zf.zf_topk_columns(norms, idx[r].numel(), idx[r])
                sels[r][li].append(set(idx[r].cpu().tolist()))
                if t == 0:
                    fixed = fixed_masks.setdefault(r, {})
                    mk = torch.zeros(m, dtype=torch.bool, device="cuda")
                    mk[idx[r].long()] = True
                    fixed[li] = mk
            if t in probes:
                a = G.float().abs()
                kk = max(1, a.numel() // 100)
                kth = torch.topk(a.view(-1), kk).values[-1]
                top = a >= kth
                for r in ratios:
                    frac = (top & fixed_masks[r][li][None, :]).sum().item() / top.sum().item()
                    elem[r].setdefault(t, []).append(frac)
    out = {"workload": "llama2-7b block-0 linears (7 matrices), synthetic column-concentrated bf16 gradients",
           "steps": T, "generator": f"per-column scale redrawn w.p. {synth.REDRAW_THRESHOLD / 2**32:.4%} per step "
                                    "(DESIGN.md §4, calibrated to P:328)", "ratios": {}}
    for r in ratios:
        cons, vs0, acrossN = [], {}, []
        for li, (n, m) in enumerate(shapes):
            k = zf.k_for(m, r)
            S = sels[r][li]
            cons += [len(S[t] & S[t - 1]) / k for t in range(1, T)]
            acrossN += [len(S[t] & S[t + 4]) / k for t in range(0, T - 4)]
            for t in (1, 4, 16, 64, T - 1):
                if t < T:
                    vs0.setdefault(t, []).append(len(S[0] & S[t]) / k)
        out["ratios"][f"{r / 1e4:g}%"] = {
            "consecutive": sum(cons) / len(cons),
            "across_refresh_N4": sum(acrossN) / len(acrossN),
            "vs_step0": {str(t): sum(v) / len(v) for t, v in sorted(vs0.items())},
            "top1pct_element_retention_fixed_step0_channels": {str(t): sum(v) / len(v) for t, v in sorted(elem[r].items())}}
    txt = json.dumps(out, indent=1)
    print(txt)
    with open(args.out, "w") as f:
        f.write(txt + "\n")


if __name__ == "__main__":
    main()
