"""Mutation test of the GPU parity suite: apply one plausible slip at a time to a scratch copy
of the CUDA / host runtime sources (libzf.so), rebuild, and run `pytest tests -m gpu -x`
against it.  A mutant the suite does not catch marks a path the parity tests do not pin.
Runs on the GPU box (sequentially; one GPU).  The product tree is never modified.

usage: python tools/mutate_gpu.py [-k SUBSTR] [--out FILE]"""
import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CS = "paper_2505_12242_b200/csrc/"
NORMS, TOPK, UPD, INT, ACC, HOST, SCAT, DRV, AUTO, PEER, ADAM = (CS + f for f in (
    "k_norms.cu", "k_topk.cu", "k_update.cu", "zf_internal.cuh", "k_accum.cu", "zf_host.cu", "k_scatter.cu",
    "zf_driver.cu", "k_auto.cu", "k_peer.cu", "k_adam.cu"))

# (name, file, [(old, new, occurrence)])  occurrence: 0-based index of `old` to replace
MUTANTS = [
    ("K1 x*|x| in the unrolled row loop", NORMS, [("acc[e] = fmaf(x, x, acc[e]);", "acc[e] = fmaf(x, fabsf(x), acc[e]) - 2.0f * fminf(x, 0.0f) * x;", 0)]),
    ("K1 tail rows dropped", NORMS, [("acc[e] = fmaf(x, x, acc[e]);", "acc[e] = acc[e];", 1)]),
    ("K1 last row block not reduced", NORMS, [("for (int b = 1; b < L.nrb; ++b)", "for (int b = 1; b + 1 < L.nrb; ++b)", 0)]),
    ("K1 last warp not reduced", NORMS, [("for (int w = 1; w < K1_WARPS; ++w) s += red[w][c];", "for (int w = 1; w + 1 < K1_WARPS; ++w) s += red[w][c];", 0)]),
    ("K2 ties to the higher index", TOPK, [("uint32_t eq_base = block_excl_scan(n_eq, warp_sums, &tot);", "uint32_t eq_base = block_excl_scan(n_eq, warp_sums, &tot);\n    const uint32_t teq = tot;", 0),
                                           ("else if (key == T) { n_sel += (e < rem); ++e; }", "else if (key == T) { n_sel += (e >= teq - rem); ++e; }", 0),
                                           ("else if (key == T) { sel = (e < rem); ++e; }", "else if (key == T) { sel = (e >= teq - rem); ++e; }", 0)]),
    ("K2 every tie selected", TOPK, [("if (key > T) ++n_sel;", "if (key >= T) ++n_sel;", 0), ("if (key > T) sel = true;", "if (key >= T) sel = true;", 0)]),
    ("K2 entering slot step count 1", TOPK, [("L.new_steps[s] = src >= 0 ? __ldg(L.old_steps + src) + old_delta : 0;", "L.new_steps[s] = src >= 0 ? __ldg(L.old_steps + src) + old_delta : 1;", 0)]),
    ("K2 remap source off by one", TOPK, [("if (word & bit) src = __ldg(L.old_prefix + (c >> 5)) + __popc(word & (bit - 1u));", "if (word & bit) src = __ldg(L.old_prefix + (c >> 5)) + __popc(word & (bit - 1u)) + (c & 1);", 0)]),
    ("K3 m with beta2", INT, [("m = __fadd_rn(__fmul_rn(h.b1, m), __fmul_rn(h.omb1, g));", "m = __fadd_rn(__fmul_rn(h.b2, m), __fmul_rn(h.omb1, g));", 0)]),
    ("K3 eps dropped", INT, [("const float den = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), bc2s), h.eps);", "const float den = __fdiv_rn(__fsqrt_rn(v), bc2s);", 0)]),
    ("K3 update sign", INT, [("p = __fsub_rn(p, __fmul_rn(ss, __fdiv_rn(m, den)));", "p = __fadd_rn(p, __fmul_rn(ss, __fdiv_rn(m, den)));", 0)]),
    ("K3 decoupled decay dropped", INT, [("if (h.wd_mode == 1) p = __fmul_rn(p, h.decay);", "if (h.wd_mode == 3) p = __fmul_rn(p, h.decay);", 0)]),
    ("K3 L2 decay sign", INT, [("else if (h.wd_mode == 2) g = __fadd_rn(g, __fmul_rn(h.wd, p));", "else if (h.wd_mode == 2) g = __fsub_rn(g, __fmul_rn(h.wd, p));", 0)]),
    ("K3 v from |g|", INT, [("v = __fadd_rn(__fmul_rn(h.b2, v), __fmul_rn(__fmul_rn(h.omb2, g), g));", "v = __fadd_rn(__fmul_rn(h.b2, v), __fmul_rn(__fmul_rn(h.omb2, g), fabsf(g)));", 0)]),
    ("K3 bias correction past the table", INT, [("return t < h.sb_len ? __ldg(h.sb_tab + t) : make_float2(h.ss_inf, 1.0f);", "return t < h.sb_len ? __ldg(h.sb_tab + t) : make_float2(h.ss_inf, 0.5f);", 0)]),
    ("K3 v stores m", UPD, [("__stcs(si.v_out + so[j], vv[j]);", "__stcs(si.v_out + so[j], mm[j]);", 0)]),
    ("K3 changed p not stored", UPD, [("if (pnew != po[j]) gP[pa[j]] = pnew;\n                    if (pmode == 1", "if (false) gP[pa[j]] = pnew;\n                    if (pmode == 1", 0)]),
    ("K3 subset block not updated", UPD, [("if (pmode == 1 || pmode == 3 || (pmode == 2 && pnew != po[j])) gS[so[j]] = pnew;", "if (pmode == 1 || pmode == 3) gS[so[j]] = pnew;", 0)]),
    ("K3 remap entering moments stale", UPD, [("mm[j] = ok ? sM[src[j]] : 0.0f;", "mm[j] = ok ? sM[src[j]] : sM[so[j] - s0];", 0)]),
    ("K3 compaction halves swapped", UPD, [("o.w = lds_u16(rowa + (u.w & 0xffffu)) | (lds_u16(rowa + (u.w >> 16)) << 16);", "o.w = lds_u16(rowa + (u.w >> 16)) | (lds_u16(rowa + (u.w & 0xffffu)) << 16);", 0)]),
    ("K3 compaction head/tail offset +1", UPD, [("const uint32_t bo = ((uint32_t)__ldg(gU + q) - base) & 0xffffu;", "const uint32_t bo = ((uint32_t)__ldg(gU + q) - base + GSZ) & 0xffffu;", 0)]),
    ("K3 last tail output dropped", UPD, [("if (e - OPL >= tail) continue;", "if (e - OPL >= tail - 1) continue;", 0)]),
    ("K7 window start not zeroed", ACC, [("if (!first) {\n            a0 = __ldcs", "if (true) {\n            a0 = __ldcs", 0)]),
    ("K7 one add dropped", ACC, [("a1.z = __fadd_rn(a1.z, x[6]);", "a1.z = x[6];", 0)]),
    ("H1 window start not zeroed (batched)", HOST, [("            for (int64_t i = 0; i < w; ++i) tmp[i] = 0.0f;", "            for (int64_t i = 0; i < w; ++i) tmp[i] = acc[c0 + i];", 0)]),
    ("H1 add dropped (batched)", HOST, [("tmp[i] = tmp[i] + f;", "tmp[i] = f;", 0)]),
    ("f1 window average by S-1", HOST, [("float g = acc[u] / Sf;", "float g = acc[u] / (Sf > 1.0f ? Sf - 1.0f : Sf);", 0)]),
    ("f1 eps dropped", HOST, [("const float den = std::sqrt(vv) / bc2s[u] + eps;", "const float den = std::sqrt(vv) / bc2s[u];", 0)]),
    ("f1 bf16 truncation", HOST, [("const uint32_t rne = (x + 0x7fffu + ((x >> 16) & 1u)) >> 16;", "const uint32_t rne = x >> 16;", 0)]),
    ("K5 scatter column shifted", SCAT, [("P[i * ldp + __ldg(unsel + u)] = buf[q];", "P[i * ldp + __ldg(unsel + (u > 0 ? u - 1 : u))] = buf[q];", 0)]),
    ("driver refresh every step", DRV, [("const bool refresh = (t % N) == 0;", "const bool refresh = true;", 0)]),
    ("driver window end off by one", DRV, [("bool end = (t + 1) % c->cfg.accum_interval == 0;", "bool end = t % c->cfg.accum_interval == 0;", 0)]),
    ("K6 gamma ignored", AUTO, [("(st.A > 0.0 && st.A >= gamma * i)", "(st.A > 0.0 && st.A >= i)", 0)]),
    # batch 2: exchange, non-finite detection, dense AdamW, Zen-auto / K7 state, f1 gather, lag ordering
    ("peer reduce drops the last rank", PEER, [("for (int q = 1; q < a.world; ++q) s = __fadd_rn", "for (int q = 1; q + 1 < a.world; ++q) s = __fadd_rn", 0)]),
    ("peer gather skips rank 0's slice", PEER, [("for (int q = 0; q < a.world; ++q) {\n        const int64_t j0 = a.M * q / a.world", "for (int q = 1; q < a.world; ++q) {\n        const int64_t j0 = a.M * q / a.world", 0)]),
    ("lagged refresh does not wait for the side-stream norms", DRV, [("if (c->lag_pending) ZF_CUDA(cudaStreamWaitEvent(s, c->norm_ready, 0));", "(void)0;", 0)]),
    ("K1 non-finite flag dropped", NORMS, [("if (!isfinite(s) && nonfinite) *nonfinite = 1;", "(void)s;", 0), ("if (!isfinite(s) && nonfinite) *nonfinite = 1;", "(void)s;", 0)]),
    ("K3 AdamW non-finite check dropped", UPD, [("if constexpr (GE::SIZE == 2) nfacc |= ((uint32_t)gb[j] & 0x7f80u) + 0x0080u;", "if constexpr (GE::SIZE == 2) (void)0;", 0)]),
    ("K3 compaction non-finite check dropped", UPD, [("nf2 = __hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.x)),", "(void)__hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.x)),", 0),
                                                    ("nf2 = __hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.z)),", "(void)__hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.z)),", 0)]),
    ("dense AdamW remap entering moment 1e-3", ADAM, [("m = src >= 0 ? L.m_in[row * L.k_in + src] : 0.0f;", "m = src >= 0 ? L.m_in[row * L.k_in + src] : 1.0e-3f;", 0),
                                                      ("m[j] = src >= 0 ? __ldcs(L.m_in + (int64_t)row * L.k_in + src) : 0.0f;", "m[j] = src >= 0 ? __ldcs(L.m_in + (int64_t)row * L.k_in + src) : 1.0e-3f;", 0)]),
    ("dense AdamW range-miss fallback skipped", ADAM, [("    if (!ok) {\n#pragma unroll\n        for (int j = 0; j < V; ++j) {", "    if (false) {\n#pragma unroll\n        for (int j = 0; j < V; ++j) {", 0)]),
    ("K6 smax off by one", AUTO, [("st.len >= smax", "st.len > smax", 0)]),
    ("K7 Zen-auto buffer parity", ACC, [("buf = (int)(st->win & 1);", "buf = (int)((st->win + 1) & 1);", 0)]),
    ("f1 refresh gather column shifted", SCAT, [("buf[q] = P[i * ldp + __ldg(cols + e)];", "buf[q] = P[i * ldp + __ldg(cols + (e > 0 ? e - 1 : e))];", 0)]),

    # batch 3: launch-table patches, remap step delta, H1 one-step adds, warm-up length, K6 statistic, X1 gate
    ("k_patch skips the last word", CS + "zf_prim.cu", [("for (int i = threadIdx.x; i < a.n; i += blockDim.x) a.base[a.off[i]] = a.val[i];", "for (int i = threadIdx.x; i + 1 < a.n; i += blockDim.x) a.base[a.off[i]] = a.val[i];", 0)]),
    ("K2 remap step delta dropped", TOPK, [("L.new_steps[s] = src >= 0 ? __ldg(L.old_steps + src) + old_delta : 0;", "L.new_steps[s] = src >= 0 ? __ldg(L.old_steps + src) : 0;", 0)]),
    ("H1 one-step add dropped", HOST, [("            acc[i] = acc[i] + x;", "            acc[i] = x;", 0)]),
    ("warm-up one step longer", DRV, [("if (t0 < tau) return warmup_step(c, t0, grads, params, s);", "if (t0 <= tau) return warmup_step(c, t0, grads, params, s);", 0)]),
    ("K6 sums squared norms", AUTO, [("const double x = sqrt((double)__ldg(L.norms + j));", "const double x = (double)__ldg(L.norms + j);", 0)]),
    ("X1 copy gated one unit early", DRV, [("c->done_target[c->L[i].chunk] += (uint32_t)(steady_geo ? c->L[i].geo_s.units : c->L[i].geo.units) *", "c->done_target[c->L[i].chunk] += (uint32_t)((steady_geo ? c->L[i].geo_s.units : c->L[i].geo.units) - 1) *", 0)]),
    # batch 4: the refresh from the previous parameter-subset block (psub_mode 3)
    ("K3 subset refresh: retained value from the new slot", UPD, [("po[j] = src[j] >= row * kin ? sPs[src[j]] : gP[pa[j] + c0 + cc[j]];", "po[j] = src[j] >= row * kin ? sPs[so[j] - s0] : gP[pa[j] + c0 + cc[j]];", 0)]),
    ("K3 subset refresh: entering value zero", UPD, [("po[j] = src[j] >= row * kin ? sPs[src[j]] : gP[pa[j] + c0 + cc[j]];", "po[j] = src[j] >= row * kin ? sPs[src[j]] : (PB)0;", 0)]),
    ("subset blocks not ping-ponged", DRV, [("t.psub_in = blk[cur];", "t.psub_in = blk[nw];", 0)]),
    ("subset refresh ignores psub_valid", DRV, [("c->have_sel && c->psub_valid &&", "c->have_sel &&", 0)]),
    ("subset refresh block not rebuilt", UPD, [("if (pmode == 1 || pmode == 3 || (pmode == 2 && pnew != po[j])) gS[so[j]] = pnew;", "if (pmode == 1 || (pmode >= 2 && pnew != po[j])) gS[so[j]] = pnew;", 0)]),
]


def apply(src, edits):
    for old, new, occ in edits:
        pos = -1
        for _ in range(occ + 1):
            pos = src.find(old, pos + 1)
            if pos < 0:
                raise ValueError(f"pattern not found: {old[:60]!r}")
        src = src[:pos] + new + src[pos + len(old):]
    return src


def run_one(mut, timeout):
    name, f, edits = mut
    d = tempfile.mkdtemp(prefix="zfgmut_")
    t0 = time.time()
    try:
        ign = shutil.ignore_patterns(".git", "gpurun_out", "baseline", "__pycache__", "*.ncu-rep")
        shutil.copytree(ROOT, os.path.join(d, "r"), ignore=ign, symlinks=True)   # copy2: mtimes kept
        r = os.path.join(d, "r")
        p = os.path.join(r, f)
        try:
            new = apply(open(p).read(), edits)
        except ValueError as e:
            return name, "BAD-PATTERN", str(e), 0.0
        open(p, "w").write(new)
        b = subprocess.run([sys.executable, "-m", "paper_2505_12242_b200._build"], cwd=r, capture_output=True, text=True)
        if b.returncode != 0:
            return name, "BUILD-FAILED", b.stderr[-300:], time.time() - t0
        try:
            t = subprocess.run([sys.executable, "-m", "pytest", "tests", "-m", "gpu", "-x", "-q", "-p", "no:cacheprovider"],
                               cwd=r, capture_output=True, text=True, timeout=timeout)
        except subprocess.TimeoutExpired:
            return name, "KILLED", "timeout (hang)", time.time() - t0
        tail = (t.stdout.strip().splitlines() or [""])[-1]
        if t.returncode == 0:
            return name, "SURVIVED", tail, time.time() - t0
        failed = [l for l in t.stdout.splitlines() if l.startswith("FAILED") or l.startswith("ERROR")]
        return name, "KILLED", (failed[0] if failed else tail)[:200], time.time() - t0
    finally:
        shutil.rmtree(d, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    ap.add_argument("--timeout", type=int, default=600)
    ap.add_argument("--check", action="store_true", help="apply + compile each mutant only (no GPU)")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "gpu_mutation.json"))
    a = ap.parse_args()
    if a.check:
        from concurrent.futures import ThreadPoolExecutor

        def chk(m):
            name, f, edits = m
            try:
                new = apply(open(os.path.join(ROOT, f)).read(), edits)
            except ValueError as e:
                return name, str(e)
            d = tempfile.mkdtemp(prefix="zfgchk_")
            try:
                shutil.copytree(os.path.join(ROOT, "paper_2505_12242_b200"), os.path.join(d, "paper_2505_12242_b200"),
                                ignore=shutil.ignore_patterns("__pycache__", "build", "*.so"))
                shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
                open(os.path.join(d, f), "w").write(new)
                src = os.path.join(d, f if f.endswith(".cu") else CS + "k_update.cu")
                r = subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17",
                                    "-I", os.path.join(d, "include"), "-I", os.environ.get("NCCL_INC", "/usr/include"),
                                    "-c", src, "-o", os.path.join(d, "x.o")], capture_output=True, text=True)
                return name, "ok" if r.returncode == 0 else r.stderr[-400:]
            finally:
                shutil.rmtree(d, ignore_errors=True)
        with ThreadPoolExecutor(8) as ex:
            for name, st in ex.map(chk, [m for m in MUTANTS if a.k in m[0]]):
                print(f"{name:42s} {st}")
        return
    res = []
    for m in MUTANTS:
        if a.k not in m[0]:
            continue
        r = run_one(m, a.timeout)
        res.append(r)
        print(f"{r[1]:12s} {r[0]:42s} {r[3]:6.0f}s {r[2]}", flush=True)
        with open(a.out, "w") as fh:
            json.dump({"suite": "pytest tests -m gpu -x", "mutants": [
                {"mutant": n, "result": s, "detail": str(i), "seconds": round(t, 1)} for n, s, i, t in res]}, fh, indent=1)
    killed = sum(1 for r in res if r[1] == "KILLED")
    print(f"{killed}/{len(res)} killed")


if __name__ == "__main__":
    main()
