"""Mutation test of the CPU oracle's pins: apply one plausible mistake at a time to a
scratch copy of oracle/ (a dropped term, a wrong sign / index / operand, an off-by-one in
the schedule) and run the CPU pin suite (tests/test_oracle_pins.py) against it.  A mutant
that passes every pin marks an unpinned part of the oracle.

usage: python tools/mutate_oracle.py [-j JOBS] [-k SUBSTR]
prints one line per mutant (KILLED / SURVIVED) and writes profiles/oracle_mutation.json."""
import argparse
import json
import os
import shutil
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP, PY = "oracle/zf_oracle.cpp", "oracle/oracle.py"

# (name, file, old text, new text) -- each `old` must occur exactly once
MUTANTS = [
    # O1 norms
    ("O1 sum of |x| instead of x^2", CPP, "s += x * x;\n        }\n        if (!std::isfinite(s)) bad = 1;", "s += std::fabs(x);\n        }\n        if (!std::isfinite(s)) bad = 1;"),
    ("O1 L2 norm (sqrt) instead of squared", CPP, "norms[j] = static_cast<float>(s);", "norms[j] = static_cast<float>(std::sqrt(s));"),
    ("O1 skips the last row", CPP, "for (int64_t i = 0; i < n; ++i) {\n            double x = static_cast<double>(load(G, dt, i * ld + j));\n            s += x * x;\n        }\n        if", "for (int64_t i = 0; i + 1 < n; ++i) {\n            double x = static_cast<double>(load(G, dt, i * ld + j));\n            s += x * x;\n        }\n        if"),
    ("O1 reads with ld = m", CPP, "double x = static_cast<double>(load(G, dt, i * ld + j));\n            s += x * x;\n        }\n        if", "double x = static_cast<double>(load(G, dt, i * m + j));\n            s += x * x;\n        }\n        if"),
    ("O1 fp32 accumulation", CPP, "double s = 0.0;\n        for (int64_t i = 0; i < n; ++i) {\n            double x = static_cast<double>(load(G, dt, i * ld + j));\n            s += x * x;\n        }\n        if", "float s = 0.0f;\n        for (int64_t i = 0; i < n; ++i) {\n            float x = load(G, dt, i * ld + j);\n            s += x * x;\n        }\n        if"),
    # O2 k
    ("O2 k = floor", CPP, "+ 999999) / 1000000;", ") / 1000000;"),
    ("O2 k = round", CPP, "+ 999999) / 1000000;", "+ 500000) / 1000000;"),
    ("O2 no k >= 1 clamp", CPP, "if (k < 1) k = 1;", ""),
    # O3 top-k
    ("O3 smallest norms", CPP, "return norms[a] > norms[b]; });", "return norms[a] < norms[b]; });"),
    ("O3 ties -> higher index", CPP, "std::iota(order.begin(), order.end(), 0);", "std::iota(order.begin(), order.end(), 0); std::reverse(order.begin(), order.end());"),
    ("O3 output in rank order", CPP, "std::sort(sel.begin(), sel.end());", ""),
    ("O3 k-1 columns + last", CPP, "std::vector<int32_t> sel(order.begin(), order.begin() + k);", "std::vector<int32_t> sel(order.begin(), order.begin() + k); if (k > 1 && m > k) sel[k - 1] = order[k];"),
    # O4 map
    ("O4 upos counts selected too", CPP, "if (slot[j] < 0) upos[j] = u++;", "{ if (slot[j] < 0) upos[j] = u; ++u; }"),
    # O5 remap
    ("O5 entering step count 1", CPP, "step_new[s] = src >= 0 ? step_old[src] : 0;", "step_new[s] = src >= 0 ? step_old[src] : 1;"),
    ("O5 retained step count reset", CPP, "step_new[s] = src >= 0 ? step_old[src] : 0;", "step_new[s] = 0;"),
    ("O5 retained v zeroed", CPP, "v_new[i * k_new + s] = src >= 0 ? v_old[i * k_old + src] : 0.0f;", "v_new[i * k_new + s] = 0.0f;"),
    ("O5 retained m zeroed", CPP, "m_new[i * k_new + s] = src >= 0 ? m_old[i * k_old + src] : 0.0f;", "m_new[i * k_new + s] = 0.0f;"),
    ("O5 slot index instead of source", CPP, "m_new[i * k_new + s] = src >= 0 ? m_old[i * k_old + src] : 0.0f;", "m_new[i * k_new + s] = (src >= 0 && s < k_old) ? m_old[i * k_old + s] : 0.0f;"),
    ("O5 m/v swapped", CPP, "m_new[i * k_new + s] = src >= 0 ? m_old[i * k_old + src] : 0.0f;\n            v_new[i * k_new + s] = src >= 0 ? v_old[i * k_old + src] : 0.0f;", "m_new[i * k_new + s] = src >= 0 ? v_old[i * k_old + src] : 0.0f;\n            v_new[i * k_new + s] = src >= 0 ? m_old[i * k_old + src] : 0.0f;"),
    # O6 AdamW
    ("O6 no decoupled decay", CPP, "if (weight_decay != 0.0 && decoupled) p = p * decay;", ""),
    ("O6 decay = 1 - wd", CPP, "const float decay = static_cast<float>(1.0 - lr * weight_decay);", "const float decay = static_cast<float>(1.0 - weight_decay);"),
    ("O6 L2 decay sign", CPP, "g = g + wp;", "g = g - wp;"),
    ("O6 L2 decay dropped", CPP, "g = g + wp;", "(void)wp;"),
    ("O6 beta1 <-> beta2 in m", CPP, "float a1 = b1 * m;", "float a1 = b2 * m;"),
    ("O6 m without (1-b1)", CPP, "float a2 = omb1 * g;", "float a2 = g;"),
    ("O6 v from |g| not g^2", CPP, "float c3 = c2 * g;", "float c3 = c2 * std::fabs(g);"),
    ("O6 v with (1-b1)", CPP, "float c2 = omb2 * g;", "float c2 = omb1 * g;"),
    ("O6 no sqrt", CPP, "float sq = std::sqrt(v);", "float sq = v;"),
    ("O6 bc2 without sqrt", CPP, "const float bc2s = static_cast<float>(std::sqrt(1.0 - std::pow(beta2, static_cast<double>(t))));", "const float bc2s = static_cast<float>(1.0 - std::pow(beta2, static_cast<double>(t)));"),
    ("O6 no bias correction 2", CPP, "float q = sq / bc2s;", "float q = sq;"),
    ("O6 bc2 multiplied", CPP, "float q = sq / bc2s;", "float q = sq * bc2s;"),
    ("O6 eps inside sqrt", CPP, "float sq = std::sqrt(v);\n            float q = sq / bc2s;\n            float den = q + eps_f;", "float sq = std::sqrt(v + eps_f);\n            float q = sq / bc2s;\n            float den = q;"),
    ("O6 eps dropped", CPP, "float den = q + eps_f;", "float den = q;"),
    ("O6 eps before bias correction", CPP, "float q = sq / bc2s;\n            float den = q + eps_f;", "float q = sq + eps_f;\n            float den = q / bc2s;"),
    ("O6 no bias correction 1", CPP, "const float ss = static_cast<float>(lr / (1.0 - std::pow(beta1, static_cast<double>(t))));", "const float ss = static_cast<float>(lr);"),
    ("O6 bias correction 1 with t-1", CPP, "lr / (1.0 - std::pow(beta1, static_cast<double>(t)))", "lr / (1.0 - std::pow(beta1, static_cast<double>(t > 1 ? t - 1 : t)))"),
    ("O6 bias correction 1 uses beta2", CPP, "const float ss = static_cast<float>(lr / (1.0 - std::pow(beta1, static_cast<double>(t))));", "const float ss = static_cast<float>(lr / (1.0 - std::pow(beta2, static_cast<double>(t))));"),
    ("O6 step count not advanced", CPP, "step[s] = t;", ""),
    ("O6 update sign", CPP, "p = p - delta;", "p = p + delta;"),
    ("O6 update from g instead of m", CPP, "float upd = m / den;", "float upd = g / den;"),
    ("O6 moments stored before update", CPP, "M[i * k + s] = m;", "M[i * k + s] = a1;"),
    # bf16 rounding
    ("bf16 round half up", CPP, "u += 0x7fffu + lsb;", "u += 0x8000u;"),
    ("bf16 truncation", CPP, "u += 0x7fffu + lsb;", "(void)lsb;"),
    # O7 compaction
    ("O7 keeps selected columns", CPP, "if (selected[static_cast<size_t>(j)]) continue;\n            copy_elem", "if (!selected[static_cast<size_t>(j)]) continue;\n            copy_elem"),
    # O8 accumulation
    ("O8 overwrite instead of add", CPP, "acc[e] = acc[e] + x;", "acc[e] = x;"),
    ("O8 adds bf16-rounded sum", CPP, "acc[e] = acc[e] + x;", "acc[e] = bf16_to_f32(f32_to_bf16_rne(acc[e] + x));"),
    # O11 / O12 Zen-auto
    ("O11 squared norms summed", CPP, "const double x = std::sqrt(static_cast<double>(norms[j]));", "const double x = static_cast<double>(norms[j]);"),
    ("O11 selected/unselected swapped", CPP, "sums[0] = sel;\n    sums[1] = unsel;", "sums[0] = unsel;\n    sums[1] = sel;"),
    ("O12 A not accumulated", CPP, "*A = *A + u;", "*A = u;"),
    ("O12 strict comparison", CPP, "return (*A > 0.0 && *A >= gamma * i) ? 1 : 0;", "return (*A > 0.0 && *A > gamma * i) ? 1 : 0;"),
    ("O12 gamma ignored", CPP, "return (*A > 0.0 && *A >= gamma * i) ? 1 : 0;", "return (*A > 0.0 && *A >= i) ? 1 : 0;"),
    ("O12 smax off by one", CPP, "if (force_end || *len >= smax) return 1;", "if (force_end || *len > smax) return 1;"),
    ("O12 force_end ignored", CPP, "if (force_end || *len >= smax) return 1;", "if (*len >= smax) return 1;"),
    ("O12 sums over all columns", CPP, "const double u = unsel_cnt > 0 ? unsel_sum / static_cast<double>(unsel_cnt) : 0.0;", "const double u = unsel_cnt > 0 ? unsel_sum / static_cast<double>(unsel_cnt + sel_cnt) : 0.0;"),
    # step driver (oracle.py)
    ("R6 refresh at t % N == 1", PY, "if t % self.refresh_interval == 0 or self.idx is None:", "if t % self.refresh_interval == 1 or self.idx is None:"),
    ("R6 refresh every step", PY, "if t % self.refresh_interval == 0 or self.idx is None:", "if True:"),
    ("R7 remap replaced by reset", PY, "self.M, self.V, self.steps = remap(self.n, self.idx, self.M, self.V, self.steps, new_idx)", "self.M = np.zeros((self.n, k), np.float32); self.V = np.zeros((self.n, k), np.float32); self.steps = np.zeros(k, np.int32)"),
    ("O8 window not zeroed", PY, "        if first:\n            self.acc[a][...] = 0.0", "        if False:\n            self.acc[a][...] = 0.0"),
    ("O8 single buffer", PY, "        a = w % 2\n", "        a = 0\n"),
    ("O8 window off by one", PY, "w, first = (t // S, t % S == 0) if window is None else window", "w, first = ((t + 1) // S, (t + 1) % S == 0) if window is None else window"),
    ("f1 g_avg = acc", PY, "g_avg = acc / np.float32(S)", "g_avg = acc"),
    ("f1 1/accum_interval", PY, "S = self.accum_interval if length is None else length", "S = self.accum_interval"),
    ("f1 entering master from zero", PY, "self.master[:, entering] = as_f32(P[:, entering])", "self.master[:, entering] = 0.0"),
    ("f1 entering moments kept", PY, "        self.Mh[:, entering] = 0.0\n", ""),
    ("f1 entering step kept", PY, "        self.th[entering] = 0\n", ""),
    ("f1 update skipped", PY, "        if self.cpu_update:\n            self._deferred_update(self.acc[w % 2], P, length)", "        pass"),
    ("f1 updates the active buffer", PY, "self._deferred_update(self.acc[w % 2], P, length)", "self._deferred_update(self.acc[(w + 1) % 2], P, length)"),
    ("f2 warm-up k = m skipped", PY, "        if t < self.warmup:\n            return self._warmup_step(G, P)\n", ""),
    ("f2 schedule not shifted by tau", PY, "        t -= self.warmup                    # R20", "        pass                    # R20"),
    ("f4 lagged uses current norms", PY, "self.last_norms = self.lag_norms if (self.lagged and self.lag_norms is not None) else column_norms(G)", "self.last_norms = column_norms(G)"),
    ("f4 lag norms taken one step early", PY, "if self.lagged and (t + 1) % self.refresh_interval == 0:", "if self.lagged and (t + 2) % self.refresh_interval == 0:"),
    ("Zen-auto window length from S_max", PY, "length = int(self.auto.len.value)", "length = self.S"),
    ("Zen-auto refresh does not force an end", PY, "force = (tr + 1) % self.N == 0", "force = False"),
    ("shard remainder to the last shards", PY, "return start, start + base + (1 if rank < rem else 0)", "start = rank * base + max(0, rank - (world - rem)); return start, start + base + (1 if rank >= world - rem else 0)"),
    # non-finite handling (R15) and NaN propagation
    ("R15 norms never flag non-finite", CPP, "if (!std::isfinite(s)) bad = 1;", ""),
    ("R15 top-k accepts non-finite norms", CPP, "if (!std::isfinite(norms[j])) return 1;", "(void)j;"),
    ("bf16 NaN not quieted", CPP, "return static_cast<uint16_t>((u >> 16) | 0x0040u);", "return static_cast<uint16_t>(u >> 16);"),
    # f1 write-back / window bookkeeping
    ("f1 writes every column", PY, "            P[:, unsel] = to_bf16(self.master[:, unsel])\n", "            P[:, :] = to_bf16(self.master)\n"),
    ("f1 fp32 write-back to all columns", PY, "            P[:, unsel] = self.master[:, unsel]\n", "            P[:, :] = self.master\n"),
    ("f1 host step counts not stored", PY, "        self.th[unsel] = tc\n", ""),
    ("f1 host v not stored", PY, "        self.Vh[:, unsel] = Vc\n", ""),
    ("sealed() returns the active buffer", PY, "w = t // S if (t + 1) % S == 0 else t // S - 1", "w = t // S"),
    ("Zen-auto next window not marked first", PY, "        self.first = end\n", "        self.first = False\n"),
    ("Zen-auto important count = m", PY, "            sel[1] += l.k\n", "            sel[1] += l.m\n"),
    ("f2 warm-up state not remapped", PY, "            self.M, self.V, self.steps = remap(self.n, self.idx, self.M, self.V, self.steps, new_idx)", "            self.M, self.V, self.steps = (np.zeros((self.n, k), np.float32), np.zeros((self.n, k), np.float32), np.zeros(k, np.int32)) if self.warmup else remap(self.n, self.idx, self.M, self.V, self.steps, new_idx)"),
]


# host-side product logic (data-parallel plumbing, byte accounting), run against the whole CPU
# suite (`-m "not gpu"`): (name, file, old, new)
DIST, BENCH = "paper_2505_12242_b200/dist.py", "bench.py"
HOST_MUTANTS = [
    ("shard_rows remainder to the last ranks", DIST, "return start, start + base + (1 if rank < rem else 0)", "start = rank * base + max(0, rank - (world - rem)); return start, start + base + (1 if rank >= world - rem else 0)"),
    ("flat_partition snaps every boundary up", DIST, "return offs[lo] + (i + (1 if 2 * o >= m else 0)) * m", "return offs[lo] + (i + (1 if o > 0 else 0)) * m"),
    ("flat_partition first row floored", DIST, "r0 = min(n, max(0, -(-(a - o) // m)))", "r0 = min(n, max(0, (a - o) // m))"),
    ("flat_partition last row floored", DIST, "r1 = min(n, max(0, -(-(b - o) // m)))", "r1 = min(n, max(0, (b - o) // m))"),
    ("segment_map stride = rows", DIST, "out.append((li, sid, base + int(c), m, rows))", "out.append((li, sid, base + int(c), rows, rows))"),
    ("segment_map base advances by n*m", DIST, "base += rows * m", "base += n * m"),
    ("gloo all-reduce MAX", DIST, "dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)", "dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)"),
    ("peer handles in reverse rank order", DIST, "ctx.peer_open(handles)", "ctx.peer_open(handles[::-1])"),
    ("algorithmic bytes: compact block m wide", BENCH, "tot += n * m * gsz + n * (m - k) * gsz + n * k * (2 * psz + 16)", "tot += n * m * gsz + n * m * gsz + n * k * (2 * psz + 16)"),
    ("algorithmic bytes: moments read only", BENCH, "tot += n * m * gsz + n * (m - k) * gsz + n * k * (2 * psz + 16)", "tot += n * m * gsz + n * (m - k) * gsz + n * k * (2 * psz + 8)"),
    ("sector bytes: 64-byte sectors", BENCH, "sectors = len(np.unique((np.asarray(idx, np.int64) * psz) // 32))", "sectors = len(np.unique((np.asarray(idx, np.int64) * psz) // 64))"),
]

# mutants that cannot change any result on the oracle's valid domain (reported, not counted)
EQUIVALENT = {
    "O2 no k >= 1 clamp": "for m >= 1 and ppm in [1, 1e6] (the validated domain), ceil(m*ppm/1e6) >= 1 already",
    "flat_partition first row floored": "the boundaries are snapped to row starts, so (a - o) is a multiple of m "
                                        "inside the matrix and clamped outside it: floor = ceil",
    "flat_partition last row floored": "as above for b",
}


def _copy(d, full):
    """Scratch copy: the whole tree for host mutants (the whole CPU suite runs), else only
    what the pin suite needs (the oracle rebuilds from source)."""
    if full:
        shutil.copytree(ROOT, d, dirs_exist_ok=True,
                        ignore=shutil.ignore_patterns(".git", "gpurun_out", "__pycache__", "build", "baseline"))
        return
    for sub in ("oracle", "tests", "synth"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub), ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "__graft_entry__.py"), d)
    shutil.copytree(os.path.join(ROOT, "paper_2505_12242_b200"), os.path.join(d, "paper_2505_12242_b200"),
                    ignore=shutil.ignore_patterns("__pycache__", "build"))
    so = "synth/libzfsynth_host.so"
    if os.path.exists(os.path.join(ROOT, so)):
        shutil.copy(os.path.join(ROOT, so), os.path.join(d, so))


def run_one(mut, keep=False):
    name, f, old, new = mut
    d = tempfile.mkdtemp(prefix="zfmut_")
    host = not f.startswith("oracle/")
    try:
        _copy(d, host)
        p = os.path.join(d, f)
        src = open(p).read()
        if src.count(old) != 1:
            return name, "BAD-PATTERN", src.count(old)
        open(p, "w").write(src.replace(old, new))
        suite = ["tests", "-m", "not gpu"] if host else ["tests/test_oracle_pins.py"]
        r = subprocess.run([sys.executable, "-m", "pytest", *suite, "-x", "-q", "-p", "no:cacheprovider"],
                           cwd=d, capture_output=True, text=True, timeout=900)
        tail = (r.stdout.strip().splitlines() or [""])[-1]
        if r.returncode == 0:
            return name, "SURVIVED", tail
        failed = [l for l in r.stdout.splitlines() if l.startswith("FAILED") or l.startswith("ERROR")]
        return name, "KILLED", (failed[0] if failed else tail)[:160]
    finally:
        if not keep:
            shutil.rmtree(d, ignore_errors=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-k", default="")
    ap.add_argument("--host", action="store_true", help="the host-side product mutants (CPU suite) instead")
    a = ap.parse_args()
    muts = [m for m in (HOST_MUTANTS if a.host else MUTANTS) if a.k in m[0]]
    with ThreadPoolExecutor(a.j) as ex:
        res = list(ex.map(run_one, muts))
    res = [(n, "EQUIVALENT" if (s == "SURVIVED" and n in EQUIVALENT) else s, EQUIVALENT.get(n, i)) for n, s, i in res]
    for name, st, info in res:
        print(f"{st:12s} {name:45s} {info}")
    eq = sum(1 for r in res if r[1] == "EQUIVALENT")
    killed = sum(1 for r in res if r[1] == "KILLED")
    print(f"{killed}/{len(res) - eq} killed ({eq} equivalent)")
    if not a.k:
        name = "host_mutation.json" if a.host else "oracle_mutation.json"
        with open(os.path.join(ROOT, "profiles", name), "w") as fh:
            json.dump({"suite": 'tests -m "not gpu"' if a.host else "tests/test_oracle_pins.py", "killed": killed, "non_equivalent": len(res) - eq,
                       "mutants": [{"mutant": n, "result": s, "detail": str(i)} for n, s, i in res]}, fh, indent=1)


if __name__ == "__main__":
    main()
