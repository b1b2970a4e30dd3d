/*
 * zf_oracle.cpp -- the CPU ORACLE for the ZenFlow data-parallel hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call this
 * code.  The product path (paper_2505_12242_b200/, libzf.so) never links,
 * imports or executes anything under oracle/, and this file shares no code,
 * header, table or constant generator with it.
 *
 * Plain, slow, single-threaded, obviously-correct C++17.  Built with
 * `-O2 -ffp-contract=off` (no FMA contraction, no fast-math), so every fp32
 * expression below is a sequence of individually rounded IEEE operations in
 * the order written.
 *
 * Citation key: P:n = PAPER.md line n (arXiv 2505.12242 LaTeX source),
 * S:n = SPEC.md line n.  Readings of silent/ambiguous passages are listed in
 * DESIGN.md "Readings" (R1..R17) and cited here as [Rn].
 *
 * Pinned by tests/test_oracle_pins.py (closed forms, worked examples,
 * invariants, brute force, library special cases).  Functions whose result
 * has no external pin say so below ("parity unpinned").
 *
 * Steps:
 *   O1 oracle_column_norms      P:486 "per-column gradient norms squared (i.e.,
 *                                the sum of squared gradient values within each
 *                                column)"
 *   O2 oracle_k_for             k = ceil(ratio*m) [R2]
 *   O3 oracle_topk              P:287 "retains the gradients with the highest
 *                                magnitudes"; ties -> lower index [R3]
 *   O4 oracle_column_map        slot / unselected-position map of a selection
 *   O5 oracle_remap             moments across a refresh [R7] (paper silent,
 *                                S:329) -- pinned only by internal consistency
 *   O6 oracle_selective_adamw   P:385 "selective-optimizer ... performs an
 *                                in-place update", "extend PyTorch's Adam
 *                                and AdamW", "AdamW ... weight decay 0.00"
 *   O7 oracle_compact           P:414 "transfers only the (1-k)·M unimportant
 *                                gradients to the CPU" [R12 layout]
 *   O11 oracle_channel_norm_sums / O12 oracle_zen_auto_decide
 *                                Zen-auto (next row f2) [R21]
 *   O8 oracle_accumulate        P:388 "offloaded to the CPU and gradually
 *                                accumulated over several iterations"
 *                                double buffering
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

enum { ORC_F32 = 0, ORC_BF16 = 1 };

// bf16 -> fp32 is exact: the bf16 bits are the top half of the fp32 bits.
float bf16_to_f32(uint16_t h) {
    uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// fp32 -> bf16, IEEE round-to-nearest-even on the dropped 16 bits; NaN stays NaN.
uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x0040u);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return static_cast<uint16_t>(u >> 16);
}

float load(const void* base, int dt, int64_t i) {
    if (dt == ORC_BF16) return bf16_to_f32(static_cast<const uint16_t*>(base)[i]);
    return static_cast<const float*>(base)[i];
}

void store(void* base, int dt, int64_t i, float x) {
    if (dt == ORC_BF16) static_cast<uint16_t*>(base)[i] = f32_to_bf16_rne(x);
    else static_cast<float*>(base)[i] = x;
}

// bit copy of one element (compaction moves bits, no arithmetic) -- O7.
void copy_elem(void* dst, int64_t di, const void* src, int64_t si, int dt) {
    if (dt == ORC_BF16) static_cast<uint16_t*>(dst)[di] = static_cast<const uint16_t*>(src)[si];
    else std::memcpy(static_cast<float*>(dst) + di, static_cast<const float*>(src) + si, 4);
}

}  // namespace

extern "C" {

float oracle_bf16_round(float x) { return bf16_to_f32(f32_to_bf16_rne(x)); }

/* fp32 -> bf16 bit patterns, round to nearest even (the bf16 parameter store of O6). */
void oracle_to_bf16(const float* x, uint16_t* out, int64_t count) {
    for (int64_t e = 0; e < count; ++e) out[e] = f32_to_bf16_rne(x[e]);
}

/* O2  k = ceil(ratio * m) with ratio = ppm / 1e6, in integer arithmetic
 * ("|channel_ids| = ceil(k_channel_ratio x m)"; reading R2: k >= 1). */
int64_t oracle_k_for(int64_t m, int32_t ppm) {
    int64_t k = (m * static_cast<int64_t>(ppm) + 999999) / 1000000;
    if (k < 1) k = 1;
    if (k > m) k = m;
    return k;
}

/* O1  norms[j] = sum_i G[i][j]^2.  Row i of G starts at i*ld.
 * Accumulated in double, in row order, rounded once to fp32 [R4].
 * Returns 0, or 1 if any element (hence any sum) is non-finite [R15]. */
int oracle_column_norms(const void* G, int dt, int64_t n, int64_t m, int64_t ld, float* norms) {
    int bad = 0;
    for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double x = static_cast<double>(load(G, dt, i * ld + j));
            s += x * x;
        }
        if (!std::isfinite(s)) bad = 1;
        norms[j] = static_cast<float>(s);
    }
    return bad;
}

/* Same sums, unrounded (double) -- used by the pins (Frobenius invariant). */
void oracle_column_norms_f64(const void* G, int dt, int64_t n, int64_t m, int64_t ld, double* norms) {
    for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double x = static_cast<double>(load(G, dt, i * ld + j));
            s += x * x;
        }
        norms[j] = s;
    }
}

/* O3  idx = the k columns with the largest norm, ties -> lower column index,
 * returned in ascending column order ([R3]).
 * A stable sort by descending norm keeps equal norms in index order.
 * Returns 1 (and writes nothing) on a non-finite norm. */
int oracle_topk(const float* norms, int64_t m, int64_t k, int32_t* idx) {
    for (int64_t j = 0; j < m; ++j)
        if (!std::isfinite(norms[j])) return 1;
    std::vector<int32_t> order(static_cast<size_t>(m));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return norms[a] > norms[b]; });
    std::vector<int32_t> sel(order.begin(), order.begin() + k);
    std::sort(sel.begin(), sel.end());
    for (int64_t s = 0; s < k; ++s) idx[s] = sel[static_cast<size_t>(s)];
    return 0;
}

/* O4  For a selection idx (ascending): slot[j] = s if idx[s] == j else -1;
 * upos[j] = position of column j among the unselected columns (ascending),
 * -1 for selected columns. */
void oracle_column_map(const int32_t* idx, int64_t k, int64_t m, int32_t* slot, int32_t* upos) {
    for (int64_t j = 0; j < m; ++j) { slot[j] = -1; upos[j] = -1; }
    for (int64_t s = 0; s < k; ++s) slot[idx[s]] = static_cast<int32_t>(s);
    int32_t u = 0;
    for (int64_t j = 0; j < m; ++j)
        if (slot[j] < 0) upos[j] = u++;
}

/* O5  Refresh remap [R7] (paper silent): a column kept across the refresh
 * carries its moments and step count to its new slot; an entering column starts
 * from zero; a leaving column's state is dropped.  M/V are [n, k] row-major.
 * Pinned on whole steps by the AdamW closed forms (entering -> step-1 move,
 * retained -> continued sequence; tests/test_oracle_pins.py); the carry/zero/drop
 * choice itself is the reading. */
void oracle_remap(int64_t n,
                  const int32_t* idx_old, int64_t k_old, const float* m_old, const float* v_old,
                  const int32_t* step_old,
                  const int32_t* idx_new, int64_t k_new, float* m_new, float* v_new, int32_t* step_new) {
    for (int64_t s = 0; s < k_new; ++s) {
        int64_t src = -1;
        for (int64_t q = 0; q < k_old; ++q)
            if (idx_old[q] == idx_new[s]) { src = q; break; }
        step_new[s] = src >= 0 ? step_old[src] : 0;
        for (int64_t i = 0; i < n; ++i) {
            m_new[i * k_new + s] = src >= 0 ? m_old[i * k_old + src] : 0.0f;
            v_new[i * k_new + s] = src >= 0 ? v_old[i * k_old + src] : 0.0f;
        }
    }
}

/* O6  Selective AdamW, in place, on the selected columns only (P:385-386,
 * P:594 "We extend PyTorch's Adam and AdamW"; AdamW P:654; reading R8).
 * Hyper-parameters are real numbers given in double; every derived constant is
 * computed in double and rounded ONCE to fp32, as PyTorch does with its Python
 * scalars.  For each slot s (column c = idx[s]) the step count is
 * t_s = step[s] + 1, shared by all rows; then for every row i, each line is ONE
 * correctly rounded fp32 operation:
 *     g = G[i][c]; p = P[i][c]; m = M[i][s]; v = V[i][s]
 *     if wd != 0 and decoupled:   p = p * decay          decay = f32(1 - lr*wd)
 *     if wd != 0 and !decoupled:  g = g + (wd_f * p)      wd_f = f32(wd)
 *     m = (b1 * m) + (omb1 * g)                           b1 = f32(beta1), omb1 = f32(1 - beta1)
 *     v = (b2 * v) + ((omb2 * g) * g)                     b2 = f32(beta2), omb2 = f32(1 - beta2)
 *     den = (sqrt(v) / bc2s[t_s]) + eps_f                 bc2s[t] = f32(sqrt(1 - beta2^t)), eps_f = f32(eps)
 *     p = p - (ss[t_s] * (m / den))                       ss[t] = f32(lr / (1 - beta1^t))
 *     P[i][c] = round(p) (fp32, or bf16 RNE) ; M[i][s] = m ; V[i][s] = v
 * and finally step[s] = t_s. */
void oracle_selective_adamw(void* P, int pdt, int64_t ldp,
                            const void* G, int gdt, int64_t ldg,
                            int64_t n, const int32_t* idx, int64_t k,
                            float* M, float* V, int32_t* step,
                            double lr, double beta1, double beta2, double eps, double weight_decay,
                            int decoupled) {
    const float decay = static_cast<float>(1.0 - lr * weight_decay);
    const float wd_f = static_cast<float>(weight_decay);
    const float b1 = static_cast<float>(beta1);
    const float b2 = static_cast<float>(beta2);
    const float omb1 = static_cast<float>(1.0 - beta1);
    const float omb2 = static_cast<float>(1.0 - beta2);
    const float eps_f = static_cast<float>(eps);
    for (int64_t s = 0; s < k; ++s) {
        const int64_t c = idx[s];
        const int32_t t = step[s] + 1;
        const float ss = static_cast<float>(lr / (1.0 - std::pow(beta1, static_cast<double>(t))));
        const float bc2s = static_cast<float>(std::sqrt(1.0 - std::pow(beta2, static_cast<double>(t))));
        for (int64_t i = 0; i < n; ++i) {
            float g = load(G, gdt, i * ldg + c);
            float p = load(P, pdt, i * ldp + c);
            float m = M[i * k + s];
            float v = V[i * k + s];
            if (weight_decay != 0.0 && decoupled) p = p * decay;
            if (weight_decay != 0.0 && !decoupled) {
                float wp = wd_f * p;
                g = g + wp;
            }
            float a1 = b1 * m;
            float a2 = omb1 * g;
            m = a1 + a2;
            float c1 = b2 * v;
            float c2 = omb2 * g;
            float c3 = c2 * g;
            v = c1 + c3;
            float sq = std::sqrt(v);
            float q = sq / bc2s;
            float den = q + eps_f;
            float upd = m / den;
            float delta = ss * upd;
            p = p - delta;
            store(P, pdt, i * ldp + c, p);
            M[i * k + s] = m;
            V[i * k + s] = v;
        }
        step[s] = t;
    }
}

/* O7  out[i][u] = G[i][j] for the u-th unselected column j of row i
 * (ascending), out is dense row-major [n, m-k] in G's dtype (bit copy;
 * P:414, reading R12). */
void oracle_compact(const void* G, int gdt, int64_t n, int64_t m, int64_t ld,
                    const int32_t* idx, int64_t k, void* out) {
    std::vector<char> selected(static_cast<size_t>(m), 0);
    for (int64_t s = 0; s < k; ++s) selected[static_cast<size_t>(idx[s])] = 1;
    const int64_t w = m - k;
    for (int64_t i = 0; i < n; ++i) {
        int64_t u = 0;
        for (int64_t j = 0; j < m; ++j) {
            if (selected[static_cast<size_t>(j)]) continue;
            copy_elem(out, i * w + u, G, i * ld + j, gdt);
            ++u;
        }
    }
}

/* O8  acc[e] += f32(stage[e]) for e < count, in element order (P:388,
 * P:437-441; the window/zeroing/swap logic lives in oracle.py). */
void oracle_accumulate(float* acc, const void* stage, int dt, int64_t count) {
    for (int64_t e = 0; e < count; ++e) {
        float x = load(stage, dt, e);
        acc[e] = acc[e] + x;
    }
}

/* O11  Zen-auto statistic of one matrix (f2, reading R21): from the
 * per-column squared norms of the current gradient (the O1 proxy -- P:447
 * "monitors gradient changes across GPUs using a lightweight coordination
 * proxy"), the sums of the per-channel L2 norms over the selected (sums[0]) and
 * the unselected (sums[1]) columns; sqrt and sums in double, column order. */
void oracle_channel_norm_sums(const float* norms, int64_t m, const int32_t* idx, int64_t k, double* sums) {
    std::vector<char> selected(static_cast<size_t>(m), 0);
    for (int64_t s = 0; s < k; ++s) selected[static_cast<size_t>(idx[s])] = 1;
    double sel = 0.0, unsel = 0.0;
    for (int64_t j = 0; j < m; ++j) {
        const double x = std::sqrt(static_cast<double>(norms[j]));
        if (selected[static_cast<size_t>(j)]) sel += x;
        else unsel += x;
    }
    sums[0] = sel;
    sums[1] = unsel;
}

/* O12  One Zen-auto decision at the end of a step ("tracks the average
 * accumulated channel gradient norm and compares it to the average one of the
 * important part.  Once the unimportant gradient part becomes comparable to
 * important ones, Zen-auto immediately triggers its CPU-side update"; reading R21):
 *   u = mean per-channel norm of the unselected columns this step (all matrices),
 *   i = mean per-channel norm of the selected columns this step,
 *   A = sum of u over the window's steps so far (the window's accumulated
 *       unimportant channel norm, averaged over channels),
 *   the window ends iff force_end (the next step refreshes the selection), or it
 *   has lasted smax steps (bounded staleness), or A > 0 and A >= gamma*i.
 * state[0] = A, *len = steps in the window; `first` starts a new window. */
int oracle_zen_auto_decide(double* A, int64_t* len, int first, double sel_sum, int64_t sel_cnt, double unsel_sum,
                           int64_t unsel_cnt, double gamma, int64_t smax, int force_end) {
    const double u = unsel_cnt > 0 ? unsel_sum / static_cast<double>(unsel_cnt) : 0.0;
    const double i = sel_cnt > 0 ? sel_sum / static_cast<double>(sel_cnt) : 0.0;
    if (first) {
        *A = 0.0;
        *len = 0;
    }
    *A = *A + u;
    *len = *len + 1;
    if (force_end || *len >= smax) return 1;
    return (*A > 0.0 && *A >= gamma * i) ? 1 : 0;
}

}  // extern "C"
