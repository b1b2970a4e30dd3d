// k_update.cu -- K3: fused selective AdamW (in place, selected columns only)
// + compaction of the unselected columns, grouped over every layer in one
// persistent launch; on refresh steps it also applies the moment remap (K4).
//
// Paper: "the pre-identified important gradients remain on the GPU,
// where a selective-optimizer, initialized only with the corresponding
// parameter subset, performs an in-place update"; "We extend PyTorch's
// Adam and AdamW optimizers to support in-place updates using selected
// important gradients"; "ZenFlow transfers only the (1-k)·M unimportant
// gradients to the CPU".  Moment carry-over across a refresh: reading R7.
//
// B200 design (DESIGN.md §5 K3).  HBM-bound: per element of G it moves 2 B of
// G, 2(1-κ) B of compact output, and for the selected columns p (the dense
// parameter-subset slab on steady steps, p's 32-byte sectors on refreshes) and
// the fp32 moments.
//  - persistent grid, one CTA per SM, warp-specialised: 4 producer warps (one
//    thread each, one stage arena each) and 28 consumer warps in two groups of 14.
//    Work units (R rows x c columns) are claimed dynamically, one atomic per unit;
//    refresh and steady steps use their own unit shapes (a steady unit holds no p tile).
//  - a producer prefetches the claimed unit's G rows / slabs into L2 while its arena is
//    still being consumed, then stages the unit's DATA into its arena with bulk copies
//    (cp.async.bulk, the TMA engine) completing on one mbarrier: the G tile, the dense
//    parameter-subset slab (steady) or the previous subset block's old rows (a refresh:
//    retained columns' p values; entering ones are loaded from p), or the p tile (a refresh
//    without a valid block, when the selection touches most of p's 32-byte sectors), and the
//    moment slabs (or the old rows on a refresh).
//    The layer's selection METADATA (selected columns, per-slot bias corrections, remap
//    sources, the unselected-column list) is not staged: every unit of a layer reads the
//    same arrays, so the consumers read them through L1 and the arenas carry only data
//    (more bytes in flight per SM).  Waits are hardware-suspended (mbarrier.try_wait).
//  - consumers: AdamW over the unit's (row, slot) pairs taken row-major (a warp's lanes hold
//    consecutive slots of one row: conflict-free slab reads, coalesced moment stores;
//    explicit round-to-nearest intrinsics in the oracle's op order; adam_unit_b), each
//    changed p value stored straight to HBM; then compaction by gather (8 bf16 outputs per
//    thread per vector store, coalesced across the warp).
//  - with offload, a unit's producer bumps its layer chunk's completion counter once the
//    stage's consumer warps all released the unit (one red.release per unit, cumulative
//    over their stores); the copy stream waits on it (cuStreamWaitValue32) to start the
//    chunk's device->host copy.
#include <cstdlib>

#include "zf_internal.cuh"

namespace zf {
namespace {

// producers prefetch a claimed unit's G / p rows and moment slabs into L2 while its arena is
// still busy
// (-DZF_K3_NO_L2PF disables)
#ifndef ZF_K3_NO_L2PF
#define ZF_K3_L2PF 1
#endif
#ifndef ZF_K3_NCW
#define ZF_K3_NCW 28   // 2 groups of 14 (64 registers per thread); measured best of 16-28 (tools/k3_flags.sh)
#endif
constexpr int K3_NCW = ZF_K3_NCW;                 // consumer warps
#ifndef ZF_K3_ROW_UNROLL
#define ZF_K3_ROW_UNROLL 2
#endif
constexpr int K3_ROW_UNROLL = ZF_K3_ROW_UNROLL;   // rows of one slot in flight per AdamW thread
#ifndef ZF_K3_GROUPS
#define ZF_K3_GROUPS 2
#endif
constexpr int K3_GROUPS = ZF_K3_GROUPS;           // independent consumer groups; group g owns stages g, g+G, ...
constexpr int K3_GW = K3_NCW / K3_GROUPS;         // warps per group
#ifndef ZF_K3_AW
#define ZF_K3_AW 0
#endif
// role split inside a group: warps [0, K3_AW) run the unit's AdamW while warps [K3_AW, K3_GW)
// run its compaction, concurrently (0: every warp runs both phases, one after the other)
constexpr int K3_AW = ZF_K3_AW;
constexpr int K3_AWARPS = K3_AW > 0 ? K3_AW : K3_GW;   // warps that run AdamW
constexpr int K3_CW0 = K3_AW > 0 ? K3_AW : 0;          // first compaction warp of a group
constexpr int K3_CWARPS = K3_GW - K3_CW0;              // warps that run the compaction
static_assert(K3_AW >= 0 && K3_AW < K3_GW, "role split");
#ifndef ZF_K3_STAGES
#define ZF_K3_STAGES 4
#endif
#ifndef ZF_K3_ARENA_KB
#define ZF_K3_ARENA_KB 48   // 4 x 48 KB of stages leaves ~60 KB of L1 for the layers' metadata
#endif
constexpr int K3_STAGES = ZF_K3_STAGES;           // stage arenas = producer warps (one chain per stage)
constexpr int K3_THREADS = 32 * (K3_NCW + K3_STAGES);
constexpr int K3_ARENA = ZF_K3_ARENA_KB * 1024;   // bytes per stage arena
constexpr int K3_SMEM = K3_STAGES * K3_ARENA;
static_assert(K3_ARENA % 128 == 0, "alignment");
static_assert(K3_SMEM <= 227 * 1024 - 512, "shared memory budget");
static_assert(K3_STAGES % K3_GROUPS == 0 && K3_NCW % K3_GROUPS == 0, "stages and warps split evenly over groups");

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Hardware-suspended wait: try_wait parks the warp until the phase completes or a
// hardware time window elapses, so waiting warps take few issue slots from working ones.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
#ifdef ZF_MBAR_HINT
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ZF_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra ZF_WAIT;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase), "r"(ZF_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "ZF_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra ZF_WAIT;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
#endif
}
#ifdef ZF_MBAR_SLEEP_NS
// consumer waits: back off with nanosleep between try_wait probes, so warps waiting for a
// stage do not take issue slots from the working ones (experiment knob)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (ok) return;
        __nanosleep(ZF_MBAR_SLEEP_NS);
    }
}
#else
#define mbar_wait_sleep mbar_wait
#endif
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// L2 prefetch of a global range by the TMA engine (no shared memory, no completion):
// lets a producer start a claimed unit's DRAM reads while its arena is still busy.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, int64_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) & ~uintptr_t(15);
    const uintptr_t b = (reinterpret_cast<uintptr_t>(src) + (uintptr_t)bytes + 15) & ~uintptr_t(15);
    for (uintptr_t q = a; q < b;) {
        const uint32_t n = (uint32_t)((b - q) < (uintptr_t)(1u << 20) ? (b - q) : (uintptr_t)(1u << 20));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(q), "r"(n) : "memory");
        q += n;
    }
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}


// Bulk-copy the ESZ-byte elements [e0, e1) of `src` to arena offset *off as an aligned
// superset (16-byte granules; the source arrays are padded).  Returns the element
// offset of e0 within the copy; advances *off.
template <int ESZ>
__device__ __forceinline__ int stage_elems(unsigned char* arena, int* off, const void* src, int64_t e0, int64_t e1,
                                           uint64_t* bar, uint32_t* tx, int* where) {
    constexpr int64_t G = 16 / ESZ;
    const int64_t a = e0 & ~(G - 1), b = (e1 + G - 1) & ~(G - 1);
    *where = *off;
    if (b > a) {
        const uint32_t bytes = (uint32_t)((b - a) * ESZ);
        bulk_g2s(arena + *off, static_cast<const unsigned char*>(src) + a * ESZ, bytes, bar, 0ull);
        *tx += bytes;
        *off += (int)bytes;
    }
    return (int)(e0 - a);
}

__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}


__device__ __forceinline__ int find_layer_from(const Table<UpdLayer>& t, int64_t u, int hint) {
    int li = hint;
    if (li >= t.n || t[li].unit_begin > u) li = 0;
    while (li + 1 < t.n && t[li + 1].unit_begin <= u) ++li;  // claims are monotonic: usually 0-1 steps
    return li;
}

struct UnitGeom {
    int64_t r0;
    int32_t Rr;
    int64_t c0, c1;
};

__device__ __forceinline__ UnitGeom unit_geom(const UpdLayer& L, int64_t lu) {
    UnitGeom g;
    const int64_t rb = lu / L.nseg, sg = lu - rb * L.nseg;
    g.r0 = rb * L.R;
    g.Rr = (int32_t)zmin<int64_t>((int64_t)L.R, L.n - g.r0);
    g.c0 = sg * L.seg_cols;
    g.c1 = zmin<int64_t>(L.m, g.c0 + L.seg_cols);
    return g;
}

// per-stage unit descriptor written by the producer (arena byte offsets; element offsets
// of the aligned supersets)
struct StageInfo {
    int64_t u;        // unit (-1: no more work)
    int32_t li;       // layer
    int32_t s0, s1;   // selected-slot range of the segment
    int32_t oG, oP, oM, oV, oPs;
    int32_t eM, eV, ePs;
    int32_t pstaged, mstaged, remap, psub_mode;
    int32_t j0, nkeep;          // segment's first output index within a row / outputs per row
    uint32_t mg_ns;             // ceil(2^24 / ns): x / ns == (x * mg_ns) >> 24 for x <= 512
    // unit geometry and layer fields, so consumers never touch the global layer table
    int32_t Rr, sw, k, kin;
    int64_t ldp, out_ld;
    int64_t r0, c0;
    void* P;                    // p + r0*ldp (row 0 of the unit)
    void* out;                  // compact block of the layer
    float* m_out;               // + r0*k
    float* v_out;
    void* psub;                 // param_subset block + r0*k (NULL: none)
    void* gsel;                 // split update: selected-gradient block + r0*k
    const float* m_in;          // layer base (non-staged path)
    const float* v_in;
    // per-layer selection metadata, read by the consumers through L1 (every unit of a layer
    // reads the same arrays, so they stay cache-resident instead of taking stage bytes)
    const int32_t* steps;       // [k] step counts at the last refresh (used when sbv is NULL)
    const float2* sbv;          // [k] per-slot {ss, bc2s} of this launch (K3 prologue), or NULL
    const int32_t* slot_src;    // [k] remap sources (refresh)
    const int32_t* idx;         // [k] selected columns
    const uint16_t* ucol;       // [m-k] byte offsets (mod 2^16) of the unselected columns
    uint32_t* done;
};

// AdamW over one unit's (row, slot) pairs by the K3_GW*32 threads of a consumer group,
// slot-major: a slot's column, bias corrections (and remap source) are read once for all of
// its rows.  PST: p tile staged; MST: moment slabs staged; REMAP: refresh step (moments come
// from the old slots); PSUB: p's current values from the staged subset slab (steady step with
// param_subset).  Without MST the remap flag is read at run time (global-load path).  Every
// changed p value is stored straight to HBM (and to the subset block).
template <int GDT, int PDT, bool PST, bool MST, bool REMAP, bool PSUB = false, int NCT = K3_AWARPS * 32>
__device__ __forceinline__ void adam_unit(const StageInfo& si, unsigned char* A, const UpdParams& prm, int ctid,
                                          uint32_t& nfacc) {
    static_assert(!PSUB || (MST && !REMAP && !PST), "the subset slab is staged on steady steps only");
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    const int sw = si.sw, Rr = si.Rr, ns = si.s1 - si.s0;
    const int k = si.k, kin = si.kin, s0 = si.s0, c0 = (int)si.c0;
    const bool remap = MST ? REMAP : (si.remap != 0);
    const GB* sG = reinterpret_cast<const GB*>(A + si.oG);
    const PB* sP = reinterpret_cast<const PB*>(A + si.oP);
    const float* sM = reinterpret_cast<const float*>(A + si.oM) + si.eM;
    const float* sV = reinterpret_cast<const float*>(A + si.oV) + si.eV;
    const PB* sPs = reinterpret_cast<const PB*>(A + si.oPs) + si.ePs;   // PSUB: staged [R, s0:s1) subset slab
    PB* gP = static_cast<PB*>(si.P);
    PB* gS = static_cast<PB*>(si.psub);                                  // subset block rows of the unit
    const int pmode = si.psub_mode;
    const int64_t ldp = si.ldp;
    const int tdelta = prm.step_delta + 1;
    uint32_t dbg_sink = 0;
    int sl, rg, nrg;
    if (ns >= NCT) {
        sl = ctid; rg = 0; nrg = 1;
    } else {  // fewer slots than threads: teams of ns threads split the rows
        rg = (int)(((uint64_t)ctid * si.mg_ns) >> 24);  // ctid / ns (exact for ctid <= 512)
        nrg = (int)(((uint64_t)NCT * si.mg_ns) >> 24);   // NCT / ns
        sl = ctid - rg * ns;
        if (rg >= nrg) return;
    }
    for (; sl < ns; sl += NCT) {
        const int s = s0 + sl;
        const int c = __ldg(si.idx + s);
        // {ss, bc2s} of the slot's step count: the prologue's per-slot array, else the tables
        const float2 sb = si.sbv ? __ldg(si.sbv + s) : adam_sb(__ldg(si.steps + s) + tdelta, prm.adam);
        const int src = remap ? __ldg(si.slot_src + s) : 0;
        const int cl = c - c0;
        const GB* g_ = sG + cl;
        float* mo = si.m_out + s;
        float* vo = si.v_out + s;
#pragma unroll K3_ROW_UNROLL
        for (int r = rg; r < Rr; r += nrg) {
            const GB gb = g_[r * sw];
            if constexpr (GE::SIZE == 2) nfacc |= ((uint32_t)gb & 0x7f80u) + 0x0080u;
            else nfacc |= ((uint32_t)gb & 0x7f800000u) + 0x00800000u;
            PB pold;
            if constexpr (PSUB) pold = sPs[r * k + sl];
            else if constexpr (PST) pold = sP[r * sw + cl];
            else pold = pmode == 2 ? gS[r * k + s] : gP[r * ldp + c];
            float p = PE::to_f(pold);
            float mm, vv;
            if constexpr (MST) {
                if constexpr (REMAP) {
                    mm = src >= 0 ? sM[r * kin + src] : 0.0f;
                    vv = src >= 0 ? sV[r * kin + src] : 0.0f;
                } else {
                    mm = sM[r * k + sl];
                    vv = sV[r * k + sl];
                }
            } else {
                const int64_t row = si.r0 + r;
                if (remap) {
                    mm = src >= 0 ? __ldcs(si.m_in + row * kin + src) : 0.0f;
                    vv = src >= 0 ? __ldcs(si.v_in + row * kin + src) : 0.0f;
                } else {
                    mm = __ldcs(si.m_in + row * k + s);
                    vv = __ldcs(si.v_in + row * k + s);
                }
            }
            adamw_elem_t(GE::to_f(gb), p, mm, vv, sb.x, sb.y, prm.adam);
            {
                // a changed value is stored straight to HBM (the memory state is that of storing
                // every value; at lr 1e-5 most bf16 values do not change); param_subset: mode 1
                // (re)builds the block, mode 2 keeps it equal to p
                const PB pnew = PE::from_f(p);
                if (pnew != pold) gP[r * ldp + c] = pnew;
                if (pmode == 1 || (pmode == 2 && pnew != pold)) gS[r * k + s] = pnew;
            }
            if (prm.debug_mode != 7) {
                __stcs(mo + r * k, mm);
                __stcs(vo + r * k, vv);
            } else {
                dbg_sink ^= __float_as_uint(mm) ^ __float_as_uint(vv);
            }
        }
    }
    asm volatile("" ::"r"(dbg_sink));  // debug mode 7 keeps the moment math live
}

#ifndef ZF_K3_NB
#define ZF_K3_NB 1
#endif
// Staged-moment AdamW (MST) in batches: each thread takes NB (row, slot) pairs at a time --
// pair q = row * ns + slot, q = ctid, ctid + NCT, ... (row-major, so the warp's 32 lanes hold
// 32 consecutive slots of one row: conflict-free slab reads and coalesced moment stores) --
// and issues every load of the batch (the slots' columns and {ss, bc2s} through L1, then g, p,
// m, v from the stage) before any arithmetic: NB independent chains per thread instead of one
// latency-bound chain per slot.
template <int GDT, int PDT, bool PST, bool REMAP, bool PSUB, int NCT = K3_AWARPS * 32, int NB = ZF_K3_NB>
__device__ __forceinline__ void adam_unit_b(const StageInfo& si, unsigned char* A, const UpdParams& prm, int ctid,
                                            uint32_t& nfacc) {
    static_assert(!PSUB || !PST, "a unit stages the p tile or a subset slab, not both");
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    const int sw = si.sw, Rr = si.Rr, ns = si.s1 - si.s0;
    const int k = si.k, kin = si.kin, s0 = si.s0, c0 = (int)si.c0;
    const GB* sG = reinterpret_cast<const GB*>(A + si.oG);
    const PB* sP = reinterpret_cast<const PB*>(A + si.oP);
    const float* sM = reinterpret_cast<const float*>(A + si.oM) + si.eM;
    const float* sV = reinterpret_cast<const float*>(A + si.oV) + si.eV;
    const PB* sPs = reinterpret_cast<const PB*>(A + si.oPs) + si.ePs;
    PB* gP = static_cast<PB*>(si.P);
    PB* gS = static_cast<PB*>(si.psub);
    const int pmode = si.psub_mode;
    const int ldp = (int)si.ldp;       // < 2^31 / Rr: unit-relative offsets fit 32 bits
    const int tdelta = prm.step_delta + 1;
    const int total = Rr * ns;
    // (row, slot) of pair ctid and the per-NCT step, by the exact multiply-shift ns reciprocal
    int r = (int)(((uint64_t)ctid * si.mg_ns) >> 24), sl = ctid - r * ns;
    const int dr = (int)(((uint64_t)NCT * si.mg_ns) >> 24), dsl = NCT - dr * ns;
    uint32_t dbg_sink = 0;
    for (int q = ctid; q < total; q += NCT * NB) {
        int so[NB], pa[NB], cc[NB], src[NB], rr[NB];
        float2 sb[NB];
        GB gb[NB];
        PB po[NB];
        float mm[NB], vv[NB];
        // (A) the batch's pairs: per-slot loads through L1
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            rr[j] = r;
            so[j] = r * k + s0 + sl;                 // [row, slot] offset in the unit's slab rows
            pa[j] = r * ldp - c0;                    // row offset in p, minus the tile's first column
            if (q + j * NCT < total) {
                const int s = s0 + sl;
                cc[j] = __ldg(si.idx + s);
                sb[j] = si.sbv ? __ldg(si.sbv + s) : adam_sb(__ldg(si.steps + s) + tdelta, prm.adam);
                if constexpr (REMAP) src[j] = __ldg(si.slot_src + s) + r * kin;
            }
            r += dr;
            sl += dsl;
            if (sl >= ns) { sl -= ns; ++r; }
        }
        // (B) stage reads (g, p, m, v) of every pair of the batch
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (q + j * NCT < total) {
                const int row = rr[j];
                const int cl = cc[j] - c0;
                gb[j] = sG[row * sw + cl];
                if constexpr (PSUB && REMAP) {
                    // refresh from the previous subset block (mode 3): a retained slot's value from
                    // its old row (staged like the old moments), an entering slot's from p
                    po[j] = src[j] >= row * kin ? sPs[src[j]] : gP[pa[j] + c0 + cc[j]];
                } else if constexpr (PSUB) po[j] = sPs[so[j] - s0];
                else if constexpr (PST) po[j] = sP[row * sw + cl];
                else po[j] = pmode == 2 ? gS[so[j]] : gP[pa[j] + c0 + cc[j]];
                if constexpr (REMAP) {
                    const bool ok = src[j] >= row * kin;
                    mm[j] = ok ? sM[src[j]] : 0.0f;
                    vv[j] = ok ? sV[src[j]] : 0.0f;
                } else {
                    mm[j] = sM[so[j] - s0];
                    vv[j] = sV[so[j] - s0];
                }
                pa[j] += c0 + cc[j];
            }
        }
        // (C) arithmetic and stores
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (q + j * NCT < total) {
                if constexpr (GE::SIZE == 2) nfacc |= ((uint32_t)gb[j] & 0x7f80u) + 0x0080u;
                else nfacc |= ((uint32_t)gb[j] & 0x7f800000u) + 0x00800000u;
                float p = PE::to_f(po[j]);
                adamw_elem_t(GE::to_f(gb[j]), p, mm[j], vv[j], sb[j].x, sb[j].y, prm.adam);
                const PB pnew = PE::from_f(p);
                if (prm.debug_mode < 9 || prm.debug_mode > 14) {
                    if (pnew != po[j]) gP[pa[j]] = pnew;
                    if (pmode == 1 || pmode == 3 || (pmode == 2 && pnew != po[j])) gS[so[j]] = pnew;  // 1, 3: rebuild
                } else if (prm.debug_mode == 12) {   // experiments: 9 no p / subset stores; 12 no subset stores
                    if (pnew != po[j]) gP[pa[j]] = pnew;
                } else if (prm.debug_mode == 13) {   // 13 no p stores
                    if (pmode == 1 || (pmode == 2 && pnew != po[j])) gS[so[j]] = pnew;
                } else if (prm.debug_mode == 14) {   // 14 every p / subset value stored (no branch)
                    gP[pa[j]] = pnew;
                    gS[so[j]] = pnew;
                } else {
                    dbg_sink ^= pnew;
                }
                if (prm.debug_mode != 7 && prm.debug_mode != 10) {   // (10: no moment stores)
                    __stcs(si.m_out + so[j], mm[j]);
                    __stcs(si.v_out + so[j], vv[j]);
                } else {
                    dbg_sink ^= __float_as_uint(mm[j]) ^ __float_as_uint(vv[j]);
                }
            }
        }
    }
    asm volatile("" ::"r"(dbg_sink));
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const void* p) {
    uint2 v;
    asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}

template <int GDT, int PDT>
__global__ void __launch_bounds__(K3_THREADS, 1) k_update(const __grid_constant__ UpdParams prm) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    constexpr int GSZ = GE::SIZE, PSZ = PE::SIZE;

    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[K3_STAGES], empty[K3_STAGES];
    __shared__ StageInfo info[K3_STAGES];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Table<UpdLayer>& table = prm.layers;

    if (tid == 0) {
        for (int st = 0; st < K3_STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], K3_GW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp < K3_STAGES) {
        // ============ producers: warp st (one thread) owns stage arena st ============
        if (lane != 0) return;
        const int st = warp;
        const uint64_t pol_first = evict_first_policy();
        const uint64_t pol_last = evict_last_policy();
        int hint = 0;
        uint32_t* prev_done = nullptr;   // completion counter of the unit last staged in this arena
        for (int it = 0;; ++it) {
            // claim and look up the next unit before waiting for its arena
            const uint32_t cl = atomicAdd(prm.claim, 1u) - prm.claim_base;
            StageInfo si{};
            si.u = (int64_t)cl < prm.total_units ? (int64_t)cl + prm.unit_offset : -1;
            const UpdLayer* Lp = nullptr;
            UnitGeom g{};
            if (si.u >= 0) {
                hint = find_layer_from(table, si.u, hint);
                si.li = hint;
                Lp = &table[hint];
                g = unit_geom(*Lp, si.u - Lp->unit_begin);
                si.s0 = g.c0 == 0 ? 0 : (g.c0 >= Lp->m ? (int32_t)Lp->k : __ldg(Lp->prefix + (g.c0 >> 5)));
                si.s1 = g.c1 >= Lp->m ? (int32_t)Lp->k : __ldg(Lp->prefix + (g.c1 >> 5));
            }
#ifdef ZF_K3_L2PF
            if (si.u >= 0 && it > 0) {
                // the arena is still being consumed: pull this unit's rows and slabs toward L2 now
                const UpdLayer& L = *Lp;
                const int sw = (int)(g.c1 - g.c0);
                if (L.tma_ok) {
                    const unsigned char* G = static_cast<const unsigned char*>(L.G);
                    if (L.nseg == 1 && L.ldg == L.m) bulk_prefetch_l2(G + g.r0 * L.m * GSZ, (int64_t)g.Rr * sw * GSZ);
                    else
                        for (int r = 0; r < g.Rr; ++r)
                            bulk_prefetch_l2(G + ((g.r0 + r) * L.ldg + g.c0) * GSZ, (int64_t)sw * GSZ);
                }
                if (prm.do_extract && si.s1 > si.s0 && L.psub_mode == 1 && L.p_tma) {
                    const unsigned char* P = static_cast<const unsigned char*>(L.P);
                    if (L.nseg == 1 && L.ldp == L.m) bulk_prefetch_l2(P + g.r0 * L.m * PSZ, (int64_t)g.Rr * sw * PSZ);
                    else
                        for (int r = 0; r < g.Rr; ++r)
                            bulk_prefetch_l2(P + ((g.r0 + r) * L.ldp + g.c0) * PSZ, (int64_t)sw * PSZ);
                }
                if (prm.do_adam && si.s1 > si.s0 && L.psub_mode == 2 && L.mv_tma)
                    bulk_prefetch_l2(static_cast<const unsigned char*>(L.psub) + (g.r0 * L.k + si.s0) * PSZ,
                                     ((g.Rr - 1) * L.k + si.s1 - si.s0) * PSZ);
                if (prm.do_adam && si.s1 > si.s0 && L.psub_mode == 3 && L.mv_tma)
                    bulk_prefetch_l2(static_cast<const unsigned char*>(L.psub_in) + g.r0 * L.k_in * PSZ,
                                     (int64_t)g.Rr * L.k_in * PSZ);
#ifndef ZF_K3_NO_PSUB_PPF
                // with the subset slab, still pull the unit's p rows into L2 when the selection
                // touches most of p's sectors: the changed values' stores then hit cached sectors
                // instead of each waiting on a partial-sector fill (measured: steady K3 9.48 ->
                // 9.36 ms at lr 1e-5, 10.33 -> 9.83 ms at lr 1e-3, Llama-2-7B k = 10%)
                if (prm.do_adam && si.s1 > si.s0 && (L.psub_mode == 2 || L.psub_mode == 3) && L.p_dense) {
                    const unsigned char* P = static_cast<const unsigned char*>(L.P);
                    for (int r = 0; r < g.Rr; ++r)
                        bulk_prefetch_l2(P + ((g.r0 + r) * L.ldp + g.c0) * PSZ, (int64_t)sw * PSZ);
                }
#endif
                if (prm.do_adam && si.s1 > si.s0 && L.p_tma) {
                    const unsigned char* P = static_cast<const unsigned char*>(L.P);
                    if (L.nseg == 1 && L.ldp == L.m) bulk_prefetch_l2(P + g.r0 * L.m * PSZ, (int64_t)g.Rr * sw * PSZ);
                    else
                        for (int r = 0; r < g.Rr; ++r)
                            bulk_prefetch_l2(P + ((g.r0 + r) * L.ldp + g.c0) * PSZ, (int64_t)sw * PSZ);
                }
                if (prm.do_adam && si.s1 > si.s0 && L.mv_tma) {  // and the moment slabs
                    int64_t e0, e1;
                    if (L.slot_src) {
                        e0 = g.r0 * L.k_in;
                        e1 = (g.r0 + g.Rr) * L.k_in;
                    } else {
                        e0 = g.r0 * L.k + si.s0;
                        e1 = (g.r0 + g.Rr - 1) * L.k + si.s1;
                    }
                    bulk_prefetch_l2(L.m_in + e0, (e1 - e0) * 4);
                    bulk_prefetch_l2(L.v_in + e0, (e1 - e0) * 4);
                }
            }
#endif
            if (it > 0) {
                mbar_wait(&empty[st], (it - 1) & 1);
                // every consumer warp of the stage's previous unit arrived (release, CTA scope;
                // this wait acquires): one GPU-scope release publishes all their compact-block
                // stores to the layer chunk's completion counter (X1's copy engine waits on it)
                if (prev_done) red_release_add(prev_done, 1u);
            }
            unsigned char* A = smem + st * K3_ARENA;
            if (si.u < 0) {
                info[st] = si;
                mbar_arrive(&full[st]);
                break;
            }
            const UpdLayer& L = *Lp;
            const int sw = (int)(g.c1 - g.c0);
            const int ns = si.s1 - si.s0;
            uint32_t tx = 0;
            int off = 0;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            // G tile
            si.oG = 0;
            if (L.tma_ok) {
                const unsigned char* G = static_cast<const unsigned char*>(L.G);
                if (L.nseg == 1 && L.ldg == L.m) {
                    bulk_g2s(A, G + g.r0 * L.m * GSZ, (uint32_t)(g.Rr * sw * GSZ), &full[st], pol_first);
                } else {
                    for (int r = 0; r < g.Rr; ++r)
                        bulk_g2s(A + r * sw * GSZ, G + ((g.r0 + r) * L.ldg + g.c0) * GSZ, (uint32_t)(sw * GSZ),
                                 &full[st], pol_first);
                }
                tx += (uint32_t)(g.Rr * sw * GSZ);
            } else {
                GB* sG = reinterpret_cast<GB*>(A);
                const GB* G = static_cast<const GB*>(L.G);
                for (int r = 0; r < g.Rr; ++r)
                    for (int c = 0; c < sw; ++c) sG[r * sw + c] = G[(g.r0 + r) * L.ldg + g.c0 + c];
            }
            off = (g.Rr * sw * GSZ + 15) & ~15;
            si.j0 = (int32_t)(g.c0 - si.s0);
            si.nkeep = sw - ns;
            if (prm.do_extract && ns > 0) {
                // split update (K3a): the AdamW inputs go to dense blocks; only a psub rebuild
                // (mode 1) needs p's values, from the p tile when the selection is dense
                si.mg_ns = (uint32_t)(((1u << 24) + (uint32_t)ns - 1u) / (uint32_t)ns);
                si.psub_mode = L.psub_mode;
                si.pstaged = L.psub_mode == 1 && L.p_tma;
                if (si.pstaged) {
                    const unsigned char* P = static_cast<const unsigned char*>(L.P);
                    si.oP = off;
                    if (L.nseg == 1 && L.ldp == L.m) {
                        bulk_g2s(A + off, P + g.r0 * L.m * PSZ, (uint32_t)(g.Rr * sw * PSZ), &full[st], pol_last);
                    } else {
                        for (int r = 0; r < g.Rr; ++r)
                            bulk_g2s(A + off + r * sw * PSZ, P + ((g.r0 + r) * L.ldp + g.c0) * PSZ,
                                     (uint32_t)(sw * PSZ), &full[st], pol_last);
                    }
                    tx += (uint32_t)(g.Rr * sw * PSZ);
                    off += (g.Rr * sw * PSZ + 15) & ~15;
                }
            } else if (prm.do_adam && ns > 0) {
                si.mg_ns = (uint32_t)(((1u << 24) + (uint32_t)ns - 1u) / (uint32_t)ns);
                si.pstaged = L.p_tma;
                si.mstaged = L.mv_tma;
                si.psub_mode = L.psub_mode;
                if (si.psub_mode == 2 && si.mstaged) {
                    // steady step: p's current selected values from the dense subset block,
                    // the [R, s0:s1) slab (same layout as the moment slab)
                    const int64_t e0 = g.r0 * L.k + si.s0, e1 = (g.r0 + g.Rr - 1) * L.k + si.s1;
                    si.ePs = stage_elems<PSZ>(A, &off, L.psub, e0, e1, &full[st], &tx, &si.oPs);
                } else if (si.psub_mode == 3 && si.mstaged) {
                    // refresh from the previous block: the unit's full old rows, like the old moments
                    si.ePs = stage_elems<PSZ>(A, &off, L.psub_in, g.r0 * L.k_in, (g.r0 + g.Rr) * L.k_in, &full[st],
                                              &tx, &si.oPs);
                }
                if (si.pstaged) {
                    const unsigned char* P = static_cast<const unsigned char*>(L.P);
                    si.oP = off;
                    if (L.nseg == 1 && L.ldp == L.m) {
                        bulk_g2s(A + off, P + g.r0 * L.m * PSZ, (uint32_t)(g.Rr * sw * PSZ), &full[st], pol_last);
                    } else {
                        for (int r = 0; r < g.Rr; ++r)
                            bulk_g2s(A + off + r * sw * PSZ, P + ((g.r0 + r) * L.ldp + g.c0) * PSZ,
                                     (uint32_t)(sw * PSZ), &full[st], pol_last);
                    }
                    tx += (uint32_t)(g.Rr * sw * PSZ);
                    off += (g.Rr * sw * PSZ + 15) & ~15;
                }
                if (si.mstaged) {
                    int64_t e0, e1;
                    if (L.slot_src) {  // refresh: the old moments of the unit's rows (full old rows)
                        e0 = g.r0 * L.k_in;
                        e1 = (g.r0 + g.Rr) * L.k_in;
                    } else {           // steady: the [R, s0:s1) slab (a superset when R > 1 and segmented)
                        e0 = g.r0 * L.k + si.s0;
                        e1 = (g.r0 + g.Rr - 1) * L.k + si.s1;
                    }
                    si.eM = stage_elems<4>(A, &off, L.m_in, e0, e1, &full[st], &tx, &si.oM);
                    si.eV = stage_elems<4>(A, &off, L.v_in, e0, e1, &full[st], &tx, &si.oV);
                }
            }
            si.Rr = g.Rr;
            si.sw = sw;
            si.k = (int32_t)L.k;
            si.kin = (int32_t)L.k_in;
            si.ldp = L.ldp;
            si.out_ld = L.out_ld;
            si.r0 = g.r0;
            si.c0 = g.c0;
            si.remap = L.slot_src != nullptr;
            si.P = static_cast<PB*>(L.P) + g.r0 * L.ldp;
            si.out = L.out;
            si.m_out = L.m_out + g.r0 * L.k;
            si.v_out = L.v_out + g.r0 * L.k;
            si.psub = L.psub ? static_cast<PB*>(L.psub) + g.r0 * L.k : nullptr;
            si.gsel = L.gsel ? static_cast<GB*>(L.gsel) + g.r0 * L.k : nullptr;
            si.m_in = L.m_in;
            si.v_in = L.v_in;
            si.steps = L.steps;
            si.sbv = L.sbv;
            si.slot_src = L.slot_src;
            si.idx = L.idx;
            si.ucol = L.ucol;
            si.done = L.done;
            info[st] = si;
            prev_done = si.done;
            mbar_expect_tx(&full[st], tx);  // the single arrival of this phase
        }
        return;
    }

    // ===================== consumer warps =====================
    // Two groups of K3_GW warps; group g consumes stages g, g+2, ...  Per unit:
    //  (1) AdamW on the unit's (row, slot) pairs by all threads of the group, row-major
    //      (adam_unit_b; the slot-major adam_unit serves the unstaged-moment paths and the
    //      ZF_K3_SLOTMAJOR build); each changed p value is stored straight to HBM;
    //  (2) compaction by gather, warp-wide windows of one row: lane l writes outputs
    //      8l..8l+7 (bf16; 4 for fp32) of the window with one 16-byte store, reading the
    //      staged tile at the unselected-column offsets (the layer's list, through L1);
    //  then each warp releases the stage.
    const int cwa = warp - K3_STAGES;          // consumer warp index
    const int grp = cwa / K3_GW;               // consumer group
    const int cw = cwa - grp * K3_GW;          // warp index within the group
    const int ctid = cw * 32 + lane;
    uint32_t dbg_sink = 0;             // debug mode 7 keeps the gathers live
    uint32_t nfacc = 0;                // non-finite detector (exponent all-ones -> carry into the top bit)
    __nv_bfloat162 nf2 = __float2bfloat162_rn(0.0f);  // bf16: NaN-propagating max of |x|
    uint32_t finished = 0, phase = 0;  // per stage: end sentinel seen / mbarrier parity

    constexpr uint32_t kMine = [] {
        uint32_t m = 0;
        for (int st = 0; st < K3_STAGES; st += K3_GROUPS) m |= 1u << st;
        return m;
    }();
    const uint32_t mine = kMine << grp;  // the stages of my group
#ifdef ZF_K3_PROF
    // per-warp cycle accounting (lane 0): wait full, AdamW, compaction, -, release
    unsigned long long pc[6] = {0, 0, 0, 0, 0, 0};
    long long tq = clock64();
#define ZF_TICK(i)                         \
    do {                                   \
        const long long tn_ = clock64();   \
        pc[i] += (unsigned long long)(tn_ - tq); \
        tq = tn_;                          \
    } while (0)
#else
#define ZF_TICK(i) \
    do {           \
    } while (0)
#endif
    for (int it = grp;; it += K3_GROUPS) {
        const int st = it % K3_STAGES;
        if ((finished >> st) & 1u) continue;
        mbar_wait_sleep(&full[st], (phase >> st) & 1u);
        ZF_TICK(0);
        phase ^= 1u << st;
        const StageInfo& si = info[st];
        if (si.u < 0) {  // this stage's producer ran out of units; others may still hold some
            finished |= 1u << st;
            if (finished == mine) break;
            continue;
        }
        if (prm.debug_mode == 1) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            continue;
        }
        const int sw = si.sw, Rr = si.Rr;
        unsigned char* A = smem + st * K3_ARENA;
        const GB* sG = reinterpret_cast<const GB*>(A + si.oG);
        const int ns = si.s1 - si.s0;
        const bool adam = prm.do_adam && (prm.debug_mode == 0 || prm.debug_mode >= 3) && ns > 0;

        // ---------------- (1) AdamW ----------------
        if (adam && cw < K3_AWARPS) {
#ifndef ZF_K3_SLOTMAJOR
            if (si.psub_mode == 2 && si.mstaged) {
                adam_unit_b<GDT, PDT, false, false, true>(si, A, prm, ctid, nfacc);
            } else if (si.psub_mode == 3 && si.mstaged) {
                adam_unit_b<GDT, PDT, false, true, true>(si, A, prm, ctid, nfacc);
            } else if (si.pstaged && si.mstaged) {
                if (si.remap) adam_unit_b<GDT, PDT, true, true, false>(si, A, prm, ctid, nfacc);
                else adam_unit_b<GDT, PDT, true, false, false>(si, A, prm, ctid, nfacc);
            } else if (si.mstaged) {
                if (si.remap) adam_unit_b<GDT, PDT, false, true, false>(si, A, prm, ctid, nfacc);
                else adam_unit_b<GDT, PDT, false, false, false>(si, A, prm, ctid, nfacc);
            } else if (si.pstaged) {
#else
            if (si.psub_mode == 2 && si.mstaged) {
                adam_unit<GDT, PDT, false, true, false, true>(si, A, prm, ctid, nfacc);
            } else if (si.pstaged && si.mstaged) {
                if (si.remap) adam_unit<GDT, PDT, true, true, true>(si, A, prm, ctid, nfacc);
                else adam_unit<GDT, PDT, true, true, false>(si, A, prm, ctid, nfacc);
            } else if (si.mstaged) {
                if (si.remap) adam_unit<GDT, PDT, false, true, true>(si, A, prm, ctid, nfacc);
                else adam_unit<GDT, PDT, false, true, false>(si, A, prm, ctid, nfacc);
            } else if (si.pstaged) {
#endif
                adam_unit<GDT, PDT, true, false, false>(si, A, prm, ctid, nfacc);
            } else {
                adam_unit<GDT, PDT, false, false, false>(si, A, prm, ctid, nfacc);
            }
        }

        if (prm.do_extract && ns > 0 && cw < K3_AWARPS) {
            // split update (K3a): the unit's selected gradients -> gsel [n, k] (and, rebuilding
            // the parameter subset, p's selected values -> psub), pairs row-major: the warp's
            // lanes write consecutive slots of one row
            const GB* sGx = reinterpret_cast<const GB*>(A + si.oG);
            const PB* sPx = reinterpret_cast<const PB*>(A + si.oP);
            const PB* gPx = static_cast<const PB*>(si.P);
            GB* gsel = static_cast<GB*>(si.gsel);
            PB* psub = static_cast<PB*>(si.psub);
            const int s0 = si.s0, k = si.k, c0 = (int)si.c0, ldp = (int)si.ldp, total = Rr * ns;
            constexpr int NCT = K3_AWARPS * 32;
            int r = (int)(((uint64_t)ctid * si.mg_ns) >> 24), sl = ctid - r * ns;
            const int dr = (int)(((uint64_t)NCT * si.mg_ns) >> 24), dsl = NCT - dr * ns;
            for (int q = ctid; q < total; q += NCT) {
                const int s = s0 + sl;
                const int c = __ldg(si.idx + s);
                const GB gb = sGx[r * sw + c - c0];
                if constexpr (GSZ == 2) nfacc |= ((uint32_t)gb & 0x7f80u) + 0x0080u;
                else nfacc |= ((uint32_t)gb & 0x7f800000u) + 0x00800000u;
                gsel[r * k + s] = gb;
                if (si.psub_mode == 1) psub[r * k + s] = si.pstaged ? sPx[r * sw + c - c0] : gPx[r * ldp + c];
                r += dr;
                sl += dsl;
                if (sl >= ns) { sl -= ns; ++r; }
            }
        }

        ZF_TICK(1);
        // ---------------- (2) compaction by gather ----------------
        const int nk = si.nkeep;
        const int cc = cw - K3_CW0;                // compaction warp index (role split)
        const int cct = cc * 32 + lane;
        if (prm.do_compact && nk > 0 && prm.debug_mode != 3 && cc >= 0) {
            constexpr int OPL = 16 / GSZ;              // outputs per lane (one 16-byte store)
            const int j0 = si.j0;
            const int old = (int)si.out_ld;
            const uint16_t* gU = si.ucol + j0;         // the segment's unselected columns (byte offsets mod 2^16)
            const uint32_t base = (uint32_t)((si.c0 * GSZ) & 0xffff);  // the tile's first byte offset
            const uint32_t base2 = base | (base << 16);
            const uint32_t sGa = smem_u32(sG);
            GB* out = static_cast<GB*>(si.out) + si.r0 * si.out_ld + j0;   // row 0, output 0 of the unit
            if (old % OPL == 0) {
                // q = qa + OPL*g has (j0 + q) % OPL == 0: aligned offset loads and stores
                const int qa = min(nk, (OPL - (j0 & (OPL - 1))) & (OPL - 1));
                const int ng = (nk - qa) / OPL;        // full groups per row
                const int tail = nk - qa - OPL * ng;
                const int nwin = (ng + 31) >> 5;       // 32-group windows per row
                if (nwin > 0) {
                    // (window, row) pairs, window-major, in one contiguous share per warp: a
                    // window's offset vector is loaded once for all its rows, and the next
                    // window's is prefetched while the current one's rows are gathered
                    const int npair = nwin * Rr;
                    const int per = (npair + K3_CWARPS - 1) / K3_CWARPS;
                    int f = cc * per;
                    const int f1 = min(npair, f + per);
                    int w = f / Rr, r = f - w * Rr;
                    auto load_u = [&](int ww) {
                        const int g = (ww << 5) + lane;
                        uint4 u = make_uint4(0u, 0u, 0u, 0u);
                        if (ww < nwin && g < ng) {
                            if constexpr (GSZ == 2) u = ldg_nc_v4(gU + qa + OPL * g);
                            else {
                                const uint2 u2 = ldg_nc_v2(gU + qa + OPL * g);
                                u.x = u2.x;
                                u.y = u2.y;
                            }
                        }
                        u.x = __vsub2(u.x, base2);    // per-halfword: offsets within the tile row
                        u.y = __vsub2(u.y, base2);
                        u.z = __vsub2(u.z, base2);
                        u.w = __vsub2(u.w, base2);
                        return u;
                    };
                    uint4 u = f < f1 ? load_u(w) : make_uint4(0u, 0u, 0u, 0u);
                    uint4 un = u;
                    for (; f < f1; ++f) {
                        if (r == Rr - 1 && f + 1 < f1) un = load_u(w + 1);   // prefetch the next window
                        const int g = (w << 5) + lane;
                        if (g < ng) {
                            const int q = qa + OPL * g;
                            const uint32_t rowa = sGa + (uint32_t)(r * sw * GSZ);
                            uint4 o;
                            if constexpr (GSZ == 2) {
                                o.x = lds_u16(rowa + (u.x & 0xffffu)) | (lds_u16(rowa + (u.x >> 16)) << 16);
                                o.y = lds_u16(rowa + (u.y & 0xffffu)) | (lds_u16(rowa + (u.y >> 16)) << 16);
                                o.z = lds_u16(rowa + (u.z & 0xffffu)) | (lds_u16(rowa + (u.z >> 16)) << 16);
                                o.w = lds_u16(rowa + (u.w & 0xffffu)) | (lds_u16(rowa + (u.w >> 16)) << 16);
                                nf2 = __hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.x)),
                                                                   __habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.y))));
                                nf2 = __hmax2_nan(nf2, __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.z)),
                                                                   __habs2(*reinterpret_cast<const __nv_bfloat162*>(&o.w))));
                            } else {
                                // fp32: 4 offsets per lane
                                o.x = lds_u32(rowa + (u.x & 0xffffu));
                                o.y = lds_u32(rowa + (u.x >> 16));
                                o.z = lds_u32(rowa + (u.y & 0xffffu));
                                o.w = lds_u32(rowa + (u.y >> 16));
                                nfacc |= ((o.x & 0x7f800000u) + 0x00800000u) | ((o.y & 0x7f800000u) + 0x00800000u) |
                                         ((o.z & 0x7f800000u) + 0x00800000u) | ((o.w & 0x7f800000u) + 0x00800000u);
                            }
                            if (prm.debug_mode != 7 && prm.debug_mode != 11) st_cs_v4(out + r * old + q, o);  // (11: no compaction stores)
                            else dbg_sink ^= o.x ^ o.y ^ o.z ^ o.w;  // keep the gather live
                        }
                        if (++r == Rr) {
                            r = 0;
                            ++w;
                            u = un;
                        }
                    }
                }
                // per row: the qa head and the tail outputs
                for (int i = cct; i < Rr * 2 * OPL; i += K3_CWARPS * 32) {
                    const int r = i / (2 * OPL), e = i - r * (2 * OPL);
                    int q;
                    if (e < OPL) {
                        if (e >= qa) continue;
                        q = e;
                    } else {
                        if (e - OPL >= tail) continue;
                        q = qa + OPL * ng + (e - OPL);
                    }
                    const uint32_t bo = ((uint32_t)__ldg(gU + q) - base) & 0xffffu;
                    const GB x = sG[r * sw + bo / GSZ];
                    if constexpr (GSZ == 2) nfacc |= ((uint32_t)x & 0x7f80u) + 0x0080u;
                    else nfacc |= ((uint32_t)x & 0x7f800000u) + 0x00800000u;
                    out[r * old + q] = x;
                }
            } else {
                // unaligned output rows (stateless primitive with a dense [n, m-k] block)
                for (int i = cct; i < Rr * nk; i += K3_CWARPS * 32) {
                    const int r = i / nk, q = i - r * nk;
                    const uint32_t bo = ((uint32_t)__ldg(gU + q) - base) & 0xffffu;
                    const GB x = sG[r * sw + bo / GSZ];
                    if constexpr (GSZ == 2) nfacc |= ((uint32_t)x & 0x7f80u) + 0x0080u;
                    else nfacc |= ((uint32_t)x & 0x7f800000u) + 0x00800000u;
                    out[r * old + q] = x;
                }
            }
        }

        ZF_TICK(2);
        // stage fully consumed by this warp
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);   // (the producer then counts the unit for X1)
        ZF_TICK(4);
#ifdef ZF_K3_PROF
        pc[5] += 1;  // units
#endif
    }
#ifdef ZF_K3_PROF
    if (lane == 0 && prm.prof)
        for (int i = 0; i < 6; ++i) atomicAdd(prm.prof + i, pc[i]);
#endif
#undef ZF_TICK
    asm volatile("" ::"r"(dbg_sink));
    if (prm.nonfinite) {
        uint32_t hit = GSZ == 2 ? (nfacc & 0x80008000u) : (nfacc & 0x80000000u);
        if constexpr (GSZ == 2) {
            const uint32_t b = *reinterpret_cast<const uint32_t*>(&nf2);
            hit |= ((b & 0xffffu) >= 0x7f80u) | ((b >> 16) >= 0x7f80u);
        }
        if (__any_sync(0xffffffffu, hit != 0) && lane == 0) *prm.nonfinite = 1;
    }
}

// K3 prologue: each slot's bias-correction pair {ss, bc2s} for this launch's step counts
// (t_s = steps[s] + step_delta + 1), so that K3 stages it with the slot's column index and
// its AdamW chain has no global table lookup.  One block row per layer.
__global__ void k_slot_consts(const UpdLayer* __restrict__ layers, int32_t step_delta, AdamK a) {
    const UpdLayer& L = layers[blockIdx.y];
    if (!L.sbv) return;
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L.k; s += (int64_t)gridDim.x * blockDim.x)
        L.sbv[s] = adam_sb(__ldg(L.steps + s) + step_delta + 1, a);
}

// Stateless AdamW-only form: (row, slot) pairs, G read at the selected columns only.
template <int GDT, int PDT>
__global__ void __launch_bounds__(256) k_adam_only(const void* __restrict__ Gv, int64_t ldg, void* Pv, int64_t ldp,
                                                   int64_t n, const int32_t* __restrict__ idx, int64_t k, float* M,
                                                   float* V, int32_t* steps, uint32_t* counter, AdamK a) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    const typename GE::bits* G = static_cast<const typename GE::bits*>(Gv);
    typename PE::bits* P = static_cast<typename PE::bits*>(Pv);
    const int64_t total = n * k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / k, s = q - i * k;
        const int32_t c = __ldg(idx + s);
        float p = PE::to_f(P[i * ldp + c]);
        float mm = M[q], vv = V[q];
        adamw_elem(GE::to_f(G[i * ldg + c]), p, mm, vv, steps[s] + 1, a);
        P[i * ldp + c] = PE::from_f(p);
        M[q] = mm;
        V[q] = vv;
    }
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = (atomicAdd(counter, 1u) + 1u == gridDim.x);
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        for (int64_t s = threadIdx.x; s < k; s += blockDim.x) steps[s] = __ldcg(steps + s) + 1;
    }
}

template <int GDT, int PDT>
void set_attr() {
    static bool done = false;
    if (!done) {
        cudaFuncSetAttribute(k_update<GDT, PDT>, cudaFuncAttributeMaxDynamicSharedMemorySize, K3_SMEM);
        done = true;
    }
}

}  // namespace

UpdLimits update_limits() {
    UpdLimits l;
    l.arena_bytes = K3_ARENA;
    l.consumer_warps = 1;      // completion-counter increments per unit (one, by the stage's producer)
    l.producers = K3_STAGES;
    return l;
}

int update_grid(int, int) {
    int dev = 0, sms = NUM_SMS_B200;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // ZF_K3_GRID: experiment knob (fewer persistent CTAs than SMs: is K3 bound per SM or globally?)
    static const int env = getenv("ZF_K3_GRID") ? atoi(getenv("ZF_K3_GRID")) : 0;
    if (env > 0 && env < sms) return env;
    return sms;
}

cudaError_t launch_update(const UpdParams& p, int gdt, int pdt, int grid, cudaStream_t s) {
    if (p.total_units <= 0) return cudaSuccess;
    int g = (int)zmin<int64_t>((int64_t)grid, p.total_units);
#define ZF_LAUNCH(GD, PD)                                            \
    do {                                                             \
        set_attr<GD, PD>();                                          \
        k_update<GD, PD><<<g, K3_THREADS, K3_SMEM, s>>>(p);          \
    } while (0)
    if (gdt == DT_BF16 && pdt == DT_BF16) ZF_LAUNCH(DT_BF16, DT_BF16);
    else if (gdt == DT_F32 && pdt == DT_F32) ZF_LAUNCH(DT_F32, DT_F32);
    else if (gdt == DT_BF16 && pdt == DT_F32) ZF_LAUNCH(DT_BF16, DT_F32);
    else ZF_LAUNCH(DT_F32, DT_BF16);
#undef ZF_LAUNCH
    return cudaGetLastError();
}

cudaError_t launch_slot_consts(const UpdLayer* layers, int32_t nl, int64_t max_k, int32_t step_delta, const AdamK& a,
                               cudaStream_t s) {
    if (nl <= 0 || max_k <= 0) return cudaSuccess;
    const dim3 grid((unsigned)zmin<int64_t>((max_k + 255) / 256, 64), (unsigned)nl);
    k_slot_consts<<<grid, 256, 0, s>>>(layers, step_delta, a);
    return cudaGetLastError();
}

cudaError_t launch_adam_only(const void* G, int gdt, int64_t ldg, void* P, int pdt, int64_t ldp, int64_t n,
                             const int32_t* idx, int64_t k, float* m, float* v, int32_t* steps, uint32_t* counter,
                             const AdamK& a, cudaStream_t s) {
    const int64_t total = n * k;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > NUM_SMS_B200 * 8) blocks = NUM_SMS_B200 * 8;
    const int gb = (int)blocks;
#define ZF_LAUNCH(GD, PD) k_adam_only<GD, PD><<<gb, 256, 0, s>>>(G, ldg, P, ldp, n, idx, k, m, v, steps, counter, a)
    if (gdt == DT_BF16 && pdt == DT_BF16) ZF_LAUNCH(DT_BF16, DT_BF16);
    else if (gdt == DT_F32 && pdt == DT_F32) ZF_LAUNCH(DT_F32, DT_F32);
    else if (gdt == DT_BF16 && pdt == DT_F32) ZF_LAUNCH(DT_BF16, DT_F32);
    else ZF_LAUNCH(DT_F32, DT_BF16);
#undef ZF_LAUNCH
    return cudaGetLastError();
}

}  // namespace zf
