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
// G, 2(1-κ) B of compact output, and for the selected columns the read-modify-
// write of p (in 32-byte sectors) and of the fp32 moments.
//  - persistent grid, one 544-thread CTA per SM, warp-specialised: warp 0 is the
//    producer, warps 1..16 consume.  Work units (R whole rows, or a 128-aligned
//    column segment of one row) are claimed dynamically, one atomic per unit.
//  - the producer stages EVERYTHING a unit needs into one of 4 shared-memory
//    stage arenas with bulk copies (cp.async.bulk, the TMA engine) completing on
//    one mbarrier: the G tile, the p tile (when the selection touches most of p's
//    32-byte sectors), the moment slabs (or the old rows on a refresh), the slot
//    step counts, the remap sources and the segment's mask/prefix words.  The
//    host sizes units so the worst case fits an arena; 3 units stay in flight.
//    Consumers issue no global loads.
//  - a consumer warp takes 256-column row chunks; lane l owns 8 consecutive
//    columns (one 16-byte shared load, one mask byte).  Its compact position is
//    8l - (selected before it in the chunk), from the prefix word and a popcount;
//    the unselected values go to a warp buffer that is streamed out with aligned
//    16-byte stores (partial edges scalar).  The selected columns are listed by
//    slot and updated with all 32 lanes busy (AdamW in shared memory, explicit
//    round-to-nearest intrinsics, the oracle's op order); moments are stored
//    coalesced; every 32-byte p sector holding a selected column is written back
//    whole from the staged tile.
//  - with offload, each consumer warp bumps a per-layer counter after its share
//    of a unit (red.release); the copy stream waits on it (cuStreamWaitValue32)
//    to start the layer's device->host copy.
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K3_NCW = 16;                        // consumer warps
constexpr int K3_GROUPS = 2;                      // independent consumer groups; group g owns stages g, g+2, ...
constexpr int K3_GW = K3_NCW / K3_GROUPS;         // warps per group
constexpr int K3_STAGES = 4;                      // stage arenas = producer warps (one chain per stage)
constexpr int K3_THREADS = 32 * (K3_NCW + K3_STAGES);
constexpr int K3_CHUNK = 512;                     // columns per warp block (32 lanes x 16)
constexpr int K3_WBUF_BYTES = (K3_CHUNK + 16) * 4;
constexpr int K3_WARP_BYTES = K3_WBUF_BYTES;
constexpr int K3_PAIRS = 3;                       // AdamW (row, slot) pairs in flight per consumer thread
constexpr int K3_ARENA = 48 * 1024;               // bytes per stage arena
constexpr int K3_SMEM = K3_STAGES * K3_ARENA + K3_NCW * K3_WARP_BYTES;
static_assert(K3_ARENA % 128 == 0 && K3_WARP_BYTES % 16 == 0, "alignment");
static_assert(K3_SMEM <= 227 * 1024 - 512, "shared memory budget");

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    // consumer-side wait: hardware try_wait, then short sleeps so that waiting warps do not
    // take issue slots from the warps still working on a stage
    uint32_t done = 0;
    int ns = 16;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
        if (done) return;
        __nanosleep(ns);
        ns = ns < 128 ? ns * 2 : 128;
    }
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    return done != 0;
}
// producer-side wait: back off with nanosleep so spinning does not steal issue slots
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
    int ns = 64;
    while (!mbar_test(bar, phase)) {
        __nanosleep(ns);
        ns = ns < 512 ? ns * 2 : 512;
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
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

__device__ __forceinline__ void sts16(void* p, uint16_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(smem_u32(p)), "h"(v) : "memory");
}
__device__ __forceinline__ void sts32(void* p, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(smem_u32(p)) : "memory");
    return v;
}
template <typename B>
__device__ __forceinline__ void sts_elem(B* p, B v) {
    if constexpr (sizeof(B) == 2) sts16(p, v);
    else sts32(p, v);
}

// Bulk-copy the 4-byte elements [e0, e1) of `src` to arena offset *off as an aligned
// superset (16-byte granules; the source arrays are padded).  Returns the element
// offset of e0 within the copy; advances *off.
__device__ __forceinline__ int stage_words(unsigned char* arena, int* off, const void* src, int64_t e0, int64_t e1,
                                           uint64_t* bar, uint32_t* tx, int* where) {
    const int64_t a = e0 & ~int64_t(3), b = (e1 + 3) & ~int64_t(3);
    *where = *off;
    if (b > a) {
        const uint32_t bytes = (uint32_t)((b - a) * 4);
        bulk_g2s(arena + *off, static_cast<const int32_t*>(src) + a, bytes, bar, 0ull);
        *tx += bytes;
        *off += (int)bytes;
    }
    return (int)(e0 - a);
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
    int32_t oG, oP, oM, oV, oS, oSrc, oMask, oPre, oIdx;
    int32_t eM, eV, eS, eSrc, eMask, ePre, eIdx;
    int32_t pstaged, mstaged, remap;
    // unit geometry and layer fields, so consumers never touch the global layer table
    int32_t Rr, sw, k, kin, ldp;
    int64_t r0, c0, mk;
    void* P;                    // p + r0*ldp (row 0 of the unit)
    void* out;                  // compact block of the layer
    float* m_out;               // + r0*k
    float* v_out;
    const float* m_in;          // layer base (non-staged path)
    const float* v_in;
    const int32_t* steps;       // layer base (non-staged path)
    const int32_t* slot_src;
    const int32_t* idx;
    uint32_t* done;
};

template <int DT>
__device__ __forceinline__ void load8(const typename Elt<DT>::bits* p, uint32_t (&w)[8 * Elt<DT>::SIZE / 4]);
template <>
__device__ __forceinline__ void load8<DT_BF16>(const uint16_t* p, uint32_t (&w)[4]) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
}
template <>
__device__ __forceinline__ void load8<DT_F32>(const uint32_t* p, uint32_t (&w)[8]) {
    const uint4 a = *reinterpret_cast<const uint4*>(p);
    const uint4 b = *reinterpret_cast<const uint4*>(p + 4);
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

template <int GDT, int PDT>
__global__ void __launch_bounds__(K3_THREADS, 1) k_update(const __grid_constant__ UpdParams prm) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    constexpr int GSZ = GE::SIZE, PSZ = PE::SIZE;
    constexpr int VEC = GE::VEC;           // elements per 16 bytes
    constexpr int NW8 = 8 * GSZ / 4;       // 32-bit words holding 8 elements

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
        for (int it = 0;; ++it) {
            // claim and look up the next unit before waiting for its arena
            const uint32_t cl = atomicAdd(prm.claim, 1u) - prm.claim_base;
            StageInfo si{};
            si.u = (int64_t)cl < prm.total_units ? (int64_t)cl : -1;
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
            if (it > 0) mbar_wait_sleep(&empty[st], (it - 1) & 1);
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
            // mask + prefix words of the segment
            const int64_t w0 = g.c0 >> 5, nwm = (sw + 31) >> 5;
            si.eMask = stage_words(A, &off, L.mask, w0, w0 + nwm, &full[st], &tx, &si.oMask);
            si.ePre = stage_words(A, &off, L.prefix, w0, w0 + nwm, &full[st], &tx, &si.oPre);
            if (prm.do_adam && ns > 0) {
                si.pstaged = L.p_tma;
                si.mstaged = L.mv_tma;
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
                    } else {           // steady: the [R, s0:s1) slab (contiguous: full rows, or R == 1)
                        e0 = g.r0 * L.k + si.s0;
                        e1 = (g.r0 + g.Rr - 1) * L.k + si.s1;
                    }
                    si.eM = stage_words(A, &off, L.m_in, e0, e1, &full[st], &tx, &si.oM);
                    si.eV = stage_words(A, &off, L.v_in, e0, e1, &full[st], &tx, &si.oV);
                    si.eS = stage_words(A, &off, L.steps, si.s0, si.s1, &full[st], &tx, &si.oS);
                    si.eIdx = stage_words(A, &off, L.idx, si.s0, si.s1, &full[st], &tx, &si.oIdx);
                    if (L.slot_src) si.eSrc = stage_words(A, &off, L.slot_src, si.s0, si.s1, &full[st], &tx, &si.oSrc);
                }
            }
            si.Rr = g.Rr;
            si.sw = sw;
            si.k = (int32_t)L.k;
            si.kin = (int32_t)L.k_in;
            si.ldp = (int32_t)L.ldp;
            si.r0 = g.r0;
            si.c0 = g.c0;
            si.mk = L.m - L.k;
            si.remap = L.slot_src != nullptr;
            si.P = static_cast<PB*>(L.P) + g.r0 * L.ldp;
            si.out = L.out;
            si.m_out = L.m_out + g.r0 * L.k;
            si.v_out = L.v_out + g.r0 * L.k;
            si.m_in = L.m_in;
            si.v_in = L.v_in;
            si.steps = L.steps;
            si.slot_src = L.slot_src;
            si.idx = L.idx;
            si.done = L.done;
            info[st] = si;
            mbar_expect_tx(&full[st], tx);  // the single arrival of this phase
        }
        return;
    }

    // ===================== consumer warps =====================
    // AdamW: the unit's (row, slot) pairs are spread over all consumer threads; their loads
    // are issued first so that their latency (global p when not staged) overlaps the
    // compaction.  Compaction: each warp takes one contiguous run of 512-column blocks
    // (row-major over the unit's rows); lane l of a block owns its columns 16l..16l+15; the
    // unselected values go to the warp buffer, flushed with aligned 16-byte stores after
    // every block (the < 16-byte remainder carries over).
    const int cwa = warp - K3_STAGES;          // consumer warp index (warp-area slot)
    const int grp = cwa / K3_GW;               // consumer group
    const int cw = cwa - grp * K3_GW;          // warp index within the group
    const int ctid = cw * 32 + lane;
    constexpr int NCT = K3_GW * 32;
    unsigned char* warea = smem + K3_STAGES * K3_ARENA + cwa * K3_WARP_BYTES;
    GB* wbuf = reinterpret_cast<GB*>(warea);
    uint32_t nfacc = 0;                // non-finite detector (exponent all-ones -> carry into the top bit)
    __nv_bfloat162 nf2 = __float2bfloat162_rn(0.0f);  // bf16 tiles: NaN-propagating max of |x|
    uint32_t finished = 0, phase = 0;  // per stage: end sentinel seen / mbarrier parity

    constexpr uint32_t kMine = [] {
        uint32_t m = 0;
        for (int st = 0; st < K3_STAGES; st += K3_GROUPS) m |= 1u << st;
        return m;
    }();
    const uint32_t mine = kMine << grp;  // the stages of my group
    for (int it = grp;; it += K3_GROUPS) {
        const int st = it % K3_STAGES;
        if ((finished >> st) & 1u) continue;
        mbar_wait(&full[st], (phase >> st) & 1u);
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
        const uint32_t* smask = reinterpret_cast<const uint32_t*>(A + si.oMask) + si.eMask;
        const int32_t* spre = reinterpret_cast<const int32_t*>(A + si.oPre) + si.ePre;

        // ---------------- AdamW pair loads (first batch) ----------------
        const int ns = si.s1 - si.s0;
        const int npairs = (prm.do_adam && prm.debug_mode == 0) ? Rr * ns : 0;
        float ag[K3_PAIRS], am[K3_PAIRS], av[K3_PAIRS];
        PB apb[K3_PAIRS];  // raw p bits: converted only in compute_pairs, so a global load's latency
                           // is not waited for before the compaction
        float ass[K3_PAIRS], abc[K3_PAIRS];  // bias corrections of each pair's step (table loads issued early)
        int32_t pidx[K3_PAIRS], midx[K3_PAIRS];  // p / moment offsets from the unit's row 0
        auto load_pairs = [&](int qb) {
            const float inv_ns = 1.0f / (float)ns;
            const int k = si.k, kin = si.kin, s0 = si.s0;
            const bool pst = si.pstaged, mst = si.mstaged, remap = si.remap;
            const PB* sP = reinterpret_cast<const PB*>(A + si.oP);
            const float* sM = reinterpret_cast<const float*>(A + si.oM) + si.eM;
            const float* sV = reinterpret_cast<const float*>(A + si.oV) + si.eV;
            const int32_t* sS = reinterpret_cast<const int32_t*>(A + si.oS) + si.eS;
            const int32_t* sSrc = reinterpret_cast<const int32_t*>(A + si.oSrc) + si.eSrc;
            const int32_t* sIdx = reinterpret_cast<const int32_t*>(A + si.oIdx) + si.eIdx;
            const int c0 = (int)si.c0;
#pragma unroll
            for (int b = 0; b < K3_PAIRS; ++b) {
                const int q = qb + b * NCT + ctid;
                pidx[b] = -1;
                if (q < npairs) {
                    int r = __float2int_rz((float)q * inv_ns);
                    if (r * ns > q) --r;
                    if ((r + 1) * ns <= q) ++r;
                    const int sl = q - r * ns;
                    const int s = s0 + sl;
                    const int c = mst ? sIdx[sl] : __ldg(si.idx + s);
                    const int cl = c - c0;
                    ag[b] = GE::to_f(sG[r * sw + cl]);
                    pidx[b] = r * si.ldp + c;
                    apb[b] = pst ? sP[r * sw + cl] : static_cast<const PB*>(si.P)[pidx[b]];
                    midx[b] = r * k + s;
                    if (mst) {
                        if (remap) {
                            const int32_t src = sSrc[sl];
                            am[b] = src >= 0 ? sM[r * kin + src] : 0.0f;
                            av[b] = src >= 0 ? sV[r * kin + src] : 0.0f;
                        } else {
                            am[b] = sM[r * k + sl];
                            av[b] = sV[r * k + sl];
                        }
                        const int32_t t = sS[sl] + prm.step_delta + 1;
                        ass[b] = adam_ss(t, prm.adam);
                        abc[b] = adam_bc2s(t, prm.adam);
                    } else {
                        const int64_t row = si.r0 + r;
                        if (remap) {
                            const int32_t src = __ldg(si.slot_src + s);
                            am[b] = src >= 0 ? __ldcs(si.m_in + row * kin + src) : 0.0f;
                            av[b] = src >= 0 ? __ldcs(si.v_in + row * kin + src) : 0.0f;
                        } else {
                            am[b] = __ldcs(si.m_in + row * k + s);
                            av[b] = __ldcs(si.v_in + row * k + s);
                        }
                        const int32_t t = __ldg(si.steps + s) + prm.step_delta + 1;
                        ass[b] = adam_ss(t, prm.adam);
                        abc[b] = adam_bc2s(t, prm.adam);
                    }
                }
            }
        };
        auto compute_pairs = [&]() {
            PB* P = static_cast<PB*>(si.P);
            float* Mo = si.m_out;
            float* Vo = si.v_out;
#pragma unroll
            for (int b = 0; b < K3_PAIRS; ++b) {
                if (pidx[b] < 0) continue;
                float p = PE::to_f(apb[b]), mm = am[b], vv = av[b];
                adamw_elem_t(ag[b], p, mm, vv, ass[b], abc[b], prm.adam);
                P[pidx[b]] = PE::from_f(p);
                __stcs(Mo + midx[b], mm);
                __stcs(Vo + midx[b], vv);
            }
        };
        // fast path: everything staged, steady step -> shared-memory operands only
        const bool fast = si.pstaged && si.mstaged && !si.remap;
        if (npairs > 0 && !fast) load_pairs(0);

        // ---------------- compaction ----------------
        const int nblk = (sw + K3_CHUNK - 1) / K3_CHUNK;
        const int nq = Rr * nblk;
        const int q0 = (nq * cw) / K3_GW, q1 = (nq * (cw + 1)) / K3_GW;
        const bool vec = (sw % 8) == 0;  // rows of the staged tile are 16-byte aligned
        GB* outp = static_cast<GB*>(si.out);
        int r = q0 / nblk, cc = q0 - r * nblk;
        int64_t obase = 0;   // global element index of wbuf[0] (16-byte aligned)
        int pend = 0;        // elements in wbuf (including `skip` leading ones we do not own)
        int skip = 0;

        auto start_row = [&]() {
            const int cl0 = cc * K3_CHUNK;
            const int64_t gpos = (si.r0 + r) * si.mk + (si.c0 + cl0 - spre[cl0 >> 5]);
            skip = (int)(gpos % VEC);
            obase = gpos - skip;
            pend = skip;
        };
        if (q0 < q1) start_row();
        for (int q = q0; q < q1; ++q) {
            const int cl0 = cc * K3_CHUNK, cl1 = min(sw, cl0 + K3_CHUNK);
            // lane l owns columns cl0 + 256h + 8l .. +7 of the block's two halves h = 0, 1:
            // 16-byte tile reads of a warp are contiguous (bank-conflict free)
            const int base0 = spre[cl0 >> 5];
            int keep_total = 0;
            int u[2], nv[2];
            uint32_t sb[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c8 = cl0 + 256 * h + 8 * lane;
                nv[h] = max(0, min(8, cl1 - c8));
                const uint32_t word = nv[h] > 0 ? smask[c8 >> 5] : 0u;
                const int sh = c8 & 31;
                sb[h] = (word >> sh) & ((1u << nv[h]) - 1u);
                const int selh = nv[h] > 0 ? (spre[c8 >> 5] - base0) + __popc(word & ((1u << sh) - 1u)) : 0;
                u[h] = pend + (256 * h + 8 * lane) - selh;
            }
            keep_total = (cl1 - cl0) - (int)__reduce_add_sync(0xffffffffu, (unsigned)(__popc(sb[0]) + __popc(sb[1])));
            const int blk_keep = keep_total;
            const GB* srow = sG + r * sw;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c8 = cl0 + 256 * h + 8 * lane;
                const uint32_t selb = sb[h];
                if (nv[h] == 8 && vec) {
                    // branch-free scatter: the address steps back over each selected column, so
                    // every kept element is one predicated store at an immediate offset from `a`
                    uint32_t a = smem_u32(wbuf + u[h]);
                    uint32_t w[NW8];
                    load8<GDT>(srow + c8, w);
#pragma unroll
                    for (int i = 0; i < NW8; ++i) {
                        if constexpr (GSZ == 2) nf2 = __hmax2_nan(nf2, __habs2(*reinterpret_cast<const __nv_bfloat162*>(&w[i])));
                        else nfacc |= (w[i] & 0x7f800000u) + 0x00800000u;
                    }
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        uint32_t x;
                        if constexpr (GSZ == 2) x = (e & 1) ? (w[e >> 1] >> 16) : w[e >> 1];
                        else x = w[e];
                        if ((selb >> e) & 1u) a -= GSZ;
                        else if constexpr (GSZ == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a + 2 * e), "r"(x) : "memory");
                        else asm volatile("st.shared.u32 [%0], %1;" ::"r"(a + 4 * e), "r"(x) : "memory");
                    }
                } else {
                    int uu = u[h];
                    for (int e = 0; e < nv[h]; ++e) {
                        const GB x = srow[c8 + e];
                        if constexpr (GSZ == 2) nfacc |= ((uint32_t)x & 0x7f80u) + 0x0080u;
                        else nfacc |= ((uint32_t)x & 0x7f800000u) + 0x00800000u;
                        if (!((selb >> e) & 1u)) sts_elem(wbuf + uu++, x);
                    }
                }
            }
            __syncwarp();
            pend += blk_keep;
            // flush: full 16-byte chunks (all at a row/run end), carry the partial remainder
            const bool fin = (cc + 1 == nblk) || (q + 1 == q1);
            const int nfull = fin ? (pend + VEC - 1) / VEC : pend / VEC;
            for (int ch = lane; ch < nfull; ch += 32) {
                const int lo = ch * VEC;
                if (lo >= skip && lo + VEC <= pend) {
                    st_cs_v4(outp + obase + lo, lds128(wbuf + lo));
                } else {
                    for (int e = max(lo, skip); e < min(lo + VEC, pend); ++e) outp[obase + e] = wbuf[e];
                }
            }
            __syncwarp();
            if (!fin) {
                const int rem = pend - nfull * VEC;
                GB v = 0;
                if (lane < rem) v = wbuf[nfull * VEC + lane];
                __syncwarp();
                if (lane < rem) sts_elem(wbuf + lane, v);
                __syncwarp();
                obase += nfull * VEC;
                pend = rem;
                if (nfull > 0) skip = 0;
            }
            if (++cc == nblk) {
                cc = 0;
                ++r;
                if (q + 1 < q1) start_row();
            }
        }

        // ---------------- AdamW compute + stores (then any further pair batches) ----------------
        if (npairs > 0 && fast) {
            const int k = si.k, s0 = si.s0, ldp = si.ldp, c0 = (int)si.c0;
            const PB* sP = reinterpret_cast<const PB*>(A + si.oP);
            const float* sM = reinterpret_cast<const float*>(A + si.oM) + si.eM;
            const float* sV = reinterpret_cast<const float*>(A + si.oV) + si.eV;
            const int32_t* sS = reinterpret_cast<const int32_t*>(A + si.oS) + si.eS;
            const int32_t* sIdx = reinterpret_cast<const int32_t*>(A + si.oIdx) + si.eIdx;
            PB* P = static_cast<PB*>(si.P);
            float* Mo = si.m_out + s0;
            float* Vo = si.v_out + s0;
            const int tdelta = prm.step_delta + 1;
            int r = ctid / ns, sl = ctid - r * ns;                 // one division per unit
            const int dr = NCT / ns, dsl = NCT - dr * ns;
            for (int q = ctid; q < npairs; q += NCT) {
                const int c = sIdx[sl];
                const int cl = c - c0;
                const float g = GE::to_f(sG[r * sw + cl]);
                float p = PE::to_f(sP[r * sw + cl]);
                float mm = sM[r * k + sl], vv = sV[r * k + sl];
                const int32_t t = sS[sl] + tdelta;
                adamw_elem_t(g, p, mm, vv, adam_ss(t, prm.adam), adam_bc2s(t, prm.adam), prm.adam);
                P[r * ldp + c] = PE::from_f(p);
                __stcs(Mo + r * k + sl, mm);
                __stcs(Vo + r * k + sl, vv);
                r += dr;
                sl += dsl;
                if (sl >= ns) { sl -= ns; ++r; }
            }
        } else if (npairs > 0) {
            compute_pairs();
            for (int qb = K3_PAIRS * NCT; qb < npairs; qb += K3_PAIRS * NCT) {
                load_pairs(qb);
                compute_pairs();
            }
        }
        // stage fully consumed by this warp
        __syncwarp();
        if (lane == 0) {
            uint32_t* done = si.done;
            mbar_arrive(&empty[st]);
            if (done) red_release_add(done, 1u);  // per-warp completion count (offload only)
        }
    }
    if (prm.nonfinite) {
        uint32_t hit = GSZ == 2 ? (nfacc & 0x80008000u) : (nfacc & 0x80000000u);
        if constexpr (GSZ == 2) {
            const uint32_t b = *reinterpret_cast<const uint32_t*>(&nf2);
            hit |= ((b & 0xffffu) >= 0x7f80u) | ((b >> 16) >= 0x7f80u);
        }
        if (__any_sync(0xffffffffu, hit != 0) && lane == 0) *prm.nonfinite = 1;
    }
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
    l.consumer_warps = K3_GW;  // warps that process (and count) each unit
    l.producers = K3_STAGES;
    return l;
}

int update_grid(int, int) {
    int dev = 0, sms = NUM_SMS_B200;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
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
