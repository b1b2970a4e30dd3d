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
// G, 2(1-κ) B of compact output, and for the κ selected columns the
// sector-scattered read-modify-write of p plus dense fp32 m, v.
//  - persistent grid, one 512-thread CTA per SM; work units (a tile of R whole
//    rows, or a column segment of one row when a row exceeds the tile) are
//    claimed dynamically with one atomic per unit, so mixed layer shapes
//    balance across the 148 SMs;
//  - G tiles are staged into a 4-deep shared-memory ring by the bulk-copy
//    engine (cp.async.bulk / TMA, completion on an mbarrier), claimed and
//    issued STAGES-1 units ahead, so HBM reads stay in flight while the CTA
//    works on the current tile;
//  - compaction reads the tile in 32-column groups (lane = column, one mask
//    word per group): the column's compact position is
//    column - (prefix[word] + popc(mask & lanemask_lt)), written into a
//    shared output tile that is then streamed out with aligned 16-byte stores
//    (the compact block of a unit is one contiguous range of the output);
//  - AdamW runs over (row, slot) pairs, so the moments [n, k] are read and
//    written fully coalesced; g comes from the staged tile; p is the only
//    scattered access (2-byte elements in 32-byte sectors).  The pair loads are
//    issued before the compaction phase so their latency overlaps it;
//  - every AdamW op is an explicit round-to-nearest intrinsic (no FMA
//    contraction), matching the oracle's op order bit for bit;
//  - when the last unit of a layer finishes (per-layer cyclic counter), its CTA
//    advances the per-slot step counts; the same counter gates the layer's
//    device->host copy (cuStreamWaitValue32) when offloading.
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K3_THREADS = 512;
constexpr int K3_WARPS = K3_THREADS / 32;
constexpr int K3_STAGES = 4;
constexpr int K3_STAGE_BYTES = 32 * 1024;
constexpr int K3_OUT_BYTES = K3_STAGE_BYTES + 64;
constexpr int K3_BATCH = 4;  // AdamW pairs in flight per thread
constexpr int K3_SMEM = K3_STAGES * K3_STAGE_BYTES + K3_OUT_BYTES + 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
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
__device__ __forceinline__ void st_cs_v4(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ int find_layer(const Table<UpdLayer>& t, int64_t u) {
    int lo = 0, hi = t.n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (t[mid].unit_begin <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

struct UnitGeom {
    int64_t r0;   // first row
    int32_t Rr;   // rows
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

// number of selected columns < c (c is 0, m, or a multiple of 32)
__device__ __forceinline__ int64_t sel_before(const UpdLayer& L, int64_t c) {
    if (c >= L.m) return L.k;
    return __ldg(L.prefix + (c >> 5));
}

template <int GDT, int PDT>
__global__ void __launch_bounds__(K3_THREADS, 1) k_update(const __grid_constant__ UpdParams prm) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    constexpr int GSZ = GE::SIZE;
    constexpr int VEC = GE::VEC;

    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* stage_buf = smem;
    GB* sOut = reinterpret_cast<GB*>(smem + K3_STAGES * K3_STAGE_BYTES);
    __shared__ __align__(8) uint64_t bars[K3_STAGES];
    __shared__ int64_t st_unit[K3_STAGES];
    __shared__ int32_t st_layer[K3_STAGES];
    __shared__ int s_bad;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const Table<UpdLayer>& table = prm.layers;
    const uint64_t policy = evict_first_policy();

    // ---- producer (thread 0): claim the next unit and start its tile copy
    bool exhausted = false;
    auto claim_issue = [&](int st) {
        int64_t u = -1;
        if (!exhausted) {
            const uint32_t c = atomicAdd(prm.claim, 1u) - prm.claim_base;
            if ((int64_t)c < prm.total_units) u = c; else exhausted = true;
        }
        st_unit[st] = u;
        if (u < 0) return;
        const int li = find_layer(table, u);
        st_layer[st] = li;
        const UpdLayer& L = table[li];
        if (!L.tma_ok) return;
        const UnitGeom g = unit_geom(L, u - L.unit_begin);
        const int64_t sw = g.c1 - g.c0;
        const uint32_t bytes = (uint32_t)(g.Rr * sw * GSZ);
        unsigned char* dst = stage_buf + st * K3_STAGE_BYTES;
        const unsigned char* G = static_cast<const unsigned char*>(L.G);
        mbar_expect_tx(&bars[st], bytes);
        if (L.nseg == 1 && L.ldg == L.m) {
            bulk_g2s(dst, G + g.r0 * L.m * GSZ, bytes, &bars[st], policy);
        } else {
            for (int r = 0; r < g.Rr; ++r)
                bulk_g2s(dst + r * sw * GSZ, G + ((g.r0 + r) * L.ldg + g.c0) * GSZ, (uint32_t)(sw * GSZ), &bars[st],
                         policy);
        }
    };

    if (tid == 0) {
        for (int st = 0; st < K3_STAGES; ++st) mbar_init(&bars[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_bad = 0;
        for (int st = 0; st < K3_STAGES; ++st) claim_issue(st);
    }
    __syncthreads();

    uint32_t phases = 0;  // per-stage mbarrier parity (bit st)
    int bad = 0;
    for (int it = 0;; ++it) {
        const int st = it % K3_STAGES;
        const int64_t u = st_unit[st];
        if (u < 0) break;
        const int li = st_layer[st];
        const UpdLayer& L = table[li];
        const UnitGeom g = unit_geom(L, u - L.unit_begin);
        const int64_t sw = g.c1 - g.c0;
        GB* sG = reinterpret_cast<GB*>(stage_buf + st * K3_STAGE_BYTES);
        const bool tma = L.tma_ok;
        if (tma) {
            mbar_wait(&bars[st], (phases >> st) & 1u);
            phases ^= 1u << st;
        } else {
            const GB* G = static_cast<const GB*>(L.G);
            for (int64_t q = tid; q < (int64_t)g.Rr * sw; q += K3_THREADS) {
                const int64_t r = q / sw, c = q - r * sw;
                sG[q] = G[(g.r0 + r) * L.ldg + g.c0 + c];
            }
            __syncthreads();
        }

        const int64_t k = L.k, m = L.m, mk = m - k;
        const int64_t s0 = sel_before(L, g.c0), s1 = sel_before(L, g.c1);
        const int64_t ns = s1 - s0;           // selected columns in the segment
        const int64_t u0 = g.c0 - s0;         // compact position of the segment's first unselected column
        const int64_t nu = sw - ns;           // unselected columns in the segment
        const int64_t o_base = g.r0 * mk + u0;
        const int head = (int)(o_base % VEC);

        // ---- AdamW pair loads (batch 0), issued before compaction to overlap latency
        const int64_t npairs = prm.do_adam ? (int64_t)g.Rr * ns : 0;
        float ag[K3_BATCH], ap[K3_BATCH], am[K3_BATCH], av[K3_BATCH];
        int32_t at[K3_BATCH];
        int64_t pidx[K3_BATCH], midx[K3_BATCH];
        const PB* Pin = static_cast<const PB*>(L.P);
        auto load_batch = [&](int64_t qb) {
#pragma unroll
            for (int b = 0; b < K3_BATCH; ++b) {
                const int64_t q = qb + (int64_t)b * K3_THREADS + tid;
                pidx[b] = -1;
                if (q < npairs) {
                    const int64_t r = q / ns, sl = q - r * ns;
                    const int64_t s = s0 + sl;
                    const int32_t c = __ldg(L.idx + s);
                    const int64_t row = g.r0 + r;
                    ag[b] = GE::to_f(sG[r * sw + (c - g.c0)]);
                    pidx[b] = row * L.ldp + c;
                    ap[b] = PE::to_f(Pin[pidx[b]]);
                    midx[b] = row * k + s;
                    if (L.slot_src) {
                        const int32_t src = __ldg(L.slot_src + s);
                        am[b] = src >= 0 ? __ldcs(L.m_in + row * L.k_in + src) : 0.0f;
                        av[b] = src >= 0 ? __ldcs(L.v_in + row * L.k_in + src) : 0.0f;
                    } else {
                        am[b] = __ldcs(L.m_in + midx[b]);
                        av[b] = __ldcs(L.v_in + midx[b]);
                    }
                    at[b] = __ldg(L.steps + s) + 1;
                }
            }
        };
        auto compute_store = [&]() {
            PB* Pout = static_cast<PB*>(L.P);
#pragma unroll
            for (int b = 0; b < K3_BATCH; ++b) {
                if (pidx[b] < 0) continue;
                float p = ap[b], mm = am[b], vv = av[b];
                adamw_elem(ag[b], p, mm, vv, at[b], prm.adam);
                Pout[pidx[b]] = PE::from_f(p);
                __stcs(L.m_out + midx[b], mm);
                __stcs(L.v_out + midx[b], vv);
            }
        };
        if (npairs > 0) load_batch(0);

        // ---- compaction into the shared output tile (+ non-finite scan of the whole tile)
        if (prm.do_compact) {
            const int64_t nw = (sw + 31) >> 5;
            const int64_t items = (int64_t)g.Rr * nw;
            const int64_t wbase = g.c0 >> 5;
            for (int64_t itm = warp; itm < items; itm += K3_WARPS) {
                const int64_t r = itm / nw, gw = itm - r * nw;
                const int64_t cl = gw * 32 + lane;  // column within the segment
                const uint32_t word = __ldg(L.mask + wbase + gw);
                const int32_t pre = __ldg(L.prefix + wbase + gw);
                if (cl < sw) {
                    const GB x = sG[r * sw + cl];
                    bad |= GE::nonfinite(x);
                    if (!((word >> lane) & 1u)) {
                        const int64_t cpos = (g.c0 + cl) - (pre + __popc(word & lanemask_lt()));  // compact column
                        sOut[head + r * nu + (cpos - u0)] = x;
                    }
                }
            }
        }
        if (npairs > 0) {
            compute_store();
            for (int64_t qb = (int64_t)K3_BATCH * K3_THREADS; qb < npairs; qb += (int64_t)K3_BATCH * K3_THREADS) {
                load_batch(qb);
                compute_store();
            }
        }
        __syncthreads();

        // ---- stream the compact tile out: aligned 16-byte stores, scalar edges
        if (prm.do_compact) {
            const int64_t total = (int64_t)g.Rr * nu;
            GB* out = static_cast<GB*>(L.out);
            const int64_t a0 = o_base - head;                      // aligned start (elements)
            const int64_t nch = (head + total + VEC - 1) / VEC;    // 16-byte chunks
            for (int64_t ch = tid; ch < nch; ch += K3_THREADS) {
                const int64_t lo = ch * VEC;                       // index into sOut
                if (lo >= head && lo + VEC <= head + total) {
                    st_cs_v4(out + a0 + lo, *reinterpret_cast<const uint4*>(sOut + lo));
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        const int64_t q = lo + e;
                        if (q >= head && q < head + total) out[a0 + q] = sOut[q];
                    }
                }
            }
        }
        __syncthreads();  // stage st and sOut free; all stores of this unit issued

        // ---- completion: layer counter, step counts, next claim
        if (warp == 0) {
            uint32_t last = 0;
            if (lane == 0) {
                if (L.done) {
                    __threadfence_system();
                    const uint32_t old = atomicAdd(L.done, 1u);
                    last = (old + 1u == (prm.epoch + 1u) * (uint32_t)L.units);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                claim_issue(st);
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last && prm.do_adam && L.steps_out) {
                __threadfence();
                for (int64_t s = lane; s < k; s += 32) L.steps_out[s] = __ldcg(L.steps + s) + 1;
            }
        }
    }
    if (bad) s_bad = 1;
    __syncthreads();
    if (tid == 0 && s_bad && prm.nonfinite) *prm.nonfinite = 1;
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

int update_stage_bytes() { return K3_STAGE_BYTES; }

int update_grid(int, int) {
    int dev = 0, sms = NUM_SMS_B200;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

cudaError_t launch_update(const UpdParams& p, int gdt, int pdt, int grid, cudaStream_t s) {
    if (p.total_units <= 0) return cudaSuccess;
    int g = (int)zmin<int64_t>((int64_t)grid, p.total_units);
#define ZF_LAUNCH(GD, PD)                                                                   \
    do {                                                                                    \
        set_attr<GD, PD>();                                                                 \
        k_update<GD, PD><<<g, K3_THREADS, K3_SMEM, s>>>(p);                                 \
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
