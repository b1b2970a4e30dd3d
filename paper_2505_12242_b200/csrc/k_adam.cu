// k_adam.cu -- K3b: the selective AdamW of row a5 as a dense streaming pass.
//
// Paper: "the pre-identified important gradients remain on the GPU, where a
// selective-optimizer, initialized only with the corresponding parameter subset, performs
// an in-place update"; P:594 (PyTorch Adam/AdamW, formula O6 / reading R8).
//
// B200 design (DESIGN.md §5 K3).  K3a (k_update.cu) streams G once: it compacts the
// unselected columns and extracts the selected ones into a dense [n, k] block gsel (and, on
// refresh steps, p's selected values into the parameter-subset block psub).  K3b then runs
// AdamW over dense, row-major [n, k] arrays -- gsel, psub, exp_avg, exp_avg_sq -- so every
// load and store is coalesced and independent: an HBM-bound elementwise pass instead of a
// latency-bound phase inside K3a's per-unit pipeline (measured: K3 with AdamW fused into the
// unit pipeline 9.5 ms on Llama-2-7B k=10%, compaction alone 4.7 ms).  A parameter value
// whose bf16 bits change is stored to psub and to its column of p (the only scattered
// access); on refresh steps the moments come from the old slots (remap R7).
//
// Work: the [n, k] blocks of a layer are one flat array; a thread takes 4 consecutive
// elements (8-byte loads of bf16 gsel / psub, 16-byte loads of exp_avg / exp_avg_sq),
// so every access is a full, aligned vector; an element's slot is its flat index mod k
// (per-slot {ss, bc2s}, column and remap source come through L1).
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K3B_THREADS = 256;
constexpr int K3B_V = 4;   // elements per thread (the vector code below is written for 4)

__device__ __forceinline__ int find_chunk_layer(const UpdLayer* __restrict__ t, int nl, int64_t ch, int hint) {
    int li = hint;
    if (li >= nl || t[li].adam_row_begin > ch) li = 0;
    while (li + 1 < nl && t[li + 1].adam_row_begin <= ch) ++li;  // chunks are visited in increasing order
    return li;
}

// One element the simple way (a layer's last, partial chunk).
template <int GDT, int PDT, bool REMAP>
__device__ __forceinline__ void adam_one(const UpdLayer& L, int64_t e, const AdamK& a, int tdelta) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    const int64_t row = e / L.k;
    const int s = (int)(e - row * L.k);
    const float2 sb = L.sbv ? __ldg(L.sbv + s) : adam_sb(__ldg(L.steps + s) + tdelta, a);
    float m, v;
    if constexpr (REMAP) {
        const int src = __ldg(L.slot_src + s);
        m = src >= 0 ? L.m_in[row * L.k_in + src] : 0.0f;
        v = src >= 0 ? L.v_in[row * L.k_in + src] : 0.0f;
    } else {
        m = L.m_in[e];
        v = L.v_in[e];
    }
    PB* ps = static_cast<PB*>(L.psub);
    const PB po = ps[e];
    float p = PE::to_f(po);
    adamw_elem_t(GE::to_f(static_cast<const GB*>(L.gsel)[e]), p, m, v, sb.x, sb.y, a);
    const PB pn = PE::from_f(p);
    if (pn != po) {
        ps[e] = pn;
        static_cast<PB*>(L.P)[row * L.ldp + __ldg(L.idx + s)] = pn;
    }
    L.m_out[e] = m;
    L.v_out[e] = v;
}

// The vector loads of one chunk (K3B_V consecutive elements of a layer's flat [n, k] blocks,
// e0 % K3B_V == 0, all < n*k), issued ahead of its arithmetic.
template <int GDT, int PDT, bool REMAP>
__device__ __forceinline__ void chunk_load(const UpdLayer& L, int64_t e0, uint4& gq, uint4& pq, float4& mq, float4& vq) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    const typename GE::bits* gs = static_cast<const typename GE::bits*>(L.gsel) + e0;
    const typename PE::bits* ps = static_cast<const typename PE::bits*>(L.psub) + e0;
    if constexpr (GE::SIZE == 2) {
        const uint2 x = __ldcs(reinterpret_cast<const uint2*>(gs));
        gq = make_uint4(x.x, x.y, 0u, 0u);
    } else {
        gq = __ldcs(reinterpret_cast<const uint4*>(gs));
    }
    if constexpr (PE::SIZE == 2) {
        const uint2 x = __ldcs(reinterpret_cast<const uint2*>(ps));
        pq = make_uint4(x.x, x.y, 0u, 0u);
    } else {
        pq = __ldcs(reinterpret_cast<const uint4*>(ps));
    }
    if constexpr (!REMAP) {
        mq = __ldcs(reinterpret_cast<const float4*>(L.m_in + e0));
        vq = __ldcs(reinterpret_cast<const float4*>(L.v_in + e0));
    }
}

// A chunk's changed p values are not stored at once: their sectors are prefetched into L2
// and the stores issued after the NEXT chunk's arithmetic, so they land on cached sectors
// instead of stalling L2 on a partial-sector read-modify-write miss each.
template <typename PB>
struct PStores {
    PB* addr[K3B_V];
    PB val[K3B_V];
    uint32_t mask = 0;
    __device__ __forceinline__ void flush() {
#pragma unroll
        for (int j = 0; j < K3B_V; ++j)
            if (mask & (1u << j)) *addr[j] = val[j];
        mask = 0;
    }
};

template <int GDT, int PDT, bool REMAP>
__device__ __forceinline__ void adam_chunk(const UpdLayer& L, int64_t e0, const uint4& gq, const uint4& pq,
                                           const float4& mq, const float4& vq, const AdamK& a, int tdelta,
                                           PStores<typename Elt<PDT>::bits>& pend) {
    using GE = Elt<GDT>;
    using PE = Elt<PDT>;
    using GB = typename GE::bits;
    using PB = typename PE::bits;
    constexpr int V = K3B_V;
    const int k = (int)L.k;
    const int row0 = (int)(e0 / k), s0 = (int)(e0 - (int64_t)row0 * k);
    uint32_t gw[V], pw[V];
    if constexpr (GE::SIZE == 2) {
        gw[0] = gq.x & 0xffffu; gw[1] = gq.x >> 16; gw[2] = gq.y & 0xffffu; gw[3] = gq.y >> 16;
    } else {
        gw[0] = gq.x; gw[1] = gq.y; gw[2] = gq.z; gw[3] = gq.w;
    }
    if constexpr (PE::SIZE == 2) {
        pw[0] = pq.x & 0xffffu; pw[1] = pq.x >> 16; pw[2] = pq.y & 0xffffu; pw[3] = pq.y >> 16;
    } else {
        pw[0] = pq.x; pw[1] = pq.y; pw[2] = pq.z; pw[3] = pq.w;
    }
    float m[V] = {mq.x, mq.y, mq.z, mq.w}, v[V] = {vq.x, vq.y, vq.z, vq.w};
    float2 sb[V];
    {
        int row = row0, s = s0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            sb[j] = L.sbv ? __ldg(L.sbv + s) : adam_sb(__ldg(L.steps + s) + tdelta, a);
            if constexpr (REMAP) {
                // refresh: the element's moments come from its column's old slot (R7)
                const int src = __ldg(L.slot_src + s);
                m[j] = src >= 0 ? __ldcs(L.m_in + (int64_t)row * L.k_in + src) : 0.0f;
                v[j] = src >= 0 ? __ldcs(L.v_in + (int64_t)row * L.k_in + src) : 0.0f;
            }
            if (++s == k) { s = 0; ++row; }
        }
    }
    // the batch branch-free (independent chains interleave); if any element left the fast
    // path's exact range, the batch again with the IEEE intrinsics from the saved inputs
    float p[V], m1[V], v1[V];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        m1[j] = m[j];
        v1[j] = v[j];
        p[j] = PE::to_f((PB)pw[j]);
        ok &= adamw_elem_fast(GE::to_f((GB)gw[j]), p[j], m1[j], v1[j], sb[j].x, sb[j].y, a);
    }
    if (!ok) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            m1[j] = m[j];
            v1[j] = v[j];
            p[j] = PE::to_f((PB)pw[j]);
            adamw_elem_t(GE::to_f((GB)gw[j]), p[j], m1[j], v1[j], sb[j].x, sb[j].y, a);
        }
    }
    {
        PB* ps = static_cast<PB*>(L.psub) + e0;
        PB* P = static_cast<PB*>(L.P);
        int row = row0, s = s0;
        PStores<PB> now;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const PB pn = PE::from_f(p[j]);
            if (pn != (PB)pw[j]) {   // same memory state as storing every value
                ps[j] = pn;
                PB* at = P + (int64_t)row * L.ldp + __ldg(L.idx + s);
#ifdef ZF_K3B_DIRECT
                *at = pn;
#else
                asm volatile("prefetch.global.L2 [%0];" ::"l"(at));
                now.addr[j] = at;
                now.val[j] = pn;
                now.mask |= 1u << j;
#endif
            }
            if (++s == k) { s = 0; ++row; }
        }
        pend.flush();          // the previous chunk's stores (their sectors were prefetched then)
        pend = now;
    }
    __stcs(reinterpret_cast<float4*>(L.m_out + e0), make_float4(m1[0], m1[1], m1[2], m1[3]));
    __stcs(reinterpret_cast<float4*>(L.v_out + e0), make_float4(v1[0], v1[1], v1[2], v1[3]));
}

// adam_row_begin holds, for K3b, the layer's first chunk (prefix of ceil(n*k / 8) over layers)
template <int GDT, int PDT>
__global__ void __launch_bounds__(K3B_THREADS, 4) k_adam_dense(const UpdLayer* __restrict__ layers, int32_t nl,
                                                            int64_t total_chunks, int32_t step_delta, AdamK a) {
    using PB = typename Elt<PDT>::bits;
    const int tdelta = step_delta + 1;
    int li = 0;
    PStores<PB> pend;
    for (int64_t ch = (int64_t)blockIdx.x * K3B_THREADS + threadIdx.x; ch < total_chunks;
         ch += (int64_t)gridDim.x * K3B_THREADS) {
        li = find_chunk_layer(layers, nl, ch, li);
        const UpdLayer& L = layers[li];
        const int64_t e0 = (ch - L.adam_row_begin) * K3B_V;
        const int64_t ne = L.n * L.k;
        uint4 gq{}, pq{};
        float4 mq{}, vq{};
        if (e0 + K3B_V <= ne) {
            if (L.slot_src) {
                chunk_load<GDT, PDT, true>(L, e0, gq, pq, mq, vq);
                adam_chunk<GDT, PDT, true>(L, e0, gq, pq, mq, vq, a, tdelta, pend);
            } else {
                chunk_load<GDT, PDT, false>(L, e0, gq, pq, mq, vq);
                adam_chunk<GDT, PDT, false>(L, e0, gq, pq, mq, vq, a, tdelta, pend);
            }
        } else {
            for (int64_t e = e0; e < ne; ++e) {
                if (L.slot_src) adam_one<GDT, PDT, true>(L, e, a, tdelta);
                else adam_one<GDT, PDT, false>(L, e, a, tdelta);
            }
        }
    }
    pend.flush();
}

}  // namespace

int adam_dense_vec() { return K3B_V; }

cudaError_t launch_adam_dense(const UpdLayer* layers, int32_t nl, int64_t total_chunks, int gdt, int pdt,
                              int32_t step_delta, const AdamK& a, cudaStream_t s) {
    if (total_chunks <= 0) return cudaSuccess;
    int dev = 0, sms = NUM_SMS_B200;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (total_chunks + K3B_THREADS - 1) / K3B_THREADS;
    const int grid = (int)zmin<int64_t>(want, (int64_t)sms * 4);    // one resident wave, grid-stride
#define ZF_LAUNCH(GD, PD) k_adam_dense<GD, PD><<<grid, K3B_THREADS, 0, s>>>(layers, nl, total_chunks, step_delta, a)
    if (gdt == DT_BF16 && pdt == DT_BF16) ZF_LAUNCH(DT_BF16, DT_BF16);
    else if (gdt == DT_F32 && pdt == DT_F32) ZF_LAUNCH(DT_F32, DT_F32);
    else if (gdt == DT_BF16 && pdt == DT_F32) ZF_LAUNCH(DT_BF16, DT_F32);
    else ZF_LAUNCH(DT_F32, DT_BF16);
#undef ZF_LAUNCH
    return cudaGetLastError();
}

}  // namespace zf
