// k_norms.cu -- K1: per-column squared L2 norms of row-major gradient matrices,
// grouped over every layer in one launch.
//
// Paper: P:486 (§3.3 "Lightweight Proxy for Gradient Ranking"): "each GPU
// computes and shares per-column gradient norms squared (i.e., the sum of
// squared gradient values within each column)".  norms[j] = sum_i G[i][j]^2.
//
// B200 design (DESIGN.md §5 K1): HBM-bound streaming read of G (2 B/elt bf16).
//  - work unit = (layer, row block of RB rows, column block of 32 lanes x VEC
//    columns); one 256-thread CTA per unit; lane l owns VEC consecutive
//    columns and reads them with one 16-byte load per row (coalesced 512 B per
//    warp-row); 8 warps stride over the rows of the block with 4 loads in
//    flight per thread; fp32 accumulation in registers.
//  - deterministic: per-thread sequential sums, then a fixed-order sum over the
//    8 warps in shared memory, then the LAST-arriving CTA of a column block sums
//    the per-row-block partials in row-block order (no fp32 atomics), so the
//    result bits do not depend on scheduling.
//  - a column sum that is NaN/Inf (from a non-finite element) sets the flag.
#include "zf_internal.cuh"

namespace zf {
namespace {

#ifndef ZF_K1_THREADS
#define ZF_K1_THREADS 256
#endif
#ifndef ZF_K1_RB
#define ZF_K1_RB 1024
#endif
#ifndef ZF_K1_UNROLL
#define ZF_K1_UNROLL 4
#endif
constexpr int K1_THREADS = ZF_K1_THREADS;
constexpr int K1_WARPS = K1_THREADS / 32;
constexpr int K1_RB = ZF_K1_RB;          // rows per row block (1024: 7B K1 2.41 -> 1.91 ms, tools/k1_cfg.sh)
constexpr int K1_UNROLL = ZF_K1_UNROLL;  // rows in flight per thread

__device__ __forceinline__ int find_layer(const Table<NormLayer>& t, int64_t u) {
    int lo = 0, hi = t.n - 1;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (t[mid].unit_begin <= u) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <int DT>
__global__ void __launch_bounds__(K1_THREADS)
k_column_norms(const __grid_constant__ Table<NormLayer> table, int32_t* nonfinite, int64_t unit_off) {
    using E = Elt<DT>;
    constexpr int VEC = E::VEC;
    constexpr int CB = 32 * VEC;
    __shared__ float red[K1_WARPS][CB];
    __shared__ int s_last;

    const int64_t u = blockIdx.x + unit_off;   // (unit_off: a launch over a subset of the layers)
    const int li = find_layer(table, u);
    const NormLayer& L = table[li];
    const int64_t lu = u - L.unit_begin;
    const int rb = (int)(lu / L.ncb), cb = (int)(lu % L.ncb);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)rb * K1_RB, r1 = zmin<int64_t>(L.n, r0 + K1_RB);
    const int64_t c0 = (int64_t)cb * CB + (int64_t)lane * VEC;

    float acc[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[e] = 0.0f;

    const typename E::bits* G = static_cast<const typename E::bits*>(L.G);
    if (L.vec_ok && c0 + VEC <= L.m) {
        // 16-byte path: row starts and c0 are 16-byte aligned (checked on the host)
        int64_t r = r0 + warp;
        for (; r + (K1_UNROLL - 1) * K1_WARPS < r1; r += K1_UNROLL * K1_WARPS) {
            uint4 v[K1_UNROLL];
#pragma unroll
            for (int q = 0; q < K1_UNROLL; ++q)
                v[q] = __ldcs(reinterpret_cast<const uint4*>(G + (r + q * K1_WARPS) * L.ld + c0));
#pragma unroll
            for (int q = 0; q < K1_UNROLL; ++q) {
                const typename E::bits* b = reinterpret_cast<const typename E::bits*>(&v[q]);
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const float x = E::to_f(b[e]);
                    acc[e] = fmaf(x, x, acc[e]);
                }
            }
        }
        for (; r < r1; r += K1_WARPS) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(G + r * L.ld + c0));
            const typename E::bits* b = reinterpret_cast<const typename E::bits*>(&v);
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const float x = E::to_f(b[e]);
                acc[e] = fmaf(x, x, acc[e]);
            }
        }
    } else if (c0 < L.m) {
        // scalar path (unaligned rows or the ragged last column block)
        for (int64_t r = r0 + warp; r < r1; r += K1_WARPS) {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                if (c0 + e < L.m) {
                    const float x = E::to_f(G[r * L.ld + c0 + e]);
                    acc[e] = fmaf(x, x, acc[e]);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < VEC; ++e) red[warp][lane * VEC + e] = acc[e];
    __syncthreads();

    const int64_t cbase = (int64_t)cb * CB;
    for (int c = threadIdx.x; c < CB; c += K1_THREADS) {
        if (cbase + c >= L.m) continue;
        float s = red[0][c];
#pragma unroll
        for (int w = 1; w < K1_WARPS; ++w) s += red[w][c];
        if (L.nrb == 1) {
            L.out[cbase + c] = s;
            if (!isfinite(s) && nonfinite) *nonfinite = 1;
        } else {
            L.partial[(int64_t)rb * L.m + cbase + c] = s;
        }
    }
    if (L.nrb == 1) return;

    // Last CTA of this column block reduces the partials in row-block order.
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t old = atomicAdd(L.counter + cb, 1u);
        s_last = (old == (uint32_t)(L.nrb - 1));
        if (s_last) L.counter[cb] = 0;  // ready for the next launch (stream-ordered)
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int c = threadIdx.x; c < CB; c += K1_THREADS) {
        if (cbase + c >= L.m) continue;
        float s = __ldcg(L.partial + cbase + c);
        for (int b = 1; b < L.nrb; ++b) s += __ldcg(L.partial + (int64_t)b * L.m + cbase + c);
        L.out[cbase + c] = s;
        if (!isfinite(s) && nonfinite) *nonfinite = 1;
    }
}

}  // namespace

int norms_rows_per_block() { return K1_RB; }
int norms_cols_per_block(int gdt) { return 32 * (gdt == DT_BF16 ? 8 : 4); }

cudaError_t launch_norms(const Table<NormLayer>& t, int64_t total_units, int gdt, int32_t* nonfinite, cudaStream_t s,
                         int64_t unit_off) {
    if (total_units <= 0) return cudaSuccess;
    if (total_units > 0x7fffffff) return cudaErrorInvalidValue;
    if (gdt == DT_BF16)
        k_column_norms<DT_BF16><<<(unsigned)total_units, K1_THREADS, 0, s>>>(t, nonfinite, unit_off);
    else
        k_column_norms<DT_F32><<<(unsigned)total_units, K1_THREADS, 0, s>>>(t, nonfinite, unit_off);
    return cudaGetLastError();
}

}  // namespace zf
