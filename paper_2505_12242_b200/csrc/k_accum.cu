// k_accum.cu -- K7: device-side window accumulation of the compacted unimportant
// gradients (row a8 on the GPU; `device_accumulate`).
//
// Paper: "offloaded to the CPU and gradually accumulated over several
// iterations"; P:437-441 double buffering.  B200 design: HBM (180 GB) holds both fp32
// window accumulators, so instead of shipping every step's bf16 compact block over the
// host link and adding it on the CPU, the GPU adds it in place and only the sealed fp32
// window crosses the link, once per window (4 B x (m-k) x n per S steps instead of
// 2 B x (m-k) x n per step).  acc = (first ? 0 : acc) + f32(x), one IEEE add per element
// in step order -- the same arithmetic as the host accumulation (bit-identical).
// HBM-bound streaming kernel: per element 2 B (bf16 x) + 4 B (acc read, skipped on a
// window's first step) + 4 B (acc write); 16-byte vector accesses, grid-stride over a
// flat element space that concatenates every layer's pitched [n, mk_pad] block.
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K7_THREADS = 256;

__device__ __forceinline__ int acc_find_layer(const AccLayer* t, int nl, int64_t v) {
    int lo = 0, hi = nl - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (t[mid].vec_begin <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// One thread per 8-element vector (bf16: 16 B in; fp32 in: two 16-byte loads).
template <int GDT>
__global__ void __launch_bounds__(K7_THREADS) k_accumulate(const AccLayer* __restrict__ layers, int32_t nl,
                                                           int64_t total_vec, int32_t first_host, int32_t buf_host,
                                                           const AutoState* __restrict__ st) {
    int first = first_host, buf = buf_host;
    if (st) {  // Zen-auto: the device window state decides (before K6 of this step runs)
        first = st->open ? 0 : 1;
        buf = (int)(st->win & 1);
    }
    int li = 0;
    for (int64_t v = blockIdx.x * (int64_t)K7_THREADS + threadIdx.x; v < total_vec;
         v += (int64_t)gridDim.x * K7_THREADS) {
        if (v < layers[li].vec_begin || (li + 1 < nl && v >= layers[li + 1].vec_begin))
            li = acc_find_layer(layers, nl, v);
        const AccLayer& L = layers[li];
        const int64_t e = (v - L.vec_begin) * 8;
        float* acc = (buf ? L.acc1 : L.acc0) + e;
        float x[8];
        if constexpr (GDT == DT_BF16) {
            const uint4 q = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(L.src) + e));
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                x[2 * i] = __uint_as_float(w[i] << 16);
                x[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
            }
        } else {
            const float4 a = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(L.src) + e));
            const float4 b = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(L.src) + e + 4));
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
            x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        }
        float4 a0 = make_float4(0.f, 0.f, 0.f, 0.f), a1 = a0;
        if (!first) {
            a0 = __ldcs(reinterpret_cast<const float4*>(acc));
            a1 = __ldcs(reinterpret_cast<const float4*>(acc + 4));
        }
        a0.x = __fadd_rn(a0.x, x[0]); a0.y = __fadd_rn(a0.y, x[1]);
        a0.z = __fadd_rn(a0.z, x[2]); a0.w = __fadd_rn(a0.w, x[3]);
        a1.x = __fadd_rn(a1.x, x[4]); a1.y = __fadd_rn(a1.y, x[5]);
        a1.z = __fadd_rn(a1.z, x[6]); a1.w = __fadd_rn(a1.w, x[7]);
        __stcs(reinterpret_cast<float4*>(acc), a0);
        __stcs(reinterpret_cast<float4*>(acc + 4), a1);
    }
}

}  // namespace

cudaError_t launch_accumulate(const AccLayer* layers, int32_t nl, int64_t total_vec, int gdt, int32_t first,
                              int32_t buf, const AutoState* st, cudaStream_t s) {
    if (total_vec <= 0) return cudaSuccess;
    int64_t blocks = (total_vec + K7_THREADS - 1) / K7_THREADS;
    if (blocks > (int64_t)NUM_SMS_B200 * 16) blocks = (int64_t)NUM_SMS_B200 * 16;
    if (gdt == DT_BF16)
        k_accumulate<DT_BF16><<<(unsigned)blocks, K7_THREADS, 0, s>>>(layers, nl, total_vec, first, buf, st);
    else
        k_accumulate<DT_F32><<<(unsigned)blocks, K7_THREADS, 0, s>>>(layers, nl, total_vec, first, buf, st);
    return cudaGetLastError();
}

}  // namespace zf
