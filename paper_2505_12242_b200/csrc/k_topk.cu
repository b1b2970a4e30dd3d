// k_topk.cu -- K2: exact per-layer top-k column selection over the norm
// proxy, plus the selection tables the fused update consumes and the refresh
// remap of optimizer state (K4 index part).
//
// Paper: "the top-k selection, which retains the gradients with the
// highest magnitudes"; applied per weight matrix to the per-column norm proxy
// (reading R5); cached between refreshes.  Ties go to the
// lower column index (reading R3); the output is ascending.
//
// B200 design (DESIGN.md §5 K2): one 1024-thread CTA per layer, all layers in
// one launch.  Norms are non-negative fp32, so their bit patterns order like
// uint32: a 4-pass MSB-first 8-bit radix select over the keys (held in shared
// memory) finds the exact k-th key T and how many keys equal to T are taken;
// two block scans then give the tie ranks (ascending index) and the output
// slots.  No floating-point comparison is involved: the result is exact.
// Also emitted: the bitmask of selected columns, its per-32-column exclusive
// popcount prefix (slot of a column = prefix + popc of lower bits; compact
// position = column - slot), and, on a refresh, for each new slot the old slot
// of the same column (or -1) with its carried step count (reading R7).
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K2_THREADS = 1024;
constexpr int K2_WARPS = K2_THREADS / 32;
constexpr int64_t K2_SMEM_KEYS_MAX = 48 * 1024;  // keys held in shared memory up to this m

// Unselected columns of one mask word, in order: ucol[j] = the column's byte offset in the
// row, modulo 2^16 (K3 subtracts its tile's first byte offset modulo 2^16, so the list serves
// every unit shape whose tile rows are shorter than 64 KB).  j0 = index of the word's first
// unselected column.
__device__ __forceinline__ void emit_ucol(uint16_t* ucol, uint32_t word, int64_t w, int64_t m, int64_t j0,
                                          int64_t /*seg_cols*/, int gsz) {
    uint32_t keep = ~word;
    const int64_t cbase = w * 32;
    if (cbase + 32 > m) keep &= (1u << (m - cbase)) - 1u;
    int64_t j = j0;
    while (keep) {
        const int b = __ffs(keep) - 1;
        keep &= keep - 1u;
        ucol[j++] = (uint16_t)(((cbase + b) * gsz) & 0xffff);
    }
}

// Exclusive block-wide scan of one uint32 per thread; returns the prefix, total in *total.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* warp_sums, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < K2_WARPS ? warp_sums[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < K2_WARPS) warp_sums[lane] = wi - w;  // exclusive warp offsets
        if (lane == 31) warp_sums[K2_WARPS] = wi;
    }
    __syncthreads();
    const uint32_t r = warp_sums[warp] + incl - x;
    *total = warp_sums[K2_WARPS];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(K2_THREADS)
k_topk(const __grid_constant__ Table<TopkLayer> table, int use_smem, int32_t old_delta, int32_t* nonfinite) {
    extern __shared__ uint32_t dyn[];
    __shared__ uint32_t hist[256];
    __shared__ uint32_t warp_sums[K2_WARPS + 1];
    __shared__ uint32_t s_digit, s_above;

    const TopkLayer& L = table[blockIdx.x];
    const int64_t m = L.m, k = L.k;
    const int tid = threadIdx.x;

    // keys: shared copy when it fits, else read in place (L2-resident)
    const uint32_t* keys;
    if (use_smem) {
        for (int64_t j = tid; j < m; j += K2_THREADS) dyn[j] = __float_as_uint(__ldg(L.norms + j));
        keys = dyn;
    } else {
        keys = reinterpret_cast<const uint32_t*>(L.norms);
    }
    uint32_t* smask = use_smem ? dyn + m : nullptr;  // W words of mask
    const int64_t W = (m + 31) >> 5;
    if (smask) for (int64_t w = tid; w < W; w += K2_THREADS) smask[w] = 0u;
    else for (int64_t w = tid; w < W; w += K2_THREADS) L.mask[w] = 0u;
    __syncthreads();

    // ---- radix select: exact k-th largest key T and number of ties to take
    uint32_t prefix = 0, pmask = 0, rem = (uint32_t)k;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int b = tid; b < 256; b += K2_THREADS) hist[b] = 0u;
        __syncthreads();
        for (int64_t j = tid; j < m; j += K2_THREADS) {
            const uint32_t key = keys[j];
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns bins [255-8l-7, 255-8l]; scan from the top bin down
            uint32_t local[8], sum = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { local[q] = hist[255 - 8 * tid - q]; sum += local[q]; }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            const uint32_t excl = incl - sum;
            if (excl < rem && incl >= rem) {  // exactly one lane
                uint32_t above = excl;
                int q = 0;
                for (; q < 8; ++q) {
                    if (above + local[q] >= rem) break;
                    above += local[q];
                }
                s_digit = 255u - 8u * tid - (uint32_t)q;
                s_above = above;
            }
        }
        __syncthreads();
        rem -= s_above;
        prefix |= s_digit << shift;
        pmask |= 255u << shift;
        __syncthreads();
    }
    const uint32_t T = prefix;
    if (tid == 0 && T >= 0x7f800000u && nonfinite) *nonfinite = 1;  // NaN/Inf among the selected norms

    // ---- tie ranks (ascending index) and output slots; thread t owns a contiguous chunk
    const int64_t C = (m + K2_THREADS - 1) / K2_THREADS;
    const int64_t j0 = zmin<int64_t>(m, (int64_t)tid * C), j1 = zmin<int64_t>(m, j0 + C);
    uint32_t n_eq = 0;
    for (int64_t j = j0; j < j1; ++j) n_eq += (keys[j] == T);
    uint32_t tot;
    uint32_t eq_base = block_excl_scan(n_eq, warp_sums, &tot);
    uint32_t n_sel = 0;
    {
        uint32_t e = eq_base;
        for (int64_t j = j0; j < j1; ++j) {
            const uint32_t key = keys[j];
            if (key > T) ++n_sel;
            else if (key == T) { n_sel += (e < rem); ++e; }
        }
    }
    uint32_t out_base = block_excl_scan(n_sel, warp_sums, &tot);
    {
        uint32_t e = eq_base, o = out_base;
        for (int64_t j = j0; j < j1; ++j) {
            const uint32_t key = keys[j];
            bool sel = false;
            if (key > T) sel = true;
            else if (key == T) { sel = (e < rem); ++e; }
            if (sel) {
                L.idx[o++] = (int32_t)j;
                if (smask) atomicOr(&smask[j >> 5], 1u << (j & 31));
                else atomicOr(&L.mask[j >> 5], 1u << (j & 31));
            }
        }
    }
    __syncthreads();
    // ---- mask words and their exclusive popcount prefix
    const int64_t WC = (W + K2_THREADS - 1) / K2_THREADS;
    const int64_t w0 = zmin<int64_t>(W, (int64_t)tid * WC), w1 = zmin<int64_t>(W, w0 + WC);
    uint32_t pc = 0;
    for (int64_t w = w0; w < w1; ++w) pc += __popc(smask ? smask[w] : __ldcg(L.mask + w));
    uint32_t pbase = block_excl_scan(pc, warp_sums, &tot);
    for (int64_t w = w0; w < w1; ++w) {
        const uint32_t word = smask ? smask[w] : __ldcg(L.mask + w);
        if (smask) L.mask[w] = word;
        L.prefix[w] = (int32_t)pbase;
        if (L.ucol) emit_ucol(L.ucol, word, w, m, w * 32 - pbase, L.seg_cols, L.gsz);
        pbase += __popc(word);
    }
    // ---- refresh remap: old slot of each new slot's column (reading R7)
    if (L.slot_src) {
        __syncthreads();  // idx written by this CTA (global writes visible after the barrier)
        for (int64_t s = tid; s < k; s += K2_THREADS) {
            const int32_t c = L.idx[s];
            int32_t src = -1;
            if (L.old_mask) {
                const uint32_t word = __ldg(L.old_mask + (c >> 5));
                const uint32_t bit = 1u << (c & 31);
                if (word & bit) src = __ldg(L.old_prefix + (c >> 5)) + __popc(word & (bit - 1u));
            }
            L.slot_src[s] = src;
            L.new_steps[s] = src >= 0 ? __ldg(L.old_steps + src) + old_delta : 0;
        }
    }
}

// Stateless helper: mask + prefix from a caller-provided ascending idx.
__global__ void k_build_mask(const int32_t* __restrict__ idx, int64_t k, int64_t m, uint32_t* mask, int32_t* prefix,
                             uint16_t* ucol, int64_t seg_cols, int gsz, int32_t* bad) {
    __shared__ uint32_t warp_sums[K2_WARPS + 1];
    const int tid = threadIdx.x;
    const int64_t W = (m + 31) >> 5;
    for (int64_t w = tid; w < W; w += K2_THREADS) mask[w] = 0u;
    __syncthreads();
    for (int64_t s = tid; s < k; s += K2_THREADS) {
        const int32_t c = idx[s];
        if (c < 0 || c >= m || (s > 0 && idx[s - 1] >= c)) {   // skipped, so never out of bounds
            if (bad) *bad = 1;
            continue;
        }
        atomicOr(&mask[c >> 5], 1u << (c & 31));
    }
    __syncthreads();
    const int64_t WC = (W + K2_THREADS - 1) / K2_THREADS;
    const int64_t w0 = zmin<int64_t>(W, (int64_t)tid * WC), w1 = zmin<int64_t>(W, w0 + WC);
    uint32_t pc = 0;
    for (int64_t w = w0; w < w1; ++w) pc += __popc(__ldcg(mask + w));
    uint32_t tot;
    uint32_t pbase = block_excl_scan(pc, warp_sums, &tot);
    for (int64_t w = w0; w < w1; ++w) {
        const uint32_t word = __ldcg(mask + w);
        prefix[w] = (int32_t)pbase;
        if (ucol) emit_ucol(ucol, word, w, m, w * 32 - pbase, seg_cols, gsz);
        pbase += __popc(word);
    }
}

__global__ void k_add_const(const int32_t* __restrict__ src, int32_t* dst, int64_t k, int32_t delta) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < k; s += (int64_t)gridDim.x * blockDim.x)
        dst[s] = src[s] + delta;
}

// Test knob (ZF_TEST_LAG_DELAY_US): holds its stream for `us` microseconds of global time, so
// a parity test can make the lagged side-stream K1 finish late and check the refresh waits.
__global__ void k_spin(uint64_t ns) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

}  // namespace

cudaError_t launch_spin(int32_t us, cudaStream_t s) {
    if (us <= 0) return cudaSuccess;
    k_spin<<<1, 1, 0, s>>>((uint64_t)us * 1000ull);
    return cudaGetLastError();
}

cudaError_t launch_add_const(const int32_t* src, int32_t* dst, int64_t k, int32_t delta, cudaStream_t s) {
    if (k <= 0) return cudaSuccess;
    k_add_const<<<(unsigned)((k + 255) / 256 < 1024 ? (k + 255) / 256 : 1024), 256, 0, s>>>(src, dst, k, delta);
    return cudaGetLastError();
}

cudaError_t launch_topk(const Table<TopkLayer>& t, int64_t max_m, int32_t old_delta, int32_t* nonfinite, cudaStream_t s) {
    if (t.n <= 0) return cudaSuccess;
    size_t smem = 0;
    const int use_smem = max_m <= K2_SMEM_KEYS_MAX;
    if (use_smem) smem = (size_t)(max_m + (max_m + 31) / 32) * sizeof(uint32_t);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(k_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((K2_SMEM_KEYS_MAX + K2_SMEM_KEYS_MAX / 32) * sizeof(uint32_t)));
        attr_set = true;
    }
    k_topk<<<t.n, K2_THREADS, smem, s>>>(t, use_smem, old_delta, nonfinite);
    return cudaGetLastError();
}

cudaError_t launch_build_mask(const int32_t* idx, int64_t k, int64_t m, uint32_t* mask, int32_t* prefix,
                              uint16_t* ucol, int64_t seg_cols, int gsz, int32_t* bad, cudaStream_t s) {
    k_build_mask<<<1, K2_THREADS, 0, s>>>(idx, k, m, mask, prefix, ucol, seg_cols, gsz, bad);
    return cudaGetLastError();
}

}  // namespace zf
