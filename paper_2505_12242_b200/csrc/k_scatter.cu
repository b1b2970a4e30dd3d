// k_scatter.cu -- K5: inverse of the compaction for the deferred CPU update (row f1):
// p[i][unsel[u]] = buf[i][u], a bit copy of the host-updated unselected columns into
// the row-major parameter ("sends back the corresponding (1-k)·M updated
// parameters"; reading R18).  Once per S-step window; scattered element stores.
#include "zf_internal.cuh"

namespace zf {
namespace {

template <typename B>
__global__ void k_scatter(B* __restrict__ P, int64_t ldp, int64_t n, int64_t mk, const int32_t* __restrict__ unsel,
                          const B* __restrict__ buf) {
    const int64_t total = n * mk;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / mk, u = q - i * mk;
        P[i * ldp + __ldg(unsel + u)] = buf[q];
    }
}

// K5': the gather the other way (f1 refresh): buf[i][e] = P[i][cols[e]], the columns
// entering the CPU-updated set, so only they cross the host link.
template <typename B>
__global__ void k_gather(const B* __restrict__ P, int64_t ldp, int64_t n, int64_t nc, const int32_t* __restrict__ cols,
                         B* __restrict__ buf) {
    const int64_t total = n * nc;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / nc, e = q - i * nc;
        buf[q] = P[i * ldp + __ldg(cols + e)];
    }
}

}  // namespace

cudaError_t launch_gather_columns(const void* P, int pdt, int64_t ldp, int64_t n, int64_t nc, const int32_t* cols,
                                  void* buf, cudaStream_t s) {
    const int64_t total = n * nc;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > NUM_SMS_B200 * 16) blocks = NUM_SMS_B200 * 16;
    if (pdt == DT_BF16)
        k_gather<uint16_t><<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint16_t*>(P), ldp, n, nc, cols,
                                                            static_cast<uint16_t*>(buf));
    else
        k_gather<uint32_t><<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint32_t*>(P), ldp, n, nc, cols,
                                                            static_cast<uint32_t*>(buf));
    return cudaGetLastError();
}

cudaError_t launch_scatter_unselected(void* P, int pdt, int64_t ldp, int64_t n, int64_t mk, const int32_t* unsel,
                                      const void* buf, cudaStream_t s) {
    const int64_t total = n * mk;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > NUM_SMS_B200 * 16) blocks = NUM_SMS_B200 * 16;
    if (pdt == DT_BF16)
        k_scatter<uint16_t><<<(unsigned)blocks, 256, 0, s>>>(static_cast<uint16_t*>(P), ldp, n, mk, unsel,
                                                             static_cast<const uint16_t*>(buf));
    else
        k_scatter<uint32_t><<<(unsigned)blocks, 256, 0, s>>>(static_cast<uint32_t*>(P), ldp, n, mk, unsel,
                                                             static_cast<const uint32_t*>(buf));
    return cudaGetLastError();
}

}  // namespace zf
