// k_peer.cu -- row a2 over peer memory (next row f4 (iii)): the ranks' partial column-norm
// vectors summed by kernels that read each other's device memory directly (CUDA IPC
// mappings: NVLink / NVSwitch peer loads between GPUs, or plain device memory when ranks
// share a GPU), instead of an NCCL all-reduce launch.
//
// Paper: "each GPU computes the local column-wise gradient norms ... then shares
// these partial norms with the other GPUs"; P:798 (the gathering overhead).
// f4 (iii): "K2 reading NVLink peer partials directly (no NCCL launch)".
//
// Each rank owns one exchange region (zf_peer_handle exports it, zf_peer_open maps the
// others):
//   flags[0] pub   : last epoch whose partials this rank published
//   flags[1] red   : last epoch whose reduced slice this rank published
//   flags[2] done  : last epoch this rank finished gathering (its reads of the peers' regions)
//   part[2][Mp]    : the rank's partial norms, double-buffered by epoch parity
//   red[2][Mp]     : the reduced slice this rank owns (columns [r*M/P, (r+1)*M/P)), by parity
// Exchange e (1, 2, ...), three kernels in stream order on every rank:
//   (a) publish:  wait until every peer's done >= e-2 (nobody still reads parity e%2), copy
//                 the local norms into part[e%2], then pub = e;
//   (b) reduce:   wait until every peer's pub >= e; for the owned slice sum the P partials in
//                 rank order 0..P-1 (one fixed fp32 order, so every rank ends with the same
//                 bits), write red[e%2], then red = e;
//   (c) gather:   wait until every peer's red >= e; norms[j] = red_owner(j)[e%2][j]; done = e.
// Per rank this moves 2·M·4 bytes over the peer links (a reduce-scatter and an all-gather),
// like a two-shot all-reduce.  Flags are written with st.release.sys after a system-scope
// fence and read with ld.acquire.sys; peer data is read with L2-only (.cg) loads.  A wait
// gives up after ZF_PEER_TIMEOUT_NS and raises the error flag (zf_sync / zf_step report
// ZF_ENCCL) instead of hanging the device.
#include "zf_internal.cuh"

namespace zf {
namespace {

#ifndef ZF_PEER_TIMEOUT_NS
#define ZF_PEER_TIMEOUT_NS 20000000000ull   // 20 s
#endif

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// every peer's flags[which] >= want (thread 0 spins, then every thread acquires once)
__device__ void wait_peers(const PeerArgs& a, int which, unsigned long long want) {
    if (threadIdx.x == 0) {
        const unsigned long long t0 = globaltimer();
        for (int q = 0; q < a.world; ++q) {
            if (q == a.rank) continue;
            const unsigned long long* f = a.flags[q] + which;
            while (ld_acquire_sys(f) < want) {
                if (globaltimer() - t0 > ZF_PEER_TIMEOUT_NS) {
                    atomicExch(a.error, 1);
                    break;
                }
                __nanosleep(256);
            }
        }
    }
    __syncthreads();
    for (int q = 0; q < a.world; ++q)
        if (q != a.rank) (void)ld_acquire_sys(a.flags[q] + which);
}

// the last block of the grid publishes flags[which] = e (self-resetting arrival counter)
__device__ void publish_last(const PeerArgs& a, int which, unsigned long long e) {
    __shared__ bool last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(a.counter, 1u) + 1u == gridDim.x;
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *a.counter = 0u;
        __threadfence_system();
        st_release_sys(a.flags[a.rank] + which, e);
    }
}

__global__ void k_peer_publish(PeerArgs a) {
    if (a.epoch > 2) wait_peers(a, 2, a.epoch - 2);
    float* dst = a.part[a.rank] + (a.epoch & 1) * a.Mp;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < a.M; j += (int64_t)gridDim.x * blockDim.x)
        dst[j] = a.norms[j];
    publish_last(a, 0, a.epoch);
}

__global__ void k_peer_reduce(PeerArgs a) {
    wait_peers(a, 0, a.epoch);
    const int64_t par = (a.epoch & 1) * a.Mp;
    const int64_t j0 = a.M * a.rank / a.world, j1 = a.M * (a.rank + 1) / a.world;
    float* dst = a.red[a.rank] + par;
    for (int64_t j = j0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < j1; j += (int64_t)gridDim.x * blockDim.x) {
        float s = __ldcg(a.part[0] + par + j);
        for (int q = 1; q < a.world; ++q) s = __fadd_rn(s, __ldcg(a.part[q] + par + j));
        dst[j] = s;
    }
    publish_last(a, 1, a.epoch);
}

__global__ void k_peer_gather(PeerArgs a) {
    wait_peers(a, 1, a.epoch);
    const int64_t par = (a.epoch & 1) * a.Mp;
    for (int q = 0; q < a.world; ++q) {
        const int64_t j0 = a.M * q / a.world, j1 = a.M * (q + 1) / a.world;
        const float* src = a.red[q] + par;
        for (int64_t j = j0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < j1;
             j += (int64_t)gridDim.x * blockDim.x)
            a.norms[j] = __ldcg(src + j);
    }
    publish_last(a, 2, a.epoch);
}

}  // namespace

cudaError_t launch_peer_allreduce(const PeerArgs& a, cudaStream_t s) {
    const int grid = (int)zmin<int64_t>((a.M + 1023) / 1024, NUM_SMS_B200);
    k_peer_publish<<<grid, 256, 0, s>>>(a);
    k_peer_reduce<<<grid, 256, 0, s>>>(a);
    k_peer_gather<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace zf
