// probe_pwrite.cu -- what does HBM charge for scattered sub-sector bf16 stores?
//
// K3 updates the selected columns of a row-major bf16 parameter in place.  At
// kappa = 0.1 a selected column hits ~81% of the 32-byte sectors of p.  This probe
// measures, on a 13.2 GB p (Llama-2-7B's element count), the time (and, under ncu,
// the DRAM bytes) of:
//   scatter_write : store the selected elements only (no read of p)
//   rmw           : read + store the selected elements
//   read_sel      : read the selected elements only
//   dense_rw      : read + write a dense [n, k] bf16 block (a "parameter subset")
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o build/probe_pwrite tools/probe_pwrite.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__global__ void scatter_write(uint16_t* P, int64_t n, int m, const int* idx, int k, uint16_t val) {
    const int64_t total = n * k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / k; const int s = (int)(q - i * k);
        P[i * m + __ldg(idx + s)] = (uint16_t)(val ^ (uint16_t)s);
    }
}
__global__ void rmw(uint16_t* P, int64_t n, int m, const int* idx, int k) {
    const int64_t total = n * k;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / k; const int s = (int)(q - i * k);
        uint16_t* a = P + i * m + __ldg(idx + s);
        *a = (uint16_t)(*a + 1);
    }
}
__global__ void read_sel(const uint16_t* P, int64_t n, int m, const int* idx, int k, unsigned* sink) {
    const int64_t total = n * k;
    unsigned acc = 0;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / k; const int s = (int)(q - i * k);
        acc += P[i * m + __ldg(idx + s)];
    }
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void dense_rw(uint16_t* D, int64_t total) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total / 8; q += (int64_t)gridDim.x * blockDim.x) {
        uint4 v = reinterpret_cast<uint4*>(D)[q];
        v.x += 1; v.y += 1; v.z += 1; v.w += 1;
        reinterpret_cast<uint4*>(D)[q] = v;
    }
}

int main(int argc, char** argv) {
    const int m = 4096;
    const double ratio = argc > 1 ? atof(argv[1]) : 0.1;
    const int64_t n = 6607077376LL / m;
    const int k = (int)((m * ratio) + 0.999999);
    std::vector<int> all(m);
    for (int j = 0; j < m; ++j) all[j] = j;
    uint64_t s = 0x250512242ULL;
    for (int j = m - 1; j > 0; --j) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; std::swap(all[j], all[(int)((s >> 33) % (uint64_t)(j + 1))]); }
    std::vector<int> idx(all.begin(), all.begin() + k);
    std::sort(idx.begin(), idx.end());
    int64_t touched = 0;
    for (int c = 0; c < m / 16; ++c) { bool t = false; for (int s2 = 0; s2 < k; ++s2) t |= idx[s2] / 16 == c; touched += t; }
    uint16_t *P, *D; int* didx; unsigned* sink;
    CK(cudaMalloc(&P, (size_t)n * m * 2));
    CK(cudaMalloc(&D, (size_t)n * k * 2));
    CK(cudaMalloc(&didx, k * 4));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(P, 0x11, (size_t)n * m * 2));
    CK(cudaMemset(D, 0x11, (size_t)n * k * 2));
    CK(cudaMemcpy(didx, idx.data(), k * 4, cudaMemcpyHostToDevice));
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int grid = sms * 8, blk = 256;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const double sel_bytes = (double)n * k * 2, sect_bytes = (double)n * (m / 16) * 32 * ((double)touched / (m / 16));
    printf("{\"m\": %d, \"k\": %d, \"n\": %lld, \"p_GB\": %.2f, \"touched_sector_frac\": %.4f}\n", m, k, (long long)n,
           n * m * 2 / 1e9, (double)touched / (m / 16));
    for (int kind = 0; kind < 4; ++kind) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (kind == 0) scatter_write<<<grid, blk>>>(P, n, m, didx, k, (uint16_t)(0x3c00 + rep));
            else if (kind == 1) rmw<<<grid, blk>>>(P, n, m, didx, k);
            else if (kind == 2) read_sel<<<grid, blk>>>(P, n, m, didx, k, sink);
            else dense_rw<<<grid, blk>>>(D, n * k);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
        }
        const char* nm[] = {"scatter_write", "rmw", "read_sel", "dense_rw"};
        printf("{\"kernel\": \"%s\", \"ms\": %.3f, \"sel_GBs\": %.1f, \"sector_GBs_one_way\": %.1f}\n", nm[kind], best,
               sel_bytes * (kind == 1 || kind == 3 ? 2 : 1) / best / 1e6, sect_bytes / best / 1e6);
    }
    CK(cudaGetLastError());
    return 0;
}
