// synth.cu -- GPU twin of synth/__init__.py: seeded synthetic inputs for the
// ZenFlow hot path.  Input generation only: no arithmetic of the method lives
// here (see synth/__init__.py for the recipe and its citations).  The integer
// recipe is identical to the numpy twin, so the outputs are bit-identical
// (tests/test_synth.py, tests/test_gpu_parity.py).
//
// C-ABI (host pointers to device memory; asynchronous on `stream`):
//   synth_col_scale_init / synth_col_scale_advance : int8 exponents [m]
//   synth_grad / synth_grad_tie / synth_param      : [n, ld] row-major, dtype 0=fp32 1=bf16,
//                                                    rows are global rows row0..row0+n-1
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace {

constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull, M1 = 0xBF58476D1CE4E5B9ull, M2 = 0x94D049BB133111EBull;
constexpr uint64_t K_TAG = 0xD1B54A32D192ED03ull, K_LAYER = 0xABC98388FB8FAC03ull, K_STEP = 0x8CB92BA72F3D8DD7ull;
enum { TAG_GRAD = 1, TAG_SCALE = 2, TAG_REDRAW = 3, TAG_PARAM = 4, TAG_TIE = 5 };

__host__ __device__ __forceinline__ uint64_t mix(uint64_t x) {
    uint64_t z = x + GOLD;
    z = (z ^ (z >> 30)) * M1;
    z = (z ^ (z >> 27)) * M2;
    return z ^ (z >> 31);
}

uint64_t stream_key(uint64_t seed, uint64_t tag, uint64_t layer, uint64_t step) {
    return mix(seed ^ (tag * K_TAG) ^ (layer * K_LAYER) ^ (step * K_STEP));
}

__device__ __forceinline__ int64_t ih4(uint64_t h) {
    return (int64_t)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + ((h >> 48) & 0xFFFF)) - 131070;
}

__device__ __forceinline__ int8_t scale_exp(int64_t z) {
    int64_t num = z * 2885 + 18918600;
    int64_t q = num / 37837200;
    if ((num % 37837200 != 0) && (num < 0)) q -= 1;  // floor division
    if (q < -24) q = -24;
    if (q > 24) q = 24;
    return (int8_t)q;
}

__device__ __forceinline__ uint16_t bf16_rne_bits(float f) {
    uint32_t u = __float_as_uint(f);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

__global__ void k_scale_init(int8_t* e, int64_t m, uint64_t key) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
        e[j] = scale_exp(ih4(mix(key + (uint64_t)j)));
}

__global__ void k_scale_advance(int8_t* e, int64_t m, uint64_t key_redraw, uint64_t key_scale) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x) {
        uint64_t hr = mix(key_redraw + (uint64_t)j);
        if ((hr & 0xFFFFFFFFull) < 1288490ull) e[j] = scale_exp(ih4(mix(key_scale + (uint64_t)j)));
    }
}

// mode 0: gradient z*2^(e_j-26); mode 1: tie-heavy ((h%5)-2)*2^-8; mode 2: param z*2^-22
template <int MODE>
__global__ void k_fill(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, uint64_t key,
                       const int8_t* e) {
    const int64_t total = n * m;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / m, j = q - i * m;
        const uint64_t h = mix(key + (uint64_t)((row0 + i) * m + j));
        float v;
        if (MODE == 0) v = (float)ih4(h) * ldexpf(1.0f, (int)e[j] - 26);
        else if (MODE == 1) v = (float)((int64_t)(h % 5ull) - 2) * 0.00390625f;
        else v = (float)ih4(h) * 2.384185791015625e-07f;  // 2^-22
        if (dtype == 1) ((uint16_t*)out)[i * ld + j] = bf16_rne_bits(v);
        else ((float*)out)[i * ld + j] = v;
    }
}

int grid_for(int64_t work) {
    int64_t g = (work + 255) / 256;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

extern "C" {

int synth_col_scale_init(int8_t* e, int64_t m, int32_t layer, uint64_t seed, cudaStream_t s) {
    k_scale_init<<<grid_for(m), 256, 0, s>>>(e, m, stream_key(seed, TAG_SCALE, (uint64_t)layer, 0));
    return (int)cudaGetLastError();
}

int synth_col_scale_advance(int8_t* e, int64_t m, int32_t layer, int64_t step, uint64_t seed, cudaStream_t s) {
    k_scale_advance<<<grid_for(m), 256, 0, s>>>(e, m, stream_key(seed, TAG_REDRAW, (uint64_t)layer, (uint64_t)step),
                                                stream_key(seed, TAG_SCALE, (uint64_t)layer, (uint64_t)step));
    return (int)cudaGetLastError();
}

int synth_grad(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, int32_t layer, int64_t step,
               const int8_t* e, uint64_t seed, cudaStream_t s) {
    k_fill<0><<<grid_for(n * m), 256, 0, s>>>(out, dtype, n, m, ld, row0,
                                              stream_key(seed, TAG_GRAD, (uint64_t)layer, (uint64_t)step), e);
    return (int)cudaGetLastError();
}

int synth_grad_tie(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, int32_t layer, int64_t step,
                   uint64_t seed, cudaStream_t s) {
    k_fill<1><<<grid_for(n * m), 256, 0, s>>>(out, dtype, n, m, ld, row0,
                                              stream_key(seed, TAG_TIE, (uint64_t)layer, (uint64_t)step), nullptr);
    return (int)cudaGetLastError();
}

int synth_param(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, int32_t layer, uint64_t seed,
                cudaStream_t s) {
    k_fill<2><<<grid_for(n * m), 256, 0, s>>>(out, dtype, n, m, ld, row0,
                                              stream_key(seed, TAG_PARAM, (uint64_t)layer, 0), nullptr);
    return (int)cudaGetLastError();
}

}  // extern "C"
