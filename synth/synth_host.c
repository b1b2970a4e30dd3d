/* synth_host.c -- host C twin of synth/__init__.py (numpy) and synth/synth.cu (GPU):
 * the same integer recipe, so the outputs are bit-identical (tests/test_synth.py).
 * Input generation only: no arithmetic of the method lives here.  It exists so that
 * the CPU-oracle timing in bench.py can generate full-size Llama-2 inputs on the host
 * in seconds (the numpy recipe needs ~100 ns per element).
 *
 * C-ABI (host memory; rows are global rows row0..row0+n-1, dtype 0=fp32 1=bf16):
 *   synth_host_col_scale_init / synth_host_col_scale_advance : int8 exponents [m]
 *   synth_host_grad / synth_host_param                        : [n, ld] row-major   */
#include <stdint.h>
#include <string.h>
#include <math.h>

#define GOLD 0x9E3779B97F4A7C15ull
#define M1 0xBF58476D1CE4E5B9ull
#define M2 0x94D049BB133111EBull
#define K_TAG 0xD1B54A32D192ED03ull
#define K_LAYER 0xABC98388FB8FAC03ull
#define K_STEP 0x8CB92BA72F3D8DD7ull
enum { TAG_GRAD = 1, TAG_SCALE = 2, TAG_REDRAW = 3, TAG_PARAM = 4 };

static inline uint64_t mix(uint64_t x) {
    uint64_t z = x + GOLD;
    z = (z ^ (z >> 30)) * M1;
    z = (z ^ (z >> 27)) * M2;
    return z ^ (z >> 31);
}
static uint64_t stream_key(uint64_t seed, uint64_t tag, uint64_t layer, uint64_t step) {
    return mix(seed ^ (tag * K_TAG) ^ (layer * K_LAYER) ^ (step * K_STEP));
}
static inline int64_t ih4(uint64_t h) {
    return (int64_t)((h & 0xFFFF) + ((h >> 16) & 0xFFFF) + ((h >> 32) & 0xFFFF) + ((h >> 48) & 0xFFFF)) - 131070;
}
static inline int8_t scale_exp(int64_t z) {
    int64_t num = z * 2885 + 18918600;
    int64_t q = num / 37837200;
    if ((num % 37837200 != 0) && (num < 0)) q -= 1; /* floor division */
    if (q < -24) q = -24;
    if (q > 24) q = 24;
    return (int8_t)q;
}
static inline uint16_t bf16_rne_bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static inline void put(void* out, int dtype, int64_t at, float v) {
    if (dtype == 1) ((uint16_t*)out)[at] = bf16_rne_bits(v);
    else ((float*)out)[at] = v;
}

void synth_host_col_scale_init(int8_t* e, int64_t m, int32_t layer, uint64_t seed) {
    const uint64_t key = stream_key(seed, TAG_SCALE, (uint64_t)layer, 0);
    for (int64_t j = 0; j < m; ++j) e[j] = scale_exp(ih4(mix(key + (uint64_t)j)));
}

void synth_host_col_scale_advance(int8_t* e, int64_t m, int32_t layer, int64_t step, uint64_t seed) {
    const uint64_t kr = stream_key(seed, TAG_REDRAW, (uint64_t)layer, (uint64_t)step);
    const uint64_t ks = stream_key(seed, TAG_SCALE, (uint64_t)layer, (uint64_t)step);
    for (int64_t j = 0; j < m; ++j)
        if ((mix(kr + (uint64_t)j) & 0xFFFFFFFFull) < 1288490ull) e[j] = scale_exp(ih4(mix(ks + (uint64_t)j)));
}

void synth_host_grad(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, int32_t layer,
                     int64_t step, const int8_t* e, uint64_t seed) {
    const uint64_t key = stream_key(seed, TAG_GRAD, (uint64_t)layer, (uint64_t)step);
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t base = key + (uint64_t)((row0 + i) * m);
        for (int64_t j = 0; j < m; ++j)
            put(out, dtype, i * ld + j, (float)ih4(mix(base + (uint64_t)j)) * ldexpf(1.0f, (int)e[j] - 26));
    }
}

void synth_host_param(void* out, int dtype, int64_t n, int64_t m, int64_t ld, int64_t row0, int32_t layer,
                      uint64_t seed) {
    const uint64_t key = stream_key(seed, TAG_PARAM, (uint64_t)layer, 0);
    for (int64_t i = 0; i < n; ++i) {
        const uint64_t base = key + (uint64_t)((row0 + i) * m);
        for (int64_t j = 0; j < m; ++j)
            put(out, dtype, i * ld + j, (float)ih4(mix(base + (uint64_t)j)) * 2.384185791015625e-07f);
    }
}
