// Host DRAM bandwidth probe for the H1 design (row a8): how fast can the host's cores run
// the window accumulation patterns?  Each pattern streams arrays far larger than the LLC.
//   read      : sum a float array                               (4 B/elt read)
//   copy      : b = a (fp32)                                     (4 read + 4 write)
//   acc1      : acc = acc + f32(x_bf16)        one step per pass (4 + 2 read, 4 write) -- H1 today
//   acc1_first: acc = 0 + f32(x_bf16)          streaming stores  (2 read, 4 write)
//   accB(b)   : acc = (...(acc + x1) + ...) + xb in one pass     (4 + 2b read, 4 write)
//   accB4_first_nt: a whole 4-step window from zero, streaming stores (8 read, 4 write)
// usage: host_membw [GiB of fp32 acc, default 4] [threads]
// build: gcc -O3 -march=native -fopenmp tools/host_membw.c -o /tmp/host_membw
#include <immintrin.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}
#define LDX(j, i) _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm256_load_si256((const __m256i*)(x[j] + (i)))), 16))
static inline float bf(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float x;
    memcpy(&x, &u, 4);
    return x;
}

int main(int argc, char** argv) {
    const double gib = argc > 1 ? atof(argv[1]) : 4.0;
    if (argc > 2) omp_set_num_threads(atoi(argv[2]));
    const int64_t n = (int64_t)(gib * (1 << 30) / 4);
    float* acc = aligned_alloc(64, n * 4);
    float* b = aligned_alloc(64, n * 4);
    uint16_t* x[4];
    for (int j = 0; j < 4; ++j) x[j] = aligned_alloc(64, n * 2);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        acc[i] = 1.0f;
        b[i] = 0.0f;
        for (int j = 0; j < 4; ++j) x[j][i] = (uint16_t)(0x3f80 + (i & 7));
    }
    printf("{\"threads\": %d, \"gib_fp32\": %.1f", omp_get_max_threads(), gib);
    for (int pat = 0; pat < 8; ++pat) {
        double best = 1e30, bytes = 0;
        volatile float sink = 0;
        for (int rep = 0; rep < 4; ++rep) {
            const double t0 = now();
            if (pat == 0) {
                float s = 0;
#pragma omp parallel reduction(+ : s)
                {
                    __m512 a0 = _mm512_setzero_ps(), a1 = a0, a2 = a0, a3 = a0;
#pragma omp for schedule(static)
                    for (int64_t i = 0; i < n; i += 64) {
                        a0 = _mm512_add_ps(a0, _mm512_load_ps(acc + i));
                        a1 = _mm512_add_ps(a1, _mm512_load_ps(acc + i + 16));
                        a2 = _mm512_add_ps(a2, _mm512_load_ps(acc + i + 32));
                        a3 = _mm512_add_ps(a3, _mm512_load_ps(acc + i + 48));
                    }
                    s += _mm512_reduce_add_ps(_mm512_add_ps(_mm512_add_ps(a0, a1), _mm512_add_ps(a2, a3)));
                }
                sink = s;
                bytes = 4.0 * n;
            } else if (pat == 1) {
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; i += 16) _mm512_store_ps(b + i, _mm512_load_ps(acc + i));
                bytes = 8.0 * n;
            } else if (pat == 3) {
#pragma omp parallel for schedule(static)
                for (int64_t i = 0; i < n; i += 16) _mm512_stream_ps(acc + i, _mm512_add_ps(_mm512_setzero_ps(), LDX(0, i)));
                bytes = 6.0 * n;
            } else {
                const int B = pat == 2 ? 1 : pat - 3;  // steps per pass
                if (B == 1) {
#pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; i += 16) _mm512_store_ps(acc + i, _mm512_add_ps(_mm512_load_ps(acc + i), LDX(0, i)));
                } else if (B == 2) {
#pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; i += 16)
                        _mm512_store_ps(acc + i, _mm512_add_ps(_mm512_add_ps(_mm512_load_ps(acc + i), LDX(0, i)), LDX(1, i)));
                } else if (B == 3) {
#pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; i += 16)
                        _mm512_store_ps(acc + i, _mm512_add_ps(_mm512_add_ps(_mm512_add_ps(_mm512_load_ps(acc + i), LDX(0, i)), LDX(1, i)), LDX(2, i)));
                } else {
#pragma omp parallel for schedule(static)
                    for (int64_t i = 0; i < n; i += 16)
                        _mm512_stream_ps(acc + i, _mm512_add_ps(_mm512_add_ps(_mm512_add_ps(_mm512_add_ps(_mm512_setzero_ps(), LDX(0, i)), LDX(1, i)), LDX(2, i)), LDX(3, i)));
                }
                bytes = (B == 4 ? 4.0 + 2.0 * B : 8.0 + 2.0 * B) * n;
            }
            const double dt = now() - t0;
            if (dt < best) best = dt;
        }
        static const char* names[] = {"read", "copy", "acc1", "acc1_first_nt", "accB1", "accB2", "accB3", "accB4_first_nt"};
        printf(", \"%s_GBs\": %.1f", names[pat], bytes / best / 1e9);
        (void)sink;
    }
    printf("}\n");
    return 0;
}
