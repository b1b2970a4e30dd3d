// k_auto.cu -- K6: the Zen-auto decision of one step (next row f2, P:445-447;
// DESIGN.md reading R21).  From the step's (all-reduced) per-column squared norms
// -- the "lightweight coordination proxy" of P:447 -- and the current selection
// mask of every layer:
//   u = mean over all layers' unselected columns of sqrt(norm[j]),
//   i = mean over all layers' selected columns of sqrt(norm[c]),
//   A = sum of u over the steps of the current window,
// and the window ends iff force_end (the next step refreshes), its length reached
// smax, or A > 0 and A >= gamma * i.  One CTA per layer sums sqrt(norm) in double
// in a fixed order (strided per thread, then a fixed tree); the last CTA to arrive
// combines the layers in layer order and updates the device-side window state, so
// the decision is deterministic and identical on every rank (same norms).
#include "zf_internal.cuh"

namespace zf {
namespace {

constexpr int K6_THREADS = 256;

__global__ void __launch_bounds__(K6_THREADS) k_zen_auto(const AutoLayer* __restrict__ layers, int32_t nl,
                                                         double* __restrict__ sums, uint32_t* counter,
                                                         AutoState* state, AutoRecord* rec, int64_t t,
                                                         double gamma, int32_t smax, int32_t force_end) {
    const AutoLayer L = layers[blockIdx.x];
    double sel = 0.0, uns = 0.0;
    for (int64_t j = threadIdx.x; j < L.m; j += K6_THREADS) {
        const double x = sqrt((double)__ldg(L.norms + j));
        if ((__ldg(L.mask + (j >> 5)) >> (j & 31)) & 1u) sel += x;
        else uns += x;
    }
    for (int o = 16; o > 0; o >>= 1) {
        sel += __shfl_xor_sync(0xffffffffu, sel, o);
        uns += __shfl_xor_sync(0xffffffffu, uns, o);
    }
    __shared__ double ws[2][K6_THREADS / 32];
    __shared__ bool last;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        ws[0][w] = sel;
        ws[1][w] = uns;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int q = 0; q < K6_THREADS / 32; ++q) {
            a += ws[0][q];
            b += ws[1][q];
        }
        sums[2 * blockIdx.x] = a;
        sums[2 * blockIdx.x + 1] = b;
        __threadfence();
        last = atomicAdd(counter, 1u) == (uint32_t)(nl - 1);
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    *counter = 0u;  // self-resetting for the next launch
    double s_sel = 0.0, s_uns = 0.0;
    int64_t c_sel = 0, c_uns = 0;
    for (int l = 0; l < nl; ++l) {
        s_sel += ((volatile double*)sums)[2 * l];
        s_uns += ((volatile double*)sums)[2 * l + 1];
        c_sel += layers[l].k;
        c_uns += layers[l].m - layers[l].k;
    }
    const double u = c_uns > 0 ? s_uns / (double)c_uns : 0.0;
    const double i = c_sel > 0 ? s_sel / (double)c_sel : 0.0;
    AutoState st = *state;
    if (!st.open) {
        st.A = 0.0;
        st.len = 0;
    }
    st.A = st.A + u;
    st.len += 1;
    const int end = (force_end || st.len >= smax || (st.A > 0.0 && st.A >= gamma * i)) ? 1 : 0;
    AutoRecord r;
    r.t = t;
    r.A = st.A;
    r.imp = i;
    r.unimp = u;
    r.len = st.len;
    r.end = end;
    st.open = end ? 0 : 1;
    if (end) st.win += 1;
    *state = st;
    volatile AutoRecord* vr = rec;
    vr->t = r.t;
    vr->A = r.A;
    vr->imp = r.imp;
    vr->unimp = r.unimp;
    vr->len = r.len;
    vr->end = r.end;
    __threadfence_system();
}

}  // namespace

cudaError_t launch_zen_auto(const AutoLayer* layers, int32_t nl, double* sums, uint32_t* counter, AutoState* state,
                            AutoRecord* rec, int64_t t, double gamma, int32_t smax, int32_t force_end,
                            cudaStream_t s) {
    k_zen_auto<<<nl, K6_THREADS, 0, s>>>(layers, nl, sums, counter, state, rec, t, gamma, smax, force_end);
    return cudaGetLastError();
}

}  // namespace zf
