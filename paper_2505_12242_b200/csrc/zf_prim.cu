// zf_prim.cu -- the C-ABI's basic calls and stateless primitives (include/zf.h rows 1-6):
// argument validation and one launch each of K1, K2, the AdamW-only kernel and K3 in
// compaction mode.  See DESIGN.md §5.
#include "zf_host.h"

// ============================================================ basic API
extern "C" const char* zf_status_string(int32_t s) {
    switch (s) {
        case ZF_OK: return "ZF_OK";
        case ZF_EINVAL: return "ZF_EINVAL: invalid argument";
        case ZF_ENONFINITE: return "ZF_ENONFINITE: non-finite gradient";
        case ZF_ECUDA: return "ZF_ECUDA: CUDA error";
        case ZF_ENCCL: return "ZF_ENCCL: NCCL error";
        case ZF_ENOMEM: return "ZF_ENOMEM: out of memory";
        case ZF_ESTATE: return "ZF_ESTATE: invalid state";
        default: return "unknown zf_status";
    }
}

extern "C" const char* zf_last_error(void) { return g_last_error.c_str(); }

extern "C" int32_t zf_version(void) { return 100; }

extern "C" int64_t zf_k_for(int64_t m, int32_t ppm) {
    if (m < 1 || ppm <= 0 || ppm > 1000000) return -1;
    int64_t k = (m * (int64_t)ppm + 999999) / 1000000;
    return std::min<int64_t>(std::max<int64_t>(k, 1), m);
}

// ============================================================ stateless primitives
extern "C" zf_status zf_column_norms(const void* G, zf_dtype gdt, int64_t n, int64_t m, int64_t ld, float* norms,
                                     int32_t* nonfinite, zf_stream_t stream) {
    g_last_error.clear();
    ZF_TRY(check_matrix(G, gdt, n, m, ld, "G"));
    if (!norms) return fail(ZF_EINVAL, "norms is NULL");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int gsz = esize(gdt);
    Table<NormLayer> t{};
    NormLayer& L = t.one;
    t.dev = nullptr;
    t.n = 1;
    L.G = G;
    L.n = n;
    L.m = m;
    L.ld = ld;
    L.out = norms;
    L.nrb = (int32_t)((n + norms_rows_per_block() - 1) / norms_rows_per_block());
    L.ncb = (int32_t)((m + norms_cols_per_block(gdt) - 1) / norms_cols_per_block(gdt));
    L.unit_begin = 0;
    L.vec_ok = aligned16(G) && ((ld * gsz) % 16 == 0);
    Scratch sc(s);
    if (L.nrb > 1) {
        ZF_TRY(sc.get(&L.partial, (size_t)L.nrb * m * sizeof(float), false));
        ZF_TRY(sc.get(&L.counter, (size_t)L.ncb * sizeof(uint32_t), true));
    }
    ZF_CUDA(launch_norms(t, (int64_t)L.nrb * L.ncb, gdt, nonfinite, s));
    return ZF_OK;
}

extern "C" zf_status zf_topk_columns(const float* norms, int64_t m, int64_t k, int32_t* idx, zf_stream_t stream) {
    g_last_error.clear();
    if (!norms || !idx) return fail(ZF_EINVAL, "norms/idx is NULL");
    if (m < 1) return fail(ZF_EINVAL, "empty norms vector (m=%lld)", (long long)m);
    if (m > 0x7fffffffLL) return fail(ZF_EINVAL, "m too large");
    if (k < 1 || k > m) return fail(ZF_EINVAL, "need 1 <= k <= m (k=%lld m=%lld)", (long long)k, (long long)m);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Scratch sc(s);
    Table<TopkLayer> t{};
    t.dev = nullptr;
    t.n = 1;
    TopkLayer& L = t.one;
    L.norms = norms;
    L.m = m;
    L.k = k;
    L.idx = idx;
    const int64_t W = (m + 31) / 32;
    ZF_TRY(sc.get(&L.mask, W * sizeof(uint32_t), false));
    ZF_TRY(sc.get(&L.prefix, W * sizeof(int32_t), false));
    ZF_CUDA(launch_topk(t, m, 0, nullptr, s));
    return ZF_OK;
}

extern "C" zf_status zf_selective_adam(void* p, zf_dtype pdt, int64_t ldp, const void* G, zf_dtype gdt, int64_t ldg,
                                       int64_t n, int64_t m, const int32_t* idx, int64_t k, float* exp_avg,
                                       float* exp_avg_sq, int32_t* step, const zf_adam_params* hp,
                                       zf_stream_t stream) {
    g_last_error.clear();
    ZF_TRY(check_matrix(G, gdt, n, m, ldg, "G"));
    ZF_TRY(check_matrix(p, pdt, n, m, ldp, "p"));
    if (!idx || !exp_avg || !exp_avg_sq || !step) return fail(ZF_EINVAL, "idx/exp_avg/exp_avg_sq/step is NULL");
    if (k < 1 || k > m) return fail(ZF_EINVAL, "need 1 <= k <= m");
    ZF_TRY(check_hp(hp));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    AdamK a = adam_scalars(*hp);
    ZF_TRY(cached_tables(*hp, s, &a));
    Scratch sc(s);
    uint32_t* counter = nullptr;
    ZF_TRY(sc.get(&counter, sizeof(uint32_t), true));
    ZF_CUDA(launch_adam_only(G, gdt, ldg, p, pdt, ldp, n, idx, k, exp_avg, exp_avg_sq, step, counter, a, s));
    return ZF_OK;
}

extern "C" zf_status zf_compact_unselected(const void* G, zf_dtype gdt, int64_t n, int64_t m, int64_t ld,
                                           const int32_t* idx, int64_t k, void* out, zf_stream_t stream) {
    g_last_error.clear();
    ZF_TRY(check_matrix(G, gdt, n, m, ld, "G"));
    if (!idx || !out) return fail(ZF_EINVAL, "idx/out is NULL");
    if (k < 1 || k > m) return fail(ZF_EINVAL, "need 1 <= k <= m");
    if (!aligned16(out)) return fail(ZF_EINVAL, "out must be 16-byte aligned");
    if (k == m) return ZF_OK;  // empty output
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int gsz = esize(gdt);
    Scratch sc(s);
    UpdParams prm{};
    prm.layers.dev = nullptr;
    prm.layers.n = 1;
    UpdLayer& L = prm.layers.one;
    const int64_t W = (m + 31) / 32;
    uint32_t* mask = nullptr;
    int32_t* prefix = nullptr;
    uint16_t* ucol = nullptr;
    ZF_TRY(sc.get(&mask, (W + 8) * sizeof(uint32_t), true));    // padded: K3 stages words in 16-byte groups
    ZF_TRY(sc.get(&prefix, (W + 8) * sizeof(int32_t), true));
    ZF_TRY(sc.get(&ucol, (m - k + 16) * sizeof(uint16_t), true));
    // k_build_mask skips entries that are out of range or not ascending, so a bad idx cannot make
    // it write out of bounds (zf.h: idx is not validated -- that would need a host round trip)
    ZF_TRY(sc.get(&prm.claim, sizeof(uint32_t), true));
    const K3Geom geo = k3_geom(n, m, k, gsz, gsz, false, false);
    ZF_CUDA(launch_build_mask(idx, k, m, mask, prefix, ucol, geo.seg_cols, gsz, nullptr, s));
    L.G = G;
    L.n = n;
    L.m = m;
    L.ldg = ld;
    L.k = k;
    L.idx = idx;
    L.mask = mask;
    L.prefix = prefix;
    L.ucol = ucol;
    L.out = out;
    L.out_ld = m - k;
    L.seg_cols = geo.seg_cols;
    L.nseg = geo.nseg;
    L.R = geo.R;
    L.units = geo.units;
    L.unit_begin = 0;
    L.tma_ok = k3_tma_ok(G, ld, m, gsz);
    prm.total_units = geo.units;
    prm.claim_base = 0;
    prm.do_adam = 0;
    prm.do_compact = 1;
    ZF_CUDA(launch_update(prm, gdt, gdt, update_grid(gdt, gdt), s));
    return ZF_OK;
}

namespace zf {
namespace {
__global__ void k_patch(const __grid_constant__ PatchArgs a) {
    for (int i = threadIdx.x; i < a.n; i += blockDim.x) a.base[a.off[i]] = a.val[i];
}
}  // namespace

cudaError_t launch_patch(const PatchArgs& a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    k_patch<<<1, 256, 0, s>>>(a);
    return cudaGetLastError();
}
}  // namespace zf
