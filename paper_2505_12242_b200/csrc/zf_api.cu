// zf_api.cu -- the C-ABI of libzf.so (include/zf.h) and the host runtime of the
// stateful driver: argument validation, the per-layer state in HBM, launch
// tables, the NCCL norm all-reduce, D2H staging on a copy stream gated per layer,
// and the host accumulation thread pool.  See DESIGN.md §5-§6.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <tuple>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zf.h"
#include "zf_internal.cuh"

using namespace zf;

// ============================================================ errors
namespace {
thread_local std::string g_last_error;

zf_status fail(zf_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define ZF_CUDA(call)                                                                                       \
    do {                                                                                                    \
        cudaError_t e_ = (call);                                                                            \
        if (e_ != cudaSuccess) return fail(ZF_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                                            cudaGetErrorString(e_));                                        \
    } while (0)

#define ZF_NCCL(call)                                                                                       \
    do {                                                                                                    \
        ncclResult_t r_ = (call);                                                                           \
        if (r_ != ncclSuccess) return fail(ZF_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                                            ncclGetErrorString(r_));                                        \
    } while (0)

#define ZF_TRY(expr)                \
    do {                            \
        zf_status s_ = (expr);      \
        if (s_ != ZF_OK) return s_; \
    } while (0)

int esize(zf_dtype d) { return d == ZF_BF16 ? 2 : 4; }
bool dtype_ok(int d) { return d == ZF_FP32 || d == ZF_BF16; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ============================================================ AdamW constants
// bias-correction tables computed on the host in double, one rounding to fp32
// (DESIGN.md §2 O6): ss[t] = f32(lr / (1 - b1^t)), bc2s[t] = f32(sqrt(1 - b2^t)).
// Both are monotone in t and reach their limits (f32(lr), 1.0f) at a finite t;
// the tables stop there and the kernel uses the limit beyond.
constexpr int64_t MAX_TAB = 1 << 24;
constexpr int64_t SS_CAP = 1 << 16;  // ss table capacity of a context (beta1 <= 0.999)

std::vector<float> make_ss(double lr, double b1) {
    std::vector<float> t(1, 0.0f);
    const float lim = (float)lr;
    for (int64_t i = 1; i < MAX_TAB; ++i) {
        const float v = (float)(lr / (1.0 - std::pow(b1, (double)i)));
        if (v == lim) break;
        t.push_back(v);
    }
    return t;
}

std::vector<float> make_bc2(double b2) {
    std::vector<float> t(1, 0.0f);
    for (int64_t i = 1; i < MAX_TAB; ++i) {
        const float v = (float)std::sqrt(1.0 - std::pow(b2, (double)i));
        if (v == 1.0f) break;
        t.push_back(v);
    }
    return t;
}

// {ss[t], bc2s[t]} interleaved over the longer of the two tables, the shorter one's limit
// filled in beyond its end (one 8-byte load per slot in K3).
std::vector<float> make_sb(const std::vector<float>& ss, const std::vector<float>& bc2, double lr) {
    const size_t n = std::max(ss.size(), bc2.size());
    std::vector<float> t(2 * n);
    for (size_t i = 0; i < n; ++i) {
        t[2 * i] = i < ss.size() ? ss[i] : (float)lr;
        t[2 * i + 1] = i < bc2.size() ? bc2[i] : 1.0f;
    }
    return t;
}

zf_status check_hp(const zf_adam_params* hp) {
    if (!hp) return fail(ZF_EINVAL, "hp is NULL");
    if (!(hp->lr >= 0.0f) || !std::isfinite(hp->lr)) return fail(ZF_EINVAL, "lr must be finite and >= 0");
    if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f)) return fail(ZF_EINVAL, "beta1 must be in [0, 1)");
    if (!(hp->beta2 >= 0.0f && hp->beta2 < 1.0f)) return fail(ZF_EINVAL, "beta2 must be in [0, 1)");
    if (!(hp->eps > 0.0f) || !std::isfinite(hp->eps)) return fail(ZF_EINVAL, "eps must be > 0");
    if (!(hp->weight_decay >= 0.0f) || !std::isfinite(hp->weight_decay)) return fail(ZF_EINVAL, "weight_decay must be >= 0");
    return ZF_OK;
}

// Scalars of AdamK (the tables are attached by the caller).
AdamK adam_scalars(const zf_adam_params& hp) {
    const double lr = hp.lr, b1 = hp.beta1, b2 = hp.beta2, eps = hp.eps, wd = hp.weight_decay;
    AdamK a{};
    a.b1 = (float)b1;
    a.b2 = (float)b2;
    a.omb1 = (float)(1.0 - b1);
    a.omb2 = (float)(1.0 - b2);
    a.eps = (float)eps;
    a.decay = (float)(1.0 - lr * wd);
    a.wd = (float)wd;
    a.wd_mode = wd == 0.0 ? 0 : (hp.decoupled ? 1 : 2);
    a.ss_inf = (float)lr;
    return a;
}

// Process-wide cache of device tables for the stateless primitive (never freed).
struct TabCache {
    std::mutex mu;
    std::map<std::tuple<int, uint64_t, uint64_t>, std::pair<float*, int>> ss;  // (dev, lr, b1)
    std::map<std::pair<int, uint64_t>, std::pair<float*, int>> bc2;              // (dev, b2)
    std::map<std::tuple<int, uint64_t, uint64_t, uint64_t>, std::pair<float*, int>> sb;  // (dev, lr, b1, b2)
};
TabCache& tab_cache() {
    static TabCache* c = new TabCache();
    return *c;
}

uint64_t dbits(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}

zf_status upload_table(const std::vector<float>& h, float** d, cudaStream_t s) {
    float* pinned = nullptr;
    ZF_CUDA(cudaMallocHost(&pinned, h.size() * sizeof(float)));  // kept alive with the table
    std::memcpy(pinned, h.data(), h.size() * sizeof(float));
    ZF_CUDA(cudaMalloc(d, h.size() * sizeof(float)));
    ZF_CUDA(cudaMemcpyAsync(*d, pinned, h.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    return ZF_OK;
}

zf_status cached_tables(const zf_adam_params& hp, cudaStream_t s, AdamK* a) {
    int dev = 0;
    ZF_CUDA(cudaGetDevice(&dev));
    TabCache& c = tab_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto ks = std::make_tuple(dev, dbits(hp.lr), dbits(hp.beta1));
    auto it = c.ss.find(ks);
    if (it == c.ss.end()) {
        auto h = make_ss(hp.lr, hp.beta1);
        float* d = nullptr;
        ZF_TRY(upload_table(h, &d, s));
        it = c.ss.emplace(ks, std::make_pair(d, (int)h.size())).first;
    }
    auto kb = std::make_pair(dev, dbits(hp.beta2));
    auto jt = c.bc2.find(kb);
    if (jt == c.bc2.end()) {
        auto h = make_bc2(hp.beta2);
        float* d = nullptr;
        ZF_TRY(upload_table(h, &d, s));
        jt = c.bc2.emplace(kb, std::make_pair(d, (int)h.size())).first;
    }
    auto kq = std::make_tuple(dev, dbits(hp.lr), dbits(hp.beta1), dbits(hp.beta2));
    auto qt = c.sb.find(kq);
    if (qt == c.sb.end()) {
        auto h = make_sb(make_ss(hp.lr, hp.beta1), make_bc2(hp.beta2), hp.lr);
        float* d = nullptr;
        ZF_TRY(upload_table(h, &d, s));
        qt = c.sb.emplace(kq, std::make_pair(d, (int)(h.size() / 2))).first;
    }
    a->ss_tab = it->second.first;
    a->ss_len = it->second.second;
    a->bc2_tab = jt->second.first;
    a->bc2_len = jt->second.second;
    a->sb_tab = reinterpret_cast<const float2*>(qt->second.first);
    a->sb_len = qt->second.second;
    return ZF_OK;
}

// ============================================================ geometry
struct K3Geom {
    int64_t seg_cols;
    int32_t nseg, R;
    int64_t units;
    bool mv_ok;
};

// p tile staging pays off when most 32-byte sectors of a row hold a selected column
bool k3_p_dense(int64_t m, int64_t k, int psz) {
    const double frac = (double)k / (double)m;
    return 1.0 - std::pow(1.0 - frac, 32.0 / psz) >= 0.5;
}

// Worst-case bytes one K3 unit stages (R rows x c columns): G tile, p tile (if dense),
// mask words, the unselected-column list, moment slabs (R*k: also covers the old rows of a refresh),
// step counts and remap sources; each as a 16-byte-granular superset.
int64_t k3_unit_bytes(int64_t R, int64_t c, int64_t k, int gsz, int psz, bool p_dense, bool mv) {
    auto a16 = [](int64_t b) { return (b + 15) & ~int64_t(15); };
    int64_t b = a16(R * c * gsz) + 2 * ((c + 31) / 32 + 8) * 4;
    if (p_dense) b += a16(R * c * psz);
    if (mv) b += 2 * (R * k + 8) * 4 + 3 * (std::min(c, k) + 8) * 4;  // moments; steps, sources, idx
    b += a16((c + 8) * 2);                                              // unselected-column offsets
    return b;
}

K3Geom k3_geom(int64_t n, int64_t m, int64_t k, int gsz, int psz, bool p_dense, bool adam = true) {
    const UpdLimits lim = update_limits();
    const int64_t A = lim.arena_bytes;
    K3Geom g{};
    // moments staged unless even one row's old moments cannot fit next to a minimal tile
    g.mv_ok = adam && k3_unit_bytes(1, std::min<int64_t>(m, 128), k, gsz, psz, p_dense, true) <= A;
    // Units are R rows x c columns (c = m, or a multiple of 128 so segments start 16-byte
    // aligned in the mask/prefix words): the shape with the fewest units per matrix (the most
    // bytes per stage), ties to full rows / wider segments.  ZF_K3_GEOM=rows keeps the older
    // rule (full rows when one fits, else single-row segments).
    // Measured (tools/k3_geom_ab.sh): the search wins with a staged p tile (Llama-2-13B K3
    // 23.90 -> 22.76 ms: m = 5120 rows go from 1-row units to 3 rows x 2688 columns) but
    // loses without one (k = 1%: 6.92 -> 7.27 ms, more exposed p loads per unit), so
    // unstaged-p layers keep the row rule.
    static const bool rows_env = getenv("ZF_K3_GEOM") && std::string(getenv("ZF_K3_GEOM")) == "rows";
    const bool rows_only = rows_env || !p_dense;
    auto rmax = [&](int64_t c) {
        int64_t R = 0;
        while (R < std::min<int64_t>(n, 127) && k3_unit_bytes(R + 1, c, k, gsz, psz, p_dense, g.mv_ok) <= A) ++R;
        return R;
    };
    int64_t best_units = -1;
    std::vector<int64_t> cands;
    cands.push_back(m);
    for (int64_t c = ((m - 1) / 128) * 128; c >= 128; c -= 128) cands.push_back(c);
    for (int64_t c : cands) {
        const int64_t R = rmax(c);
        if (R < 1) continue;
        const int64_t nseg = (m + c - 1) / c;
        if (rows_only && best_units >= 0) break;
        if (rows_only && nseg > 1) {  // older rule: widest single-row segment
            const int64_t u = n * nseg;
            g.seg_cols = c; g.nseg = (int32_t)nseg; g.R = 1; best_units = u;
            break;
        }
        const int64_t u = ((n + R - 1) / R) * nseg;
        if (best_units < 0 || u < best_units) {
            best_units = u;
            g.seg_cols = c;
            g.nseg = (int32_t)nseg;
            g.R = (int32_t)R;
        }
    }
    if (best_units < 0) {  // nothing fits (tiny arena): single-row minimal segments
        g.seg_cols = 128;
        g.nseg = (int32_t)((m + 127) / 128);
        g.R = 1;
    }
    g.units = ((n + g.R - 1) / g.R) * g.nseg;
    return g;
}

bool k3_tma_ok(const void* G, int64_t ldg, int64_t m, int gsz) {
    return aligned16(G) && ((ldg * gsz) % 16 == 0) && ((m * gsz) % 16 == 0);
}

// Stream-ordered scratch (freed asynchronously on the same stream).
struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    template <typename T>
    zf_status get(T** p, size_t bytes, bool zero) {
        void* q = nullptr;
        ZF_CUDA(cudaMallocAsync(&q, std::max<size_t>(bytes, 16), s));
        ptrs.push_back(q);
        if (zero) ZF_CUDA(cudaMemsetAsync(q, 0, std::max<size_t>(bytes, 16), s));
        *p = static_cast<T*>(q);
        return ZF_OK;
    }
    ~Scratch() {
        for (void* q : ptrs) cudaFreeAsync(q, s);
    }
};

zf_status check_matrix(const void* G, int gdt, int64_t n, int64_t m, int64_t ld, const char* what) {
    if (!G) return fail(ZF_EINVAL, "%s is NULL", what);
    if (!dtype_ok(gdt)) return fail(ZF_EINVAL, "%s: unsupported dtype %d", what, gdt);
    if (n < 1 || m < 1) return fail(ZF_EINVAL, "%s: need n >= 1 and m >= 1 (got n=%lld m=%lld)", what, (long long)n,
                                    (long long)m);
    if (m > 0x7fffffffLL) return fail(ZF_EINVAL, "%s: m too large", what);
    if (ld < m) return fail(ZF_EINVAL, "%s: ld (%lld) < m (%lld)", what, (long long)ld, (long long)m);
    return ZF_OK;
}

}  // namespace

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
    int32_t* bad = nullptr;
    uint16_t* ucol = nullptr;
    ZF_TRY(sc.get(&mask, (W + 8) * sizeof(uint32_t), true));    // padded: K3 stages words in 16-byte groups
    ZF_TRY(sc.get(&prefix, (W + 8) * sizeof(int32_t), true));
    ZF_TRY(sc.get(&ucol, (m - k + 16) * sizeof(uint16_t), true));
    ZF_TRY(sc.get(&bad, sizeof(int32_t), true));
    ZF_TRY(sc.get(&prm.claim, sizeof(uint32_t), true));
    const K3Geom geo = k3_geom(n, m, k, gsz, gsz, false, false);
    ZF_CUDA(launch_build_mask(idx, k, m, mask, prefix, ucol, geo.seg_cols, gsz, bad, s));
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

// ============================================================ stateful driver
namespace {

typedef CUresult (*PFN_waitValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct LayerState {
    zf_layer_desc d{};
    int64_t k = 0, W = 0, mk = 0;
    int64_t mk_pad = 0;               // device compact block row pitch (16-byte rows)
    // K1
    int32_t nrb = 0, ncb = 0;
    int64_t norm_off = 0, norm_unit_begin = 0;
    float* partial = nullptr;
    uint32_t* k1_counter = nullptr;
    // selection sets (double-buffered for the refresh remap)
    int32_t* idx[2] = {nullptr, nullptr};
    uint32_t* mask[2] = {nullptr, nullptr};
    int32_t* prefix[2] = {nullptr, nullptr};
    uint16_t* ucol[2] = {nullptr, nullptr};
    int32_t* steps[2] = {nullptr, nullptr};
    int32_t* slot_src = nullptr;
    float* mom[2] = {nullptr, nullptr};
    float* vel[2] = {nullptr, nullptr};
    void* stage_dev[2] = {nullptr, nullptr};
    void* stage_host[2] = {nullptr, nullptr};
    float* acc[2] = {nullptr, nullptr};
    float* dacc[2] = {nullptr, nullptr};  // device_accumulate: [n, mk_pad] fp32 window accumulators
    float* acc_sealed_h = nullptr;        // device_accumulate: pinned dense [n, mk] copy of the sealed window
    // K3 geometry
    K3Geom geo{};
    int64_t unit_begin = 0;
    cudaEvent_t d2h_ev[2] = {nullptr, nullptr};
    // f1: deferred CPU AdamW (reading R18)
    float* master = nullptr;          // [n, m] fp32 host master (valid on CPU-updated columns)
    float* mh = nullptr;              // [n, m] host moments
    float* vh = nullptr;
    std::vector<int32_t> th;          // [m] host step count per column
    std::vector<int32_t> idx_host;    // current selection (ascending), host copy
    std::vector<int32_t> unsel_host;  // its complement (ascending)
    void* p_mirror = nullptr;         // pinned [n, m] copy of p at a refresh
    void* p_up = nullptr;             // pinned [n, m-k] updated unselected params
    void* p_up_dev = nullptr;         // device [n, m-k]
    int32_t* unsel_dev = nullptr;     // device [m-k]
    // f2: warm-up selection set (all m columns; reading R20)
    int32_t* idx_w = nullptr;
    uint32_t* mask_w = nullptr;
    int32_t* prefix_w = nullptr;
    int32_t* steps_w = nullptr;
    float* mom_w = nullptr;           // [n, m]
    float* vel_w = nullptr;
    K3Geom geo_w{};
    int64_t unit_begin_w = 0;
};

// Simple pool for the host accumulation (row 8, H1).
class Pool {
   public:
    explicit Pool(int n) : n_(n) {
        for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { run(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // fn(begin, end) over [0, count) split into n_ contiguous slices; callers from several
    // threads (H1 and the f1 host update) are serialised.
    template <typename F>
    void parallel_for(int64_t count, F&& fn) {
        std::lock_guard<std::mutex> call(call_mu_);
        std::unique_lock<std::mutex> lk(mu_);
        job_ = [&](int i) {
            const int64_t per = (count + n_ - 1) / n_;
            const int64_t b = std::min<int64_t>(count, per * i), e = std::min<int64_t>(count, b + per);
            if (b < e) fn(b, e);
        };
        pending_ = n_;
        ++gen_;
        cv_.notify_all();
        done_cv_.wait(lk, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

   private:
    void run(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(int)> job;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                job = job_;
            }
            if (job) job(i);
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (--pending_ == 0) done_cv_.notify_all();
            }
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    std::function<void(int)> job_;
    uint64_t gen_ = 0;
    int pending_ = 0;
    bool stop_ = false;
};

}  // namespace

struct zf_ctx {
    int device = 0;
    zf_config cfg{};
    int world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    zf_host_allreduce_fn host_allreduce = nullptr;  // world > 1 without NCCL
    void* host_allreduce_user = nullptr;
    float* norms_host = nullptr;
    int gdt = 0, pdt = 0, gsz = 2, psz = 2;
    std::vector<LayerState> L;
    int64_t total_m = 0, max_m = 0, k1_units = 0, k3_units = 0;
    bool has_empty = false;       // some layer has n = 0 rows on this rank
    int n_stage = 1;
    float* norms = nullptr;
    std::vector<void*> dev_allocs, host_pinned;
    std::vector<float*> host_plain;
    int32_t* nonfinite_h = nullptr;  // mapped pinned
    int32_t* nonfinite_d = nullptr;
    uint32_t* claim = nullptr;
    uint32_t* done = nullptr;  // [n_layers]
    uint32_t claim_base = 0;
    int32_t since = 0;            // K3 launches since the last refresh (step-count delta)
    std::vector<uint32_t> done_target;  // expected per-layer completion count after the last step
    cudaStream_t aux = nullptr;   // inspection copies (zf_optimizer_state)
    std::vector<int32_t*> steps_view;
    int grid = 148;
    // launch tables
    NormLayer* d_norm_tab = nullptr;
    std::vector<NormLayer> h_norm_tab, up_norm_tab;
    TopkLayer* d_topk_tab[3] = {nullptr, nullptr, nullptr};  // [new set 0 | new set 1 | first (new 1, no old)]
    UpdLayer* d_upd_tab[8] = {};                              // [(cur)*4 + refresh*2 + stage]
    std::vector<UpdLayer> h_upd_tab[8], up_upd_tab[8];
    // f2 warm-up (reading R20): K3 table of the all-columns set, K2 table of the first
    // regular refresh (old = warm-up set) and K3 tables of that step (remap from [n, m])
    int64_t tau = 0, k3_units_w = 0;
    UpdLayer* d_upd_w = nullptr;
    std::vector<UpdLayer> h_upd_w, up_upd_w;
    TopkLayer* d_topk_w = nullptr;
    UpdLayer* d_upd_x[2] = {};
    std::vector<UpdLayer> h_upd_x[2], up_upd_x[2];
    int64_t last_step = -1;       // t of the last zf_step call (warm-up included)
    // table uploads through a small pinned ring
    std::vector<unsigned char*> ring;
    std::vector<cudaEvent_t> ring_ev;
    size_t ring_bytes = 0;
    int ring_pos = 0;
    // AdamW tables (ss depends on lr; may change via zf_set_lr)
    AdamK adam{};
    float* d_ss = nullptr;
    float* d_bc2 = nullptr;
    float* d_sb = nullptr;
    std::vector<float> bc2_host;
    double lr_cur = 0.0, lr_uploaded = -1.0;
    // step state
    int cur = 0;
    bool have_sel = false;
    int64_t last_t = -1;          // regular-schedule index (t - tau) of the last regular step
    int64_t launches = 0;
    cudaEvent_t step_done = nullptr, k3_done = nullptr;
    // offload
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t d2h_all[2] = {nullptr, nullptr};
    bool d2h_issued[2] = {false, false};
    PFN_waitValue32 wait_value = nullptr;
    // host accumulation
    Pool* pool = nullptr;
    std::thread h1;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<int64_t> jobs;
    int64_t h1_done = -1;
    bool stopping = false;
    // accumulation windows as H1 sees them (fixed S, or Zen-auto decisions), and the log
    int64_t h1_win = 0;           // index of the window the next processed step belongs to
    bool h1_first = true;         // the next processed step starts a window
    int h1_last_buf = -1;         // buffer the last processed step accumulated into
    int h1_sealed_buf = -1;       // buffer of the last ended window
    std::vector<int64_t> log_t;
    std::vector<int32_t> log_end;
    std::vector<double> log_A, log_i, log_u;
    // the same windows as zf_step sees them (f1 updates at window ends)
    int64_t mw = 0, mw_len = 0;
    // f2 Zen-auto (reading R21): K6 tables per current set, device state, decision records
    bool autoz = false;
    AutoLayer* d_auto_tab[2] = {nullptr, nullptr};
    double* auto_sums = nullptr;
    uint32_t* auto_counter = nullptr;
    AutoState* auto_state = nullptr;
    AutoRecord* auto_rec_h = nullptr;   // mapped pinned ring [AUTO_RING]
    AutoRecord* auto_rec_d = nullptr;
    cudaEvent_t auto_ev[8] = {};
    static constexpr int AUTO_RING = 8;
    // device-side window accumulation (K7; device_accumulate)
    bool devacc = false;
    AccLayer* d_acc_tab = nullptr;
    int64_t acc_vecs = 0;
    cudaEvent_t acc_d2h_ev[2] = {nullptr, nullptr};
    cudaEvent_t k7_done = nullptr;
    // per-phase timing (zf_profile)
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
    struct Pending { int phase; cudaEvent_t a, b; };
    std::vector<Pending> pending;
    static constexpr int NPHASE = 7;
    double prof_ms[NPHASE] = {};
    int64_t prof_n[NPHASE] = {};

    ~zf_ctx();
    zf_status prof_begin(int phase, cudaStream_t s, Pending* p) {
        p->phase = phase;
        p->a = p->b = nullptr;
        if (!profiling) return ZF_OK;
        if (ev_pool.empty()) {
            cudaEvent_t a, b;
            ZF_CUDA(cudaEventCreate(&a));
            ZF_CUDA(cudaEventCreate(&b));
            ev_pool.push_back({a, b});
        }
        p->a = ev_pool.back().first;
        p->b = ev_pool.back().second;
        ev_pool.pop_back();
        ZF_CUDA(cudaEventRecord(p->a, s));
        return ZF_OK;
    }
    zf_status prof_end(Pending* p, cudaStream_t s) {
        if (!p->a) return ZF_OK;
        ZF_CUDA(cudaEventRecord(p->b, s));
        pending.push_back(*p);
        return ZF_OK;
    }
    zf_status dev_alloc(void** p, size_t bytes) {
        void* q = nullptr;
        ZF_CUDA(cudaMalloc(&q, std::max<size_t>(bytes, 256)));
        dev_allocs.push_back(q);
        *p = q;
        return ZF_OK;
    }
    template <typename T>
    zf_status dalloc(T** p, size_t bytes, bool zero = true) {
        void* q = nullptr;
        ZF_TRY(dev_alloc(&q, bytes));
        if (zero) ZF_CUDA(cudaMemset(q, 0, std::max<size_t>(bytes, 256)));
        *p = static_cast<T*>(q);
        return ZF_OK;
    }
    zf_status upload(void* dst, const void* src, size_t bytes, cudaStream_t s) {
        if (bytes > ring_bytes) return fail(ZF_ESTATE, "table upload larger than ring slot");
        unsigned char* buf = ring[ring_pos];
        ZF_CUDA(cudaEventSynchronize(ring_ev[ring_pos]));  // slot free once its last copy finished
        std::memcpy(buf, src, bytes);
        ZF_CUDA(cudaMemcpyAsync(dst, buf, bytes, cudaMemcpyHostToDevice, s));
        ZF_CUDA(cudaEventRecord(ring_ev[ring_pos], s));
        ring_pos = (ring_pos + 1) % (int)ring.size();
        return ZF_OK;
    }
    // optimizer-state storage: HBM, or mapped pinned host memory (state_offload, row f3)
    zf_status state_alloc(float** p, size_t elems) {
        if (!cfg.state_offload) return dalloc(p, elems * sizeof(float));
        void* h = nullptr;
        ZF_CUDA(cudaHostAlloc(&h, std::max<size_t>(elems * sizeof(float), 256), cudaHostAllocMapped));
        host_pinned.push_back(h);
        std::memset(h, 0, std::max<size_t>(elems * sizeof(float), 256));
        void* d = nullptr;
        ZF_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        *p = static_cast<float*>(d);
        return ZF_OK;
    }
    void h1_loop();
};

zf_ctx::~zf_ctx() {
    if (h1.joinable()) {
        {
            std::lock_guard<std::mutex> lk(mu);
            stopping = true;
        }
        cv.notify_all();
        h1.join();
    }
    delete pool;
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    if (comm) ncclCommDestroy(comm);
    for (void* p : dev_allocs) cudaFree(p);
    for (void* p : host_pinned) cudaFreeHost(p);
    for (float* p : host_plain) std::free(p);
    for (auto& l : L)
        for (int i = 0; i < 2; ++i)
            if (l.d2h_ev[i]) cudaEventDestroy(l.d2h_ev[i]);
    for (auto e : ring_ev) cudaEventDestroy(e);
    for (auto e : d2h_all)
        if (e) cudaEventDestroy(e);
    for (auto e : auto_ev)
        if (e) cudaEventDestroy(e);
    for (auto e : acc_d2h_ev)
        if (e) cudaEventDestroy(e);
    if (k7_done) cudaEventDestroy(k7_done);
    for (auto& e : ev_pool) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
    for (auto& e : pending) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    if (step_done) cudaEventDestroy(step_done);
    if (k3_done) cudaEventDestroy(k3_done);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (aux) cudaStreamDestroy(aux);
}

// One row of H1 (fp32 adds in step order; a window's first step writes 0 + x).  Cloned for
// the host's vector ISA; -ffp-contract=off keeps every add a single IEEE operation.
__attribute__((target_clones("avx512f", "avx2", "default")))
void acc_row_bf16(float* __restrict__ acc, const uint16_t* __restrict__ src, int64_t n, bool first) {
    if (first) {
        for (int64_t i = 0; i < n; ++i) {
            uint32_t u = (uint32_t)src[i] << 16;
            float x;
            std::memcpy(&x, &u, 4);
            acc[i] = 0.0f + x;
        }
    } else {
        for (int64_t i = 0; i < n; ++i) {
            uint32_t u = (uint32_t)src[i] << 16;
            float x;
            std::memcpy(&x, &u, 4);
            acc[i] = acc[i] + x;
        }
    }
}
__attribute__((target_clones("avx512f", "avx2", "default")))
void acc_row_f32(float* __restrict__ acc, const float* __restrict__ src, int64_t n, bool first) {
    if (first) {
        for (int64_t i = 0; i < n; ++i) acc[i] = 0.0f + src[i];
    } else {
        for (int64_t i = 0; i < n; ++i) acc[i] = acc[i] + src[i];
    }
}

// H1: accumulate each layer's staged compact block into the window's fp32 buffer
// as soon as its D2H copy completed (DESIGN.md §2 O8).
void zf_ctx::h1_loop() {
    cudaSetDevice(device);
    const int S = cfg.accum_interval;
    for (;;) {
        int64_t t;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return stopping || !jobs.empty(); });
            if (jobs.empty()) return;
            t = jobs.front();
        }
        const int a = (int)(h1_win % 2);
        const bool first = h1_first;
        const int sb = (int)(t % n_stage);
        for (auto& l : L) {
            cudaEventSynchronize(l.d2h_ev[sb]);
            const int64_t mk = l.mk, ld = l.mk_pad;
            float* acc = l.acc[a];
            const void* stage = l.stage_host[sb];
            const bool bf = gdt == ZF_BF16;
            pool->parallel_for(l.d.n, [&](int64_t b, int64_t e) {
                for (int64_t r = b; r < e; ++r) {
                    if (bf) acc_row_bf16(acc + r * mk, static_cast<const uint16_t*>(stage) + r * ld, mk, first);
                    else acc_row_f32(acc + r * mk, static_cast<const float*>(stage) + r * ld, mk, first);
                }
            });
        }
        // the window decision of step t: fixed S, or K6's record (Zen-auto, reading R21)
        bool end = (t + 1) % S == 0;
        double rA = NAN, ri = NAN, ru = NAN;
        if (autoz) {
            const int slot = (int)(t % AUTO_RING);
            cudaEventSynchronize(auto_ev[slot]);
            const volatile AutoRecord* r = auto_rec_h + slot;
            end = r->end != 0;
            rA = r->A;
            ri = r->imp;
            ru = r->unimp;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            h1_last_buf = a;
            if (end) {
                h1_sealed_buf = a;
                ++h1_win;
            }
            h1_first = end;
            log_t.push_back(t + tau);
            log_end.push_back(end ? 1 : 0);
            log_A.push_back(rA);
            log_i.push_back(ri);
            log_u.push_back(ru);
            jobs.pop_front();
            h1_done = t;
        }
        cv.notify_all();
    }
}

extern "C" zf_status zf_nccl_unique_id(void* out128) {
    g_last_error.clear();
    if (!out128) return fail(ZF_EINVAL, "out is NULL");
    ncclUniqueId id;
    ZF_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, 128);
    return ZF_OK;
}

namespace {

zf_status build_tables(zf_ctx* c) {
    const int nl = (int)c->L.size();
    // K1 table
    c->h_norm_tab.resize(nl);
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        NormLayer& t = c->h_norm_tab[i];
        t = NormLayer{};
        t.n = l.d.n;
        t.m = l.d.m;
        t.ld = l.d.ld_grad;
        t.out = c->norms + l.norm_off;
        t.partial = l.partial;
        t.counter = l.k1_counter;
        t.nrb = l.nrb;
        t.ncb = l.ncb;
        t.unit_begin = l.norm_unit_begin;
    }
    ZF_TRY(c->dalloc(&c->d_norm_tab, nl * sizeof(NormLayer)));
    c->up_norm_tab.assign(nl, NormLayer{});
    // K2 tables
    for (int v = 0; v < 3; ++v) {
        std::vector<TopkLayer> h(nl);
        const int nw = v == 2 ? 1 : v, old = v == 2 ? -1 : (v ^ 1);
        for (int i = 0; i < nl; ++i) {
            LayerState& l = c->L[i];
            TopkLayer& t = h[i];
            t = TopkLayer{};
            t.norms = c->norms + l.norm_off;
            t.m = l.d.m;
            t.k = l.k;
            t.idx = l.idx[nw];
            t.mask = l.mask[nw];
            t.prefix = l.prefix[nw];
            if (old >= 0) {
                t.old_mask = l.mask[old];
                t.old_prefix = l.prefix[old];
                t.old_steps = l.steps[old];
            }
            t.slot_src = l.slot_src;
            t.new_steps = l.steps[nw];
            t.ucol = l.ucol[nw];
            t.seg_cols = l.geo.seg_cols;
            t.gsz = c->gsz;
        }
        ZF_TRY(c->dalloc(&c->d_topk_tab[v], nl * sizeof(TopkLayer)));
        ZF_CUDA(cudaMemcpy(c->d_topk_tab[v], h.data(), nl * sizeof(TopkLayer), cudaMemcpyHostToDevice));
    }
    // K3 tables: variant (cur, refresh, stage)
    for (int v = 0; v < 8; ++v) {
        const int cur = v >> 2, refresh = (v >> 1) & 1, sb = v & 1;
        const int nw = refresh ? (cur ^ 1) : cur;
        auto& h = c->h_upd_tab[v];
        h.resize(nl);
        for (int i = 0; i < nl; ++i) {
            LayerState& l = c->L[i];
            UpdLayer& t = h[i];
            t = UpdLayer{};
            t.n = l.d.n;
            t.m = l.d.m;
            t.ldg = l.d.ld_grad;
            t.ldp = l.d.ld_param;
            t.k = l.k;
            t.idx = l.idx[nw];
            t.mask = l.mask[nw];
            t.prefix = l.prefix[nw];
            t.m_in = l.mom[cur];
            t.v_in = l.vel[cur];
            t.m_out = l.mom[nw];
            t.v_out = l.vel[nw];
            t.slot_src = refresh ? l.slot_src : nullptr;
            t.k_in = l.k;
            t.steps = l.steps[nw];
            t.out = l.stage_dev[sb < c->n_stage ? sb : 0];
            t.out_ld = l.mk_pad;
            t.ucol = l.ucol[nw];
            t.done = c->cfg.offload ? c->done + i : nullptr;
            t.seg_cols = l.geo.seg_cols;
            t.nseg = l.geo.nseg;
            t.R = l.geo.R;
            t.units = l.geo.units;
            t.unit_begin = l.unit_begin;
            t.mv_tma = l.geo.mv_ok ? 1 : 0;
        }
        ZF_TRY(c->dalloc(&c->d_upd_tab[v], nl * sizeof(UpdLayer)));
        c->up_upd_tab[v].assign(nl, UpdLayer{});
    }
    if (c->tau > 0) {
        // warm-up steps: every column selected, moments [n, m] updated in place, no compaction
        c->h_upd_w.resize(nl);
        for (int i = 0; i < nl; ++i) {
            LayerState& l = c->L[i];
            UpdLayer& t = c->h_upd_w[i];
            t = UpdLayer{};
            t.n = l.d.n;
            t.m = l.d.m;
            t.ldg = l.d.ld_grad;
            t.ldp = l.d.ld_param;
            t.k = l.d.m;
            t.idx = l.idx_w;
            t.mask = l.mask_w;
            t.prefix = l.prefix_w;
            t.m_in = t.m_out = l.mom_w;
            t.v_in = t.v_out = l.vel_w;
            t.k_in = l.d.m;
            t.steps = l.steps_w;
            t.seg_cols = l.geo_w.seg_cols;
            t.nseg = l.geo_w.nseg;
            t.R = l.geo_w.R;
            t.units = l.geo_w.units;
            t.unit_begin = l.unit_begin_w;
            t.mv_tma = l.geo_w.mv_ok ? 1 : 0;
        }
        ZF_TRY(c->dalloc(&c->d_upd_w, nl * sizeof(UpdLayer)));
        c->up_upd_w.assign(nl, UpdLayer{});
        // first regular refresh: new set 1, old = the warm-up set
        std::vector<TopkLayer> h(nl);
        for (int i = 0; i < nl; ++i) {
            LayerState& l = c->L[i];
            TopkLayer& t = h[i];
            t = TopkLayer{};
            t.norms = c->norms + l.norm_off;
            t.m = l.d.m;
            t.k = l.k;
            t.idx = l.idx[1];
            t.mask = l.mask[1];
            t.prefix = l.prefix[1];
            t.old_mask = l.mask_w;
            t.old_prefix = l.prefix_w;
            t.old_steps = l.steps_w;
            t.slot_src = l.slot_src;
            t.new_steps = l.steps[1];
            t.ucol = l.ucol[1];
            t.seg_cols = l.geo.seg_cols;
            t.gsz = c->gsz;
        }
        ZF_TRY(c->dalloc(&c->d_topk_w, nl * sizeof(TopkLayer)));
        ZF_CUDA(cudaMemcpy(c->d_topk_w, h.data(), nl * sizeof(TopkLayer), cudaMemcpyHostToDevice));
        // its K3: the regular refresh variant with the old moments read from the [n, m] set
        // (not staged: one old row is m wide)
        for (int sb = 0; sb < 2; ++sb) {
            c->h_upd_x[sb] = c->h_upd_tab[0 * 4 + 2 + sb];
            for (int i = 0; i < nl; ++i) {
                UpdLayer& t = c->h_upd_x[sb][i];
                t.m_in = c->L[i].mom_w;
                t.v_in = c->L[i].vel_w;
                t.k_in = c->L[i].d.m;
                t.mv_tma = 0;
            }
            ZF_TRY(c->dalloc(&c->d_upd_x[sb], nl * sizeof(UpdLayer)));
            c->up_upd_x[sb].assign(nl, UpdLayer{});
        }
    }
    return ZF_OK;
}

zf_status upload_ss(zf_ctx* c, cudaStream_t s) {
    if (c->lr_cur == c->lr_uploaded) return ZF_OK;
    auto h = make_ss(c->lr_cur, c->cfg.adam.beta1);
    if ((int64_t)h.size() > SS_CAP)
        return fail(ZF_EINVAL, "bias-correction table too long for beta1=%g", (double)c->cfg.adam.beta1);
    // one device table, rewritten in stream order: launches already enqueued on the
    // context's (ordered) stream read the old values before the copy lands
    if (!c->d_ss) ZF_TRY(c->dalloc(&c->d_ss, SS_CAP * sizeof(float), false));
    ZF_TRY(c->upload(c->d_ss, h.data(), h.size() * sizeof(float), s));
    c->adam.ss_tab = c->d_ss;
    c->adam.ss_len = (int)h.size();
    auto sb = make_sb(h, c->bc2_host, c->lr_cur);
    if (!c->d_sb) ZF_TRY(c->dalloc(&c->d_sb, (std::max<int64_t>(SS_CAP, (int64_t)c->bc2_host.size())) * 2 * sizeof(float), false));
    ZF_TRY(c->upload(c->d_sb, sb.data(), sb.size() * sizeof(float), s));
    c->adam.sb_tab = reinterpret_cast<const float2*>(c->d_sb);
    c->adam.sb_len = (int)(sb.size() / 2);
    c->adam.ss_inf = (float)c->lr_cur;
    c->adam.decay = (float)(1.0 - c->lr_cur * c->cfg.adam.weight_decay);
    c->lr_uploaded = c->lr_cur;
    return ZF_OK;
}

}  // namespace

extern "C" zf_status zf_create(const zf_layer_desc* layers, int32_t n_layers, const zf_config* cfg, int32_t world,
                               int32_t rank, const void* nccl_id128, int32_t device, zf_ctx** out) {
    g_last_error.clear();
    if (!out) return fail(ZF_EINVAL, "out is NULL");
    *out = nullptr;
    if (!layers || n_layers < 1) return fail(ZF_EINVAL, "need at least one layer");
    if (!cfg) return fail(ZF_EINVAL, "cfg is NULL");
    if (!dtype_ok(cfg->grad_dtype) || !dtype_ok(cfg->param_dtype)) return fail(ZF_EINVAL, "unsupported dtype");
    if (cfg->topk_ppm <= 0 || cfg->topk_ppm > 1000000) return fail(ZF_EINVAL, "topk_ppm must be in (0, 1e6]");
    if (cfg->refresh_interval < 1 || cfg->accum_interval < 1) return fail(ZF_EINVAL, "intervals must be >= 1");
    if (cfg->host_accumulate && !cfg->offload) return fail(ZF_EINVAL, "host_accumulate requires offload");
    if (cfg->host_accumulate && (cfg->refresh_interval % cfg->accum_interval) != 0)
        return fail(ZF_EINVAL, "host_accumulate requires refresh_interval %% accum_interval == 0");
    if (cfg->cpu_update && !cfg->host_accumulate) return fail(ZF_EINVAL, "cpu_update requires host_accumulate");
    if (cfg->cpu_update && cfg->refresh_interval % cfg->accum_interval != 0)
        return fail(ZF_EINVAL, "cpu_update requires refresh_interval to be a multiple of accum_interval");
    if (cfg->warmup_steps < 0) return fail(ZF_EINVAL, "warmup_steps must be >= 0");
    if (!(cfg->auto_gamma >= 0.0f) || !std::isfinite(cfg->auto_gamma))
        return fail(ZF_EINVAL, "auto_gamma must be finite and >= 0");
    if (cfg->auto_gamma > 0.0f && !cfg->host_accumulate) return fail(ZF_EINVAL, "auto_gamma requires host_accumulate");
    if (cfg->device_accumulate && !cfg->host_accumulate)
        return fail(ZF_EINVAL, "device_accumulate requires host_accumulate (it moves that accumulation onto the GPU)");
    ZF_TRY(check_hp(&cfg->adam));
    if (world < 1 || rank < 0 || rank >= world) return fail(ZF_EINVAL, "bad world/rank");
    // world > 1 without an NCCL id: the norm exchange goes through a host all-reduce callback
    // registered with zf_set_host_allreduce before the first step
    for (int i = 0; i < n_layers; ++i) {
        const zf_layer_desc& d = layers[i];
        if (d.n < 0 || d.m < 1 || d.m > 0x7fffffffLL || d.ld_grad < d.m || d.ld_param < d.m)
            return fail(ZF_EINVAL, "layer %d: bad shape (n=%lld m=%lld ld_grad=%lld ld_param=%lld)", i, (long long)d.n,
                        (long long)d.m, (long long)d.ld_grad, (long long)d.ld_param);
    }
    ZF_CUDA(cudaSetDevice(device));
    zf_ctx* c = new zf_ctx();
    auto bail = [&](zf_status st) {
        std::string keep = g_last_error;
        delete c;
        g_last_error = keep;
        return st;
    };
#define ZF_CTRY(expr)                         \
    do {                                      \
        zf_status s_ = (expr);                \
        if (s_ != ZF_OK) return bail(s_);     \
    } while (0)
    c->device = device;
    c->cfg = *cfg;
    c->world = world;
    c->rank = rank;
    c->gdt = cfg->grad_dtype;
    c->pdt = cfg->param_dtype;
    c->gsz = esize(cfg->grad_dtype);
    c->psz = esize(cfg->param_dtype);
    c->devacc = cfg->device_accumulate != 0;
    c->n_stage = cfg->offload && !c->devacc ? 2 : 1;
    c->lr_cur = cfg->adam.lr;
    c->tau = cfg->warmup_steps;
    c->grid = update_grid(c->gdt, c->pdt);
    c->L.resize(n_layers);
    const int rb = norms_rows_per_block(), cb = norms_cols_per_block(c->gdt);
    for (int i = 0; i < n_layers; ++i) {
        LayerState& l = c->L[i];
        l.d = layers[i];
        l.k = zf_k_for(l.d.m, cfg->topk_ppm);
        l.W = (l.d.m + 31) / 32;
        l.mk = l.d.m - l.k;
        l.mk_pad = (l.mk + 7) & ~int64_t(7);
        l.nrb = (int32_t)((l.d.n + rb - 1) / rb);
        l.ncb = (int32_t)((l.d.m + cb - 1) / cb);
        l.norm_off = c->total_m;
        if (l.d.n == 0) c->has_empty = true;
        l.norm_unit_begin = c->k1_units;
        c->total_m += l.d.m;
        c->max_m = std::max(c->max_m, l.d.m);
        c->k1_units += (int64_t)l.nrb * l.ncb;
        l.geo = k3_geom(l.d.n, l.d.m, l.k, c->gsz, c->psz, k3_p_dense(l.d.m, l.k, c->psz));
        l.unit_begin = c->k3_units;
        c->k3_units += l.geo.units;
        if (c->tau > 0) {  // warm-up geometry: k = m
            l.geo_w = k3_geom(l.d.n, l.d.m, l.d.m, c->gsz, c->psz, true);
            l.unit_begin_w = c->k3_units_w;
            c->k3_units_w += l.geo_w.units;
        }
    }
    if (c->k3_units_w > 0x3fffffffLL) return bail(fail(ZF_EINVAL, "model too large"));
    if (c->k1_units > 0x7fffffffLL || c->k3_units > 0x3fffffffLL) return bail(fail(ZF_EINVAL, "model too large"));
    // ---- device state
    ZF_CTRY(c->dalloc(&c->norms, c->total_m * sizeof(float)));
    ZF_CTRY(c->dalloc(&c->claim, sizeof(uint32_t)));
    ZF_CTRY(c->dalloc(&c->done, n_layers * sizeof(uint32_t)));
    for (auto& l : c->L) {
        const int64_t n = l.d.n, k = l.k;
        if (l.nrb > 1) ZF_CTRY(c->dalloc(&l.partial, (size_t)l.nrb * l.d.m * sizeof(float), false));
        ZF_CTRY(c->dalloc(&l.k1_counter, l.ncb * sizeof(uint32_t)));
        for (int s = 0; s < 2; ++s) {
            ZF_CTRY(c->dalloc(&l.idx[s], (k + 16) * sizeof(int32_t)));  // padded (K3 bulk copies)
            ZF_CTRY(c->dalloc(&l.mask[s], (l.W + 8) * sizeof(uint32_t)));   // padded (K3 bulk copies)
            ZF_CTRY(c->dalloc(&l.prefix[s], (l.W + 8) * sizeof(int32_t)));
            ZF_CTRY(c->dalloc(&l.ucol[s], (l.mk + 16) * sizeof(uint16_t)));  // padded (K3 bulk copies)
            // padded by 16 elements: K3 stages these with 16-byte-granular bulk copies
            ZF_CTRY(c->dalloc(&l.steps[s], (k + 16) * sizeof(int32_t)));
            ZF_CTRY(c->state_alloc(&l.mom[s], (size_t)n * k + 16));
            ZF_CTRY(c->state_alloc(&l.vel[s], (size_t)n * k + 16));
        }
        ZF_CTRY(c->dalloc(&l.slot_src, (k + 16) * sizeof(int32_t)));
        if (c->tau > 0) {
            // the warm-up set: all m columns selected (slot = column), zero moments and counts
            const int64_t m = l.d.m;
            ZF_CTRY(c->dalloc(&l.idx_w, (m + 16) * sizeof(int32_t)));
            ZF_CTRY(c->dalloc(&l.mask_w, (l.W + 8) * sizeof(uint32_t)));
            ZF_CTRY(c->dalloc(&l.prefix_w, (l.W + 8) * sizeof(int32_t)));
            ZF_CTRY(c->dalloc(&l.steps_w, (m + 16) * sizeof(int32_t)));
            ZF_CTRY(c->state_alloc(&l.mom_w, (size_t)n * m + 16));
            ZF_CTRY(c->state_alloc(&l.vel_w, (size_t)n * m + 16));
            std::vector<int32_t> iw(m), pw(l.W);
            std::vector<uint32_t> mw(l.W, 0xffffffffu);
            for (int64_t j = 0; j < m; ++j) iw[j] = (int32_t)j;
            for (int64_t w = 0; w < l.W; ++w) pw[w] = (int32_t)(32 * w);
            if (m % 32) mw[l.W - 1] = (1u << (m % 32)) - 1u;
            ZF_CUDA(cudaMemcpy(l.idx_w, iw.data(), m * sizeof(int32_t), cudaMemcpyHostToDevice));
            ZF_CUDA(cudaMemcpy(l.mask_w, mw.data(), l.W * sizeof(uint32_t), cudaMemcpyHostToDevice));
            ZF_CUDA(cudaMemcpy(l.prefix_w, pw.data(), l.W * sizeof(int32_t), cudaMemcpyHostToDevice));
        }
        for (int s = 0; s < c->n_stage; ++s) ZF_CTRY(c->dalloc(&l.stage_dev[s], (size_t)n * l.mk_pad * c->gsz, false));
    }
    {
        int32_t* h = nullptr;
        ZF_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
        c->host_pinned.push_back(h);
        *h = 0;
        c->nonfinite_h = h;
        ZF_CUDA(cudaHostGetDevicePointer(&c->nonfinite_d, h, 0));
    }
    // ---- AdamW tables
    c->adam = adam_scalars(cfg->adam);
    // ---- table upload ring
    c->bc2_host = make_bc2(cfg->adam.beta2);
    c->ring_bytes = std::max<size_t>({n_layers * sizeof(UpdLayer), n_layers * sizeof(NormLayer), SS_CAP * sizeof(float),
                                      std::max<size_t>(SS_CAP, c->bc2_host.size()) * 2 * sizeof(float)});
    for (int i = 0; i < 4; ++i) {
        unsigned char* b = nullptr;
        ZF_CUDA(cudaMallocHost(&b, c->ring_bytes));
        c->host_pinned.push_back(b);
        c->ring.push_back(b);
        cudaEvent_t e;
        ZF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->ring_ev.push_back(e);
    }
    {
        const auto& h = c->bc2_host;
        ZF_CTRY(c->dalloc(&c->d_bc2, h.size() * sizeof(float), false));
        ZF_CUDA(cudaMemcpy(c->d_bc2, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
        c->adam.bc2_tab = c->d_bc2;
        c->adam.bc2_len = (int)h.size();
    }
    ZF_CTRY(build_tables(c));
    // ---- f2 Zen-auto (reading R21): K6 tables over the two selection sets, window state
    c->autoz = cfg->auto_gamma > 0.0f;
    if (c->autoz) {
        for (int v = 0; v < 2; ++v) {
            std::vector<AutoLayer> h(n_layers);
            for (int i = 0; i < n_layers; ++i) {
                const LayerState& l = c->L[i];
                h[i].norms = c->norms + l.norm_off;
                h[i].mask = l.mask[v];
                h[i].m = l.d.m;
                h[i].k = l.k;
            }
            ZF_CTRY(c->dalloc(&c->d_auto_tab[v], n_layers * sizeof(AutoLayer)));
            ZF_CUDA(cudaMemcpy(c->d_auto_tab[v], h.data(), n_layers * sizeof(AutoLayer), cudaMemcpyHostToDevice));
        }
        ZF_CTRY(c->dalloc(&c->auto_sums, 2 * n_layers * sizeof(double)));
        ZF_CTRY(c->dalloc(&c->auto_counter, sizeof(uint32_t)));
        ZF_CTRY(c->dalloc(&c->auto_state, sizeof(AutoState)));  // zero: no open window
        ZF_CUDA(cudaHostAlloc(&c->auto_rec_h, zf_ctx::AUTO_RING * sizeof(AutoRecord), cudaHostAllocMapped));
        c->host_pinned.push_back(c->auto_rec_h);
        std::memset(c->auto_rec_h, 0, zf_ctx::AUTO_RING * sizeof(AutoRecord));
        ZF_CUDA(cudaHostGetDevicePointer(&c->auto_rec_d, c->auto_rec_h, 0));
        for (auto& e : c->auto_ev) ZF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
    }
    c->done_target.assign(n_layers, 0u);
    ZF_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
    for (auto& l : c->L) {
        int32_t* v = nullptr;
        ZF_CTRY(c->dalloc(&v, (c->tau > 0 ? l.d.m : l.k) * sizeof(int32_t)));
        c->steps_view.push_back(v);
    }
    ZF_CUDA(cudaEventCreateWithFlags(&c->step_done, cudaEventDisableTiming));
    ZF_CUDA(cudaEventCreateWithFlags(&c->k3_done, cudaEventDisableTiming));
    // ---- offload: copy stream, pinned host staging, per-layer events, host accumulators
    if (cfg->offload) {
        ZF_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int s = 0; s < 2; ++s) ZF_CUDA(cudaEventCreateWithFlags(&c->d2h_all[s], cudaEventDisableTiming));
        for (auto& l : c->L) {
            for (int s = 0; s < (c->devacc ? 0 : 2); ++s) {  // per-step compact D2H (not with K7)
                void* h = nullptr;
                ZF_CUDA(cudaHostAlloc(&h, std::max<size_t>((size_t)l.d.n * l.mk_pad * c->gsz, 64), cudaHostAllocDefault));
                c->host_pinned.push_back(h);
                l.stage_host[s] = h;
                ZF_CUDA(cudaEventCreateWithFlags(&l.d2h_ev[s], cudaEventDisableTiming | cudaEventBlockingSync));
            }
        }
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            c->wait_value = reinterpret_cast<PFN_waitValue32>(fn);
        if (cfg->host_accumulate && c->devacc) {
            // K7 accumulates on the device; one pinned dense copy of the sealed window per layer
            std::vector<AccLayer> h(c->L.size());
            for (size_t i = 0; i < c->L.size(); ++i) {
                LayerState& l = c->L[i];
                const size_t e = (size_t)l.d.n * l.mk_pad;
                for (int s = 0; s < 2; ++s) ZF_CTRY(c->dalloc(&l.dacc[s], e * sizeof(float), false));
                ZF_CUDA(cudaHostAlloc(&l.acc_sealed_h, std::max<size_t>((size_t)l.d.n * l.mk * sizeof(float), 64),
                                      cudaHostAllocDefault));
                c->host_pinned.push_back(l.acc_sealed_h);
                h[i].src = l.stage_dev[0];
                h[i].acc0 = l.dacc[0];
                h[i].acc1 = l.dacc[1];
                h[i].vec_begin = c->acc_vecs;
                c->acc_vecs += (int64_t)(e / 8);
            }
            ZF_CTRY(c->dalloc(&c->d_acc_tab, h.size() * sizeof(AccLayer)));
            ZF_CUDA(cudaMemcpy(c->d_acc_tab, h.data(), h.size() * sizeof(AccLayer), cudaMemcpyHostToDevice));
            for (auto& e : c->acc_d2h_ev) ZF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ZF_CUDA(cudaEventCreateWithFlags(&c->k7_done, cudaEventDisableTiming));
        }
        if (cfg->host_accumulate && !c->devacc) {
            for (auto& l : c->L) {
                for (int s = 0; s < 2; ++s) {
                    const size_t bytes = std::max<size_t>((size_t)l.d.n * l.mk * sizeof(float), 64);
                    float* p = static_cast<float*>(std::aligned_alloc(64, (bytes + 63) / 64 * 64));
                    if (!p) return bail(fail(ZF_ENOMEM, "host accumulator allocation failed"));
                    std::memset(p, 0, bytes);
                    c->host_plain.push_back(p);
                    l.acc[s] = p;
                }
            }
        }
        if (cfg->host_accumulate && cfg->cpu_update) {
            {
                for (auto& l : c->L) {
                    const size_t nm = (size_t)l.d.n * l.d.m;
                    for (float** pp : {&l.master, &l.mh, &l.vh}) {
                        float* q = static_cast<float*>(std::aligned_alloc(64, (nm * sizeof(float) + 63) / 64 * 64));
                        if (!q) return bail(fail(ZF_ENOMEM, "host optimizer state allocation failed"));
                        std::memset(q, 0, nm * sizeof(float));
                        c->host_plain.push_back(q);
                        *pp = q;
                    }
                    l.th.assign(l.d.m, 0);
                    ZF_CUDA(cudaHostAlloc(&l.p_mirror, std::max<size_t>(nm * c->psz, 64), cudaHostAllocDefault));
                    c->host_pinned.push_back(l.p_mirror);
                    ZF_CUDA(cudaHostAlloc(&l.p_up, std::max<size_t>((size_t)l.d.n * l.mk * c->psz, 64),
                                          cudaHostAllocDefault));
                    c->host_pinned.push_back(l.p_up);
                    ZF_CTRY(c->dalloc(&l.p_up_dev, (size_t)l.d.n * l.mk * c->psz, false));
                    ZF_CTRY(c->dalloc(&l.unsel_dev, (l.mk + 16) * sizeof(int32_t)));
                }
            }
        }
        if (cfg->host_accumulate) {
            int nt = cfg->host_threads > 0 ? cfg->host_threads
                                           : (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            c->pool = new Pool(nt);
            if (!c->devacc) c->h1 = std::thread([c] { c->h1_loop(); });
        }
    }
    // ---- NCCL (collective across ranks), or a pinned host buffer for the host all-reduce
    if (world > 1 && !nccl_id128) {
        ZF_CUDA(cudaHostAlloc(&c->norms_host, std::max<size_t>(c->total_m * sizeof(float), 64), cudaHostAllocDefault));
        c->host_pinned.push_back(c->norms_host);
    }
    if (world > 1 && nccl_id128) {
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof id);
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) return bail(fail(ZF_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
    }
    ZF_CUDA(cudaDeviceSynchronize());
    *out = c;
    return ZF_OK;
#undef ZF_CTRY
}

namespace {

zf_status refresh_pointer_tables(zf_ctx* c, int variant, bool refresh, void* const* grads, void* const* params,
                                 cudaStream_t s) {
    const int nl = (int)c->L.size();
    if (refresh) {
        for (int i = 0; i < nl; ++i) {
            NormLayer& t = c->h_norm_tab[i];
            t.G = grads[i];
            t.vec_ok = aligned16(grads[i]) && ((c->L[i].d.ld_grad * c->gsz) % 16 == 0);
        }
        if (std::memcmp(c->h_norm_tab.data(), c->up_norm_tab.data(), nl * sizeof(NormLayer)) != 0) {
            ZF_TRY(c->upload(c->d_norm_tab, c->h_norm_tab.data(), nl * sizeof(NormLayer), s));
            c->up_norm_tab = c->h_norm_tab;
        }
    }
    // variant >= 0: regular table; -1: warm-up table; -2 - sb: first refresh after warm-up
    std::vector<UpdLayer>& h = variant >= 0 ? c->h_upd_tab[variant] : variant == -1 ? c->h_upd_w : c->h_upd_x[-2 - variant];
    std::vector<UpdLayer>& up =
        variant >= 0 ? c->up_upd_tab[variant] : variant == -1 ? c->up_upd_w : c->up_upd_x[-2 - variant];
    UpdLayer* d = variant >= 0 ? c->d_upd_tab[variant] : variant == -1 ? c->d_upd_w : c->d_upd_x[-2 - variant];
    for (int i = 0; i < nl; ++i) {
        h[i].G = grads[i];
        h[i].P = params[i];
        h[i].tma_ok = k3_tma_ok(grads[i], c->L[i].d.ld_grad, c->L[i].d.m, c->gsz);
        h[i].p_tma = k3_tma_ok(params[i], c->L[i].d.ld_param, c->L[i].d.m, c->psz) &&
                     k3_p_dense(c->L[i].d.m, h[i].k, c->psz);
    }
    if (std::memcmp(h.data(), up.data(), nl * sizeof(UpdLayer)) != 0) {
        ZF_TRY(c->upload(d, h.data(), nl * sizeof(UpdLayer), s));
        up = h;
    }
    return ZF_OK;
}

}  // namespace

// ============================================================ f1: deferred CPU AdamW (reading R18)
namespace {

uint16_t host_bf16_rne(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float host_widen(const void* p, int dt, size_t i) {
    if (dt == ZF_BF16) {
        uint32_t u = (uint32_t) static_cast<const uint16_t*>(p)[i] << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
    return static_cast<const float*>(p)[i];
}

// At a refresh: columns entering the CPU-updated set take the parameter's current value as
// their fp32 master with zero host moments/step count; then the new selection is recorded.
zf_status f1_refresh(zf_ctx* c, void* const* params, cudaStream_t s) {
    const int nl = (int)c->L.size();
    std::vector<std::vector<int32_t>> nidx(nl);
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        nidx[i].resize(l.k);
        ZF_CUDA(cudaMemcpyAsync(nidx[i].data(), l.idx[c->cur], l.k * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        if (l.d.n > 0)
        ZF_CUDA(cudaMemcpy2DAsync(l.p_mirror, l.d.m * c->psz, params[i], l.d.ld_param * c->psz, l.d.m * c->psz, l.d.n,
                                  cudaMemcpyDeviceToHost, s));
    }
    ZF_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        const int64_t m = l.d.m, n = l.d.n;
        std::vector<char> was_cpu(m, 0), now_cpu(m, 1);
        if (!l.idx_host.empty()) {
            std::fill(was_cpu.begin(), was_cpu.end(), 1);
            for (int32_t col : l.idx_host) was_cpu[col] = 0;
        }
        for (int32_t col : nidx[i]) now_cpu[col] = 0;
        std::vector<int32_t> entering;
        for (int64_t col = 0; col < m; ++col)
            if (now_cpu[col] && !was_cpu[col]) entering.push_back((int32_t)col);
        const int pdt = c->pdt;
        c->pool->parallel_for(n, [&](int64_t b, int64_t e) {
            for (int64_t r = b; r < e; ++r)
                for (int32_t col : entering) {
                    l.master[r * m + col] = host_widen(l.p_mirror, pdt, (size_t)(r * m + col));
                    l.mh[r * m + col] = 0.0f;
                    l.vh[r * m + col] = 0.0f;
                }
        });
        for (int32_t col : entering) l.th[col] = 0;
        l.idx_host = nidx[i];
        l.unsel_host.clear();
        for (int64_t col = 0; col < m; ++col)
            if (now_cpu[col]) l.unsel_host.push_back((int32_t)col);
        if (!l.unsel_host.empty())
            ZF_CUDA(cudaMemcpy(l.unsel_dev, l.unsel_host.data(), l.unsel_host.size() * sizeof(int32_t),
                               cudaMemcpyHostToDevice));
    }
    return ZF_OK;
}

// At a window end: one AdamW step (O6 op order, double-derived constants rounded once) with
// the window's average gradient acc/S on the fp32 master of the unselected columns; the
// rounded results are uploaded and scattered into the parameters.
zf_status f1_window_end(zf_ctx* c, int64_t t, int buf, int64_t len, void* const* params, cudaStream_t s) {
    if (c->devacc) {
        ZF_CUDA(cudaEventSynchronize(c->acc_d2h_ev[buf]));  // the sealed window's host copy
    } else {
        std::unique_lock<std::mutex> lk(c->mu);
        c->cv.wait(lk, [&] { return c->h1_done >= t; });
    }
    const zf_adam_params& hp = c->cfg.adam;
    const double lr = c->lr_cur, b1d = hp.beta1, b2d = hp.beta2;
    const float b1 = (float)b1d, b2 = (float)b2d, omb1 = (float)(1.0 - b1d), omb2 = (float)(1.0 - b2d);
    const float eps = (float)hp.eps, wd_f = (float)hp.weight_decay, decay = (float)(1.0 - lr * hp.weight_decay);
    const int wd_mode = hp.weight_decay == 0.0 ? 0 : (hp.decoupled ? 1 : 2);
    const float Sf = (float)len;  // the window's length: S, or Zen-auto's interval (R21)
    const int nl = (int)c->L.size();
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        const int64_t m = l.d.m, n = l.d.n, mk = l.mk;
        if (mk == 0) continue;
        const float* acc = c->devacc ? l.acc_sealed_h : l.acc[buf];
        std::vector<float> ss(mk), bc2s(mk);
        for (int64_t u = 0; u < mk; ++u) {
            const double tt = (double)(l.th[l.unsel_host[u]] + 1);
            ss[u] = (float)(lr / (1.0 - std::pow(b1d, tt)));
            bc2s[u] = (float)std::sqrt(1.0 - std::pow(b2d, tt));
        }
        const int pdt = c->pdt;
        c->pool->parallel_for(n, [&](int64_t b, int64_t e) {
            for (int64_t r = b; r < e; ++r) {
                for (int64_t u = 0; u < mk; ++u) {
                    const int64_t col = l.unsel_host[u];
                    float g = acc[r * mk + u] / Sf;
                    float p = l.master[r * m + col];
                    float mm = l.mh[r * m + col], vv = l.vh[r * m + col];
                    if (wd_mode == 1) p = p * decay;
                    else if (wd_mode == 2) {
                        const float wp = wd_f * p;
                        g = g + wp;
                    }
                    const float a1 = b1 * mm, a2 = omb1 * g;
                    mm = a1 + a2;
                    const float c1 = b2 * vv, c2 = omb2 * g, c3 = c2 * g;
                    vv = c1 + c3;
                    const float den = std::sqrt(vv) / bc2s[u] + eps;
                    const float upd = mm / den;
                    const float delta = ss[u] * upd;
                    p = p - delta;
                    l.master[r * m + col] = p;
                    l.mh[r * m + col] = mm;
                    l.vh[r * m + col] = vv;
                    if (pdt == ZF_BF16) static_cast<uint16_t*>(l.p_up)[r * mk + u] = host_bf16_rne(p);
                    else static_cast<float*>(l.p_up)[r * mk + u] = p;
                }
            }
        });
        for (int64_t u = 0; u < mk; ++u) l.th[l.unsel_host[u]] += 1;
        ZF_CUDA(cudaMemcpyAsync(l.p_up_dev, l.p_up, (size_t)n * mk * c->psz, cudaMemcpyHostToDevice, s));
        ZF_CUDA(launch_scatter_unselected(params[i], pdt, l.d.ld_param, n, mk, l.unsel_dev, l.p_up_dev, s));
        c->launches++;
    }
    ZF_CUDA(cudaStreamSynchronize(s));  // pinned upload buffers are reused next window
    return ZF_OK;
}

// f2 warm-up step (reading R20): every column selected, moments [n, m] updated in place by
// K3 (no compaction, nothing offloaded).  K3 launches since the set was made = t.
zf_status warmup_step(zf_ctx* c, int64_t t, void* const* grads, void* const* params, cudaStream_t s) {
    const int nl = (int)c->L.size();
    ZF_TRY(upload_ss(c, s));
    ZF_TRY(refresh_pointer_tables(c, -1, false, grads, params, s));
    UpdParams prm{};
    prm.layers.dev = c->d_upd_w;
    prm.layers.n = nl;
    prm.total_units = c->k3_units_w;
    prm.claim = c->claim;
    prm.claim_base = c->claim_base;
    prm.step_delta = c->since;
    prm.do_adam = 1;
    prm.do_compact = 0;
    prm.nonfinite = c->nonfinite_d;
    prm.adam = c->adam;
    const int grid = (int)std::min<int64_t>(c->grid, c->k3_units_w);
    zf_ctx::Pending pe3;
    ZF_TRY(c->prof_begin(3, s, &pe3));
    ZF_CUDA(launch_update(prm, c->gdt, c->pdt, grid, s));
    ZF_TRY(c->prof_end(&pe3, s));
    c->launches++;
    c->claim_base += (uint32_t)(c->k3_units_w + (int64_t)grid * update_limits().producers);
    c->since += 1;
    c->last_step = t;
    ZF_CUDA(cudaEventRecord(c->step_done, s));
    return ZF_OK;
}

}  // namespace

extern "C" zf_status zf_step(zf_ctx* c, int64_t t0, void* const* grads, void* const* params, zf_stream_t stream) {
    g_last_error.clear();
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    if (!grads || !params) return fail(ZF_EINVAL, "grads/params is NULL");
    const int nl = (int)c->L.size();
    for (int i = 0; i < nl; ++i)
        if ((!grads[i] || !params[i]) && c->L[i].d.n > 0)
            return fail(ZF_EINVAL, "layer %d: NULL gradient or parameter", i);
    if (t0 < 0) return fail(ZF_EINVAL, "t must be >= 0");
    const int N = c->cfg.refresh_interval;
    const int64_t tau = c->tau;
    if (c->last_step >= 0) {
        if (t0 != c->last_step + 1)
            return fail(ZF_ESTATE, "steps must be consecutive (last %lld, got %lld)", (long long)c->last_step,
                        (long long)t0);
    } else if (tau > 0) {
        if (t0 != 0) return fail(ZF_ESTATE, "with warm-up steps the first step must be t = 0");
    } else if (t0 % N != 0) {
        return fail(ZF_ESTATE, "first step must be a refresh step (t %% N == 0)");
    }
    if (c->world > 1 && !c->comm && !c->host_allreduce)
        return fail(ZF_ESTATE, "world > 1 needs an NCCL id at zf_create or zf_set_host_allreduce");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ZF_CUDA(cudaSetDevice(c->device));
    if (t0 < tau) return warmup_step(c, t0, grads, params, s);
    // the regular schedule (refreshes, windows, offload stages) counts from step tau (R20)
    const int64_t t = t0 - tau;
    const bool refresh = (t % N) == 0;
    const int sb = (int)(t % c->n_stage);
    // the first refresh after a warm-up remaps from the [n, m] warm-up set (tables -2 - sb)
    const bool from_warmup = !c->have_sel && tau > 0;
    const int variant = from_warmup ? -2 - (sb & 1) : c->cur * 4 + (refresh ? 2 : 0) + (sb & 1);
    ZF_TRY(upload_ss(c, s));
    const bool norms_now = refresh || c->autoz;  // Zen-auto reads every step's norms (R21)
    ZF_TRY(refresh_pointer_tables(c, variant, norms_now, grads, params, s));

    if (c->cfg.offload) {
        // (K3 counts per-layer completions only when offloading; see build_tables)
        // the device staging buffer sb is free once the D2H copies issued two steps ago finished
        if (c->d2h_issued[sb]) ZF_CUDA(cudaStreamWaitEvent(s, c->d2h_all[sb], 0));
        if (c->cfg.host_accumulate && !c->devacc) {
            // host staging buffer sb is free once H1 consumed step t-2
            std::unique_lock<std::mutex> lk(c->mu);
            c->cv.wait(lk, [&] { return c->h1_done >= t - 2 || c->last_t < t - 2; });
        }
    }
    if (norms_now) {
        zf_ctx::Pending pe;
        // layers with no rows on this rank (flat partitions, row f3) contribute zero norms
        if (c->has_empty) ZF_CUDA(cudaMemsetAsync(c->norms, 0, c->total_m * sizeof(float), s));
        Table<NormLayer> tn{};
        tn.dev = c->d_norm_tab;
        tn.n = nl;
        ZF_TRY(c->prof_begin(0, s, &pe));
        ZF_CUDA(launch_norms(tn, c->k1_units, c->gdt, c->nonfinite_d, s));
        ZF_TRY(c->prof_end(&pe, s));
        c->launches++;
        if (c->world > 1) {
            ZF_TRY(c->prof_begin(1, s, &pe));
            if (c->comm) {
                ZF_NCCL(ncclAllReduce(c->norms, c->norms, (size_t)c->total_m, ncclFloat32, ncclSum, c->comm, s));
            } else {
                // host all-reduce (e.g. torch.distributed gloo): stream-synchronous round trip
                ZF_CUDA(cudaMemcpyAsync(c->norms_host, c->norms, c->total_m * sizeof(float), cudaMemcpyDeviceToHost, s));
                ZF_CUDA(cudaStreamSynchronize(s));
                if (c->host_allreduce(c->norms_host, c->total_m, c->host_allreduce_user) != 0)
                    return fail(ZF_ENCCL, "host all-reduce callback failed");
                ZF_CUDA(cudaMemcpyAsync(c->norms, c->norms_host, c->total_m * sizeof(float), cudaMemcpyHostToDevice, s));
            }
            ZF_TRY(c->prof_end(&pe, s));
        }
    }
    if (refresh) {
        zf_ctx::Pending pe;
        Table<TopkLayer> tk{};
        tk.dev = c->have_sel ? c->d_topk_tab[c->cur ^ 1] : (from_warmup ? c->d_topk_w : c->d_topk_tab[2]);
        tk.n = nl;
        ZF_TRY(c->prof_begin(2, s, &pe));
        ZF_CUDA(launch_topk(tk, c->max_m, c->since, c->nonfinite_d, s));
        c->since = 0;
        ZF_TRY(c->prof_end(&pe, s));
        c->launches++;
    }
    // first refresh writes set 1 (variant built with cur=0, refresh=1 -> new set 1)
    UpdParams prm{};
    prm.layers.dev = from_warmup ? c->d_upd_x[sb & 1] : c->d_upd_tab[variant];
    prm.layers.n = nl;
    prm.total_units = c->k3_units;
    prm.claim = c->claim;
    prm.claim_base = c->claim_base;
    prm.step_delta = c->since;
    prm.do_adam = 1;
    prm.do_compact = 1;
    prm.nonfinite = c->nonfinite_d;
    prm.adam = c->adam;
    {
        static const int dbg = getenv("ZF_K3_DEBUG_MODE") ? atoi(getenv("ZF_K3_DEBUG_MODE")) : 0;
        prm.debug_mode = dbg;
    }
    const int grid = (int)std::min<int64_t>(c->grid, c->k3_units);
    zf_ctx::Pending pe3;
    ZF_TRY(c->prof_begin(3, s, &pe3));
    ZF_CUDA(launch_update(prm, c->gdt, c->pdt, grid, s));
    ZF_TRY(c->prof_end(&pe3, s));
    c->launches++;
    c->claim_base += (uint32_t)(c->k3_units + (int64_t)grid * update_limits().producers);
    c->since += 1;
    for (int i = 0; i < nl; ++i) c->done_target[i] += (uint32_t)c->L[i].geo.units * (uint32_t)update_limits().consumer_warps;
    if (refresh) {
        c->cur ^= 1;
        c->have_sel = true;
    }
    if (c->devacc) {
        // K7: add this step's compact block into the window's device accumulator (before K6,
        // which decides whether this step ends the window); a window's first step overwrites
        // the buffer, so it waits for that buffer's last D2H (two windows ago)
        const int b = (int)(c->mw % 2);
        if (c->mw_len == 0) ZF_CUDA(cudaStreamWaitEvent(s, c->acc_d2h_ev[b], 0));
        zf_ctx::Pending pe6;
        ZF_TRY(c->prof_begin(6, s, &pe6));
        ZF_CUDA(launch_accumulate(c->d_acc_tab, nl, c->acc_vecs, c->gdt, c->mw_len == 0 ? 1 : 0, b,
                                  c->autoz ? c->auto_state : nullptr, s));
        ZF_TRY(c->prof_end(&pe6, s));
        c->launches++;
    }
    if (c->autoz) {
        // K6: the step's Zen-auto decision from its norms and the (new) current selection
        const int slot = (int)(t % zf_ctx::AUTO_RING);
        ZF_CUDA(launch_zen_auto(c->d_auto_tab[c->cur], nl, c->auto_sums, c->auto_counter, c->auto_state,
                                c->auto_rec_d + slot, t0, (double)c->cfg.auto_gamma, c->cfg.accum_interval,
                                (t + 1) % N == 0 ? 1 : 0, s));
        c->launches++;
        ZF_CUDA(cudaEventRecord(c->auto_ev[slot], s));
    }
    c->last_t = t;
    c->last_step = t0;
    ZF_CUDA(cudaEventRecord(c->step_done, s));

    if (c->cfg.offload && !c->devacc) {
        // X1: per-layer D2H as soon as the layer's last unit finished (cyclic counter)
        if (!c->wait_value) ZF_CUDA(cudaStreamWaitEvent(c->copy_stream, c->step_done, 0));
        zf_ctx::Pending pe4;
        bool pe4_open = false;
        for (int i = 0; i < nl; ++i) {
            LayerState& l = c->L[i];
            if (c->wait_value) {
                const uint32_t target = c->done_target[i];
                CUresult r = c->wait_value(reinterpret_cast<CUstream>(c->copy_stream),
                                           reinterpret_cast<CUdeviceptr>(c->done + i), target,
                                           CU_STREAM_WAIT_VALUE_GEQ);
                if (r != CUDA_SUCCESS) {  // stream memory ops unavailable: gate on the whole step
                    c->wait_value = nullptr;
                    ZF_CUDA(cudaStreamWaitEvent(c->copy_stream, c->step_done, 0));
                }
            }
            // one flat copy of the pitched block (H1 reads the rows at the same pitch)
            if (l.mk && l.d.n) {
                if (!pe4_open) {  // phase 4: the step's D2H span, from the first copy's start
                    ZF_TRY(c->prof_begin(4, c->copy_stream, &pe4));
                    pe4_open = true;
                }
                ZF_CUDA(cudaMemcpyAsync(l.stage_host[sb], l.stage_dev[sb], (size_t)l.d.n * l.mk_pad * c->gsz,
                                        cudaMemcpyDeviceToHost, c->copy_stream));
            }
            ZF_CUDA(cudaEventRecord(l.d2h_ev[sb], c->copy_stream));
        }
        if (pe4_open) ZF_TRY(c->prof_end(&pe4, c->copy_stream));
        ZF_CUDA(cudaEventRecord(c->d2h_all[sb], c->copy_stream));
        c->d2h_issued[sb] = true;
        if (c->cfg.host_accumulate) {
            {
                std::lock_guard<std::mutex> lk(c->mu);
                c->jobs.push_back(t);
            }
            c->cv.notify_all();
        }
    }
    if (c->cfg.cpu_update && refresh) ZF_TRY(f1_refresh(c, params, s));
    if (c->cfg.host_accumulate) {
        // the window decision of step t (fixed S, or Zen-auto's record) and, with f1, the
        // CPU update of an ended window (synchronous, reading R18)
        c->mw_len += 1;
        bool end = (t + 1) % c->cfg.accum_interval == 0;
        double rA = NAN, ri = NAN, ru = NAN;
        if (c->autoz && (c->cfg.cpu_update || c->devacc)) {
            const int slot = (int)(t % zf_ctx::AUTO_RING);
            ZF_CUDA(cudaEventSynchronize(c->auto_ev[slot]));
            const volatile AutoRecord* r = c->auto_rec_h + slot;
            end = r->end != 0;
            rA = r->A;
            ri = r->imp;
            ru = r->unimp;
        } else if (c->autoz) {
            end = false;  // not needed on this thread without f1 (H1 tracks the windows)
        }
        const int b = (int)(c->mw % 2);
        if (c->devacc) {
            // this thread plays H1's bookkeeping role; a sealed window goes to the host once
            if (end) {
                ZF_CUDA(cudaEventRecord(c->k7_done, s));
                ZF_CUDA(cudaStreamWaitEvent(c->copy_stream, c->k7_done, 0));
                zf_ctx::Pending pe5;
                ZF_TRY(c->prof_begin(5, c->copy_stream, &pe5));  // phase 5: the sealed window's D2H
                for (auto& l : c->L)
                    if (l.mk && l.d.n)
                        ZF_CUDA(cudaMemcpy2DAsync(l.acc_sealed_h, l.mk * sizeof(float), l.dacc[b],
                                                  l.mk_pad * sizeof(float), l.mk * sizeof(float), l.d.n,
                                                  cudaMemcpyDeviceToHost, c->copy_stream));
                ZF_TRY(c->prof_end(&pe5, c->copy_stream));
                ZF_CUDA(cudaEventRecord(c->acc_d2h_ev[b], c->copy_stream));
            }
            std::lock_guard<std::mutex> lk(c->mu);
            c->h1_last_buf = b;
            if (end) c->h1_sealed_buf = b;
            c->log_t.push_back(t0);
            c->log_end.push_back(end ? 1 : 0);
            c->log_A.push_back(rA);
            c->log_i.push_back(ri);
            c->log_u.push_back(ru);
        }
        if (c->cfg.cpu_update && end) ZF_TRY(f1_window_end(c, t, b, c->mw_len, params, s));
        if (end) {
            c->mw += 1;
            c->mw_len = 0;
        }
    }
    return ZF_OK;
}

extern "C" zf_status zf_sync(zf_ctx* c) {
    g_last_error.clear();
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    ZF_CUDA(cudaSetDevice(c->device));
    ZF_CUDA(cudaEventSynchronize(c->step_done));
    if (c->copy_stream) ZF_CUDA(cudaStreamSynchronize(c->copy_stream));
    if (c->cfg.host_accumulate) {
        std::unique_lock<std::mutex> lk(c->mu);
        c->cv.wait(lk, [&] { return c->jobs.empty(); });
    }
    volatile int32_t* f = c->nonfinite_h;
    if (*f) {
        *f = 0;
        return fail(ZF_ENONFINITE, "non-finite gradient value seen");
    }
    return ZF_OK;
}

extern "C" zf_status zf_selected(zf_ctx* c, int32_t layer, const int32_t** idx, int64_t* k) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    if (!c->have_sel && c->tau > 0 && c->last_step >= 0) {  // warm-up: all columns
        if (idx) *idx = c->L[layer].idx_w;
        if (k) *k = c->L[layer].d.m;
        return ZF_OK;
    }
    if (!c->have_sel) return fail(ZF_ESTATE, "no selection yet");
    if (idx) *idx = c->L[layer].idx[c->cur];
    if (k) *k = c->L[layer].k;
    return ZF_OK;
}

extern "C" zf_status zf_norms(zf_ctx* c, int32_t layer, const float** norms) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    if (norms) *norms = c->norms + c->L[layer].norm_off;
    return ZF_OK;
}

extern "C" zf_status zf_optimizer_state(zf_ctx* c, int32_t layer, const float** exp_avg, const float** exp_avg_sq,
                                        const int32_t** step) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    const bool warm = !c->have_sel && c->tau > 0 && c->last_step >= 0;
    if (!c->have_sel && !warm) return fail(ZF_ESTATE, "no state yet");
    const LayerState& l = c->L[layer];
    if (exp_avg) *exp_avg = warm ? l.mom_w : l.mom[c->cur];
    if (exp_avg_sq) *exp_avg_sq = warm ? l.vel_w : l.vel[c->cur];
    if (step) {
        // device keeps base counts at the last refresh; materialize base + delta
        ZF_CUDA(cudaSetDevice(c->device));
        ZF_CUDA(cudaEventSynchronize(c->step_done));
        ZF_CUDA(launch_add_const(warm ? l.steps_w : l.steps[c->cur], c->steps_view[layer], warm ? l.d.m : l.k,
                                 c->since, c->aux));
        ZF_CUDA(cudaStreamSynchronize(c->aux));
        *step = c->steps_view[layer];
    }
    return ZF_OK;
}

extern "C" zf_status zf_compact_buffer(zf_ctx* c, int32_t layer, const void** dev, int64_t* dev_ld,
                                       const void** host) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    if (c->last_t < 0) return fail(ZF_ESTATE, "no step yet");
    const int sb = (int)(c->last_t % c->n_stage);
    if (dev) *dev = c->L[layer].stage_dev[sb];
    if (dev_ld) *dev_ld = c->L[layer].mk_pad;
    if (host) *host = c->cfg.offload && !c->devacc ? c->L[layer].stage_host[sb] : nullptr;
    return ZF_OK;
}

extern "C" zf_status zf_host_accumulator(zf_ctx* c, int32_t layer, int32_t which, const float** host, int64_t* rows,
                                         int64_t* cols) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    if (!c->cfg.host_accumulate) return fail(ZF_ESTATE, "host accumulation is off");
    const LayerState& l = c->L[layer];
    const float* p = nullptr;
    {
        // windows as the host accumulation processed them (fixed S or Zen-auto)
        std::lock_guard<std::mutex> lk(c->mu);
        const int b = which == 0 ? c->h1_last_buf : c->h1_sealed_buf;
        if (c->devacc) {
            if (which == 1 && b >= 0) p = l.acc_sealed_h;  // the active window lives on the device
        } else if (b >= 0) {
            p = l.acc[b];
        }
    }
    if (host) *host = p;
    if (rows) *rows = l.d.n;
    if (cols) *cols = l.mk;
    return ZF_OK;
}

extern "C" zf_status zf_device_accumulator(zf_ctx* c, int32_t layer, int32_t which, const float** dev,
                                           int64_t* ld) {
    if (!c || layer < 0 || layer >= (int)c->L.size()) return fail(ZF_EINVAL, "bad ctx/layer");
    if (!c->devacc) return fail(ZF_ESTATE, "device accumulation is off");
    const LayerState& l = c->L[layer];
    std::lock_guard<std::mutex> lk(c->mu);
    const int b = which == 0 ? c->h1_last_buf : c->h1_sealed_buf;
    if (dev) *dev = b >= 0 ? l.dacc[b] : nullptr;
    if (ld) *ld = l.mk_pad;
    return ZF_OK;
}

extern "C" zf_status zf_window_log(zf_ctx* c, int64_t cap, int64_t* t, int32_t* end, double* A, double* imp,
                                   double* unimp, int64_t* count) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    if (!c->cfg.host_accumulate) return fail(ZF_ESTATE, "host accumulation is off");
    std::lock_guard<std::mutex> lk(c->mu);
    const int64_t n = (int64_t)c->log_t.size();
    for (int64_t i = 0; i < std::min(cap, n); ++i) {
        if (t) t[i] = c->log_t[i];
        if (end) end[i] = c->log_end[i];
        if (A) A[i] = c->log_A[i];
        if (imp) imp[i] = c->log_i[i];
        if (unimp) unimp[i] = c->log_u[i];
    }
    if (count) *count = n;
    return ZF_OK;
}

extern "C" zf_status zf_set_host_allreduce(zf_ctx* c, zf_host_allreduce_fn fn, void* user) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    if (c->world < 2 || c->comm) return fail(ZF_ESTATE, "host all-reduce needs world > 1 created without an NCCL id");
    c->host_allreduce = fn;
    c->host_allreduce_user = user;
    return ZF_OK;
}

extern "C" zf_status zf_set_lr(zf_ctx* c, double lr) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    if (!(lr >= 0.0f) || !std::isfinite(lr)) return fail(ZF_EINVAL, "lr must be finite and >= 0");
    c->lr_cur = lr;
    return ZF_OK;
}

extern "C" int64_t zf_kernel_launches(zf_ctx* c) { return c ? c->launches : -1; }

extern "C" zf_status zf_profile(zf_ctx* c, int32_t enable) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    c->profiling = enable != 0;
    return ZF_OK;
}

extern "C" zf_status zf_profile_read(zf_ctx* c, double* ms, int64_t* count) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    for (auto& p : c->pending) {
        ZF_CUDA(cudaEventSynchronize(p.b));
        float e = 0.0f;
        ZF_CUDA(cudaEventElapsedTime(&e, p.a, p.b));
        c->prof_ms[p.phase] += e;
        c->prof_n[p.phase] += 1;
        c->ev_pool.push_back({p.a, p.b});
    }
    c->pending.clear();
    for (int i = 0; i < zf_ctx::NPHASE; ++i) {
        if (ms) ms[i] = c->prof_ms[i];
        if (count) count[i] = c->prof_n[i];
        c->prof_ms[i] = 0;
        c->prof_n[i] = 0;
    }
    return ZF_OK;
}

extern "C" zf_status zf_destroy(zf_ctx* c) {
    if (!c) return ZF_OK;
    delete c;
    return ZF_OK;
}
