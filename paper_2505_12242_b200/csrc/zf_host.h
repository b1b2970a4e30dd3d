// zf_host.h -- private host-side declarations of libzf.so: error reporting, AdamW
// constant tables, K3 work-unit geometry, the per-layer state and the context struct
// behind the opaque zf_ctx of include/zf.h.  Shared by zf_prim.cu (stateless
// primitives), zf_driver.cu (zf_create / zf_step / views) and zf_host.cu (host
// accumulation threads, deferred CPU AdamW).  Product code only.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
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
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <pthread.h>
#include <sched.h>
#include <cctype>

#include "../../include/zf.h"
#include "zf_internal.cuh"


namespace zfh {
using namespace zf;

// ============================================================ errors
inline thread_local std::string g_last_error;

inline zf_status fail(zf_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

// A failed runtime call is reported once: the thread's last-error state is reset so a
// later launch check (cudaGetLastError) does not report it again (e.g. an out-of-memory
// zf_create followed by a successful one).
#define ZF_CUDA(call)                                                                                       \
    do {                                                                                                    \
        cudaError_t e_ = (call);                                                                            \
        if (e_ != cudaSuccess) {                                                                            \
            (void)cudaGetLastError();                                                                       \
            return fail(ZF_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));       \
        }                                                                                                   \
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

inline int esize(zf_dtype d) { return d == ZF_BF16 ? 2 : 4; }
inline bool dtype_ok(int d) { return d == ZF_FP32 || d == ZF_BF16; }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ============================================================ AdamW constants
// bias-correction tables computed on the host in double, one rounding to fp32
// (DESIGN.md §2 O6): ss[t] = f32(lr / (1 - b1^t)), bc2s[t] = f32(sqrt(1 - b2^t)).
// Both are monotone in t and reach their limits (f32(lr), 1.0f) at a finite t;
// the tables stop there and the kernel uses the limit beyond.
#define ZF_MAX_HSTAGE 16   // host staging slots a context may ask for (zf_config.host_stages)
constexpr int64_t MAX_TAB = 1 << 24;
constexpr int64_t SS_CAP = 1 << 16;  // ss table capacity of a context (beta1 <= 0.999)

inline std::vector<float> make_ss(double lr, double b1) {
    std::vector<float> t(1, 0.0f);
    const float lim = (float)lr;
    for (int64_t i = 1; i < MAX_TAB; ++i) {
        const float v = (float)(lr / (1.0 - std::pow(b1, (double)i)));
        if (v == lim) break;
        t.push_back(v);
    }
    return t;
}

inline std::vector<float> make_bc2(double b2) {
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
inline std::vector<float> make_sb(const std::vector<float>& ss, const std::vector<float>& bc2, double lr) {
    const size_t n = std::max(ss.size(), bc2.size());
    std::vector<float> t(2 * n);
    for (size_t i = 0; i < n; ++i) {
        t[2 * i] = i < ss.size() ? ss[i] : (float)lr;
        t[2 * i + 1] = i < bc2.size() ? bc2[i] : 1.0f;
    }
    return t;
}

inline zf_status check_hp(const zf_adam_params* hp) {
    if (!hp) return fail(ZF_EINVAL, "hp is NULL");
    if (!(hp->lr >= 0.0f) || !std::isfinite(hp->lr)) return fail(ZF_EINVAL, "lr must be finite and >= 0");
    if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f)) return fail(ZF_EINVAL, "beta1 must be in [0, 1)");
    if (!(hp->beta2 >= 0.0f && hp->beta2 < 1.0f)) return fail(ZF_EINVAL, "beta2 must be in [0, 1)");
    if (!(hp->eps > 0.0f) || !std::isfinite(hp->eps)) return fail(ZF_EINVAL, "eps must be > 0");
    if (!(hp->weight_decay >= 0.0f) || !std::isfinite(hp->weight_decay)) return fail(ZF_EINVAL, "weight_decay must be >= 0");
    return ZF_OK;
}

// Scalars of AdamK (the tables are attached by the caller).
inline AdamK adam_scalars(const zf_adam_params& hp) {
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
inline TabCache& tab_cache() {
    static TabCache* c = new TabCache();
    return *c;
}

inline uint64_t dbits(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}

inline zf_status upload_table(const std::vector<float>& h, float** d, cudaStream_t s) {
    float* pinned = nullptr;
    ZF_CUDA(cudaMallocHost(&pinned, h.size() * sizeof(float)));  // kept alive with the table
    std::memcpy(pinned, h.data(), h.size() * sizeof(float));
    ZF_CUDA(cudaMalloc(d, h.size() * sizeof(float)));
    ZF_CUDA(cudaMemcpyAsync(*d, pinned, h.size() * sizeof(float), cudaMemcpyHostToDevice, s));
    return ZF_OK;
}

inline zf_status cached_tables(const zf_adam_params& hp, cudaStream_t s, AdamK* a) {
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
inline bool k3_p_dense(int64_t m, int64_t k, int psz) {
    const double frac = (double)k / (double)m;
    return 1.0 - std::pow(1.0 - frac, 32.0 / psz) >= 0.5;
}

// Worst-case bytes one K3 unit stages (R rows x c columns): the G tile, the p tile (refresh
// units with a dense selection), the parameter-subset slab (steady units with param_subset)
// and the moment slabs (R*k: also covers the old rows of a refresh); each a 16-byte-granular
// superset.  The layer's selection metadata is read through L1, not staged.
inline int64_t k3_unit_bytes(int64_t R, int64_t c, int64_t k, int gsz, int psz, bool p_tile, bool mv,
                             bool psub = false) {
    auto a16 = [](int64_t b) { return (b + 15) & ~int64_t(15); };
    int64_t b = a16(R * c * gsz);
    if (p_tile) b += a16(R * c * psz);
    if (psub && mv) b += a16((R * k + 8) * psz) + 16;
    if (mv) b += 2 * (a16((R * k + 8) * 4) + 16);
    return b;
}

inline K3Geom k3_geom(int64_t n, int64_t m, int64_t k, int gsz, int psz, bool p_dense, bool adam = true,
                      bool psub = false) {
    const UpdLimits lim = update_limits();
    const int64_t A = lim.arena_bytes;
    K3Geom g{};
    // moments staged unless even one row's old moments cannot fit next to a minimal tile
    g.mv_ok = adam && k3_unit_bytes(1, std::min<int64_t>(m, 128), k, gsz, psz, p_dense, true, psub) <= A;
    // Units are R rows x c columns (c = m, or a multiple of 128 so segments start 16-byte
    // aligned in the mask/prefix words): the shape with the fewest units per matrix (the most
    // bytes per stage), ties to full rows / wider segments.  ZF_K3_GEOM=rows keeps the older
    // rule (full rows when one fits, else single-row segments).
    // Measured (tools/k3_geom_ab.sh): the search wins with a staged p tile (Llama-2-13B K3
    // 23.90 -> 22.76 ms: m = 5120 rows go from 1-row units to 3 rows x 2688 columns) but
    // loses without one (k = 1%: 6.92 -> 7.27 ms, more exposed p loads per unit), so
    // unstaged-p layers keep the row rule.
    static const bool rows_env = getenv("ZF_K3_GEOM") && std::string(getenv("ZF_K3_GEOM")) == "rows";
    const bool rows_only = rows_env || (!p_dense && !psub);
    auto rmax = [&](int64_t c) {
        int64_t R = 0;
        while (R < std::min<int64_t>(n, 127) && k3_unit_bytes(R + 1, c, k, gsz, psz, p_dense, g.mv_ok, psub) <= A)
            ++R;
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

inline bool k3_tma_ok(const void* G, int64_t ldg, int64_t m, int gsz) {
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

inline zf_status check_matrix(const void* G, int gdt, int64_t n, int64_t m, int64_t ld, const char* what) {
    if (!G) return fail(ZF_EINVAL, "%s is NULL", what);
    if (!dtype_ok(gdt)) return fail(ZF_EINVAL, "%s: unsupported dtype %d", what, gdt);
    if (n < 1 || m < 1) return fail(ZF_EINVAL, "%s: need n >= 1 and m >= 1 (got n=%lld m=%lld)", what, (long long)n,
                                    (long long)m);
    if (m > 0x7fffffffLL) return fail(ZF_EINVAL, "%s: m too large", what);
    if (ld < m) return fail(ZF_EINVAL, "%s: ld (%lld) < m (%lld)", what, (long long)ld, (long long)m);
    return ZF_OK;
}


// ============================================================ stateful driver state
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
    void* psub = nullptr;             // param_subset: [n, k] dense copy of p[:, idx] (HBM)
    void* psub2 = nullptr;            // its ping-pong partner (blocks follow the moment sets' cur)
    float2* sbv = nullptr;            // [max(k, m during warm-up)] per-slot {ss, bc2s} of the next K3
    void* gsel = nullptr;             // split update: [n, k] selected gradients (K3a -> K3b)
    int64_t row_begin = 0;            // K3b: prefix of ceil(n*k / 8) over layers (its chunks)
    void* stage_dev[2] = {nullptr, nullptr};
    void* stage_host[ZF_MAX_HSTAGE] = {};   // pinned compact blocks, one per host staging slot
    float* acc[2] = {nullptr, nullptr};
    float* dacc[2] = {nullptr, nullptr};  // device_accumulate: [n, mk_pad] fp32 window accumulators
    float* acc_sealed_h = nullptr;        // device_accumulate: pinned dense [n, mk] copy of the sealed window
    // K3 geometry
    K3Geom geo{};                     // refresh units (p tile when the selection is dense)
    int64_t unit_begin = 0;
    K3Geom geo_s{};                   // steady units (param_subset: the subset slab instead of a p tile)
    int64_t unit_begin_s = 0;
    int32_t chunk = 0;                // X1 copy chunk (consecutive layers, one D2H per chunk)
    int64_t stage_off = 0;            // byte offset of this layer's compact block in a staging slot
    // f1: deferred CPU AdamW (reading R18)
    // dense over the current unselected columns (position u = column unsel_host[u]), remapped
    // at every refresh: the window update is then a contiguous, vectorised row loop
    float* master = nullptr;          // [n, m-k] fp32 host master of the CPU-updated columns
    float* mh = nullptr;              // [n, m-k] host moments
    float* vh = nullptr;
    std::vector<int32_t> th;          // [m-k] host step count per unselected column
    std::vector<int32_t> idx_host;    // current selection (ascending), host copy
    std::vector<int32_t> unsel_host;  // its complement (ascending)
    void* p_mirror = nullptr;         // pinned [n, <= m-k]: the entering columns of p at a refresh
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

// NUMA placement of the host side (rows a7/a8, f1): the CPUs of the NUMA node the GPU hangs
// off (sysfs numa_node of its PCI function, then that node's cpulist).  Empty when the
// platform reports no node (-1, e.g. a single-node VM) -- then nothing is pinned.
inline std::vector<int> gpu_numa_cpus(int device, int* node_out) {
    std::vector<int> cpus;
    *node_out = -1;
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, device) != cudaSuccess) return cpus;
    std::string id(bus);
    for (auto& ch : id) ch = (char)std::tolower((unsigned char)ch);
    FILE* f = std::fopen(("/sys/bus/pci/devices/" + id + "/numa_node").c_str(), "r");
    if (!f) return cpus;
    int node = -1;
    if (std::fscanf(f, "%d", &node) != 1) node = -1;
    std::fclose(f);
    *node_out = node;
    if (node < 0) return cpus;
    f = std::fopen(("/sys/devices/system/node/node" + std::to_string(node) + "/cpulist").c_str(), "r");
    if (!f) return cpus;
    char buf[4096] = {0};
    if (std::fgets(buf, sizeof buf, f)) {
        const char* p = buf;
        while (*p) {                      // "0-15,32-47"
            char* e = nullptr;
            const long a = std::strtol(p, &e, 10);
            if (e == p) break;
            long b = a;
            if (*e == '-') { p = e + 1; b = std::strtol(p, &e, 10); }
            for (long c = a; c <= b; ++c) cpus.push_back((int)c);
            p = (*e == ',') ? e + 1 : e;
            if (*p == '\n') break;
        }
    }
    std::fclose(f);
    return cpus;
}
inline void pin_thread_to(const std::vector<int>& cpus) {
    if (cpus.empty()) return;
    cpu_set_t set;
    CPU_ZERO(&set);
    for (int c : cpus)
        if (c < CPU_SETSIZE) CPU_SET(c, &set);
    pthread_setaffinity_np(pthread_self(), sizeof set, &set);
}

// Simple pool for the host accumulation (row 8, H1); its threads run on the GPU's NUMA node.
class Pool {
   public:
    explicit Pool(int n, std::vector<int> cpus = {}) : n_(n), cpus_(std::move(cpus)) {
        for (int i = 0; i < n_; ++i) th_.emplace_back([this, i] { pin_thread_to(cpus_); run(i); });
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
    std::vector<int> cpus_;
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


}  // namespace zfh

using namespace zfh;

struct zf_ctx {
    int device = 0;
    zf_config cfg{};
    int world = 1, rank = 0;
    ncclComm_t comm = nullptr;
    zf_host_allreduce_fn host_allreduce = nullptr;  // world > 1 without NCCL
    // f4 (iii): norm exchange over peer memory (k_peer.cu; zf_peer_handle / zf_peer_open)
    bool peer = false;
    void* peer_region = nullptr;               // this rank's exchange region (cudaMalloc, IPC-exported)
    void* peer_mapped[ZF_MAX_PEERS] = {};      // the peers' regions opened in this process
    PeerArgs peer_args{};
    unsigned long long peer_epoch = 0;
    int32_t* peer_err_h = nullptr;             // mapped: a peer wait timed out
    void* host_allreduce_user = nullptr;
    float* norms_host = nullptr;
    int gdt = 0, pdt = 0, gsz = 2, psz = 2;
    std::vector<LayerState> L;
    int64_t total_m = 0, max_m = 0, k1_units = 0, k3_units = 0, k3_units_s = 0;
    bool has_empty = false;       // some layer has n = 0 rows on this rank
    int n_stage = 1;              // device compact blocks (ring over steps)
    int n_hstage = 2;             // pinned host staging slots (ring over steps; host_stages)
    // X1 in chunks: the layers' compact blocks sit back to back in one device / host block per
    // staging slot, so a run of consecutive layers is ONE copy gated by ONE counter -- a few
    // dozen copy-stream commands per step instead of three per layer (a deep queue of per-layer
    // commands stalls the issuing thread once the previous step's copies still fill it)
    struct Chunk {
        int32_t first = 0, last = 0;      // layers [first, last)
        int64_t off = 0, bytes = 0;       // byte range in a staging slot
        cudaEvent_t ev[ZF_MAX_HSTAGE] = {};   // per host slot: this chunk's D2H landed
    };
    std::vector<Chunk> chunks;
    // f4 (i): refresh in groups of layers (refresh_group_mb): layers [a, b), their K1 / K3 units
    struct RGroup {
        int32_t a = 0, b = 0;
        int64_t k1_off = 0, k1_units = 0, k3_off = 0, k3_units = 0;
    };
    std::vector<RGroup> rgroups;
    // X1 issue thread (x1_loop): one job per offloaded step
    struct X1Job {
        int64_t t = 0;
        int hs = 0, sb = 0;
        std::vector<uint32_t> targets;   // per-chunk completion counts of this step's K3
    };
    std::thread x1;
    std::mutex x1_mu;
    std::condition_variable x1_cv;
    std::deque<X1Job> x1_jobs;
    int64_t x1_issued = -1;           // last step whose D2H commands are issued
    bool x1_stop = false;
    zf_status x1_status = ZF_OK;
    std::string x1_error;
    cudaEvent_t k3_step_ev[2] = {nullptr, nullptr};   // per device slot: the step's K3 done
    std::mutex prof_mu;               // prof_begin / prof_end from the X1 thread
    void x1_loop();
    zf_status x1_issue(const X1Job& j);
    // wait until step t's D2H commands are issued (and report an X1 thread error)
    zf_status x1_wait_issued(int64_t t) {
        std::unique_lock<std::mutex> lk(x1_mu);
        x1_cv.wait(lk, [&] { return x1_issued >= t || x1_status != ZF_OK; });
        if (x1_status != ZF_OK) return fail(x1_status, "X1 thread: %s", x1_error.c_str());
        return ZF_OK;
    }
    int64_t stage_bytes = 0;      // one staging slot (every layer's compact block)
    void* stage_dev_blk[2] = {nullptr, nullptr};
    void* stage_host_blk[ZF_MAX_HSTAGE] = {};
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
    bool psub_valid = false;      // param_subset: the block holds p[:, idx] (set by a K3 in mode 1)
    bool subset_refresh = false;  // this step's refresh reads retained p values from the old block (mode 3)
    bool split = false;           // regular steps run K3a (compaction + extraction) then K3b (dense AdamW)
    bool lagged = false;          // f4 (ii): refresh norms from the previous step (K1 on lag_stream)
    cudaStream_t lag_stream = nullptr;
    cudaEvent_t lag_in = nullptr, norm_ready = nullptr;
    bool lag_pending = false;     // a lagged K1 was enqueued and not yet waited for
    int32_t lag_delay_us = 0;     // test knob ZF_TEST_LAG_DELAY_US: delay before the lagged K1
    int numa_node = -1;           // NUMA node of the GPU (-1: not reported)
    std::vector<int> numa_cpus;   // its CPUs: host threads and first-touch allocations run there
    int64_t total_rows = 0;       // K3b chunks over all layers
    int64_t last_t = -1;          // regular-schedule index (t - tau) of the last regular step
    int64_t launches = 0;
    // ZF_TRACE_STEP=1: host time spent in each part of zf_step, printed by zf_sync
    bool trace = getenv("ZF_TRACE_STEP") != nullptr;
    double trace_ms[10] = {};
    int64_t trace_n = 0;
    std::chrono::steady_clock::time_point trace_t;
    void tmark(int i) {
        if (!trace) return;
        const auto now = std::chrono::steady_clock::now();
        if (i >= 0) trace_ms[i] += std::chrono::duration<double, std::milli>(now - trace_t).count();
        trace_t = now;
    }
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
    int h1_waiters = 0;           // threads blocked on H1 progress: H1 then processes what it has
    int64_t h1_batches = 0, h1_batched_steps = 0;   // H1 passes and the steps they covered

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
    // f1 host update: upload-done event; cpu_update_async worker (reading R23)
    cudaEvent_t f1_up_ev = nullptr;
    std::thread f1_worker;
    bool f1_pending = false;
    zf_status f1_status = ZF_OK;
    std::string f1_error;
    std::vector<void*> f1_params;
    cudaStream_t last_stream = nullptr;  // stream of the last zf_step
    unsigned long long* k3_prof = nullptr;  // -DZF_K3_PROF builds only
    // f2 Zen-auto (reading R21): K6 tables per current set, device state, decision records
    bool autoz = false;
    AutoLayer* d_auto_tab[2] = {nullptr, nullptr};
    double* auto_sums = nullptr;
    uint32_t* auto_counter = nullptr;
    AutoState* auto_state = nullptr;
    AutoRecord* auto_rec_h = nullptr;   // mapped pinned ring [AUTO_RING]
    AutoRecord* auto_rec_d = nullptr;
    static constexpr int AUTO_RING = 2 * ZF_MAX_HSTAGE;   // > the steps H1 may lag behind zf_step (host_stages)
    cudaEvent_t auto_ev[AUTO_RING] = {};
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
    static constexpr int NPHASE = 8;
    double prof_ms[NPHASE] = {};
    int64_t prof_n[NPHASE] = {};

    ~zf_ctx();
    zf_status prof_begin(int phase, cudaStream_t s, Pending* p) {
        p->phase = phase;
        p->a = p->b = nullptr;
        if (!profiling) return ZF_OK;
        std::lock_guard<std::mutex> lk(prof_mu);
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
        std::lock_guard<std::mutex> lk(prof_mu);
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
    // dst holds `old` (bytes, a multiple of 8): write the changed words of src by patch
    // kernels (k_patch) in stream order -- no copy engine, no ring slot wait
    std::unique_ptr<PatchArgs> patch;
    zf_status upload_diff(void* dst, const void* src, const void* old, size_t bytes, cudaStream_t s) {
        if (bytes % 8 != 0) return upload(dst, src, bytes, s);
        if (!patch) patch.reset(new PatchArgs);
        PatchArgs& a = *patch;
        a.base = static_cast<unsigned long long*>(dst);
        a.n = 0;
        const unsigned long long* x = static_cast<const unsigned long long*>(src);
        const unsigned long long* y = static_cast<const unsigned long long*>(old);
        for (size_t w = 0; w < bytes / 8; ++w) {
            if (x[w] == y[w]) continue;
            a.off[a.n] = (uint32_t)w;
            a.val[a.n] = x[w];
            if (++a.n == ZF_PATCH_N) {
                ZF_CUDA(launch_patch(a, s));
                ++launches;
                a.n = 0;
            }
        }
        if (a.n) {
            ZF_CUDA(launch_patch(a, s));
            ++launches;
        }
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


namespace zfh {
// zf_host.cu
void acc_row_bf16(float* acc, const uint16_t* src, int64_t n, bool first);
void acc_row_f32(float* acc, const float* src, int64_t n, bool first);
// b steps of one window in one pass: acc = (((first ? 0 : acc) + x_0) + x_1) ... + x_{b-1}
void acc_row_multi(float* acc, const void* const* src, int b, int64_t n, bool first, bool bf16);
zf_status f1_refresh(zf_ctx* c, void* const* params, cudaStream_t s);
zf_status f1_window_end(zf_ctx* c, int64_t t, int buf, int64_t len, void* const* params, cudaStream_t s);
zf_status f1_launch(zf_ctx* c, int64_t t, int buf, int64_t len, void* const* params);
zf_status f1_finish(zf_ctx* c, cudaStream_t s);
}  // namespace zfh
