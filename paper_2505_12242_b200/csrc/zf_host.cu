// zf_host.cu -- the host side of the stateful driver: context teardown, the host
// accumulation thread (row a8, H1) and the deferred CPU AdamW of the unselected columns
// (next row f1, reading R18).  See DESIGN.md §5.
#include "zf_host.h"

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
void zfh::acc_row_bf16(float* __restrict__ acc, const uint16_t* __restrict__ src, int64_t n, bool first) {
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
void zfh::acc_row_f32(float* __restrict__ acc, const float* __restrict__ src, int64_t n, bool first) {
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

// ============================================================ f1: deferred CPU AdamW (reading R18)
namespace zfh {

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

}  // namespace zfh
