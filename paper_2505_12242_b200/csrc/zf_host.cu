// zf_host.cu -- the host side of the stateful driver: context teardown, the host
// accumulation thread (row a8, H1) and the deferred CPU AdamW of the unselected columns
// (next row f1, reading R18).  See DESIGN.md §5.
#include "zf_host.h"

zf_ctx::~zf_ctx() {
    if (f1_worker.joinable()) f1_worker.join();
    if (x1.joinable()) {
        {
            std::lock_guard<std::mutex> lk(x1_mu);
            x1_stop = true;
        }
        x1_cv.notify_all();
        x1.join();
    }
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
    for (void* p : peer_mapped)
        if (p) cudaIpcCloseMemHandle(p);
    for (void* p : dev_allocs) cudaFree(p);
    for (void* p : host_pinned) cudaFreeHost(p);
    for (float* p : host_plain) std::free(p);
    for (auto e : k3_step_ev)
        if (e) cudaEventDestroy(e);
    for (auto& ch : chunks)
        for (int i = 0; i < ZF_MAX_HSTAGE; ++i)
            if (ch.ev[i]) cudaEventDestroy(ch.ev[i]);
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
    if (lag_stream) cudaStreamDestroy(lag_stream);
    if (lag_in) cudaEventDestroy(lag_in);
    if (norm_ready) cudaEventDestroy(norm_ready);
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

// X1: issue one step's D2H of the compact blocks -- per chunk of consecutive layers, wait on
// the device until the chunk's K3 units are done (cuStreamWaitValue32 on its completion
// counter; the whole step's K3 without stream memory ops), one copy into host slot hs, one
// event -- then hand the step to H1.
zf_status zf_ctx::x1_issue(const X1Job& j) {
    if (!wait_value) ZF_CUDA(cudaStreamWaitEvent(copy_stream, k3_step_ev[j.sb], 0));
    Pending pe4;
    bool pe4_open = false;
    for (size_t ci = 0; ci < chunks.size(); ++ci) {
        Chunk& ch = chunks[ci];
        if (wait_value) {
            CUresult r = wait_value(reinterpret_cast<CUstream>(copy_stream), reinterpret_cast<CUdeviceptr>(done + ci),
                                    j.targets[ci], CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) {  // stream memory ops unavailable: gate on the whole step
                wait_value = nullptr;
                ZF_CUDA(cudaStreamWaitEvent(copy_stream, k3_step_ev[j.sb], 0));
            }
        }
        if (ch.bytes > 0) {
            if (!pe4_open) {  // phase 4: the step's D2H span, from the first copy's start
                ZF_TRY(prof_begin(4, copy_stream, &pe4));
                pe4_open = true;
            }
            ZF_CUDA(cudaMemcpyAsync(static_cast<unsigned char*>(stage_host_blk[j.hs]) + ch.off,
                                    static_cast<unsigned char*>(stage_dev_blk[j.sb]) + ch.off, (size_t)ch.bytes,
                                    cudaMemcpyDeviceToHost, copy_stream));
        }
        ZF_CUDA(cudaEventRecord(ch.ev[j.hs], copy_stream));
    }
    if (pe4_open) ZF_TRY(prof_end(&pe4, copy_stream));
    ZF_CUDA(cudaEventRecord(d2h_all[j.sb], copy_stream));
    if (cfg.host_accumulate) {
        {
            std::lock_guard<std::mutex> lk(mu);
            jobs.push_back(j.t);
        }
        cv.notify_all();
    }
    return ZF_OK;
}

void zf_ctx::x1_loop() {
    cudaSetDevice(device);
    for (;;) {
        X1Job j;
        {
            std::unique_lock<std::mutex> lk(x1_mu);
            x1_cv.wait(lk, [&] { return x1_stop || !x1_jobs.empty(); });
            if (x1_jobs.empty()) return;
            j = std::move(x1_jobs.front());
            x1_jobs.pop_front();
        }
        const zf_status st = x1_status == ZF_OK ? x1_issue(j) : x1_status;
        {
            std::lock_guard<std::mutex> lk(x1_mu);
            if (st != ZF_OK && x1_status == ZF_OK) {
                x1_status = st;
                x1_error = zf_last_error();
            }
            x1_issued = j.t;
        }
        x1_cv.notify_all();
    }
}

// b staged steps of one window in one pass over the accumulator: the host-DRAM traffic of a
// batch is (first ? 0 : 4) + 2b + 4 bytes per element instead of b x 10 (H1 is host-DRAM
// bound).  The adds stay in step order per element, so the sums are bit-identical to one
// step at a time.  Rows are walked in chunks that stay in L1.
__attribute__((target_clones("avx512f", "avx2", "default")))
void zfh::acc_row_multi(float* __restrict__ acc, const void* const* src, int b, int64_t n, bool first, bool bf16) {
    constexpr int64_t CH = 512;
    float tmp[CH];
    for (int64_t c0 = 0; c0 < n; c0 += CH) {
        const int64_t w = n - c0 < CH ? n - c0 : CH;
        if (first)
            for (int64_t i = 0; i < w; ++i) tmp[i] = 0.0f;
        else
            for (int64_t i = 0; i < w; ++i) tmp[i] = acc[c0 + i];
        for (int j = 0; j < b; ++j) {
            if (bf16) {
                const uint16_t* x = static_cast<const uint16_t*>(src[j]) + c0;
                for (int64_t i = 0; i < w; ++i) {
                    uint32_t u = (uint32_t)x[i] << 16;
                    float f;
                    std::memcpy(&f, &u, 4);
                    tmp[i] = tmp[i] + f;
                }
            } else {
                const float* x = static_cast<const float*>(src[j]) + c0;
                for (int64_t i = 0; i < w; ++i) tmp[i] = tmp[i] + x[i];
            }
        }
        for (int64_t i = 0; i < w; ++i) acc[c0 + i] = tmp[i];
    }
}

// H1: accumulate the staged compact blocks into the window's fp32 buffer as their D2H copies
// complete (DESIGN.md §2 O8).  Steps are taken in batches: every queued
// step of the current window, up to its last step.  A batch that does not reach the window's
// end waits for more steps while the producer can still stage them (free host slots) and
// nobody waits on H1 (zf_step on a slot, zf_sync, f1) -- then it runs with what it has.
void zf_ctx::h1_loop() {
    cudaSetDevice(device);
    const int S = cfg.accum_interval;
    std::vector<int64_t> batch;
    std::vector<char> ends;
    for (;;) {
        batch.clear();
        ends.clear();
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return stopping || !jobs.empty(); });
            if (jobs.empty()) return;
        }
        // grow the batch: queued steps of the current window, stopping after a window end
        for (;;) {
            std::vector<int64_t> q;
            {
                std::lock_guard<std::mutex> lk(mu);
                q.assign(jobs.begin(), jobs.end());
            }
            for (size_t i = batch.size(); i < q.size(); ++i) {
                const int64_t t = q[i];
                bool end = (t + 1) % S == 0;
                if (autoz) {
                    // the window decision of step t: K6's record (Zen-auto, reading R21)
                    const int slot = (int)(t % AUTO_RING);
                    cudaEventSynchronize(auto_ev[slot]);
                    end = auto_rec_h[slot].end != 0;
                }
                batch.push_back(t);
                ends.push_back(end ? 1 : 0);
                if (end || (int)batch.size() >= n_hstage) break;
            }
            if (ends.back() || (int)batch.size() >= n_hstage || n_hstage <= 2) break;
            // more steps of this window can still be staged: wait for one, unless someone waits on us
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return stopping || h1_waiters > 0 || jobs.size() > batch.size(); });
            if (jobs.size() <= batch.size()) break;   // stopping or a waiter: run what we have
        }
        const int b = (int)batch.size();
        const int a = (int)(h1_win % 2);
        const bool first = h1_first;
        const bool bf = gdt == ZF_BF16;
        for (auto& l : L) {
            const void* srcs[ZF_MAX_HSTAGE];
            for (int j = 0; j < b; ++j) {
                const int hs = (int)(batch[j] % n_hstage);
                cudaEventSynchronize(chunks[l.chunk].ev[hs]);
                srcs[j] = l.stage_host[hs];
            }
            const int64_t mk = l.mk, ld = l.mk_pad;
            float* acc = l.acc[a];
            pool->parallel_for(l.d.n, [&](int64_t rb, int64_t re) {
                const void* rs[ZF_MAX_HSTAGE];
                for (int64_t r = rb; r < re; ++r) {
                    if (b == 1) {
                        if (bf) acc_row_bf16(acc + r * mk, static_cast<const uint16_t*>(srcs[0]) + r * ld, mk, first);
                        else acc_row_f32(acc + r * mk, static_cast<const float*>(srcs[0]) + r * ld, mk, first);
                    } else {
                        for (int j = 0; j < b; ++j)
                            rs[j] = static_cast<const unsigned char*>(srcs[j]) + r * ld * (bf ? 2 : 4);
                        acc_row_multi(acc + r * mk, rs, b, mk, first, bf);
                    }
                }
            });
        }
        const bool end = ends.back() != 0;
        {
            std::lock_guard<std::mutex> lk(mu);
            for (int j = 0; j < b; ++j) {
                double rA = NAN, ri = NAN, ru = NAN;
                if (autoz) {
                    const volatile AutoRecord* r = auto_rec_h + (int)(batch[j] % AUTO_RING);
                    rA = r->A;
                    ri = r->imp;
                    ru = r->unimp;
                }
                log_t.push_back(batch[j] + tau);
                log_end.push_back(ends[j]);
                log_A.push_back(rA);
                log_i.push_back(ri);
                log_u.push_back(ru);
                jobs.pop_front();
            }
            h1_last_buf = a;
            if (end) {
                h1_sealed_buf = a;
                ++h1_win;
            }
            h1_first = end;
            h1_done = batch.back();
            h1_batches += 1;
            h1_batched_steps += b;
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
    }
    ZF_CUDA(cudaStreamSynchronize(s));
    // new unselected lists, the retained columns' old positions, and the entering columns,
    // whose current parameter values are gathered on the device and read back (K5')
    std::vector<std::vector<int32_t>> unew(nl), src(nl), ent(nl);
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        const int64_t m = l.d.m, mk = l.mk;
        std::vector<char> now_cpu(m, 1);
        for (int32_t col : nidx[i]) now_cpu[col] = 0;
        unew[i].reserve(mk);
        for (int64_t col = 0; col < m; ++col)
            if (now_cpu[col]) unew[i].push_back((int32_t)col);
        // src[u] = position of column unew[u] in the old unselected list (retained), or
        // -(1 + e) for the e-th entering column (was selected, or the first refresh)
        const std::vector<int32_t>& uold = l.unsel_host;
        src[i].assign(mk, 0);
        for (size_t u = 0, v = 0; u < unew[i].size(); ++u) {
            while (v < uold.size() && uold[v] < unew[i][u]) ++v;
            if (v < uold.size() && uold[v] == unew[i][u]) {
                src[i][u] = (int32_t)v;
            } else {
                src[i][u] = -1 - (int32_t)ent[i].size();
                ent[i].push_back(unew[i][u]);
            }
        }
        const int64_t ne = (int64_t)ent[i].size();
        if (ne > 0 && l.d.n > 0) {
            // ordered on s (a caller's non-blocking stream too); ent[i] outlives the sync below
            ZF_CUDA(cudaMemcpyAsync(l.unsel_dev, ent[i].data(), ne * sizeof(int32_t), cudaMemcpyHostToDevice, s));
            ZF_CUDA(launch_gather_columns(params[i], c->pdt, l.d.ld_param, l.d.n, ne, l.unsel_dev, l.p_up_dev, s));
            c->launches++;
            ZF_CUDA(cudaMemcpyAsync(l.p_mirror, l.p_up_dev, (size_t)l.d.n * ne * c->psz, cudaMemcpyDeviceToHost, s));
            ZF_CUDA(cudaStreamSynchronize(s));  // unsel_dev / p_up_dev are reused by the next layer
        }
    }
    for (int i = 0; i < nl; ++i) {
        LayerState& l = c->L[i];
        const int64_t n = l.d.n, mk = l.mk, ne = (int64_t)ent[i].size();
        const std::vector<int32_t>& sr = src[i];
        const int pdt = c->pdt;
        // runs of consecutive retained positions (u0, v0, len) move with memmove; entering
        // positions are filled from the gathered parameter values
        struct Run { int64_t u0, v0, len; };
        std::vector<Run> runs;
        std::vector<int64_t> enter_pos;
        for (int64_t u = 0; u < mk; ++u) {
            const int32_t v = sr[u];
            if (v < 0) {
                enter_pos.push_back(u);
            } else if (!runs.empty() && runs.back().u0 + runs.back().len == u && runs.back().v0 + runs.back().len == v) {
                ++runs.back().len;
            } else {
                runs.push_back({u, (int64_t)v, 1});
            }
        }
        // retained columns only move toward lower positions or stay (both lists ascending,
        // the new one drops old columns before adding), so an in-place forward pass is safe
        // for runs with u0 <= v0; runs moving up are copied from a row snapshot
        bool all_down = true;
        for (const Run& q : runs) all_down = all_down && q.u0 <= q.v0;
        if (mk > 0)
            c->pool->parallel_for(n, [&](int64_t b, int64_t e) {
                std::vector<float> tmp(all_down ? 0 : 3 * (size_t)mk);
                for (int64_t r = b; r < e; ++r) {
                    float* A3[3] = {l.master + r * mk, l.mh + r * mk, l.vh + r * mk};
                    if (all_down) {
                        for (const Run& q : runs)
                            for (float* A : A3) std::memmove(A + q.u0, A + q.v0, q.len * sizeof(float));
                    } else {
                        for (int a = 0; a < 3; ++a) std::memcpy(tmp.data() + a * mk, A3[a], mk * sizeof(float));
                        for (const Run& q : runs)
                            for (int a = 0; a < 3; ++a)
                                std::memcpy(A3[a] + q.u0, tmp.data() + a * mk + q.v0, q.len * sizeof(float));
                    }
                    for (int64_t u : enter_pos) {  // entering: the parameter's value, zero moments
                        A3[0][u] = host_widen(l.p_mirror, pdt, (size_t)(r * ne + (-1 - sr[u])));
                        A3[1][u] = 0.0f;
                        A3[2][u] = 0.0f;
                    }
                }
            });
        std::vector<int32_t> thn(mk, 0);
        for (int64_t u = 0; u < mk; ++u)
            if (sr[u] >= 0) thn[u] = l.th[sr[u]];
        l.th.swap(thn);
        l.idx_host = nidx[i];
        l.unsel_host.swap(unew[i]);
        if (!l.unsel_host.empty())
            ZF_CUDA(cudaMemcpyAsync(l.unsel_dev, l.unsel_host.data(), l.unsel_host.size() * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, s));  // ordered before the K5 scatter on s
    }
    return ZF_OK;
}

// One row of the window update (O6 op order, every operation one IEEE fp32 op; the host
// build uses -ffp-contract=off, so the vectorised clones keep the rounding of the scalar
// code: vdivps / vsqrtps are correctly rounded).
template <int WD, bool BF>
static inline void f1_row_impl(float* __restrict__ M, float* __restrict__ Mh, float* __restrict__ Vh,
                               const float* __restrict__ acc, const float* __restrict__ ss,
                               const float* __restrict__ bc2s, void* __restrict__ out, int64_t mk, float Sf,
                               float b1, float b2, float omb1, float omb2, float eps, float wd_f, float decay) {
    for (int64_t u = 0; u < mk; ++u) {
        float g = acc[u] / Sf;
        float p = M[u];
        float mm = Mh[u], vv = Vh[u];
        if (WD == 1) p = p * decay;
        if (WD == 2) {
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
        M[u] = p;
        Mh[u] = mm;
        Vh[u] = vv;
        if (BF) {
            uint32_t x;
            std::memcpy(&x, &p, 4);
            const uint32_t rne = (x + 0x7fffu + ((x >> 16) & 1u)) >> 16;
            const uint32_t nan = (x >> 16) | 0x40u;
            static_cast<uint16_t*>(out)[u] = (uint16_t)(((x & 0x7fffffffu) > 0x7f800000u) ? nan : rne);
        } else {
            static_cast<float*>(out)[u] = p;
        }
    }
}

__attribute__((target_clones("avx512f", "avx2", "default")))
void f1_row(int wd_mode, bool bf, float* M, float* Mh, float* Vh, const float* acc, const float* ss,
            const float* bc2s, void* out, int64_t mk, float Sf, float b1, float b2, float omb1, float omb2, float eps,
            float wd_f, float decay) {
#define ZF_F1_ROW(W, B) f1_row_impl<W, B>(M, Mh, Vh, acc, ss, bc2s, out, mk, Sf, b1, b2, omb1, omb2, eps, wd_f, decay)
    if (bf) {
        if (wd_mode == 0) ZF_F1_ROW(0, true);
        else if (wd_mode == 1) ZF_F1_ROW(1, true);
        else ZF_F1_ROW(2, true);
    } else {
        if (wd_mode == 0) ZF_F1_ROW(0, false);
        else if (wd_mode == 1) ZF_F1_ROW(1, false);
        else ZF_F1_ROW(2, false);
    }
#undef ZF_F1_ROW
}

// The host half: one AdamW step of every unselected column from the sealed window `buf` of
// `len` steps (waits for that window's accumulation first); results in the pinned p_up
// blocks and the host master/moments.  Runs on the caller's thread (sync) or on the f1
// worker thread (cpu_update_async, reading R23).
zf_status f1_compute(zf_ctx* c, int64_t t, int buf, int64_t len, double lr) {
    if (c->f1_up_ev) ZF_CUDA(cudaEventSynchronize(c->f1_up_ev));  // the previous upload read p_up
    if (c->devacc) {
        ZF_CUDA(cudaEventSynchronize(c->acc_d2h_ev[buf]));  // the sealed window's host copy
    } else {
        std::unique_lock<std::mutex> lk(c->mu);
        ++c->h1_waiters;
        c->cv.notify_all();
        c->cv.wait(lk, [&] { return c->h1_done >= t; });
        --c->h1_waiters;
    }
    const zf_adam_params& hp = c->cfg.adam;
    const double b1d = hp.beta1, b2d = hp.beta2;
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
            const double tt = (double)(l.th[u] + 1);
            ss[u] = (float)(lr / (1.0 - std::pow(b1d, tt)));
            bc2s[u] = (float)std::sqrt(1.0 - std::pow(b2d, tt));
        }
        const bool bf = c->pdt == ZF_BF16;
        c->pool->parallel_for(n, [&](int64_t b, int64_t e) {
            for (int64_t r = b; r < e; ++r)
                f1_row(wd_mode, bf, l.master + r * mk, l.mh + r * mk, l.vh + r * mk, acc + r * mk, ss.data(),
                       bc2s.data(), static_cast<unsigned char*>(l.p_up) + (size_t)r * mk * c->psz, mk, Sf, b1, b2, omb1,
                       omb2, eps, wd_f, decay);
        });
        for (int64_t u = 0; u < mk; ++u) l.th[u] += 1;
    }
    return ZF_OK;
}

// The device half: upload every layer's p_up block and scatter it into the parameter's
// unselected columns (K5), on stream s; f1_up_ev marks when p_up may be rewritten.
zf_status f1_apply(zf_ctx* c, void* const* params, cudaStream_t s) {
    for (size_t i = 0; i < c->L.size(); ++i) {
        LayerState& l = c->L[i];
        const int64_t n = l.d.n, mk = l.mk;
        if (mk == 0 || n == 0) continue;
        ZF_CUDA(cudaMemcpyAsync(l.p_up_dev, l.p_up, (size_t)n * mk * c->psz, cudaMemcpyHostToDevice, s));
        ZF_CUDA(launch_scatter_unselected(params[i], c->pdt, l.d.ld_param, n, mk, l.unsel_dev, l.p_up_dev, s));
        c->launches++;
    }
    if (!c->f1_up_ev) ZF_CUDA(cudaEventCreateWithFlags(&c->f1_up_ev, cudaEventDisableTiming));
    ZF_CUDA(cudaEventRecord(c->f1_up_ev, s));
    return ZF_OK;
}

// Synchronous window end (reading R18): compute, apply, and wait.
zf_status f1_window_end(zf_ctx* c, int64_t t, int buf, int64_t len, void* const* params, cudaStream_t s) {
    ZF_TRY(f1_compute(c, t, buf, len, c->lr_cur));
    ZF_TRY(f1_apply(c, params, s));
    ZF_CUDA(cudaStreamSynchronize(s));
    return ZF_OK;
}

// cpu_update_async (reading R23): start the host half on the worker thread and return; the
// update is applied by f1_finish at the start of the next zf_step (or in zf_sync).
zf_status f1_launch(zf_ctx* c, int64_t t, int buf, int64_t len, void* const* params) {
    c->f1_params.assign(params, params + c->L.size());
    c->f1_status = ZF_OK;
    const double lr = c->lr_cur;
    c->f1_worker = std::thread([c, t, buf, len, lr] {
        cudaSetDevice(c->device);
        const zf_status st = f1_compute(c, t, buf, len, lr);
        c->f1_status = st;
        if (st != ZF_OK) c->f1_error = g_last_error;
    });
    c->f1_pending = true;
    return ZF_OK;
}

zf_status f1_finish(zf_ctx* c, cudaStream_t s) {
    if (!c->f1_pending) return ZF_OK;
    c->f1_worker.join();
    c->f1_pending = false;
    if (c->f1_status != ZF_OK) return fail(c->f1_status, "deferred CPU update: %s", c->f1_error.c_str());
    return f1_apply(c, c->f1_params.data(), s);
}

}  // namespace zfh
