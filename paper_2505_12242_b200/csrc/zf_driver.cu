// zf_driver.cu -- the stateful driver of the C-ABI (include/zf.h): zf_create (per-layer
// state in HBM, launch tables, NCCL communicator, offload buffers), zf_step (K1 -> norm
// all-reduce -> K2 -> K3 -> K7/K6, per-layer D2H, window bookkeeping, f1), zf_sync and
// the views of library-owned state.  See DESIGN.md §5-§6.
#include "zf_host.h"

zf_status peer_allreduce(zf_ctx* c, cudaStream_t s);   // f4 (iii), below

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
            t.done = c->cfg.offload ? c->done + l.chunk : nullptr;
            const K3Geom& gg = refresh ? l.geo : l.geo_s;
            t.seg_cols = gg.seg_cols;
            t.nseg = gg.nseg;
            t.R = gg.R;
            t.units = gg.units;
            t.unit_begin = refresh ? l.unit_begin : l.unit_begin_s;
            t.mv_tma = gg.mv_ok ? 1 : 0;
            {   // subset blocks ping-pong with the moment sets (a refresh writes the other one)
                void* blk[2] = {l.psub, l.psub2 ? l.psub2 : l.psub};
                t.psub = blk[nw];
                t.psub_in = blk[cur];
            }
            t.psub_mode = l.psub ? 1 : 0;   // set per step (refresh_pointer_tables)
            t.sbv = l.sbv;
            t.gsel = l.gsel;
            t.adam_row_begin = l.row_begin;
            if (c->split) t.mv_tma = 0;     // K3a never stages moments
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
            t.sbv = l.sbv;
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
    if (cfg->cpu_update_async && !cfg->cpu_update) return fail(ZF_EINVAL, "cpu_update_async requires cpu_update");
    if (cfg->cpu_update && cfg->refresh_interval % cfg->accum_interval != 0)
        return fail(ZF_EINVAL, "cpu_update requires refresh_interval to be a multiple of accum_interval");
    if (cfg->warmup_steps < 0) return fail(ZF_EINVAL, "warmup_steps must be >= 0");
    if (!(cfg->auto_gamma >= 0.0f) || !std::isfinite(cfg->auto_gamma))
        return fail(ZF_EINVAL, "auto_gamma must be finite and >= 0");
    if (cfg->auto_gamma > 0.0f && !cfg->host_accumulate) return fail(ZF_EINVAL, "auto_gamma requires host_accumulate");
    if (cfg->lagged_selection && cfg->auto_gamma > 0.0f)
        return fail(ZF_EINVAL, "lagged_selection and auto_gamma are exclusive (Zen-auto reads every step's norms)");
    if (cfg->device_accumulate && !cfg->host_accumulate)
        return fail(ZF_EINVAL, "device_accumulate requires host_accumulate (it moves that accumulation onto the GPU)");
    ZF_TRY(check_hp(&cfg->adam));
    if (cfg->refresh_group_mb < 0) return fail(ZF_EINVAL, "refresh_group_mb must be >= 0");
    if (cfg->refresh_group_mb > 0 && (world > 1 || cfg->auto_gamma > 0.0f || cfg->lagged_selection))
        return fail(ZF_EINVAL, "refresh_group_mb: world 1 only, not with auto_gamma or lagged_selection");
    if (cfg->host_stages < 0 || cfg->host_stages > ZF_MAX_HSTAGE)
        return fail(ZF_EINVAL, "host_stages must be in [0, %d]", ZF_MAX_HSTAGE);
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
    c->n_hstage = cfg->host_stages > 0 ? cfg->host_stages : 2;
    c->lr_cur = cfg->adam.lr;
    c->tau = cfg->warmup_steps;
    c->grid = update_grid(c->gdt, c->pdt);
    // ZF_K3_SPLIT: the split update (K3a compaction + extraction, K3b dense AdamW, k_adam.cu)
    // instead of AdamW inside K3's unit pipeline.  Measured slower on Llama-2-7B k = 10% (K3a
    // 4.65 + K3b 5.7 ms vs 9.4 ms fused): K3b's scattered stores of the changed p values miss
    // L2 and each waits on a partial-sector fill, 3 ms of its time at lr 1e-5 (3.3 ms without
    // them), where the fused kernel's stores hit the p rows it pulled into L2
    c->split = getenv("ZF_K3_SPLIT") != nullptr;
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
        l.row_begin = c->total_rows;   // K3b: the layer's first chunk of adam_dense_vec() elements
        c->total_rows += (l.d.n * l.k + adam_dense_vec() - 1) / adam_dense_vec();
        if (c->split) {
            // split update: K3a stages the G tile (and on refresh steps the p tile, to rebuild the
            // parameter subset); the moments never enter its stages (K3b streams them)
            l.geo = k3_geom(l.d.n, l.d.m, l.k, c->gsz, c->psz, k3_p_dense(l.d.m, l.k, c->psz), false);
            l.geo_s = cfg->param_subset ? k3_geom(l.d.n, l.d.m, l.k, c->gsz, c->psz, false, false) : l.geo;
        } else {
            l.geo = k3_geom(l.d.n, l.d.m, l.k, c->gsz, c->psz, k3_p_dense(l.d.m, l.k, c->psz));
            // steady steps with param_subset stage the dense subset slab instead of a p tile, so
            // their units hold more rows (more bytes in flight per stage)
            l.geo_s = cfg->param_subset ? k3_geom(l.d.n, l.d.m, l.k, c->gsz, c->psz, false, true, true) : l.geo;
        }
        l.unit_begin = c->k3_units;
        c->k3_units += l.geo.units;
        l.unit_begin_s = c->k3_units_s;
        c->k3_units_s += l.geo_s.units;
        if (c->tau > 0) {  // warm-up geometry: k = m
            l.geo_w = k3_geom(l.d.n, l.d.m, l.d.m, c->gsz, c->psz, true);
            l.unit_begin_w = c->k3_units_w;
            c->k3_units_w += l.geo_w.units;
        }
    }
    if (c->k3_units_w > 0x3fffffffLL) return bail(fail(ZF_EINVAL, "model too large"));
    if (c->k1_units > 0x7fffffffLL || c->k3_units > 0x3fffffffLL || c->k3_units_s > 0x3fffffffLL)
        return bail(fail(ZF_EINVAL, "model too large"));
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
        // per-slot {ss, bc2s} of the next K3 (prologue), padded for K3's bulk copies
        ZF_CTRY(c->dalloc(&l.sbv, ((c->tau > 0 ? l.d.m : k) + 16) * sizeof(float2)));
        // padded: K3 stages the subset with 16-byte-granular bulk copies.  The split update keeps
        // p's selected values in this dense block even without param_subset (rebuilt every step)
        if ((cfg->param_subset || c->split) && n > 0) ZF_CTRY(c->dalloc(&l.psub, ((size_t)n * k + 16) * c->psz, false));
#if ZF_REFRESH_SUBSET
        // refresh steps read the retained columns' p values from the previous block (mode 3)
        if (cfg->param_subset && !c->split && n > 0) ZF_CTRY(c->dalloc(&l.psub2, ((size_t)n * k + 16) * c->psz, false));
#endif
        if (c->split && n > 0) ZF_CTRY(c->dalloc(&l.gsel, ((size_t)n * k + 16) * c->gsz, false));
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
        l.stage_off = c->stage_bytes;
        c->stage_bytes += ((int64_t)n * l.mk_pad * c->gsz + 255) / 256 * 256;
    }
    if (cfg->refresh_group_mb > 0) {
        // f4 (i): consecutive layers whose gradients fit the budget refresh together
        const int64_t budget = (int64_t)cfg->refresh_group_mb << 20;
        zf_ctx::RGroup g;
        int64_t bytes = 0;
        const int nl_ = (int)c->L.size();
        for (int i = 0; i < nl_; ++i) {
            const LayerState& l = c->L[i];
            const int64_t lb = l.d.n * l.d.m * c->gsz;
            if (i > g.a && bytes + lb > budget) {
                g.b = i;
                c->rgroups.push_back(g);
                g = zf_ctx::RGroup{};
                g.a = i;
                bytes = 0;
            }
            bytes += lb;
        }
        g.b = nl_;
        c->rgroups.push_back(g);
        for (auto& gg : c->rgroups) {
            gg.k1_off = c->L[gg.a].norm_unit_begin;
            gg.k1_units = (gg.b < nl_ ? c->L[gg.b].norm_unit_begin : c->k1_units) - gg.k1_off;
            gg.k3_off = c->L[gg.a].unit_begin;
            gg.k3_units = (gg.b < nl_ ? c->L[gg.b].unit_begin : c->k3_units) - gg.k3_off;
        }
    }
    // the compact blocks of every layer back to back per staging slot; X1 copies chunks of
    // consecutive layers (~512 MB) with one command each
    for (int s = 0; s < c->n_stage; ++s) {
        ZF_CTRY(c->dalloc(&c->stage_dev_blk[s], std::max<int64_t>(c->stage_bytes, 256), false));
        for (auto& l : c->L) l.stage_dev[s] = static_cast<unsigned char*>(c->stage_dev_blk[s]) + l.stage_off;
    }
    {
        // ZF_X1_CHUNK_KB: chunk size override (tests use tiny chunks to exercise many counters)
        const int64_t chunk_target = getenv("ZF_X1_CHUNK_KB") ? atoll(getenv("ZF_X1_CHUNK_KB")) << 10 : 512ll << 20;
        zf_ctx::Chunk ch;
        for (int i = 0; i < (int)c->L.size(); ++i) {
            LayerState& l = c->L[i];
            if (ch.last == ch.first) ch.off = l.stage_off;
            l.chunk = (int32_t)c->chunks.size();
            ch.last = i + 1;
            ch.bytes = l.stage_off + ((int64_t)l.d.n * l.mk_pad * c->gsz + 255) / 256 * 256 - ch.off;
            if (ch.bytes >= chunk_target || i + 1 == (int)c->L.size()) {
                c->chunks.push_back(ch);
                ch = zf_ctx::Chunk{};
                ch.first = ch.last = i + 1;
            }
        }
    }
    {
        int32_t* h = nullptr;
        ZF_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
        c->host_pinned.push_back(h);
        *h = 0;
        c->nonfinite_h = h;
        ZF_CUDA(cudaHostGetDevicePointer(&c->nonfinite_d, h, 0));
        c->peer_err_h = h + 4;   // f4 (iii): peer-exchange timeout flag, same mapped block
        *c->peer_err_h = 0;
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
    c->lagged = cfg->lagged_selection != 0;
    if (c->lagged) {
        c->lag_delay_us = getenv("ZF_TEST_LAG_DELAY_US") ? atoi(getenv("ZF_TEST_LAG_DELAY_US")) : 0;
        ZF_CUDA(cudaStreamCreateWithFlags(&c->lag_stream, cudaStreamNonBlocking));
        ZF_CUDA(cudaEventCreateWithFlags(&c->lag_in, cudaEventDisableTiming));
        ZF_CUDA(cudaEventCreateWithFlags(&c->norm_ready, cudaEventDisableTiming));
    }
    for (auto& l : c->L) {
        int32_t* v = nullptr;
        ZF_CTRY(c->dalloc(&v, (c->tau > 0 ? l.d.m : l.k) * sizeof(int32_t)));
        c->steps_view.push_back(v);
    }
    ZF_CUDA(cudaEventCreateWithFlags(&c->step_done, cudaEventDisableTiming));
    ZF_CUDA(cudaEventCreateWithFlags(&c->k3_done, cudaEventDisableTiming));
    // host buffers on the GPU's NUMA node: this thread runs there while it allocates and
    // first-touches them (pinned staging, accumulators, f1 state), then its affinity returns
    c->numa_cpus = gpu_numa_cpus(device, &c->numa_node);
    cpu_set_t saved;
    const bool pinned_here = !c->numa_cpus.empty() &&
                             pthread_getaffinity_np(pthread_self(), sizeof saved, &saved) == 0;
    if (pinned_here) pin_thread_to(c->numa_cpus);
    struct Restore {
        bool on;
        cpu_set_t set;
        ~Restore() {
            if (on) pthread_setaffinity_np(pthread_self(), sizeof set, &set);
        }
    } restore{pinned_here, saved};
    // ---- offload: copy stream, pinned host staging, per-layer events, host accumulators
    if (cfg->offload) {
        ZF_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        for (int s = 0; s < 2; ++s) ZF_CUDA(cudaEventCreateWithFlags(&c->d2h_all[s], cudaEventDisableTiming));
        for (int s = 0; s < (c->devacc ? 0 : c->n_hstage); ++s) {  // per-step compact D2H (not with K7)
            void* h = nullptr;
            ZF_CUDA(cudaHostAlloc(&h, std::max<size_t>((size_t)c->stage_bytes, 64), cudaHostAllocDefault));
            c->host_pinned.push_back(h);
            c->stage_host_blk[s] = h;
            for (auto& l : c->L) l.stage_host[s] = static_cast<unsigned char*>(h) + l.stage_off;
            for (auto& ch : c->chunks)
                ZF_CUDA(cudaEventCreateWithFlags(&ch.ev[s], cudaEventDisableTiming | cudaEventBlockingSync));
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
                    const size_t nm = (size_t)l.d.n * l.d.m, nmk = std::max<size_t>((size_t)l.d.n * l.mk, 16);
                    for (float** pp : {&l.master, &l.mh, &l.vh}) {
                        float* q = static_cast<float*>(std::aligned_alloc(64, (nmk * sizeof(float) + 63) / 64 * 64));
                        if (!q) return bail(fail(ZF_ENOMEM, "host optimizer state allocation failed"));
                        std::memset(q, 0, nmk * sizeof(float));
                        c->host_plain.push_back(q);
                        *pp = q;
                    }
                    l.th.assign(l.mk, 0);
                    (void)nm;
                    ZF_CUDA(cudaHostAlloc(&l.p_mirror, std::max<size_t>(nmk * c->psz, 64), cudaHostAllocDefault));
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
            // H1 / f1 pool: the GPU node's cores (all hardware threads when no node is reported)
            const int avail = c->numa_cpus.empty() ? (int)std::max(1u, std::thread::hardware_concurrency())
                                                   : (int)c->numa_cpus.size();
            int nt = cfg->host_threads > 0 ? cfg->host_threads : std::min(avail, 64);
            c->pool = new Pool(nt, c->numa_cpus);
            if (!c->devacc) c->h1 = std::thread([c] { pin_thread_to(c->numa_cpus); c->h1_loop(); });
        }
        if (!c->devacc) {
            for (auto& e : c->k3_step_ev) ZF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->x1 = std::thread([c] { pin_thread_to(c->numa_cpus); c->x1_loop(); });
        }
    }
    // ---- NCCL (collective across ranks), or a pinned host buffer for the host all-reduce
    if (world > 1 && !nccl_id128) {
        ZF_CUDA(cudaHostAlloc(&c->norms_host, std::max<size_t>(c->total_m * sizeof(float), 64), cudaHostAllocDefault));
        c->host_pinned.push_back(c->norms_host);
    }
    if (nccl_id128) {   // (world 1 with an id: a one-rank communicator, the NCCL path on one GPU)
        ncclUniqueId id;
        std::memcpy(&id, nccl_id128, sizeof id);
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) return bail(fail(ZF_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
    }
    ZF_CUDA(cudaDeviceSynchronize());
    {
        // leave room for kernel launches (local memory, launch resources): a context that
        // fills HBM to the brim would fail at its first zf_step instead of here
        size_t fr = 0, tot = 0;
        ZF_CUDA(cudaMemGetInfo(&fr, &tot));
        if (fr < ((size_t)256 << 20))
            return bail(fail(ZF_ENOMEM, "device memory nearly exhausted after allocating the context (%zu MB free)",
                             fr >> 20));
    }
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
            ZF_TRY(c->upload_diff(c->d_norm_tab, c->h_norm_tab.data(), c->up_norm_tab.data(), nl * sizeof(NormLayer), s));
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
        h[i].p_dense = k3_p_dense(c->L[i].d.m, h[i].k, c->psz) ? 1 : 0;
        h[i].p_tma = k3_tma_ok(params[i], c->L[i].d.ld_param, c->L[i].d.m, c->psz) && h[i].p_dense;
        if (h[i].psub && variant != -1) {
            // param_subset: a steady step with a valid block reads p's selected values from it
            // (no p tile: steady units are sized without one); refreshes (and the step after
            // zf_params_changed, which reads p from global memory) rebuild it from p.  The split
            // update without param_subset rebuilds it every step (steady units keep the p tile)
            const bool steady = variant >= 0 && ((variant >> 1) & 1) == 0;
            h[i].psub_mode = steady && c->psub_valid && c->cfg.param_subset ? 2 : 1;
            if (steady && c->cfg.param_subset) h[i].p_tma = 0;
            if (variant >= 0 && !steady && c->subset_refresh) {
                h[i].psub_mode = 3;
                h[i].p_tma = 0;
            }
        }
        if (variant >= 0 && ((variant >> 1) & 1) == 1 && !c->split) {
            // a refresh: the steady unit shapes (no p tile) when it reads the retained columns'
            // values from the previous subset block (mode 3), else its own (p tile) -- for every
            // layer, rows-less ones included, so the unit ranges stay one consistent sequence
            const LayerState& l = c->L[i];
            const K3Geom& gg = c->subset_refresh ? l.geo_s : l.geo;
            h[i].seg_cols = gg.seg_cols;
            h[i].nseg = gg.nseg;
            h[i].R = gg.R;
            h[i].units = gg.units;
            h[i].unit_begin = c->subset_refresh ? l.unit_begin_s : l.unit_begin;
            h[i].mv_tma = gg.mv_ok ? 1 : 0;
        }
    }
    if (std::memcmp(h.data(), up.data(), nl * sizeof(UpdLayer)) != 0) {
        ZF_TRY(c->upload_diff(d, h.data(), up.data(), nl * sizeof(UpdLayer), s));
        up = h;
    }
    return ZF_OK;
}

}  // namespace

namespace {

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
    ZF_CUDA(launch_slot_consts(c->d_upd_w, nl, c->max_m, prm.step_delta, c->adam, s));
    c->launches++;
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
    if (c->world > 1 && !c->comm && !c->host_allreduce && !c->peer)
        return fail(ZF_ESTATE, "world > 1 needs an NCCL id at zf_create, zf_peer_open or zf_set_host_allreduce");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    c->last_stream = s;
    c->tmark(-1);
    c->trace_n++;
    ZF_CUDA(cudaSetDevice(c->device));
    // R23: the previous window's CPU update (computed while the caller ran its next forward /
    // backward) lands before this step touches any parameter
    ZF_TRY(f1_finish(c, s));
    c->tmark(0);
    if (t0 < tau) return warmup_step(c, t0, grads, params, s);
    // the regular schedule (refreshes, windows, offload stages) counts from step tau (R20)
    const int64_t t = t0 - tau;
    const bool refresh = (t % N) == 0;
    const int sb = (int)(t % c->n_stage);
    // the first refresh after a warm-up remaps from the [n, m] warm-up set (tables -2 - sb)
    const bool from_warmup = !c->have_sel && tau > 0;
    const int variant = from_warmup ? -2 - (sb & 1) : c->cur * 4 + (refresh ? 2 : 0) + (sb & 1);
    ZF_TRY(upload_ss(c, s));
    // f4 (ii), reading R24: a lagged refresh (not the first) takes the norms K1 computed from the
    // previous step's gradient on the side stream; a pre-refresh step launches that K1
    const bool lag_refresh = c->lagged && refresh && c->have_sel;
    const bool lag_pre = c->lagged && (t + 1) % N == 0;
    const bool norms_now = (refresh && !lag_refresh) || c->autoz;  // Zen-auto reads every step's norms (R21)
    // f4 (i): this refresh runs K1 -> K2 -> K3 per group of layers (G re-read from L2)
    const bool grouped = refresh && !c->rgroups.empty() && c->have_sel && !c->split;
    // a refresh with a valid subset block builds the new one from it (mode 3, steady unit shapes)
    c->subset_refresh = ZF_REFRESH_SUBSET && refresh && !from_warmup && !grouped && c->have_sel && c->psub_valid &&
                        c->cfg.param_subset && !c->split;
    ZF_TRY(refresh_pointer_tables(c, variant, norms_now || lag_pre, grads, params, s));
    c->tmark(1);

    if (c->cfg.offload) {
        // (K3 counts per-layer completions only when offloading; see build_tables)
        // the device staging buffer sb is free once the D2H copies issued two steps ago finished
        if (c->d2h_issued[sb]) {
            if (!c->devacc) ZF_TRY(c->x1_wait_issued(t - c->n_stage));   // d2h_all[sb] of step t - 2 recorded
            ZF_CUDA(cudaStreamWaitEvent(s, c->d2h_all[sb], 0));
        }
        if (c->cfg.host_accumulate && !c->devacc) {
            // host staging buffer sb is free once H1 consumed step t-2
            std::unique_lock<std::mutex> lk(c->mu);
            const int64_t need = t - c->n_hstage;
            if (!(c->h1_done >= need || c->last_t < need)) {
                ++c->h1_waiters;
                c->cv.notify_all();
                c->cv.wait(lk, [&] { return c->h1_done >= need || c->last_t < need; });
                --c->h1_waiters;
            }
        }
    }
    c->tmark(2);
    if (norms_now && !grouped) {
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
        if (c->world > 1 || c->comm) {
            ZF_TRY(c->prof_begin(1, s, &pe));
            if (c->comm) {
                ZF_NCCL(ncclAllReduce(c->norms, c->norms, (size_t)c->total_m, ncclFloat32, ncclSum, c->comm, s));
            } else if (c->peer) {
                ZF_TRY(peer_allreduce(c, s));
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
    if (lag_refresh) {
        // the norms of step t-1 (and, with NCCL, their all-reduce) were made on the side stream
        if (c->lag_pending) ZF_CUDA(cudaStreamWaitEvent(s, c->norm_ready, 0));
        c->lag_pending = false;
        if (c->world > 1 && !c->comm && !c->peer) {
            zf_ctx::Pending pe;
            ZF_TRY(c->prof_begin(1, s, &pe));
            ZF_CUDA(cudaMemcpyAsync(c->norms_host, c->norms, c->total_m * sizeof(float), cudaMemcpyDeviceToHost, s));
            ZF_CUDA(cudaStreamSynchronize(s));
            if (c->host_allreduce(c->norms_host, c->total_m, c->host_allreduce_user) != 0)
                return fail(ZF_ENCCL, "host all-reduce callback failed");
            ZF_CUDA(cudaMemcpyAsync(c->norms, c->norms_host, c->total_m * sizeof(float), cudaMemcpyHostToDevice, s));
            ZF_TRY(c->prof_end(&pe, s));
        }
    }
    const int32_t old_delta = c->since;   // K2's remap: launches since the old selection was made
    if (refresh && !grouped) {
        zf_ctx::Pending pe;
        Table<TopkLayer> tk{};
        tk.dev = c->have_sel ? c->d_topk_tab[c->cur ^ 1] : (from_warmup ? c->d_topk_w : c->d_topk_tab[2]);
        tk.n = nl;
        ZF_TRY(c->prof_begin(2, s, &pe));
        ZF_CUDA(launch_topk(tk, c->max_m, old_delta, c->nonfinite_d, s));
        ZF_TRY(c->prof_end(&pe, s));
        c->launches++;
    }
    if (refresh) c->since = 0;
    // first refresh writes set 1 (variant built with cur=0, refresh=1 -> new set 1)
    UpdParams prm{};
    prm.layers.dev = from_warmup ? c->d_upd_x[sb & 1] : c->d_upd_tab[variant];
    prm.layers.n = nl;
    // (a first refresh after warm-up is a refresh; a mode-3 refresh runs the steady unit shapes)
    const bool steady_geo = (!refresh || c->subset_refresh) && !from_warmup;
    const int64_t units = steady_geo ? c->k3_units_s : c->k3_units;
    prm.total_units = units;
    prm.claim = c->claim;
    prm.claim_base = c->claim_base;
    prm.step_delta = c->since;
    prm.do_adam = c->split ? 0 : 1;
    prm.do_extract = c->split ? 1 : 0;
    prm.do_compact = 1;
    prm.nonfinite = c->nonfinite_d;
    prm.adam = c->adam;
    {
        static const int dbg = getenv("ZF_K3_DEBUG_MODE") ? atoi(getenv("ZF_K3_DEBUG_MODE")) : 0;
        prm.debug_mode = dbg;
    }
#ifdef ZF_K3_PROF
    {
        // experiment builds: K3 consumer cycle breakdown, printed to stderr by zf_sync
        static unsigned long long* prof = nullptr;
        if (!prof) {
            cudaMalloc(&prof, 8 * sizeof(unsigned long long));
            cudaMemset(prof, 0, 8 * sizeof(unsigned long long));
        }
        prm.prof = prof;
        c->k3_prof = prof;
    }
#endif
    const int grid = (int)std::min<int64_t>(c->grid, units);
    if (lag_pre) {
        // f4 (ii): this step's gradient gives the next refresh's norms: K1 (and the NCCL
        // all-reduce) on the side stream, ordered after everything above on s (the K1 table
        // upload, K2's reading of the previous norms), concurrent with K3 and whatever the
        // caller enqueues next
        ZF_CUDA(cudaEventRecord(c->lag_in, s));
        ZF_CUDA(cudaStreamWaitEvent(c->lag_stream, c->lag_in, 0));
        zf_ctx::Pending pe;
        if (c->has_empty) ZF_CUDA(cudaMemsetAsync(c->norms, 0, c->total_m * sizeof(float), c->lag_stream));
        Table<NormLayer> tn{};
        tn.dev = c->d_norm_tab;
        tn.n = nl;
        if (c->lag_delay_us > 0) ZF_CUDA(launch_spin(c->lag_delay_us, c->lag_stream));   // test knob
        ZF_TRY(c->prof_begin(0, c->lag_stream, &pe));
        ZF_CUDA(launch_norms(tn, c->k1_units, c->gdt, c->nonfinite_d, c->lag_stream));
        ZF_TRY(c->prof_end(&pe, c->lag_stream));
        c->launches++;
        if (c->comm || (c->world > 1 && c->peer)) {
            ZF_TRY(c->prof_begin(1, c->lag_stream, &pe));
            if (c->comm)
                ZF_NCCL(ncclAllReduce(c->norms, c->norms, (size_t)c->total_m, ncclFloat32, ncclSum, c->comm, c->lag_stream));
            else
                ZF_TRY(peer_allreduce(c, c->lag_stream));
            ZF_TRY(c->prof_end(&pe, c->lag_stream));
        }
        ZF_CUDA(cudaEventRecord(c->norm_ready, c->lag_stream));
        c->lag_pending = true;
    }
    if (grouped) {
        // f4 (i): per group of layers K1 -> K2 -> K3 prologue -> K3, so K3 finds the group's G
        // in L2 where K1 just read it (same tables, unit ranges offset to the group)
        if (c->has_empty) ZF_CUDA(cudaMemsetAsync(c->norms, 0, c->total_m * sizeof(float), s));
        const TopkLayer* tkd = c->d_topk_tab[c->cur ^ 1];
        for (const auto& g : c->rgroups) {
            const int gn = g.b - g.a;
            zf_ctx::Pending pa, pb, pc;
            Table<NormLayer> tn{};
            tn.dev = c->d_norm_tab + g.a;
            tn.n = gn;
            ZF_TRY(c->prof_begin(0, s, &pa));
            ZF_CUDA(launch_norms(tn, g.k1_units, c->gdt, c->nonfinite_d, s, g.k1_off));
            ZF_TRY(c->prof_end(&pa, s));
            Table<TopkLayer> tk{};
            tk.dev = tkd + g.a;
            tk.n = gn;
            ZF_TRY(c->prof_begin(2, s, &pb));
            ZF_CUDA(launch_topk(tk, c->max_m, old_delta, c->nonfinite_d, s));
            ZF_TRY(c->prof_end(&pb, s));
            UpdParams pg = prm;
            pg.layers.dev = prm.layers.dev + g.a;
            pg.layers.n = gn;
            pg.total_units = g.k3_units;
            pg.unit_offset = g.k3_off;
            pg.claim_base = c->claim_base;
            const int gg = (int)std::min<int64_t>(c->grid, std::max<int64_t>(g.k3_units, 1));
            ZF_TRY(c->prof_begin(3, s, &pc));
            ZF_CUDA(launch_slot_consts(pg.layers.dev, gn, c->max_m, pg.step_delta, c->adam, s));
            ZF_CUDA(launch_update(pg, c->gdt, c->pdt, gg, s));
            ZF_TRY(c->prof_end(&pc, s));
            c->launches += g.k3_units > 0 ? 4 : 3;
            if (g.k3_units > 0) c->claim_base += (uint32_t)(g.k3_units + (int64_t)gg * update_limits().producers);
        }
    } else {
        zf_ctx::Pending pe3;
        ZF_TRY(c->prof_begin(3, s, &pe3));
        // prologue: the slots' {ss, bc2s} for this launch (after K2 wrote a refresh's step counts)
        ZF_CUDA(launch_slot_consts(prm.layers.dev, nl, c->max_m, prm.step_delta, c->adam, s));
        c->launches++;
        c->tmark(3);
        ZF_CUDA(launch_update(prm, c->gdt, c->pdt, grid, s));
        c->tmark(4);
        ZF_TRY(c->prof_end(&pe3, s));
        c->launches++;
    }
    if (c->split) {
        // K3b: AdamW over the dense [n, k] blocks K3a filled (phase 7)
        zf_ctx::Pending pe7;
        ZF_TRY(c->prof_begin(7, s, &pe7));
        ZF_CUDA(launch_adam_dense(prm.layers.dev, nl, c->total_rows, c->gdt, c->pdt, prm.step_delta, c->adam, s));
        ZF_TRY(c->prof_end(&pe7, s));
        c->launches++;
    }
    if (!grouped) c->claim_base += (uint32_t)(units + (int64_t)grid * update_limits().producers);
    c->since += 1;
    c->psub_valid = c->cfg.param_subset != 0;  // this K3 (re)built or kept the subset block
    for (int i = 0; i < nl; ++i)
        c->done_target[c->L[i].chunk] += (uint32_t)(steady_geo ? c->L[i].geo_s.units : c->L[i].geo.units) *
                                         (uint32_t)update_limits().consumer_warps;
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
        // X1: this step's D2H commands (per chunk: wait for its layers' K3 units, copy, event)
        // are issued by the X1 thread (x1_loop): submitting copies while the previous step's
        // are still running can block the submitting thread for most of a step, which would
        // hold the caller's next H2D back
        ZF_CUDA(cudaEventRecord(c->k3_step_ev[sb], s));
        zf_ctx::X1Job j;
        j.t = t;
        j.hs = (int)(t % c->n_hstage);
        j.sb = sb;
        j.targets = c->done_target;
        {
            std::lock_guard<std::mutex> lk(c->x1_mu);
            c->x1_jobs.push_back(std::move(j));
        }
        c->x1_cv.notify_all();
        c->d2h_issued[sb] = true;
    }
    c->tmark(5);
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
        if (c->cfg.cpu_update && end) {
            if (c->cfg.cpu_update_async) ZF_TRY(f1_launch(c, t, b, c->mw_len, params));
            else ZF_TRY(f1_window_end(c, t, b, c->mw_len, params, s));
        }
        if (end) {
            c->mw += 1;
            c->mw_len = 0;
        }
    }
    c->tmark(6);
    return ZF_OK;
}

extern "C" zf_status zf_sync(zf_ctx* c) {
    g_last_error.clear();
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    ZF_CUDA(cudaSetDevice(c->device));
    ZF_CUDA(cudaEventSynchronize(c->step_done));
    if (c->f1_pending) {  // R23: land the pending CPU update so the state is complete
        // on the stream of the last zf_step: after whatever the caller queued there since
        ZF_TRY(f1_finish(c, c->last_stream));
        ZF_CUDA(cudaStreamSynchronize(c->last_stream));
    }
    if (c->cfg.offload && !c->devacc && c->last_t >= 0) ZF_TRY(c->x1_wait_issued(c->last_t));
    if (c->copy_stream) ZF_CUDA(cudaStreamSynchronize(c->copy_stream));
    if (c->lag_stream) ZF_CUDA(cudaStreamSynchronize(c->lag_stream));   // a lagged K1 (f4 ii)
    if (c->cfg.host_accumulate) {
        std::unique_lock<std::mutex> lk(c->mu);
        ++c->h1_waiters;
        c->cv.notify_all();
        c->cv.wait(lk, [&] { return c->jobs.empty(); });
        --c->h1_waiters;
    }
    if (c->k3_prof && getenv("ZF_K3_PROF_PRINT")) {
        unsigned long long h[6];
        ZF_CUDA(cudaMemcpy(h, c->k3_prof, sizeof h, cudaMemcpyDeviceToHost));
        ZF_CUDA(cudaMemset(c->k3_prof, 0, 8 * sizeof(unsigned long long)));
        const double u = h[5] ? (double)h[5] : 1.0;
        fprintf(stderr, "[k3 prof] per warp-unit cycles: wait_full %.0f adam %.0f compact %.0f gbar_wait %.0f "
                        "writeback+release %.0f (warp-units %llu)\n",
                h[0] / u, h[1] / u, h[2] / u, h[3] / u, h[4] / u, h[5]);
    }
    if (c->peer_err_h && *(volatile int32_t*)c->peer_err_h) {
        *c->peer_err_h = 0;
        return fail(ZF_ENCCL, "peer-memory norm exchange: a peer did not arrive within the timeout");
    }
    if (c->trace && c->trace_n) {
        fprintf(stderr, "[zf_step host ms/step over %lld] f1_finish %.2f tables %.2f waits %.2f norms+topk %.2f "
                "k3_launch %.2f d2h_issue %.2f tail %.2f\n", (long long)c->trace_n, c->trace_ms[0] / c->trace_n,
                c->trace_ms[1] / c->trace_n, c->trace_ms[2] / c->trace_n, c->trace_ms[3] / c->trace_n,
                c->trace_ms[4] / c->trace_n, c->trace_ms[5] / c->trace_n, c->trace_ms[6] / c->trace_n);
        std::fill(c->trace_ms, c->trace_ms + 10, 0.0);
        c->trace_n = 0;
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
    if (host) *host = c->cfg.offload && !c->devacc ? c->L[layer].stage_host[c->last_t % c->n_hstage] : nullptr;
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

// ---- f4 (iii): the norm exchange over peer memory (k_peer.cu)
static int64_t peer_stride(const zf_ctx* c) { return (c->total_m + 63) / 64 * 64; }
static size_t peer_region_bytes(const zf_ctx* c) { return 256 + 4 * (size_t)peer_stride(c) * sizeof(float); }

zf_status peer_allreduce(zf_ctx* c, cudaStream_t s) {
    PeerArgs a = c->peer_args;
    a.epoch = ++c->peer_epoch;
    ZF_CUDA(launch_peer_allreduce(a, s));
    c->launches += 3;
    return ZF_OK;
}

extern "C" zf_status zf_peer_handle(zf_ctx* c, void* out64) {
    g_last_error.clear();
    if (!c || !out64) return fail(ZF_EINVAL, "ctx/out is NULL");
    if (c->world < 2 || c->comm) return fail(ZF_ESTATE, "peer exchange needs world > 1 created without an NCCL id");
    if (c->world > ZF_MAX_PEERS) return fail(ZF_EINVAL, "peer exchange supports world <= %d", ZF_MAX_PEERS);
    ZF_CUDA(cudaSetDevice(c->device));
    if (!c->peer_region) {
        ZF_CUDA(cudaMalloc(&c->peer_region, peer_region_bytes(c)));
        c->dev_allocs.push_back(c->peer_region);
        ZF_CUDA(cudaMemset(c->peer_region, 0, peer_region_bytes(c)));
        ZF_CUDA(cudaDeviceSynchronize());
    }
    cudaIpcMemHandle_t h;
    ZF_CUDA(cudaIpcGetMemHandle(&h, c->peer_region));
    static_assert(sizeof(h) == 64, "IPC handle size");
    std::memcpy(out64, &h, 64);
    return ZF_OK;
}

extern "C" zf_status zf_peer_open(zf_ctx* c, const void* handles) {
    g_last_error.clear();
    if (!c || !handles) return fail(ZF_EINVAL, "ctx/handles is NULL");
    if (!c->peer_region) return fail(ZF_ESTATE, "zf_peer_handle first");
    if (c->peer) return fail(ZF_ESTATE, "peer exchange already open");
    ZF_CUDA(cudaSetDevice(c->device));
    PeerArgs& a = c->peer_args;
    a = PeerArgs{};
    a.world = c->world;
    a.rank = c->rank;
    a.M = c->total_m;
    a.Mp = peer_stride(c);
    a.norms = c->norms;
    for (int q = 0; q < c->world; ++q) {
        unsigned char* base;
        if (q == c->rank) {
            base = static_cast<unsigned char*>(c->peer_region);
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, static_cast<const unsigned char*>(handles) + 64 * q, 64);
            void* p = nullptr;
            ZF_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            c->peer_mapped[q] = p;
            base = static_cast<unsigned char*>(p);
        }
        a.flags[q] = reinterpret_cast<unsigned long long*>(base);
        a.part[q] = reinterpret_cast<float*>(base + 256);
        a.red[q] = a.part[q] + 2 * a.Mp;
    }
    uint32_t* counter = nullptr;
    ZF_TRY(c->dalloc(&counter, sizeof(uint32_t) * 8, true));
    a.counter = counter;
    int32_t* err_d = nullptr;
    ZF_CUDA(cudaHostGetDevicePointer(&err_d, c->peer_err_h, 0));
    a.error = err_d;
    c->peer = true;
    return ZF_OK;
}

extern "C" zf_status zf_params_changed(zf_ctx* c) {
    g_last_error.clear();
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    c->psub_valid = false;
    return ZF_OK;
}

extern "C" zf_status zf_set_lr(zf_ctx* c, double lr) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    if (!(lr >= 0.0f) || !std::isfinite(lr)) return fail(ZF_EINVAL, "lr must be finite and >= 0");
    c->lr_cur = lr;
    return ZF_OK;
}

extern "C" int64_t zf_kernel_launches(zf_ctx* c) { return c ? c->launches : -1; }

extern "C" zf_status zf_host_stats(zf_ctx* c, int64_t* passes, int64_t* steps) {
    g_last_error.clear();
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    std::lock_guard<std::mutex> lk(c->mu);
    if (passes) *passes = c->h1_batches;
    if (steps) *steps = c->h1_batched_steps;
    return ZF_OK;
}

extern "C" zf_status zf_profile(zf_ctx* c, int32_t enable) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    c->profiling = enable != 0;
    return ZF_OK;
}

extern "C" zf_status zf_profile_read(zf_ctx* c, double* ms, int64_t* count) {
    if (!c) return fail(ZF_EINVAL, "ctx is NULL");
    std::lock_guard<std::mutex> lk(c->prof_mu);   // the X1 thread records phase 4
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
