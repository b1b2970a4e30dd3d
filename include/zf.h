/*
 * zf.h -- C-ABI of libzf.so, the B200-native (sm_100a) hot path of ZenFlow
 * (arXiv 2505.12242): importance-based gradient partitioning.
 *
 * For every linear layer's weight gradient G ([n, m], row-major, n = output
 * rows, m = input channels / columns) the path
 *   1. computes per-column squared L2 norms                (§3.3 "Lightweight Proxy")
 *   2. sums them across data-parallel ranks (NCCL)          (fig. gradient_gathering)
 *   3. selects the top-k columns, cached for N steps        ("cache and reuse")
 *   4. applies AdamW in place to the selected columns only
 *   5. compacts the unselected columns for the CPU side     ("(1-k)·M unimportant")
 *   6. stages them to pinned host memory, where they are
 *      accumulated in a double-buffered fp32 window         (fig. zero_bubble_pipeline)
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; Rn = reading n in
 * DESIGN.md §3.
 *
 * Conventions (every function):
 *  - Pointers are DEVICE pointers unless marked [host].  Device pointers must
 *    be valid CUDA device (or managed) memory of the current device.
 *  - Matrices are row-major with a leading dimension (elements) ld >= m; row i
 *    of G starts at G + i*ld.  Vector (16-byte) paths are used when row starts
 *    are 16-byte aligned; otherwise a slower scalar path runs (same results).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is
 *    asynchronous and ordered on `stream`; none synchronizes the device unless
 *    documented.
 *  - Argument errors are detected synchronously, before anything is enqueued,
 *    and return ZF_EINVAL with a message in zf_last_error().  CUDA/NCCL launch
 *    failures return ZF_ECUDA / ZF_ENCCL.  No C++ exception crosses the ABI.
 *  - Non-finite gradient values (NaN/Inf; the oracle and SPEC S:44 reject them)
 *    are detected on the device and OR-ed into a flag; results of such a step
 *    are unspecified (reading R15).
 *  - fp32 arithmetic of the AdamW update is IEEE round-to-nearest with no
 *    contraction, in the op order of DESIGN.md §2 O6, so results are
 *    reproducible bit for bit.
 */
#ifndef ZF_H_
#define ZF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* zf_stream_t; /* == cudaStream_t */

typedef enum {
    ZF_OK = 0,
    ZF_EINVAL = 1,     /* bad argument (checked before enqueueing anything)           */
    ZF_ENONFINITE = 2, /* NaN/Inf seen in a gradient (reported by zf_sync)             */
    ZF_ECUDA = 3,      /* CUDA runtime/driver error; detail in zf_last_error()         */
    ZF_ENCCL = 4,      /* NCCL error                                                   */
    ZF_ENOMEM = 5,     /* device or host allocation failed                             */
    ZF_ESTATE = 6      /* call not valid in the context's current state                */
} zf_status;

typedef enum { ZF_FP32 = 0, ZF_BF16 = 1 } zf_dtype;

/* AdamW hyper-parameters [host] (reading R8: PyTorch AdamW; paper P:653-654 uses
 * lr 1e-5, weight decay 0).  Real numbers in double: every fp32 constant of the
 * update is derived from them in double and rounded once, as PyTorch does with
 * its Python scalars.  decoupled=1: p *= (1 - lr*wd) (AdamW); decoupled=0:
 * g += wd*p (Adam with L2). */
typedef struct {
    double lr, beta1, beta2, eps, weight_decay;
    int32_t decoupled;
} zf_adam_params;

/* Human-readable name of a status code; never NULL. */
const char* zf_status_string(int32_t status);
/* Detail of the last failure on the calling thread ("" if none); never NULL. */
const char* zf_last_error(void);
/* ABI version (major*100 + minor). */
int32_t zf_version(void);
/* k = ceil(m * ratio_ppm / 1e6) in integer arithmetic, clamped to [1, m]
 * ("|channel_ids| = ceil(k_channel_ratio x m)"; reading R2).  Returns -1 if
 * m < 1 or ratio_ppm is outside (0, 1e6]. */
int64_t zf_k_for(int64_t m, int32_t ratio_ppm);

/* =========================== stateless primitives ===========================
 * The caller owns every buffer.  Scratch memory, when needed, is taken from the
 * stream-ordered allocator (cudaMallocAsync) on `stream`. */

/* Row 1 of §8(a) -- P:486 "each GPU computes and shares per-column gradient norms
 * squared (i.e., the sum of squared gradient values within each column)".
 *   G       [n, ld] row-major, dtype gdt (ZF_BF16 or ZF_FP32), read only.
 *   norms   [m] fp32, OVERWRITTEN with sum_i G[i][j]^2 (fp32 accumulation in a
 *           fixed, deterministic order: identical bits run to run).
 *   nonfinite  [1] int32 or NULL; set to 1 (never cleared) if any norm is NaN/Inf.
 * Requires n >= 1, m >= 1, ld >= m. */
zf_status zf_column_norms(const void* G, zf_dtype gdt, int64_t n, int64_t m, int64_t ld,
                          float* norms, int32_t* nonfinite, zf_stream_t stream);

/* Row 3 -- P:287 "top-k selection, which retains the gradients with the highest
 * magnitudes", applied to the per-column proxy.
 *   norms   [m] fp32, finite and >= 0 (the output of zf_column_norms, possibly
 *           summed over ranks).
 *   idx     [k] int32, OVERWRITTEN with the k columns of largest norm, ties broken
 *           toward the lower column index (reading R3), in ASCENDING column order.
 * Requires 1 <= k <= m <= 2^31-1.  Exact: selection compares fp32 bit patterns. */
zf_status zf_topk_columns(const float* norms, int64_t m, int64_t k, int32_t* idx, zf_stream_t stream);

/* Row 5 -- P:385 "a selective-optimizer, initialized only with the corresponding
 * parameter subset, performs an in-place update"; "We extend PyTorch's
 * Adam and AdamW".  For every row i < n and slot s < k (column c = idx[s]):
 * AdamW (DESIGN.md §2 O6) on p[i][c] with gradient G[i][c] and moments
 * exp_avg[i][s], exp_avg_sq[i][s], step count t_s = step[s] + 1; afterwards
 * step[s] = t_s.
 *   p        [n, ldp] dtype pdt, updated in place (bf16: RNE store).
 *   G        [n, ldg] dtype gdt, read only.
 *   idx      [k] int32, strictly ascending, each in [0, m).
 *   exp_avg, exp_avg_sq  [n, k] fp32 row-major, updated in place.
 *   step     [k] int32, updated in place.
 *   hp       [host] hyper-parameters; beta1, beta2 in [0, 1), eps > 0.
 * Other columns of p are not touched. */
zf_status zf_selective_adam(void* p, zf_dtype pdt, int64_t ldp, const void* G, zf_dtype gdt, int64_t ldg,
                            int64_t n, int64_t m, const int32_t* idx, int64_t k, float* exp_avg,
                            float* exp_avg_sq, int32_t* step, const zf_adam_params* hp, zf_stream_t stream);

/* Row 6 -- P:414 "ZenFlow transfers only the (1-k)·M unimportant gradients to the
 * CPU".  out[i][u] = G[i][j] where j is the u-th column NOT in idx (ascending):
 * a bit copy into a dense row-major [n, m-k] buffer of dtype gdt (reading R12).
 *   out      device memory, or mapped pinned host memory; 16-byte aligned for the
 *            vector path.  k == m gives an empty output (nothing written).
 *   idx      [k] int32 device data, strictly ascending, each in [0, m).  Its contents
 *            are NOT validated (that would need a host round trip): an idx violating
 *            this leaves out unspecified, without any out-of-bounds access. */
zf_status zf_compact_unselected(const void* G, zf_dtype gdt, int64_t n, int64_t m, int64_t ld,
                                const int32_t* idx, int64_t k, void* out, zf_stream_t stream);

/* ============================ stateful driver ===============================
 * One context per (process, GPU).  It owns: the flat norm buffer, the selected
 * index sets (double-buffered for the refresh remap), the AdamW moments
 * [n_local, k] (double-buffered), per-slot step counts, the device compaction
 * buffers, pinned host staging buffers, the fp32 host accumulators, a copy
 * stream, host accumulation threads and (world > 1) an NCCL communicator. */

typedef struct {
    int64_t n;          /* rows of this rank's shard (n_local >= 0; all ranks same m;
                           0: the matrix has no rows on this rank -- flat partitions,
                           row f3 -- its pointers may be NULL, it contributes zero norms) */
    int64_t m;          /* columns (input channels)                                */
    int64_t ld_grad;    /* leading dim of the gradient passed to zf_step (>= m)     */
    int64_t ld_param;   /* leading dim of the parameter passed to zf_step (>= m)    */
} zf_layer_desc;

typedef struct {
    zf_dtype grad_dtype, param_dtype; /* the same for every layer of a context        */
    int32_t topk_ppm;                 /* k = zf_k_for(m, topk_ppm) per layer           */
    int32_t refresh_interval;         /* N: selection refreshed iff t % N == 0 */
    int32_t accum_interval;           /* S: host accumulation window (S=4)      */
    zf_adam_params adam;
    int32_t offload;                  /* 1: D2H of each layer's compact block to pinned
                                         host as soon as it is written (row 7)        */
    int32_t host_accumulate;          /* 1: fp32 accumulation on the host (row 8);
                                         requires offload and N % S == 0             */
    int32_t host_threads;             /* host accumulation threads (0: default)        */
    int32_t cpu_update;               /* 1: deferred CPU AdamW of the unselected columns
                                         at every window end (next row f1, P:519-531,
                                         reading R18); requires host_accumulate. The
                                         window's average gradient acc/S updates an fp32
                                         host master with host moments; the result is
                                         uploaded into the parameters before zf_step
                                         returns (synchronous: zf_step blocks at window
                                         ends and refreshes)                          */
    int32_t warmup_steps;             /* tau >= 0: steps 0..tau-1 are synchronous warm-up
                                         steps with every column selected (k = m: full
                                         AdamW on the GPU, moments [n, m], nothing
                                         offloaded; next row f2, reading R20).
                                         The regular schedule (refresh iff (t-tau) % N
                                         == 0, windows of S steps) starts at step tau,
                                         whose refresh keeps the moments of the columns
                                         it selects (R7).  With tau > 0 the first step
                                         must be t = 0.                              */
    float auto_gamma;                 /* > 0: Zen-auto (next row f2, reading
                                         R21): the accumulation windows end adaptively,
                                         for the whole model at once, when the window's
                                         accumulated mean unimportant channel norm A
                                         reaches auto_gamma x the step's mean important
                                         channel norm (norms from K1, which then runs on
                                         every step, all-reduced when world > 1), after
                                         accum_interval (= S_max) steps, or before a
                                         refresh.  With cpu_update a window of L steps
                                         applies acc / L.  Requires host_accumulate.
                                         0: fixed S-step windows.                     */
    int32_t state_offload;            /* 1: swap the selective optimizer's state out of
                                         HBM (next row f3, "swap out its
                                         optimizer states to CPU and swap back in before
                                         next update on GPU"): the moments live in
                                         mapped pinned host memory and K3 streams each
                                         unit's slab in over the host link with the same
                                         bulk copies and writes it back with streaming
                                         stores -- no moment bytes resident in HBM, at
                                         the cost of 16 B per selected element per step on
                                         the host link.  Results are bit-identical.     */
    int32_t device_accumulate;        /* 1: the window accumulation (row 8) runs on the GPU
                                         (K7): both fp32 window accumulators [n, m-k] live
                                         in HBM, each step's compact block is added in
                                         place, and only the sealed window is copied to
                                         pinned host memory, once per window (4 B x (m-k)
                                         x n per S steps on the host link instead of 2 B x
                                         (m-k) x n per step; no host accumulation
                                         traffic).  Requires host_accumulate; with offload
                                         the per-step compact D2H is replaced by the
                                         per-window one.  Bit-identical sums.           */
    int32_t cpu_update_async;         /* 1 (with cpu_update): the window-end CPU AdamW runs
                                         on a worker thread while the caller goes on (its
                                         next forward/backward), and lands at the start
                                         of the next zf_step or in zf_sync (reading R23,
                                         the paper's overlapped "zero-stall" update,
                                         P:437-441).  Every zf_step / zf_sync leaves the
                                         same state as the synchronous mode; between a
                                         window's last zf_step and the next call the
                                         unselected columns are one window stale.  The
                                         parameter buffers of that last step must stay
                                         valid until then.                              */
    int32_t param_subset;             /* 1: the selective optimizer keeps its parameter
                                         subset p[:, idx] as a dense [n, k] block in HBM
                                         ("a selective-optimizer, initialized only
                                         with the corresponding parameter subset"): every
                                         refresh step re-reads the selected columns from
                                         p and rewrites the block; steady steps read p's
                                         current value from the block instead of p's
                                         row-major sectors (2 B per selected element
                                         instead of most of p: a selected column touches
                                         ~83% of p's 32-byte sectors at k = 10%), and
                                         store an updated value to both p and the block
                                         when its bits change.  Results are bit-identical.
                                         Contract: between refreshes the library is the
                                         only writer of the selected columns of p; a
                                         caller that writes them calls zf_params_changed
                                         before the next zf_step.  0: read p itself.    */
    int32_t lagged_selection;         /* 1: one-step-lagged selection (next row f4 (ii),
                                         P:505-508 "cache and reuse selected channel
                                         indices", reading R24): a refresh at regular step
                                         t > 0 selects by the column norms of step t-1's
                                         gradient, which K1 (and the norm exchange when
                                         world > 1) computes on the library's side stream
                                         during step t-1 (enqueued with that step's K3, it
                                         overlaps K3's tail and whatever the caller runs
                                         next) -- the refresh step makes a single pass
                                         over G.  The first refresh uses its own step's
                                         gradient.  Contract: the gradient buffers of a
                                         step t with (t+1) % N == 0 must stay valid until
                                         the next zf_step or zf_sync (e.g. double-buffered
                                         gradients).  Not with auto_gamma.             */
    int32_t host_stages;              /* pinned host staging slots of the per-step D2H
                                         (offload without device_accumulate), each one
                                         compact block of every layer; 0 = 2.  H1 (row a8)
                                         accumulates every staged step of the current window
                                         in ONE pass over the fp32 accumulator (the adds
                                         stay in step order: bit-identical sums), so more
                                         slots cut its host-DRAM traffic from ~10 B per
                                         element and step towards 3 (2·accum_interval slots:
                                         whole windows, overlapped with the next window's
                                         copies).  Range [0, 16]; ZF_EINVAL otherwise.   */
    int32_t refresh_group_mb;         /* > 0: next row f4 (i) -- a refresh step runs K1 ->
                                         K2 -> K3 per group of consecutive layers whose
                                         gradients total <= this many MB, so K3 re-reads a
                                         group's G while it is still in the 126 MB L2 from
                                         K1, instead of K1 over the whole model and then K3
                                         over it.  Results are identical.  world 1 only,
                                         not with auto_gamma / lagged_selection / the
                                         split update; 0 (default) = whole-model passes
                                         (measured faster on Llama-2-7B).  */
} zf_config;

typedef struct zf_ctx zf_ctx;

/* Rank 0 creates the NCCL unique id; the caller broadcasts its 128 bytes.  One id per
 * zf_create: a NCCL unique id bootstraps exactly one communicator. */
zf_status zf_nccl_unique_id(void* out128 /* [host] 128 bytes */);

/* Create a context on CUDA device `device`.  layers [host] [n_layers].
 * world/rank: data-parallel group; with world > 1, nccl_id128 [host] makes zf_create
 * a collective call that joins an NCCL communicator (every rank must call it); NULL
 * selects the host all-reduce callback (zf_set_host_allreduce) or the peer-memory
 * exchange (zf_peer_open).  With world == 1 an id is optional: it creates a one-rank
 * communicator, so the NCCL exchange path runs (as a copy) on a single GPU.  Each rank
 * passes the row shard it owns (reading R13: rows [r*n/P, (r+1)*n/P) of every matrix). */
zf_status zf_create(const zf_layer_desc* layers, int32_t n_layers, const zf_config* cfg, int32_t world,
                    int32_t rank, const void* nccl_id128, int32_t device, zf_ctx** out);

/* One step of the hot path at global step t (t >= 0, increasing by 1 per call;
 * the first call must be a refresh, i.e. t % N == 0, or t = 0 with warm-up).
 *   grads  [host] array of n_layers DEVICE pointers (G of each layer, [n, ld_grad])
 *   params [host] array of n_layers DEVICE pointers (p of each layer, [n, ld_param])
 * Refresh step (t % N == 0): column norms -> (world > 1) NCCL all-reduce(sum)
 * of the flat norm vector -> per-layer top-k -> moment remap (R7) -> fused
 * selective AdamW + compaction.  Other steps: fused selective AdamW +
 * compaction with the cached selection.  With offload, each layer's compact
 * block is copied to pinned host memory on the context's copy stream as soon as
 * the layer is done; with host_accumulate, host threads add it into the active
 * fp32 accumulator of window floor(t/S).  grads/params may be reused by the
 * caller once `stream` passes this call. */
zf_status zf_step(zf_ctx* ctx, int64_t t, void* const* grads, void* const* params, zf_stream_t stream);

/* Block until every D2H copy and host accumulation issued so far has finished.
 * Returns ZF_ENONFINITE if a non-finite gradient was seen since the last call. */
zf_status zf_sync(zf_ctx* ctx);

/* Views of library-owned state (valid until the next zf_step / zf_destroy). */
zf_status zf_selected(zf_ctx* ctx, int32_t layer, const int32_t** idx, int64_t* k);   /* device [k] */
zf_status zf_norms(zf_ctx* ctx, int32_t layer, const float** norms);                  /* device [m], last refresh */
zf_status zf_optimizer_state(zf_ctx* ctx, int32_t layer, const float** exp_avg, const float** exp_avg_sq,
                             const int32_t** step);                                   /* device [n,k],[n,k],[k] */
/* Compact block of the last step: device [n, m-k] with row pitch *ld elements
 * (m-k rounded up to a multiple of 8, so every row starts 16-byte aligned), and,
 * with offload, its pinned host copy (same layout and pitch) once zf_sync returned
 * (NULL otherwise).  The host accumulators are dense [n, m-k].  Any out pointer may
 * be NULL. */
zf_status zf_compact_buffer(zf_ctx* ctx, int32_t layer, const void** dev, int64_t* ld, const void** host);
/* Host accumulator [host] fp32 [rows, cols] = [n, m-k]: which = 0 the active
 * window's buffer, 1 the last sealed window's buffer (NULL if none yet). */
zf_status zf_host_accumulator(zf_ctx* ctx, int32_t layer, int32_t which, const float** host, int64_t* rows,
                              int64_t* cols);
/* device_accumulate: the device accumulator [n, m-k] fp32 with row pitch *ld elements
 * of the active window (which = 0: the buffer the last step added into) or of the
 * last sealed window (which = 1); NULL before any.  With device_accumulate,
 * zf_host_accumulator(which = 1) is the pinned host copy of the sealed window (valid
 * after zf_sync, until the next window seals) and which = 0 gives NULL. */
zf_status zf_device_accumulator(zf_ctx* ctx, int32_t layer, int32_t which, const float** dev, int64_t* ld);
/* Accumulation-window log, one entry per regular step the host accumulation has
 * processed (call after zf_sync): global step t, whether a window ended there, and
 * (Zen-auto only, else NaN) the decision's inputs: A = the window's accumulated mean
 * unimportant channel norm, imp / unimp = the step's mean important / unimportant
 * channel norm (reading R21).  Entries [0, min(cap, count)) are written to the
 * [host] arrays that are not NULL; *count = the number of entries so far. */
zf_status zf_window_log(zf_ctx* ctx, int64_t cap, int64_t* t, int32_t* end, double* A, double* imp, double* unimp,
                        int64_t* count);
/* Row a2 without NCCL: a context created with world > 1 and nccl_id128 == NULL sums the
 * ranks' partial norm vectors through this callback instead of ncclAllReduce -- zf_step
 * copies the flat fp32 norm vector [count] to a pinned host buffer, calls fn(buf, count,
 * user), which must replace it in place by the element-wise sum over all ranks (and
 * return 0; nonzero -> ZF_ENCCL), and copies it back.  Stream-synchronous; meant for
 * host-side process groups (e.g. torch.distributed over gloo) and for running several
 * ranks on one GPU.  Must be set before the first zf_step of such a context. */
typedef int32_t (*zf_host_allreduce_fn)(float* buf, int64_t count, void* user);
zf_status zf_set_host_allreduce(zf_ctx* ctx, zf_host_allreduce_fn fn, void* user);
/* Change the learning rate used from the next zf_step on (schedules). */
zf_status zf_set_lr(zf_ctx* ctx, double lr);
/* Per-phase device timing: when enabled, zf_step records CUDA events around each
 * phase on the stream it runs on (0: K1 column norms, 1: NCCL norm all-reduce,
 * 2: K2 top-k, 3: K3 fused selective AdamW + compaction, 4: a step's per-layer D2H
 * of the compact blocks on the copy stream -- first copy start to last copy end,
 * 5: a sealed window's D2H (device_accumulate), 6: K7 device accumulation,
 * 7: K3b dense selective AdamW of the split update; phase 3 is then K3a, the
 * compaction + extraction pass).  zf_profile_read waits for the recorded events,
 * writes the summed milliseconds ms[8] and occurrence counts count[8] [host] since
 * the previous read, and resets them. */
zf_status zf_profile(zf_ctx* ctx, int32_t enable);
zf_status zf_profile_read(zf_ctx* ctx, double* ms, int64_t* count);
/* Row a2 over peer memory (next row f4 (iii), "shares these partial norms with the
 * other GPUs"): instead of an NCCL all-reduce (or the host callback), the ranks' kernels
 * sum the partial norm vectors by reading each other's device memory directly -- over
 * NVLink / NVSwitch between GPUs (CUDA IPC mappings with peer access), or plain device
 * memory when ranks share a GPU.  Two-shot: each rank sums its 1/world slice of the
 * columns over the ranks in rank order 0..world-1 (one fixed fp32 order, so every rank
 * holds the same bits), then every rank gathers the slices; flags in the regions order
 * the phases and double buffers let the next exchange start while a slow peer still
 * reads the previous one.  Setup, on every rank of a context created with world > 1 and
 * no NCCL id (world <= 8):
 *   zf_peer_handle writes this rank's 64-byte IPC handle [host];
 *   the caller all-gathers the handles (e.g. torch.distributed) in rank order;
 *   zf_peer_open(handles [host] world x 64 bytes) maps the others' regions.
 * A wait that sees no peer for 20 s gives up and zf_sync reports ZF_ENCCL.
 * ZF_ESTATE: NCCL context, world < 2, zf_peer_open before zf_peer_handle or twice. */
zf_status zf_peer_handle(zf_ctx* ctx, void* out64);
zf_status zf_peer_open(zf_ctx* ctx, const void* handles);

/* param_subset: the caller wrote p (e.g. loaded a checkpoint) outside zf_step; the next
 * zf_step re-reads the selected columns from p (as a refresh does) before using them. */
zf_status zf_params_changed(zf_ctx* c);

/* H1 (row a8) statistics [host]: accumulation passes run and the steps they covered
 * (steps / passes = the mean batch of window steps one pass accumulated; host_stages).
 * Counts the passes finished so far (zf_sync first for a complete count). */
zf_status zf_host_stats(zf_ctx* ctx, int64_t* h1_passes, int64_t* h1_steps);

/* Number of this library's kernel launches issued so far by the context. */
int64_t zf_kernel_launches(zf_ctx* ctx);
zf_status zf_destroy(zf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* ZF_H_ */
