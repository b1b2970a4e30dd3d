#!/usr/bin/env python
"""Benchmark of the ZenFlow hot path on B200 (BASELINE.json metric):
"Llama-2-7B select+update ms/step; achieved HBM GB/s vs B200 peak, 1-8 GPU".

One step = one zf_step over every nn.Linear gradient of the model (225 for
Llama-2-7B): on refresh steps (t % 4 == 0) column norms (K1) -> NCCL norm
all-reduce (N>1) -> top-k (K2) -> fused selective AdamW + compaction with
moment remap (K3); on the other steps K3 alone with the cached selection.
``value`` is device time per step averaged over the K timed steps (which mix
refresh and steady steps in the 1:3 ratio of N=4), inputs resident in HBM,
compaction into the device staging buffer.  ``e2e`` is the same metric through
the same public API with HOST buffers: every step uploads G from pinned host
memory, and the compact blocks go device->host and are accumulated on the host
(rows 7-8 of the path).

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N  (row shards, strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Llama-2-7B select+update ms/step; achieved HBM GB/s vs B200 peak, 1-8 GPU"
UNIT = "ms/step"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--impl", default="zenflow", choices=["zenflow", "reference"])
    ap.add_argument("--model", default="llama2-7b", choices=["llama2-7b", "llama2-13b", "gpt2-small"])
    ap.add_argument("--ratio-ppm", type=int, default=100000)
    ap.add_argument("--refresh", type=int, default=4)
    ap.add_argument("--lr", type=float, default=1e-5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=48)
    ap.add_argument("--host-stages", type=int, default=0,
                    help="pinned host staging slots for the host-accumulation e2e line (0: 2*S, capped by "
                         "the host memory available)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k1pct", action="store_true", help="skip the k = 1%% line (reported as the k1pct field)")
    ap.add_argument("--no-lr1e3", action="store_true",
                    help="skip timing the main config at lr 1e-3 (nearly every bf16 value changes; field lr_1e-3)")
    ap.add_argument("--also-state-offload", action="store_true",
                    help="also time the f3 state swap-out mode (moments in mapped pinned host memory)")
    ap.add_argument("--also-auto", type=float, default=0.0, metavar="GAMMA",
                    help="also time Zen-auto (f2) with this gamma (K1 every step + K6 decision; offload + H1)")
    ap.add_argument("--partition", default="rows", choices=["rows", "flat"],
                    help="N>1 data layout: every matrix split by rows (R13), or a row-snapped flat ZeRO partition (f3)")
    ap.add_argument("--shard-of", type=int, default=1, metavar="P",
                    help="time rank 0's row shard of a P-GPU data-parallel run on this one GPU (no all-reduce): "
                         "per-rank evidence for the multi-GPU configs on a one-GPU box")
    ap.add_argument("--also-cpu-update", action="store_true",
                    help="also time e2e with the deferred CPU AdamW (f1), synchronous vs overlapped (R23)")
    ap.add_argument("--no-lagged", action="store_true",
                    help="skip the f4 (ii) lagged-selection line (device time, and a training-loop proxy "
                         "with a synthetic compute-bound backward between steps)")
    ap.add_argument("--refresh-group-mb", type=int, default=64,
                    help="the f4 (i) line: refresh steps run K1 -> K2 -> K3 per group of layers of at most "
                         "this many MB of gradients (G re-read from L2); 0 skips the line")
    ap.add_argument("--exchange", choices=["auto", "nccl", "host", "peer"], default="auto",
                    help="N>1 norm exchange (row a2): NCCL all-reduce, the host callback over gloo, or "
                         "peer-memory kernels (f4 iii, k_peer.cu); auto = nccl, or host with --colocate")
    ap.add_argument("--colocate", action="store_true",
                    help="N > 1 ranks share the visible GPU(s) (rank r on cuda:r %% device_count): gloo process group "
                         "and the library's host all-reduce instead of NCCL -- runs the multi-rank path (launcher, "
                         "sharding, norm exchange, max-over-ranks timing) on a one-GPU box; not a scaling number")
    ap.add_argument("--json-out", default=None)
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: 1 Gi bf16 copy, read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------ clocks sampler
class Clocks:
    def __init__(self):
        self.proc = None
        self.path = f"/tmp/zf_clocks_{os.getpid()}.csv"

    def start(self, index=0):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader",
                                          "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                smax.append(float(f[2].split()[0]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ byte accounting
def algorithmic_bytes(shapes, ks, gsz=2, psz=2):
    """Element-algorithmic bytes of one K3 launch: read G; write the compact block;
    read+write p, m, v at the selected columns (5.80 B/elt at k=10%)."""
    tot = 0
    for (n, m), k in zip(shapes, ks):
        tot += n * m * gsz + n * (m - k) * gsz + n * k * (2 * psz + 16)
    return tot


def sector_bytes(shapes, idxs, gsz=2, psz=2):
    """Sector-compulsory bytes of one K3 launch with the actual selection: p moves in
    32-byte sectors (every sector holding a selected column is read and written)."""
    tot = 0
    for (n, m), idx in zip(shapes, idxs):
        k = len(idx)
        sectors = len(np.unique((np.asarray(idx, np.int64) * psz) // 32))
        tot += n * m * gsz + n * (m - k) * gsz + n * k * 16 + n * sectors * 32 * 2
    return tot


# ------------------------------------------------------------ CPU oracle timing (baseline)
def _oracle_worker(wid, core, mats, ratio_ppm, refresh, lr, steps, barrier, q):
    """One process of the oracle timing: pinned to `core`, owns the matrices `mats`
    [(layer, n, m)], generates their inputs (host C twin of the generator), then runs the
    oracle's step sequence on them in lock step with the other workers (a barrier after
    every step), so each step's wall time is the slowest worker's."""
    try:
        os.sched_setaffinity(0, {core})
    except (AttributeError, OSError):
        pass
    from oracle import oracle as orc
    from synth import host
    hp = orc.AdamHP(lr=lr)
    st = []
    for li, n, m in mats:
        G = host.grad(n, m, li, 0, host.col_scale_at(m, 0, li))
        st.append({"n": n, "G": G, "P": host.param(n, m, li), "k": orc.k_for(m, ratio_ppm), "idx": None})
    times = []
    barrier.wait()
    for t in range(steps):
        t0 = time.perf_counter()
        for s_ in st:
            if t % refresh == 0:         # O1 norms -> O3 top-k -> O5 remap
                idx = orc.topk(orc.column_norms(s_["G"]), s_["k"])
                if s_["idx"] is None:
                    s_["M"] = np.zeros((s_["n"], s_["k"]), np.float32)
                    s_["V"] = np.zeros((s_["n"], s_["k"]), np.float32)
                    s_["steps"] = np.zeros(s_["k"], np.int32)
                else:
                    s_["M"], s_["V"], s_["steps"] = orc.remap(s_["n"], s_["idx"], s_["M"], s_["V"], s_["steps"], idx)
                s_["idx"] = idx
            orc.selective_adamw(s_["P"], s_["G"], s_["idx"], s_["M"], s_["V"], s_["steps"], hp)   # O6
            orc.compact(s_["G"], s_["idx"])                                                        # O7
        barrier.wait()
        times.append(time.perf_counter() - t0)
    if wid == 0:
        q.put(times)


def oracle_ms_per_step(model, ratio_ppm, refresh, steps, warmup, lr=1e-5, max_frac_mem=0.6):
    """Time the CPU oracle (as it stands: oracle/zf_oracle.cpp through oracle.py, one thread
    per process) on the FULL model, one process per host core (pinned), matrices balanced
    over the processes by element count; the GPU arm's step sequence (refresh every N, then
    selective AdamW + compaction; no host accumulation, which the GPU line does not run
    either).  If the host cannot hold the model's state, a stated prefix of the matrices is
    timed and scaled by element count.  Returns (ms_per_step, sample, cores)."""
    import multiprocessing as mp

    import synth
    names = synth.MODELS[model]()
    mats = [(li, n, m) for li, (_nm, n, m) in enumerate(names)]
    total = sum(n * m for _, n, m in mats)
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else list(range(os.cpu_count()))
    k_frac = ratio_ppm / 1e6
    need = lambda elems: elems * (2 + 2 + 8 * k_frac + 2 * 2 + 2)   # G, P, M+V, compact + temporaries (bytes)
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # noqa: BLE001
        avail = 1 << 62
    frac = 1.0
    if need(total) > max_frac_mem * avail:
        keep, acc = [], 0
        for x in mats:
            if need(acc + x[1] * x[2]) > max_frac_mem * avail:
                break
            keep.append(x)
            acc += x[1] * x[2]
        mats, frac = keep, acc / total
    nw = max(1, min(len(cores), len(mats)))
    bins = [[] for _ in range(nw)]
    load = [0] * nw
    for x in sorted(mats, key=lambda x: -x[1] * x[2]):   # longest-processing-time first
        w = load.index(min(load))
        bins[w].append(x)
        load[w] += x[1] * x[2]
    ctx = mp.get_context("spawn")
    barrier, q = ctx.Barrier(nw), ctx.Queue()
    procs = [ctx.Process(target=_oracle_worker, args=(w, cores[w], bins[w], ratio_ppm, refresh, lr,
                                                      warmup + steps, barrier, q)) for w in range(nw)]
    for p in procs:
        p.start()
    times = q.get()
    for p in procs:
        p.join()
    timed = times[warmup:] or times
    ms = sum(timed) / len(timed) * 1e3 / frac
    elems = sum(n * m for _, n, m in mats)
    desc = (f"{'full model' if frac == 1.0 else f'first {len(mats)} of {len(names)} matrices'}: "
            f"{len(mats)} matrices, {elems / 1e9:.3f} G elements ({frac:.1%} of the model"
            f"{'' if frac == 1.0 else ', time scaled by element count'}); {len(timed)} timed steps after "
            f"{min(warmup, len(times) - len(timed)) if len(times) > len(timed) else 0} warm-up (refresh every "
            f"{refresh}); {nw} single-threaded oracle processes pinned one per core, lock-stepped per step")
    return ms, desc, nw


def run_reference(args, rank, world):
    if rank != 0:
        return
    ms, desc, cores = oracle_ms_per_step(args.model, args.ratio_ppm, args.refresh, max(1, args.steps),
                                         args.warmup, lr=args.lr)
    line = {"impl": "reference", "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.model}-all-linear-k{args.ratio_ppm // 10000}pct", "model": args.model,
                       "ratio_ppm": args.ratio_ppm, "refresh_interval": args.refresh, "lr": args.lr},
            "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                             "host_cores": os.cpu_count()},
            "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def host_dram_probe():
    """Host DRAM bandwidth of this box's cores on H1's access patterns (tools/host_membw.c,
    built here with the host compiler, all cores, 2 GiB fp32 arrays); {} if unavailable."""
    import subprocess as _sp
    exe = f"/tmp/zf_host_membw_{os.getpid()}"
    src = os.path.join(ROOT, "tools", "host_membw.c")
    try:
        _sp.run(["gcc", "-O3", "-march=native", "-fopenmp", src, "-o", exe], check=True, capture_output=True,
                timeout=120)
        out = _sp.run([exe, "2", str(os.cpu_count())], capture_output=True, text=True, timeout=300).stdout
        os.remove(exe)
        return json.loads(out.strip().splitlines()[-1])
    except Exception as ex:  # noqa: BLE001
        return {"error": str(ex)[-120:]}


def max_over_ranks(vals, world):
    """Element-wise max over ranks (CPU tensor: works for the nccl and the gloo group)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64)
    if world > 1:
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().tolist()


def run_zenflow(args, rank, world):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2505_12242_b200 import _build
    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()
    from paper_2505_12242_b200 import zf
    from synth import gpu as sgpu
    from paper_2505_12242_b200.dist import flat_partition, shard_rows

    dev = int(os.environ.get("LOCAL_RANK", 0))
    if args.colocate:
        dev %= torch.cuda.device_count()
    torch.cuda.set_device(dev)
    hbm_peak, peak_src = peaks()
    names = synth.MODELS[args.model]()
    full_shapes = [(n, m) for _, n, m in names]

    sim = args.shard_of if (args.shard_of > 1 and world == 1) else 1
    if args.partition == "flat":
        spans = flat_partition(full_shapes, max(world, sim), rank)
    else:
        spans = [shard_rows(n, max(world, sim), rank) for n, _ in full_shapes]
    shapes = [(b - a, m) for (a, b), (_, m) in zip(spans, full_shapes)]
    row0s = [a for a, _ in spans]
    ks = [zf.k_for(m, args.ratio_ppm) for _, m in shapes]

    # ---- inputs resident in HBM: two gradient versions (alternating steps), params
    def alloc_flat(shp, dtype):
        tot = sum(n * m for n, m in shp)
        buf = torch.empty(tot, dtype=dtype, device="cuda")
        views, off = [], 0
        for n, m in shp:
            views.append(buf[off:off + n * m].view(n, m))
            off += n * m
        return buf, views

    _g0, G0 = alloc_flat(shapes, torch.bfloat16)
    _g1, G1 = alloc_flat(shapes, torch.bfloat16)
    _p, Ps = alloc_flat(shapes, torch.bfloat16)
    for li, (n, m) in enumerate(shapes):
        sc = sgpu.ColScale(m, li)
        sgpu.fill_grad(G0[li], li, 0, sc, row0=row0s[li])
        sc.advance_to(1)
        sgpu.fill_grad(G1[li], li, 1, sc, row0=row0s[li])
        sgpu.fill_param(Ps[li], li, row0=row0s[li])
        del sc
    torch.cuda.synchronize()
    host_ar = None
    exch = args.exchange if args.exchange != "auto" else ("host" if args.colocate else "nccl")

    def nccl_id():
        # a NCCL unique id serves ONE communicator: every context gets a fresh one (rank 0
        # makes it, torch.distributed broadcasts it; all ranks create contexts in the same order)
        if world > 1 and exch == "nccl":
            from paper_2505_12242_b200.dist import broadcast_nccl_id
            return broadcast_nccl_id()
        return None

    if world > 1 and exch == "host":
        from paper_2505_12242_b200.dist import gloo_allreduce
        host_ar = gloo_allreduce()

    def make_ctx(ratio_ppm, offload, **kw):
        ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=ratio_ppm,
                         refresh_interval=args.refresh, accum_interval=args.refresh,
                         adam=zf.adam_params(lr=args.lr), offload=offload, host_accumulate=offload,
                         world=world, rank=rank, nccl_id=nccl_id(), device=dev, host_allreduce=host_ar, **kw)
        if world > 1 and exch == "peer":
            from paper_2505_12242_b200.dist import open_peer_exchange
            open_peer_exchange(ctx)
        return ctx

    import ctypes
    nl = len(shapes)
    gp = [(ctypes.c_void_p * nl)(*[g.data_ptr() for g in G0]), (ctypes.c_void_p * nl)(*[g.data_ptr() for g in G1])]
    pp = (ctypes.c_void_p * nl)(*[p.data_ptr() for p in Ps])
    stream = torch.cuda.current_stream()

    def timed_run(ctx, K, W, tag):
        for t in range(W):
            ctx.step_ptrs(t, gp[t % 2], pp, stream)
        ctx.sync()
        ctx.profile_read()
        ctx.profile(True)
        l0 = ctx.kernel_launches()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for t in range(W, W + K):
            ctx.step_ptrs(t, gp[t % 2], pp, stream)
        ev1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        prof = ctx.profile_read()
        ctx.profile(False)
        ctx.sync()
        return ms, prof, ctx.kernel_launches() - l0

    # ---- main measurement: k = ratio, offload off (device staging)
    ctx = make_ctx(args.ratio_ppm, False)
    clocks = Clocks()
    clocks.start(dev)
    ms_total, prof, launches = timed_run(ctx, args.steps, args.warmup, "main")
    clk = clocks.stop()
    idxs = [ctx.selected(li).cpu().numpy() for li in range(nl)]
    ctx.close()
    del ctx
    mine = {"rank": rank, "device": dev, "k3_ms": prof["k3_update"][0] / max(1, prof["k3_update"][1]),
            "k3_alg_GBs": algorithmic_bytes(shapes, ks) / (prof["k3_update"][0] / max(1, prof["k3_update"][1]) * 1e-3)
            / 1e9 if prof["k3_update"][1] else None, "ms_per_step": ms_total / args.steps,
            "elements": sum(n * m for n, m in shapes),
            # the last selection of every layer, hashed: identical on every rank
            "selection_sha1": __import__("hashlib").sha1(b"".join(i.tobytes() for i in idxs)).hexdigest()[:16]}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    ms_total, k3_ms, k1_ms, k2_ms, ar_ms = max_over_ranks(
        [ms_total, prof["k3_update"][0], prof["k1_norms"][0], prof["k2_topk"][0], prof["allreduce"][0]], world)
    ms_per_step = ms_total / args.steps
    n_k3 = prof["k3_update"][1]
    n_k1 = prof["k1_norms"][1]
    k3_avg = k3_ms / max(1, n_k3)
    alg = algorithmic_bytes(shapes, ks)
    sec = sector_bytes(shapes, idxs)
    g_bytes = sum(n * m * 2 for n, m in shapes)
    if sim > 1:
        par_desc = f"rank 0 of dp{sim} ({args.partition}) timed alone on 1 GPU, no all-reduce"
    else:
        par_desc = (f"dp{world} ({'flat ZeRO partition' if args.partition == 'flat' else 'row shards'}, "
                    + {"host": "norm all-reduce over gloo via the host callback",
                       "peer": "norm exchange over peer memory (k_peer)",
                       "nccl": "NCCL norm all-reduce"}[exch]
                    + (f", ranks co-located on {torch.cuda.device_count()} GPU(s))" if args.colocate else ")"))
    result = {
        "metric": METRIC, "value": ms_per_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded column-concentrated bf16 gradients, bf16 params, fp32 AdamW state)",
        "config": {"workload": f"{args.model}-all-linear-k{args.ratio_ppm // 10000}pct"
                               + (f"-rank0-of-dp{sim}" if sim > 1 else ""), "model": args.model,
                   "linears": nl, "elements": sum(n * m for n, m in full_shapes), "ratio_ppm": args.ratio_ppm,
                   "refresh_interval": args.refresh, "parallelism": par_desc,
                   "l2": "inputs larger than L2 (working set > 100 GB vs 126 MB L2); no flush needed",
                   "lr": args.lr},
        "phases_ms_per_launch": {"k3_update": k3_avg, "k1_norms": k1_ms / max(1, n_k1),
                                 "k2_topk": k2_ms / max(1, prof["k2_topk"][1]),
                                 "allreduce": (ar_ms / max(1, prof["allreduce"][1])) if world > 1 else None},
        "gpu_launches": launches,
        "per_rank": per_rank if world > 1 else None,
        "selection_identical_across_ranks": (len({r["selection_sha1"] for r in per_rank}) == 1) if world > 1 else None,
        "clocks": clk,
    }
    if world > 1 and prof["allreduce"][1]:
        # row a2 on NVLink: the flat fp32 norm vector, once per refresh (nccl-tests conventions)
        ar_bytes = 4 * sum(m for _n, m in full_shapes)
        ar_avg = ar_ms / prof["allreduce"][1]
        algbw = ar_bytes / (ar_avg * 1e-3) / 1e9
        result["nvlink_allreduce"] = {"bytes": ar_bytes, "ms": ar_avg, "algbw_GBs": algbw,
                                      "busbw_GBs": algbw * 2 * (world - 1) / world,
                                      "peak_GBs_per_direction": 900.0}
    achieved = alg / (k3_avg * 1e-3) / 1e9
    result["roofline"] = {"bound": "hbm", "kernel": "k_update (K3 fused selective AdamW + compaction)",
                          "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                          "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
                          "sector_compulsory_bytes_per_launch": sec,
                          "achieved_sector_GBs": sec / (k3_avg * 1e-3) / 1e9,
                          "frac_sector": sec / (k3_avg * 1e-3) / 1e9 / hbm_peak, "traffic": None}
    def add_traffic(roof, workload, k3_ms):
        # DRAM bytes the kernel actually moves per launch (committed ncu captures) over its
        # live average duration: the launch-list average of the default command, else the
        # one-launch full capture of the workload
        tr, src = None, None
        p1 = os.path.join(ROOT, "profiles", "k3_dram_traffic.json")
        p2 = os.path.join(ROOT, "profiles", "k3_dram_traffic_ncu_full.json")
        if os.path.exists(p1):
            d = json.load(open(p1))
            if d.get("workload") == workload:
                tr, src = d.get("traffic_bytes_per_launch"), d.get("source")
        if tr is None and os.path.exists(p2):
            d = json.load(open(p2))
            e = d.get("by_workload", {}).get(workload)
            if e:
                tr, src = e["traffic_bytes_per_launch"], d.get("source")
        if tr is not None and world == 1:
            roof["traffic"] = tr
            roof["traffic_source"] = src
            roof["achieved_dram_GBs"] = tr / (k3_ms * 1e-3) / 1e9
            roof["frac_dram"] = tr / (k3_ms * 1e-3) / 1e9 / hbm_peak

    add_traffic(result["roofline"], result["config"]["workload"], k3_avg)
    if n_k1:
        k1_avg = k1_ms / n_k1
        result["k1_roofline"] = {"bound": "hbm", "achieved": g_bytes / (k1_avg * 1e-3) / 1e9, "peak": hbm_peak,
                                 "unit": "GB/s", "frac": g_bytes / (k1_avg * 1e-3) / 1e9 / hbm_peak}

    def k3_line(ctx_ppm, lr=None, tag="", **kw):
        ctx = make_ctx(ctx_ppm, False, **kw) if lr is None else zf.Context(
            [zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=ctx_ppm, refresh_interval=args.refresh,
            accum_interval=args.refresh, adam=zf.adam_params(lr=lr), world=world, rank=rank, nccl_id=nccl_id(),
            device=dev, host_allreduce=host_ar)
        msx, profx, _ = timed_run(ctx, args.steps, args.warmup, tag)
        idxx = [ctx.selected(li).cpu().numpy() for li in range(nl)]
        ctx.close()
        del ctx
        ksx = [zf.k_for(m, ctx_ppm) for _, m in shapes]
        msx, k3x, k1x = max_over_ranks([msx, profx["k3_update"][0], profx["k1_norms"][0]], world)
        k3a = k3x / max(1, profx["k3_update"][1])
        algx = algorithmic_bytes(shapes, ksx)
        secx = sector_bytes(shapes, idxx)
        return {"ms_per_step": msx / args.steps, "k3_ms": k3a, "k1_ms": k1x / max(1, profx["k1_norms"][1]),
                "roofline": {"bound": "hbm", "kernel": "k_update", "achieved": algx / (k3a * 1e-3) / 1e9,
                             "peak": hbm_peak, "unit": "GB/s", "frac": algx / (k3a * 1e-3) / 1e9 / hbm_peak,
                             "algorithmic_bytes_per_launch": algx, "sector_compulsory_bytes_per_launch": secx,
                             "frac_sector": secx / (k3a * 1e-3) / 1e9 / hbm_peak}}

    # ---- k = 1% (config 3's second ratio) with its own K3 roofline
    if not args.no_k1pct and args.ratio_ppm != 10000:
        result["k1pct"] = k3_line(10000, tag="k1pct")
        result["k1pct"]["workload"] = f"{args.model}-all-linear-k1pct"
        add_traffic(result["k1pct"]["roofline"], result["k1pct"]["workload"], result["k1pct"]["k3_ms"])
    # ---- the main config at lr 1e-3: nearly every selected bf16 value changes, so K3 stores
    #      (and read-modify-writes) the p sectors the lr 1e-5 headline mostly skips
    if not args.no_lr1e3 and args.lr != 1e-3:
        result["lr_1e-3"] = k3_line(args.ratio_ppm, lr=1e-3, tag="lr1e3")

    # ---- f4 (i): refresh steps in groups of layers (K1 -> K2 -> K3 per group, G re-read from L2)
    if args.refresh_group_mb > 0 and world == 1:
        rg = k3_line(args.ratio_ppm, tag="rgroup", refresh_group_mb=args.refresh_group_mb)
        result["refresh_in_groups"] = {"group_mb": args.refresh_group_mb, "ms_per_step": rg["ms_per_step"],
                                       "k1_ms": rg["k1_ms"], "k3_ms": rg["k3_ms"],
                                       "note": "K1/K3 ms are per group launch here; compare ms_per_step with "
                                               "the whole-model passes of the main line"}

    # ---- f4 (ii) lagged selection: device time of the same loop, and a training-loop proxy in
    #      which each step is preceded by a compute-bound "backward" (bf16 GEMMs on the caller's
    #      stream); with the lag, a pre-refresh step's K1 runs on the library's side stream under
    #      the next backward instead of on the refresh step's critical path
    if not args.no_lagged and world == 1:
        def loop_with_backward(lagged, K, W):
            ctx = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=args.ratio_ppm,
                             refresh_interval=args.refresh, accum_interval=args.refresh,
                             adam=zf.adam_params(lr=args.lr), device=dev, lagged_selection=lagged)
            a = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
            b = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
            c_ = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")

            def backward():
                for _ in range(3):
                    torch.matmul(a, b, out=c_)
            for t in range(W):
                backward()
                ctx.step_ptrs(t, gp[t % 2], pp, stream)
            ctx.sync()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for t in range(W, W + K):
                backward()
                ctx.step_ptrs(t, gp[t % 2], pp, stream)
            ctx.sync()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            ctx.close()
            e0.record(stream)
            for _ in range(K):
                backward()
            e1.record(stream)
            torch.cuda.synchronize()
            bw = e0.elapsed_time(e1) / K
            del a, b, c_
            return ms, bw
        ctxl = zf.Context([zf.LayerShape(n, m) for n, m in shapes], topk_ratio_ppm=args.ratio_ppm,
                          refresh_interval=args.refresh, accum_interval=args.refresh,
                          adam=zf.adam_params(lr=args.lr), device=dev, lagged_selection=True)
        msl, profl, _ = timed_run(ctxl, args.steps, args.warmup, "lagged")
        ctxl.close()
        del ctxl
        Kp = max(8, args.steps)
        plain_ms, bw_ms = loop_with_backward(False, Kp, 4)
        lag_ms, _ = loop_with_backward(True, Kp, 4)
        result["lagged_selection"] = {
            "ms_per_step": msl / args.steps,
            "k1_launches": profl["k1_norms"][1],
            "training_loop_proxy": {"backward_ms": bw_ms, "plain_ms_per_step": plain_ms,
                                    "lagged_ms_per_step": lag_ms, "steps": Kp,
                                    "backward": "3 x bf16 GEMM 8192^3 on the caller's stream before every zf_step; "
                                                "gradient buffers alternate (the lagged K1 reads the other one)"},
            "delta_loop_ms_per_step": msl / args.steps - ms_per_step,
            "delta_proxy_ms_per_step": lag_ms - plain_ms,
            "note": "same work per N steps (one K1 per refresh either way).  zf_step loop alone: the lagged K1 runs "
                    "on the library's side stream next to the pre-refresh step's K3 and fills its tail "
                    "(delta_loop_ms_per_step < 0 means faster).  Training-loop proxy: a full-occupancy GEMM "
                    "backward leaves the side-stream K1 no SMs, so the norm pass is not hidden there "
                    "(delta_proxy_ms_per_step ~ 0)"}

    # ---- f3 state swap-out: moments in mapped pinned host memory (extra field)
    if args.also_state_offload:
        ctx = make_ctx(args.ratio_ppm, False, state_offload=True)
        mss, profs, _ = timed_run(ctx, args.steps, args.warmup, "state_offload")
        ctx.close()
        del ctx
        mv = sum(n * k * 16 for (n, _m), k in zip(shapes, ks))  # m, v read + written per step
        k3s = profs["k3_update"][0] / max(1, profs["k3_update"][1])
        result["state_offload"] = {"ms_per_step": mss / args.steps, "k3_ms": k3s,
                                   "host_link_moment_bytes_per_step": mv,
                                   "host_link_GBs": mv / (k3s * 1e-3) / 1e9}

    # ---- f2 Zen-auto: K1 every step + K6, with offload and host accumulation (extra field)
    if args.also_auto > 0:
        ctx = make_ctx(args.ratio_ppm, True, auto_gamma=args.also_auto)
        msa, profa, la = timed_run(ctx, args.steps, args.warmup, "auto")
        log = ctx.window_log()
        ctx.close()
        del ctx
        ends = [t for (t, e, *_r) in log if e]
        dev_ms = sum(profa[p][0] for p in ("k1_norms", "k2_topk", "k3_update", "k7_accumulate")) / args.steps
        result["zen_auto"] = {"gamma": args.also_auto, "kernel_ms_per_step": dev_ms,
                              "wall_ms_per_step": msa / args.steps,
                              "k1_launches": profa["k1_norms"][1], "gpu_launches": la,
                              "window_ends": ends[-12:],
                              "note": "kernel_ms = K1+K2+K3 event time per step (K6 not profiled, ~us); "
                                      "wall includes waiting on the host accumulation (offload + H1)"}

    # ---- e2e: host buffers through the same API.  Two offload modes, both measured:
    #   device_accumulate (K7: fp32 window accumulators in HBM, one D2H of the sealed window
    #   per S steps) -- the headline e2e; host accumulation (per-step bf16 compact D2H + CPU
    #   fp32 accumulation, the paper's layout) -- reported beside it.
    if not args.no_e2e:
        del _g1, G1
        torch.cuda.empty_cache()
        host_g = torch.empty(sum(n * m for n, m in shapes), dtype=torch.bfloat16, pin_memory=True)
        host_g.copy_(_g0)
        h2d = host_g.numel() * 2
        gpp = (ctypes.c_void_p * nl)(*[g.data_ptr() for g in G0])
        d2h_host = sum(n * (m - k) * 2 for (n, m), k in zip(shapes, ks))
        d2h_dev = sum(n * (m - k) * 4 for (n, m), k in zip(shapes, ks)) / args.refresh  # one fp32 window per S
        K = args.e2e_steps

        # host-link peaks on this box: 1 GiB pinned <-> device copies, CUDA events
        def link_peak(d2h):
            nb = 1 << 30
            hb = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
            db = torch.empty(nb, dtype=torch.uint8, device="cuda")
            for _ in range(2):
                (hb.copy_(db, non_blocking=True) if d2h else db.copy_(hb, non_blocking=True))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(4):
                (hb.copy_(db, non_blocking=True) if d2h else db.copy_(hb, non_blocking=True))
            e1.record()
            torch.cuda.synchronize()
            del hb, db
            return 4 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9

        def link_bidir():
            # both directions at once (1 GiB each way on two streams): the host link's combined
            # rate when the H2D of G and the offload D2H overlap
            nb = 1 << 30
            hb = [torch.empty(nb, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            db = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
            st = [torch.cuda.Stream(), torch.cuda.Stream()]
            best = None
            for rep in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                with torch.cuda.stream(st[0]):
                    for _ in range(2):
                        hb[0].copy_(db[0], non_blocking=True)
                with torch.cuda.stream(st[1]):
                    for _ in range(2):
                        db[1].copy_(hb[1], non_blocking=True)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                if rep and (best is None or dt < best):
                    best = dt
            del hb, db
            return 4 * nb / best / 1e9

        link = {"d2h_peak_GBs": link_peak(True), "h2d_peak_GBs": link_peak(False),
                "bidir_peak_GBs": link_bidir(),
                "peak_source": "measured in this run: 1 GiB pinned <-> device cudaMemcpyAsync, CUDA events "
                               "(bidir: 1 GiB each way concurrently on two streams, wall clock)"}
        torch.cuda.empty_cache()  # return the 1 GiB probe to the device before the contexts

        # two device gradient buffers: the H2D of step t+1's G (side stream) overlaps step t's
        # kernels, as a training loop that uploads the next gradients would
        # (falls back to one buffer, uploaded in stream order, when HBM cannot hold a second copy
        # next to the context -- Llama-2-13B with K7 on one GPU)
        state = {"double": True}
        gbufs = [_g0, torch.empty_like(_g0)]   # the list holds the only reference to the second copy
        gpps = [gpp, (ctypes.c_void_p * nl)(*[gbufs[1].data_ptr() + (g.data_ptr() - _g0.data_ptr()) for g in G0])]
        h2d_stream = torch.cuda.Stream()

        def e2e_loop(ctx, t_begin, t_end):
            if not state["double"]:
                for t in range(t_begin, t_end):
                    _g0.copy_(host_g, non_blocking=True)
                    ctx.step_ptrs(t, gpp, pp, stream)
                return
            up = [torch.cuda.Event(), torch.cuda.Event()]
            used = [torch.cuda.Event(), torch.cuda.Event()]
            with torch.cuda.stream(h2d_stream):
                gbufs[t_begin % 2].copy_(host_g, non_blocking=True)
                up[t_begin % 2].record(h2d_stream)
            for t in range(t_begin, t_end):
                b = t % 2
                stream.wait_event(up[b])
                ctx.step_ptrs(t, gpps[b], pp, stream)
                used[b].record(stream)
                if t + 1 < t_end:
                    nb = (t + 1) % 2
                    with torch.cuda.stream(h2d_stream):
                        h2d_stream.wait_event(used[nb])   # step t-1 finished reading that buffer
                        gbufs[nb].copy_(host_g, non_blocking=True)
                        up[nb].record(h2d_stream)

        def e2e_run(devacc, **kw):
            try:
                ctx = make_ctx(args.ratio_ppm, True, device_accumulate=devacc, **kw)
            except zf.ZFError:
                if not state["double"]:
                    raise
                state["double"] = False
                gbufs[1] = None
                gpps[1] = None
                torch.cuda.empty_cache()
                ctx = make_ctx(args.ratio_ppm, True, device_accumulate=devacc, **kw)
            try:
                return _e2e_timed(ctx, devacc)
            finally:
                ctx.close()
                del ctx
                torch.cuda.empty_cache()

        def _e2e_timed(ctx, devacc):
            W2 = args.refresh   # warm-up: one accumulation window
            e2e_loop(ctx, 0, W2)
            ctx.sync()
            h1_0 = ctx.host_stats()
            ctx.profile_read()
            ctx.profile(True)
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_loop(ctx, W2, W2 + K)
            ctx.sync()
            e2e_s = time.perf_counter() - t0
            h1_1 = ctx.host_stats()
            if not devacc:
                link["h1_passes"] = h1_1[0] - h1_0[0]
                link["h1_steps"] = h1_1[1] - h1_0[1]
            prof_e = ctx.profile_read()
            ctx.profile(False)
            if devacc:
                ms_w, n_w = prof_e["d2h_window"]
                wbytes = sum(n * (m - k) * 4 for (n, m), k in zip(shapes, ks))
                link["window_d2h_GBs"] = wbytes / (ms_w / n_w * 1e-3) / 1e9 if n_w else None
                link["window_d2h_ms"] = ms_w / n_w if n_w else None
                link["k7_ms"] = prof_e["k7_accumulate"][0] / max(1, prof_e["k7_accumulate"][1])
            else:
                ms_s, n_s = prof_e["d2h_step"]
                link["x1_d2h_GBs"] = d2h_host / (ms_s / n_s * 1e-3) / 1e9 if n_s else None
                link["x1_d2h_ms_per_step"] = ms_s / n_s if n_s else None
            return max_over_ranks([e2e_s], world)[0] * 1e3 / K

        try:
            ms_dev = e2e_run(True)
        except zf.ZFError as ex:   # K7's two fp32 accumulators do not fit (e.g. Llama-2-13B on one GPU)
            ms_dev = None
            result["e2e_note"] = f"device_accumulate does not fit in HBM here ({str(ex)[-60:]}); e2e = host accumulation"
            torch.cuda.empty_cache()
        # host staging slots for the per-step D2H: H1 accumulates every staged step of a window
        # in one pass (2*S slots: whole windows, overlapped with the next window's copies),
        # as many as the host memory holds next to the accumulators and the pinned G
        S_ = args.refresh
        acc_bytes = 2 * 4 * sum(n * (m - k) for (n, m), k in zip(shapes, ks))
        try:
            avail = int([l.split()[1] for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0]) * 1024
        except Exception:  # noqa: BLE001
            avail = 0
        # every rank of this node allocates at once: each takes its share of what is available
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
        hstages = args.host_stages or 2 * S_
        while hstages > 2 and hstages * d2h_host + acc_bytes + h2d > 0.85 * avail / max(1, local_world):
            hstages -= 1
        link["host_stages"] = hstages
        ms_host = e2e_run(False, host_stages=hstages)
        if not state["double"]:
            result["e2e_note"] = (result.get("e2e_note", "") + "; one device gradient buffer "
                                  "(a second copy does not fit next to the context)").lstrip("; ")
        if args.also_cpu_update:
            # f1 at every window end: synchronous (R18) vs overlapped with the next step's H2D (R23)
            result["e2e_cpu_update"] = {
                "sync_ms_per_step": e2e_run(True, cpu_update=True),
                "async_ms_per_step": e2e_run(True, cpu_update=True, cpu_update_async=True),
                "note": "device_accumulate + deferred CPU AdamW of the unselected columns every S steps; "
                        "async overlaps it with the caller's next H2D of G"}
        for key in ("x1_d2h_GBs", "window_d2h_GBs"):
            if link.get(key):
                link[key.replace("_GBs", "_frac")] = link[key] / link["d2h_peak_GBs"]
        # H1's host-memory traffic per step: per unselected element every staged bf16 value is
        # read once (2 B); each H1 pass writes the fp32 accumulator once (4 B) and reads it
        # unless the pass starts its window (4 B); windows = steps / S in the timed region
        E_ = sum(n * (m - k) for (n, m), k in zip(shapes, ks))
        p_, s_ = link.get("h1_passes") or K, link.get("h1_steps") or K
        h1_bytes = E_ * (2 * s_ + 4 * p_ + 4 * max(0, p_ - s_ / S_)) / s_
        link["h1_host_dram_bytes_per_step"] = h1_bytes
        link["h1_host_dram_GBs"] = h1_bytes / (ms_host * 1e-3) / 1e9
        link["host_link_floor_ms"] = h2d / (link["h2d_peak_GBs"] * 1e9) * 1e3
        # the per-step D2H host-accumulation mode moves G up and the compact block down every
        # step: its floor is the slower of each direction alone and both through the shared link
        link["host_link_floor_bidir_ms"] = max(h2d / link["h2d_peak_GBs"], d2h_host / link["d2h_peak_GBs"],
                                               (h2d + d2h_host) / link["bidir_peak_GBs"]) / 1e9 * 1e3
        link["host_link_floor_k7_ms"] = max(h2d / link["h2d_peak_GBs"], d2h_dev / link["d2h_peak_GBs"],
                                            (h2d + d2h_dev) / link["bidir_peak_GBs"]) / 1e9 * 1e3
        link["host_dram"] = host_dram_probe() if rank == 0 else {"skipped": "rank 0 probes the host"}
        if link["host_dram"].get("accB1_GBs"):
            # H1's floor on this host: its bytes per step at the probe's one-step-pass rate
            link["h1_floor_ms"] = h1_bytes / (link["host_dram"]["accB1_GBs"] * 1e9) * 1e3
        node = None
        try:
            import glob as _glob
            import subprocess as _sp
            bid = _sp.run(["nvidia-smi", f"--id={dev}", "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                          capture_output=True, text=True, timeout=20).stdout.strip().lower()
            bid = bid[4:] if bid.count(":") == 2 and len(bid.split(":")[0]) == 8 else bid
            for f in _glob.glob(f"/sys/bus/pci/devices/*{bid[-7:]}/numa_node"):
                node = int(open(f).read().strip())
        except Exception:  # noqa: BLE001
            pass
        link["gpu_numa_node"] = node
        link["host_cpus"] = os.cpu_count()
        result["host_link"] = link
        result["e2e"] = {"value": ms_dev if ms_dev is not None else ms_host, "unit": UNIT, "h2d_bytes_per_step": h2d,
                         "d2h_bytes_per_step": int(d2h_dev) if ms_dev is not None else d2h_host, "steps": K,
                         "path": ("pinned host G -> H2D (side stream, double-buffered, overlapping the previous "
                                  "step) -> zf_step (offload, device_accumulate: K7 fp32 window accumulators in HBM, "
                                  "sealed window D2H once per S steps) -> zf_sync") if ms_dev is not None else
                                 ("pinned host G -> H2D -> zf_step (offload: per-step bf16 compact D2H, host fp32 "
                                  "accumulation) -> zf_sync")}
        result["e2e_host_accumulate"] = {"value": ms_host, "unit": UNIT, "h2d_bytes_per_step": h2d,
                                         "d2h_bytes_per_step": d2h_host, "steps": K,
                                         "path": "pinned host G -> H2D -> zf_step (offload: per-step bf16 compact "
                                                 "D2H, host fp32 accumulation) -> zf_sync"}
    else:
        result["e2e"] = None

    # ---- CPU oracle baseline (rank 0, N=1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ms, desc, cores = oracle_ms_per_step(args.model, args.ratio_ppm, args.refresh, args.refresh, 0, lr=args.lr)
        result["cpu_baseline"] = {"value": ms, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                                  "host_cores": os.cpu_count()}
    if rank == 0:
        line = json.dumps(result)
        print(line, flush=True)
        if args.json_out:
            open(args.json_out, "w").write(line + "\n")


def _free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """`bench.py --gpus N` (N > 1) without a torchrun environment: re-run this script as N
    ranks under torch.distributed.run on 127.0.0.1 (one process per GPU, or per rank with
    --colocate) and return its exit code.  Only rank 0 prints the JSON line."""
    if args.impl == "zenflow" and not args.colocate:
        import torch
        nd = torch.cuda.device_count()
        if nd < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but {nd} CUDA device(s) visible; use --colocate to run "
                  f"{args.gpus} ranks on the visible GPU(s)", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    if not args.colocate:
        env.setdefault("NCCL_DEBUG", "INFO")        # communicator lines (nranks) on stderr
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "zenflow":
        sys.exit(self_launch(args))
    if os.environ.get("ZF_BENCH_LAUNCH_PROBE"):
        # launcher test hook (tests/test_bench_cpu.py): report the rank layout, do no work
        print(json.dumps({"rank": rank, "world": world, "local_rank": int(os.environ.get("LOCAL_RANK", 0))}),
              flush=True)
        return
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if args.impl == "reference":
        if world > 1 and rank != 0:
            return
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.colocate:
            dist.init_process_group("gloo")
        else:
            if torch.cuda.device_count() < world:
                print(f"bench.py: WORLD_SIZE={world} but {torch.cuda.device_count()} CUDA device(s); "
                      "use --colocate", file=sys.stderr)
                sys.exit(2)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            dist.init_process_group("nccl")
    run_zenflow(args, rank, world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
