#!/usr/bin/env python
"""bench.py -- paged decode-attention step on B200: achieved HBM GB/s, us/step.

One step = copy_blocks (when the step has copy-on-write pairs) +
reshape_and_cache + paged_attention (with its split-context merge) for ONE attention
layer over the whole batch, all on one stream; by default the cache write is fused
into the attention kernel (pa_paged_attention_decode; --unfused runs the separate
reshape_and_cache launch); at N > 1 GPUs heads are sharded
tensor-parallel style and the per-rank output head slices are all-gathered
with NCCL (+ permute to [S][H][D]).

value = logical K/V bytes read per step by all ranks / device step time (GB/s); the
roofline object reports the dominant call (pa_paged_attention) against
MEASURED_PEAKS.json's HBM copy bandwidth.  Inputs are seeded synthetic data with the
BASELINE.json shapes (synth/), resident in HBM.  R layer caches (each with its own
seeded values) are rotated step by step, R chosen so that R x the K/V one step reads on
this rank >= 4 x the L2 size queried at run time (R >= 2), so every step streams its
cache from HBM (no flush; stated in config.l2).  The JSON line carries p10/p50/p90 of
the per-step and per-launch event times, the same-run read-only HBM ceiling
(pa_hbm_read_probe) beside the copy peak, and, at N > 1, per-rank GB/s and gather us.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_sharegpt] [--impl ours|reference]
Under torchrun (N > 1) every rank runs its head shard; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "paged decode-attention achieved HBM GB/s (% of peak), \u00b5s/step at 1/2/4/8 GPUs"  # BASELINE.json metric
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_traffic(config: str, n: int):
    """ncu dram bytes per launch of the dominant kernel, from the committed profile summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(config, {}).get(str(n))
    except Exception:
        return None


class ClockSampler:
    """NVML samples of SM clock + throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="c2_sharegpt")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--partition-tokens", type=int, default=0)
    ap.add_argument("--block-size", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="separate reshape_and_cache launch (ablation)")
    ap.add_argument("--grouped", type=int, default=-1,
                    help="sharing-aware decode on the tensor cores over groups of this many sequences "
                         "(tcgen05 kernel, SURVEY 8(f) N1; 0 = off; -1 = auto: C5's beam groups of 4, where it "
                         "measured fastest; coop elsewhere)")
    ap.add_argument("--shared", type=int, default=0,
                    help="sharing-aware decode on the CUDA cores over groups of this many sequences "
                         "(pa_paged_attention_decode_shared, SURVEY 8(f) N1; ablation, 0 = off)")
    ap.add_argument("--layers", type=int, default=0,
                    help="rotated layer caches (0 = auto: R x K/V read per step >= 4 x L2, R >= 2)")
    ap.add_argument("--no-plan", action="store_true",
                    help="natural grid order instead of pa_decode_plan's longest-first order (coop decode)")
    ap.add_argument("--shard-of", type=int, default=0,
                    help="run rank 0's head shard of a P-way tensor-parallel split on this one GPU (no exchange): "
                         "the per-rank kernel time of TP=P, a scaling proxy on a single-GPU box")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-prefill", action="store_true", help="skip the N4 prompt-phase context line")
    ap.add_argument("--extra", action="store_true", help="also print per-config lines for the other configs")
    ap.add_argument("--tp-gather", default="auto", choices=["auto", "fused", "nccl"],
                    help="N>1 output exchange: fused (attention stores into every rank's buffer over "
                         "CUDA IPC / NVLink, pa_paged_attention_decode_tp) or an NCCL all-gather; auto = fused "
                         "if the IPC setup succeeds")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("PA_BENCH_SAME_DEVICE") == "1":  # test only: every rank on cuda:0 (gloo)
        local = 0
    return world, rank, local


# --------------------------------------------------------------------- reference arm ---

def oracle_sample(wl, budget_s: float, steps_total: int):
    """Pick a bounded sample (sequences x heads) of the workload for the oracle."""
    import oracle
    from synth import materialize_numpy, shard, subset
    rs = np.random.default_rng(wl.seed)
    order = rs.permutation(wl.S)
    # heads: a slice of the heads keeps input generation small
    world = 1
    for w in (10, 8, 6, 5, 4, 3, 2, 1):
        if wl.H % w == 0 and wl.H_kv % w == 0 and wl.H // w >= 2:
            world = w
            break
    nseq = 8
    while True:
        sub = shard(subset(wl, sorted(order[:nseq].tolist())), 0, world)
        x = materialize_numpy(sub)
        args = (x["query"], x["key_cache"], x["value_cache"], sub.block_tables, sub.context_lens, sub.scale, sub.B,
                sub.H_kv, sub.dtype)
        t0 = time.perf_counter()
        oracle.paged_attention(*args)
        dt = time.perf_counter() - t0
        if dt * steps_total <= budget_s or nseq == 1:
            return sub, args, dt
        nseq = max(1, nseq // 2)


def run_reference(a, wl, world, rank):
    if rank != 0:
        return
    import oracle
    threads = oracle.max_threads()
    sub, args, dt = oracle_sample(wl, budget_s=150.0, steps_total=a.steps + a.warmup)
    for _ in range(a.warmup):
        oracle.paged_attention(*args)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        oracle.paged_attention(*args)
    el = time.perf_counter() - t0
    kv = sub.logical_kv_bytes()
    gbs = kv * a.steps / el / 1e9
    sample = f"{sub.S} of {wl.S} sequences x {sub.H} of {wl.H} heads per step (ctx sum {int(sub.context_lens.sum())})"
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": el / a.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": wl.name, "seqs": wl.S, "heads": wl.H, "head_dim": wl.D, "block_size": wl.B,
                       "kv_dtype": wl.dtype},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- our arm ---------

def layer_count(kv_layer_bytes: int, l2_bytes: int, cache_alloc_bytes: int, free_bytes: int, forced: int = 0):
    """R rotated layer caches: R x (K/V bytes one layer-step reads) >= 4 x L2,
    R >= 2, at most 96 (OPT-175B's layer count; only tiny configs such as C1, which make no
    HBM claim, hit it), and the R caches fit in 60% of the free device memory."""
    if forced > 0:
        return forced
    r = min(96, max(2, math.ceil(4 * l2_bytes / max(1, kv_layer_bytes))))
    fit = max(1, int(0.6 * free_bytes // max(1, cache_alloc_bytes)))
    return max(1, min(r, fit))


def pct(xs, q):
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


def run_ours(a, wl_full, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2309_06180_b200 as pa
    from paper_2309_06180_b200.tp import gather_heads
    from synth import materialize_torch, shard, tables_torch

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    props = torch.cuda.get_device_properties(dev)
    l2_bytes = int(getattr(props, "L2_cache_size", 0) or 126 * (1 << 20))
    if a.shard_of > 1 and world > 1:
        raise SystemExit("--shard-of simulates one rank on one GPU; run it without torchrun")
    wl = shard(wl_full, rank, world) if world > 1 else (shard(wl_full, 0, a.shard_of) if a.shard_of > 1 else wl_full)
    tb = tables_torch(wl, dev)
    bt, cl, sm, bm = tb["block_tables"], tb["context_lens"], tb["slot_mapping"], tb["block_mapping"]
    # R layer caches rotated step by step, so consecutive steps never re-read a cache that
    # could still sit in L2 (the rank's shard can be smaller than L2 at TP=8)
    kv_unique_rank = wl.unique_kv_bytes()
    cache_alloc = 2 * wl.num_blocks * wl.H_kv * wl.B * wl.D * wl.elem_bytes
    free_b, _ = torch.cuda.mem_get_info(dev)
    R = layer_count(min(kv_unique_rank, wl.logical_kv_bytes()), l2_bytes, cache_alloc, free_b, a.layers)
    layers = [materialize_torch(wl, dev, layer=l) for l in range(R)]
    x = layers[0]
    q = x["query"]
    out = torch.empty_like(q)
    mcl = wl.max_context_len
    ws_n = pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, mcl, a.partition_tokens)
    ws = torch.zeros(max(ws_n, 16), dtype=torch.uint8, device=dev)
    gathered = torch.empty((world * wl.S, wl.H, wl.D), dtype=q.dtype, device=dev) if world > 1 else None
    full_out = torch.empty((wl.S, wl.H * world, wl.D), dtype=q.dtype, device=dev) if world > 1 else None
    tp_gather, ftp = "none", None
    if world > 1:
        tp_gather = "nccl"
        if a.tp_gather in ("auto", "fused") and not a.unfused:
            from paper_2309_06180_b200.tp import FusedTP
            try:
                ftp = FusedTP(None, wl.S, wl.H * world, wl.D, q.dtype, dev)
                tp_gather = "fused"
            except Exception as exc:  # e.g. CUDA IPC not permitted in this container
                if a.tp_gather == "fused":
                    raise
                tp_gather = f"nccl (fused setup failed: {type(exc).__name__}: {exc})"
    has_pairs = len(wl.block_mapping) > 0
    # the tcgen05 N1 kernel on the sharing configs: C5's beams, and c3_fork (samples right
    # after the fork share all but their last block); c3_parallel (samples diverged:
    # unique/logical 0.72) stays on coop (258 vs 328 us).  TP shards of C5 have few (group,
    # 4 heads) items per SM, which the kernel's split context covers: TP=8/4/2 shards 66.6 /
    # 102 / 174 us vs coop 76.7 / 141 / 275 (profiles/r02_tp_shard_n1_split.jsonl)
    auto_grouped = {"c5_beam": 4, "c3_fork": 6}.get(wl_full.name, 0)
    grouped = a.grouped if a.grouped >= 0 else auto_grouped
    if a.shared > 0 or ftp is not None or a.unfused:
        grouped = 0 if a.grouped < 0 else grouped
    if grouped and (ftp is not None or a.unfused):
        raise SystemExit("--grouped runs the single-GPU fused decode step only")
    shared_g = a.shared
    if ftp is not None or a.unfused or grouped:
        if a.shared > 0:
            raise SystemExit("--shared runs the single-GPU fused decode step only")
        shared_g = 0
    stream = torch.cuda.current_stream(dev)

    # longest-first grid order from the host context lengths, once per decode iteration
    # (every layer reuses it, like the block tables): scheduling only, bit-identical output
    use_plan = not a.no_plan and not shared_g
    plan = pa.decode_plan(wl.context_lens) if use_plan else None
    if ftp is not None:
        # the fused gather (N2) is checked once against the NCCL all-gather of the same step on
        # every rank before anything is timed: a bitwise mismatch or a flag-wait timeout on this
        # node's peer links makes every rank fall back to NCCL (the decision is all-reduced)
        L0 = layers[0]
        bad = 0
        try:
            got = ftp.decode(L0["query"], L0["key"], L0["value"], L0["key_cache"], L0["value_cache"], bt, cl, wl.scale,
                             max_context_len=mcl, workspace=ws, seq_order=plan).clone()
            torch.cuda.synchronize(dev)
            pa.paged_attention_decode(out, L0["query"], L0["key"], L0["value"], L0["key_cache"], L0["value_cache"], bt,
                                      cl, wl.scale, max_context_len=mcl, workspace=ws, seq_order=plan)
            want = gather_heads(out, buffer=gathered)
            torch.cuda.synchronize(dev)
            bad = int(int(ftp.status.item()) != 0 or not torch.equal(got, want))
        except Exception as exc:  # noqa: BLE001 -- any failure of the fused path means: use NCCL
            print(f"rank {rank}: fused TP gather check failed: {type(exc).__name__}: {exc}", file=sys.stderr)
            bad = 1
        flag = torch.tensor([bad], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if int(flag.item()) != 0:
            if a.tp_gather == "fused":
                raise SystemExit("--tp-gather fused: the fused gather does not match the NCCL all-gather here")
            ftp = None
            tp_gather = "nccl (the fused gather's check against NCCL failed on this node)"
    # every launch of the step prepared once per layer cache (pa.prepare: Python checks and
    # argument marshalling done up front), so the timed loop is not bound by host overhead
    def layer_calls(L):
        q, kn, vn, kc, vc = L["query"], L["key"], L["value"], L["key_cache"], L["value_cache"]
        pre = []
        if has_pairs:
            pre.append(pa.prepare(pa.copy_blocks, [kc], [vc], bm))
        if a.unfused:
            pre.append(pa.prepare(pa.reshape_and_cache, kn, vn, kc, vc, sm))
        if ftp is not None:  # attention + fused all-gather: rows stored into every rank's buffer
            attn = lambda: ftp.decode(q, kn, vn, kc, vc, bt, cl, wl.scale, max_context_len=mcl,  # noqa: E731
                                      workspace=ws, seq_order=plan)
        elif a.unfused:
            attn = pa.prepare(pa.paged_attention, out, q, kc, vc, bt, cl, wl.scale, max_context_len=mcl,
                              partition_tokens=a.partition_tokens, workspace=ws, seq_order=plan)
        elif grouped:  # N1: groups of sequences sharing blocks, QK^T / PV on the tensor cores
            attn = pa.prepare(pa.paged_attention_decode_grouped, out, q, kn, vn, kc, vc, bt, cl, wl.scale, grouped,
                              max_context_len=mcl, workspace=ws, seq_order=plan)
        elif shared_g:  # N1: groups of sequences sharing blocks, each distinct block staged once
            attn = pa.prepare(pa.paged_attention_decode_shared, out, q, kn, vn, kc, vc, bt, cl, wl.scale, shared_g,
                              max_context_len=mcl, workspace=ws)
        else:  # the decode step's cache write fused into the attention kernel
            attn = pa.prepare(pa.paged_attention_decode, out, q, kn, vn, kc, vc, bt, cl, wl.scale,
                              max_context_len=mcl, workspace=ws, seq_order=plan)
        return pre, attn

    calls = [layer_calls(L) for L in layers]
    post = world > 1 and ftp is None  # the one exchange: all-gather of the output head slices (NCCL)
    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]  # noqa: E731
    ev_s0, ev_a1 = mk(), mk()
    ev_a0 = mk() if calls[0][0] else ev_s0  # attention starts the step when nothing precedes it
    ev_s1 = mk() if post else ev_a1

    def step(j, i=None):
        pre, attn = calls[j % R]
        if i is not None:
            ev_s0[i].record(stream)
        for c in pre:
            c()
        if i is not None and ev_a0 is not ev_s0:
            ev_a0[i].record(stream)
        attn()
        if i is not None:
            ev_a1[i].record(stream)
        if post:
            full_out.copy_(gather_heads(out, buffer=gathered))
            if i is not None:
                ev_s1[i].record(stream)

    # warm-up behind a GPU sleep: the host's unblocked cost to issue one step is measured
    # here (in the timed loop the launch queue fills and the host waits on the GPU)
    for j in range(2):  # first launches load modules lazily (implicitly synchronising)
        step(j)
    torch.cuda.synchronize()
    torch.cuda._sleep(50_000_000)
    hw = time.perf_counter()
    for j in range(max(3, a.warmup)):
        step(j)
    host_issue_us = (time.perf_counter() - hw) / max(3, a.warmup) * 1e6
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    pa.take_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda._sleep(50_000_000)  # ~25 ms head start (untimed): the host queues steps ahead of the GPU
        e0.record(stream)
        h0 = time.perf_counter()
        for i in range(a.steps):
            step(i, i)
        host_us = (time.perf_counter() - h0) / a.steps * 1e6
        e1.record(stream)
        torch.cuda.synchronize()
    launches = pa.take_launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    step_ms = [ev_s0[i].elapsed_time(ev_s1[i]) for i in range(a.steps)]
    attn_l = [ev_a0[i].elapsed_time(ev_a1[i]) for i in range(a.steps)]
    gath_l = [ev_a1[i].elapsed_time(ev_s1[i]) for i in range(a.steps)] if post else [0.0]
    attn_ms = float(np.mean(attn_l))
    stats = [ms_total, attn_ms, pct(step_ms, 10), pct(step_ms, 50), pct(step_ms, 90), pct(attn_l, 10),
             pct(attn_l, 50), pct(attn_l, 90), float(np.mean(gath_l))]
    t = torch.tensor(stats, dtype=torch.float64, device=dev)
    per_rank = None
    if world > 1:
        allr = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allr, t)
        per_rank = torch.stack(allr).cpu().numpy()
        t = torch.as_tensor(per_rank.max(axis=0))
    stats = [float(v) for v in t.tolist()]
    ms_total, attn_ms = stats[0], stats[1]
    ms_step = ms_total / a.steps
    if ftp is not None:
        status = int(ftp.status.item())
        if status != 0:
            raise RuntimeError("fused TP all-gather: a flag wait timed out")
        ftp.close()

    # ---- e2e: the same step through pa_decode_step with pinned host buffers ----------
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, wl, world, dev, {"query": q, "key": x["key"], "value": x["value"]}, x["key_cache"],
                      x["value_cache"], mcl, ws, stream)

    del layers, x
    probe = read_probe(dev)
    n4 = None
    if world == 1 and not a.no_prefill:
        n4 = prefill_summary(dev)
    if rank != 0:
        return
    peak, peak_src = load_peaks()
    kv_all = wl_full.logical_kv_bytes() if a.shard_of <= 1 else wl.logical_kv_bytes()
    sb = wl.step_bytes()
    # per launch of the attention call on this rank: K/V read + q/out + tables (+ the fused new-token write)
    attn_bytes = sb["kv_logical"] + sb["q_out"] + sb["tables"] + (0 if a.unfused else sb["cache_write"] // 2)
    achieved = attn_bytes / (attn_ms * 1e-3) / 1e9
    # sequences that share physical blocks (parallel samples, beams: C3 / C5) read each
    # shared block once from HBM at best; SURVEY §8(d) quotes those configs' % of peak on
    # the UNIQUE K/V bytes, with the logical figure beside it
    kv_unique = kv_unique_rank
    shared = kv_unique < 0.99 * sb["kv_logical"]
    attn_bytes_u = attn_bytes - sb["kv_logical"] + kv_unique
    achieved_u = attn_bytes_u / (attn_ms * 1e-3) / 1e9
    value = kv_all / (ms_step * 1e-3) / 1e9
    ach = achieved_u if shared else achieved
    # ncu_traffic.json keys: the workload for its default kernel, _grouped / _coop otherwise
    default_kernel = grouped == auto_grouped and not shared_g
    traffic = None if a.shard_of > 1 else load_traffic(
        wl_full.name + ("" if default_kernel else "_grouped" if grouped else "_shared" if shared_g else "_coop"), world)
    read_kv = min(kv_unique, sb["kv_logical"])
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_step, "us_per_step": ms_step * 1e3, "higher_is_better": True,
        "scaling": "strong",  # heads of a fixed batch sharded over the ranks
        "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic (seeded; shapes of BASELINE.json configs)",
        "config": {"workload": wl_full.name, "seqs": wl_full.S, "heads": wl_full.H, "kv_heads": wl_full.H_kv,
                   "head_dim": wl_full.D, "block_size": wl_full.B, "kv_dtype": wl_full.dtype,
                   "mean_ctx": float(wl_full.context_lens.mean()), "max_ctx": int(wl_full.max_context_len),
                   "cow_pairs": int(len(wl_full.block_mapping)), "parallelism": (f"tp{world}" if a.shard_of <= 1 else
                                   f"rank 0 of tp{a.shard_of}, simulated on one GPU (no exchange)"),
                   "tp_gather": tp_gather,
                   "decode_kernel": (f"grouped{grouped} (N1, tensor cores)" if grouped else
                                     f"shared{shared_g} (N1, CUDA cores)" if shared_g else "coop"),
                   "partition_tokens": a.partition_tokens or pa.DEFAULT_PARTITION_TOKENS,
                   "layer_caches": R,
                   "grid_order": ("longest-first (pa_decode_plan from the host context lengths, once per iteration; "
                                  "scheduling only)" if use_plan else "natural"),
                   "l2": (f"{'inputs larger than L2' if R * read_kv >= 4 * l2_bytes else 'WORKING SET NOT >= 4x L2'}: "
                          f"{R} layer caches rotated step by step, each step reads "
                          f"{read_kv / 1e6:.1f} MB of K/V per rank ({R} x = {R * read_kv / 1e6:.0f} MB vs "
                          f"{l2_bytes / 1e6:.0f} MB L2 = {R * read_kv / l2_bytes:.1f}x); no flush")},
        "tokens_per_s": wl_full.S / (ms_step * 1e-3),
        "kv_tokens_per_s": float(wl_full.context_lens.sum()) / (ms_step * 1e-3),
        "frac_of_peak": value / peak,
        "step_us": {"mean": ms_step * 1e3, "p10": stats[2] * 1e3, "p50": stats[3] * 1e3, "p90": stats[4] * 1e3,
                    "host_issue_us": round(host_issue_us, 2), "host_loop_us": round(host_us, 2),
                    "note": "mean = whole timed region / steps; p10/p50/p90 of per-step CUDA events; max over ranks; "
                            "host_issue_us = rank 0's CPU time to issue one step (prepared calls) while the GPU is "
                            "busy elsewhere (warm-up behind a sleep): the loop is device-bound when it is below the "
                            "step time; host_loop_us = the timed loop's CPU time per step (blocks on a full queue)"},
        "roofline": {"bound": "hbm", "kernel": (f"paged_attention_group_tc_kernel (pa_paged_attention_decode_grouped, "
                                                 f"groups of {grouped}: each distinct block piece loaded once, QK^T "
                                                 f"and PV as tcgen05 MMAs; cache write fused)") if grouped else
                     (f"paged_attention_shared_kernel (pa_paged_attention_decode_shared, groups of {shared_g}: each "
                      f"distinct block staged once for the group's members; cache write fused)") if shared_g else
                     "paged_attention_kernel (pa_paged_attention_decode: cache write + attention + split-context "
                     "merge in one launch)" if not a.unfused else "paged_attention_kernel (pa_paged_attention)",
                     "achieved": ach, "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
                     "read_peak": probe["gbs"], "frac_of_read_peak": ach / probe["gbs"],
                     "algorithmic_bytes_per_launch": attn_bytes_u if shared else attn_bytes,
                     "basis": ("unique K/V bytes (blocks shared by samples/beams counted once; SURVEY 8(d))"
                               if shared else "logical K/V bytes (no sharing)"),
                     "achieved_logical": achieved, "frac_logical": achieved / peak,
                     "kv_unique_over_logical": kv_unique / sb["kv_logical"],
                     "avg_launch_ms": attn_ms,
                     "launch_us": {"p10": stats[5] * 1e3, "p50": stats[6] * 1e3, "p90": stats[7] * 1e3}},
        "read_probe": probe,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    if per_rank is not None:
        rb = attn_bytes_u if shared else attn_bytes
        line["per_rank"] = {
            "attention_gbs": [round(rb / (r[1] * 1e-3) / 1e9, 1) for r in per_rank],
            "frac_of_peak": [round(rb / (r[1] * 1e-3) / 1e9 / peak, 4) for r in per_rank],
            "step_us_p50": [round(r[3] * 1e3, 2) for r in per_rank],
            "gather_us": ([round(r[8] * 1e3, 2) for r in per_rank] if ftp is None else None),
            "gather_note": ("NCCL all_gather_into_tensor + permute, CUDA events after the attention launch"
                            if ftp is None else "fused: the all-gather stores happen inside the attention kernel "
                            "and its flag handshake; attention_gbs includes them")}
    if e2e is not None:
        line["e2e"] = e2e
    if n4 is not None:
        line["n4_prefill"] = n4
    if not a.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(wl_full)
    print(json.dumps(line), flush=True)


def prefill_summary(dev, name: str = "p_2k", iters: int = 20):
    """Context only (not the headline): the N4 prompt-phase kernel on one synth.prefill
    workload, timed the same way as scripts/prefill_bench.py (CUDA events, mean of
    `iters` launches after 3 warm-up), algorithmic TFLOP/s vs the measured bf16 peak."""
    import torch

    import paper_2309_06180_b200 as pa
    from synth.prefill import algorithmic_flops, make_prefill
    c = make_prefill(name)
    dt = torch.float16 if c["dtype"] == "f16" else torch.bfloat16
    g = torch.Generator(device=dev)
    g.manual_seed(c["seed"])
    D = 128
    kc = (torch.rand((c["num_blocks"], c["H_kv"], c["B"], D), generator=g, device=dev) * 2 - 1).to(dt)
    vc = (torch.rand(tuple(kc.shape), generator=g, device=dev) * 2 - 1).to(dt)
    T = int(c["qlen"].sum())
    q = (torch.rand((T, c["H"], D), generator=g, device=dev) * 2 - 1).to(dt)
    qs = torch.as_tensor(np.concatenate([[0], np.cumsum(c["qlen"])]).astype(np.int32), device=dev)
    bt = torch.as_tensor(c["block_tables"], device=dev)
    cl = torch.as_tensor(c["ctx"].astype(np.int32), device=dev)
    out = torch.empty_like(q)
    mql = int(c["qlen"].max())
    ws = torch.empty(16, dtype=torch.uint8, device=dev)
    for _ in range(3):
        pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, D ** -0.5, max_query_len=mql, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, D ** -0.5, max_query_len=mql, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tflops = algorithmic_flops(c["ctx"], c["qlen"], c["H"], D) / (ms * 1e-3) / 1e12
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak = float(json.load(f)["bf16_tflops"])
    except Exception:
        peak = 2250.0
    return {"workload": name, "ms": round(ms, 4), "tflops": round(tflops, 1), "peak_tflops": peak,
            "frac": round(tflops / peak, 3), "bound": "tensor", "query_tokens": T,
            "note": "tcgen05 prompt-phase kernel (SURVEY §8(f) N4), context only; see DESIGN.md §8c"}


PROBE_SHAPES = ((8192, 3, 4), (32768, 2, 2), (65536, 2, 1))  # (chunk B, stages, CTAs/SM): the best of
# scripts/read_probe.py's sweep on a B200 (profiles/r02_read_probe.txt), 7.37-7.39 TB/s


def read_probe(dev, gib: float = 4.0):
    """Same-run read-only HBM ceiling: pa_hbm_read_probe streams a 4 GiB
    buffer into shared memory with 1-D bulk copies (the attention kernel's load path) and
    writes nothing but one word per CTA; best of 6.  Beside it, torch's copy (read+write,
    the MEASURED_PEAKS method) in the same run."""
    import torch

    import paper_2309_06180_b200 as pa
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    x = torch.empty(int(gib * (1 << 30)), dtype=torch.uint8, device=dev)
    x.fill_(1)
    sink = torch.zeros(8 * sms, dtype=torch.int32, device=dev)

    def best_of(fn, nbytes, n=6):
        b = 0.0
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            b = max(b, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        return round(b, 1)

    shapes = {}
    for chunk, stages, cps in PROBE_SHAPES:
        shapes[f"{chunk}x{stages}x{cps}"] = best_of(
            lambda: pa.hbm_read_probe(x, sink, chunk=chunk, stages=stages, ctas=cps * sms), x.numel())
    gbs = max(shapes.values())
    half = x.numel() // 2
    a_, b_ = x[:half], x[half:]
    copy = best_of(lambda: b_.copy_(a_), 2 * half)
    del x, a_, b_
    return {"gbs": gbs, "copy_gbs": copy, "shapes": shapes,
            "how": f"pa_hbm_read_probe: {gib:g} GiB streamed into shared memory by bulk copies (chunk B x stages x "
                   "CTAs/SM as keyed in shapes), no global writes, best of 6 each, gbs = the max; copy_gbs = torch "
                   "copy_ of 2 GiB (read+write bytes)"}


def run_e2e(a, wl, world, dev, x, kc, vc, mcl, ws, stream):
    """Same metric measured through pa_decode_step: per step H2D of the step's inputs
    from pinned host memory, the kernels, and D2H of the output."""
    import torch

    import paper_2309_06180_b200 as pa
    pin = {k: x[k].cpu().pin_memory() for k in ("query", "key", "value")}
    host = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory() for k, v in
            dict(slot=wl.slot_mapping, bt=wl.block_tables, cl=wl.context_lens,
                 bm=wl.block_mapping.reshape(-1, 2)).items()}
    out = torch.empty(pin["query"].shape, dtype=pin["query"].dtype).pin_memory()
    st = torch.empty(pa.decode_step_staging_size(wl.S, wl.H, wl.H_kv, wl.D, wl.W, len(wl.block_mapping),
                                                 pin["query"].dtype), dtype=torch.uint8, device=dev)
    # bytes pa_decode_step copies: q, k, v, block tables, context lengths, CoW pairs (the
    # slot mapping is implied by the tables and not sent)
    h2d = sum(t.numel() * t.element_size() for t in list(pin.values()) + [host["bt"], host["cl"]]) + \
        (host["bm"].numel() * host["bm"].element_size() if len(wl.block_mapping) else 0)
    d2h = out.numel() * out.element_size()
    steps = max(10, min(a.steps, 200))

    def one():
        pa.decode_step(out, pin["query"], pin["key"], pin["value"], host["slot"], host["bt"], host["cl"], host["bm"],
                       kc, vc, wl.scale, st, ws, max_context_len=mcl, stream=stream)

    for _ in range(3):
        one()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h0 = time.perf_counter()
    for _ in range(steps):
        one()
    host_us = (time.perf_counter() - h0) / steps * 1e6  # CPU time to enqueue one step
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0])
    kv_all = wl.logical_kv_bytes() * world
    return {"value": kv_all / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms, "steps": steps,
            "host_enqueue_us_per_step": round(host_us, 1),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": "pa_decode_step (C ABI, pinned host buffers)",
            "transfer": ("zero-copy: kernel reads q/k/v and writes out over the host link; tables copied"
                         if os.environ.get("PA_E2E_MODE") == "zerocopy" else
                         "copy-engine chunks (PA_E2E_CHUNKS, default 4) overlapped with the chunk kernels" +
                         ("; the step is captured once into a CUDA graph and replayed"
                          if os.environ.get("PA_E2E_GRAPH") == "1" else ""))}


def cpu_baseline(wl, target_s: float = 10.0):
    """The oracle as it stands, on the host cores, over a bounded sample of the same
    workload: every sequence, a slice of the heads; repeated for ~target_s seconds."""
    import oracle
    from synth import materialize_numpy, shard
    world = 1
    for w in (10, 8, 6, 5, 4, 3, 2, 1):
        if wl.H % w == 0 and wl.H_kv % w == 0:
            world = w
            break
    sub = shard(wl, 0, world)
    x = materialize_numpy(sub)
    args = (x["query"], x["key_cache"], x["value_cache"], sub.block_tables, sub.context_lens, sub.scale, sub.B,
            sub.H_kv, sub.dtype)
    oracle.paged_attention(*args)
    reps, t0 = 0, time.perf_counter()
    while True:
        oracle.paged_attention(*args)
        reps += 1
        el = time.perf_counter() - t0
        if el >= target_s:
            break
    per = el / reps
    res = {"value": sub.logical_kv_bytes() / per / 1e9, "unit": "GB/s", "cores": oracle.max_threads(),
           "kind": "oracle", "sample": f"all {wl.S} sequences x {sub.H} of {wl.H} heads (heads {sub.q_head0}.."
                                       f"{sub.q_head0 + sub.H - 1}), {reps} reps x {per:.3f} s (fp64 C, OpenMP)"}
    # the same oracle on ONE host thread (one head of the sample, ~target_s / 4 seconds)
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        n_all = oracle.max_threads()
        gomp.omp_set_num_threads(1)
        try:
            one = shard(wl, 0, wl.H)  # one query head
            x1 = materialize_numpy(one)
            a1 = (x1["query"], x1["key_cache"], x1["value_cache"], one.block_tables, one.context_lens, one.scale,
                  one.B, one.H_kv, one.dtype)
            reps1, t1 = 0, time.perf_counter()
            while True:
                oracle.paged_attention(*a1)
                reps1 += 1
                el1 = time.perf_counter() - t1
                if el1 >= target_s / 4:
                    break
            res["single_core"] = {"value": one.logical_kv_bytes() / (el1 / reps1) / 1e9, "unit": "GB/s", "cores": 1,
                                  "sample": f"all {wl.S} sequences x 1 head, {reps1} reps"}
        finally:
            gomp.omp_set_num_threads(n_all)
    except OSError:
        pass
    return res


def main():
    a = parse()
    world, rank, local = dist_env()
    from synth import make_config
    over = {"B": a.block_size} if a.block_size else {}
    wl = make_config(a.config, **over)
    if a.impl == "reference":
        run_reference(a, wl, world, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        backend = os.environ.get("PA_BENCH_BACKEND", "nccl")  # gloo: multi-rank test on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(a, wl, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
