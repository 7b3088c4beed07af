"""Prompt-phase (N4) benchmark: pa_paged_prefill_attention on the synth.prefill workloads.

Per config, one JSON line: kernel time (CUDA events on the launching stream, mean over
`--iters` back-to-back launches after warm-up), algorithmic TFLOP/s (4*D flops per
(query row, head, attended token), causal) against the measured dense bf16 peak of
MEASURED_PEAKS.json (f16 has the same nominal tensor rate), query tokens/s, and as
context torch's scaled_dot_product_attention on the same prompts with CONTIGUOUS K/V
(no paging; library kernels, padded batch) where the prompts are uniform (p_2k), and the
fp64 oracle (oracle.prefill_attention, as it stands) timed on the host cores on a bounded
sample of the same workload (`cpu_baseline`, TFLOP/s of the sample's algorithmic flops).
Caches hold U(-1,1) values; unused slots are NaN.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)  # the oracle (cpu_baseline only) and tests.pathutil live at the repo root

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from synth.prefill import PREFILL_CONFIGS, algorithmic_flops, make_prefill  # noqa: E402

D = 128


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["bf16_tflops"]), "MEASURED_PEAKS.json bf16_tflops (burst)"
    except Exception:
        return 2250.0, "nominal dense bf16 (B200_PROFILING.md fallback)"


def time_it(fn, iters, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / iters


def build(c, dev="cuda"):
    dt = torch.float16 if c["dtype"] == "f16" else torch.bfloat16
    g = torch.Generator(device=dev)
    g.manual_seed(c["seed"])
    H, Hk, B, NB = c["H"], c["H_kv"], c["B"], c["num_blocks"]
    kc = (torch.rand((NB, Hk, B, D), generator=g, device=dev) * 2 - 1).to(dt)
    vc = (torch.rand((NB, Hk, B, D), generator=g, device=dev) * 2 - 1).to(dt)
    T = int(c["qlen"].sum())
    q = (torch.rand((T, H, D), generator=g, device=dev) * 2 - 1).to(dt)
    qs = torch.as_tensor(np.concatenate([[0], np.cumsum(c["qlen"])]).astype(np.int32), device=dev)
    return q, kc, vc, torch.as_tensor(c["block_tables"], device=dev), \
        torch.as_tensor(c["ctx"].astype(np.int32), device=dev), qs


def oracle_baseline(c, q, kc, vc, bt, cl, budget_rows=512, heads=4):
    """The fp64 oracle on a bounded sample: the last `budget_rows` query rows of the
    longest sequence (the most expensive rows) x `heads` query heads (and their kv heads)."""
    import time

    import oracle
    from tests.pathutil import bits
    s = int(np.argmax(c["ctx"]))
    ql, ctx = int(c["qlen"][s]), int(c["ctx"][s])
    n = min(budget_rows, ql)
    qs_all = np.concatenate([[0], np.cumsum(c["qlen"])])
    rows = bits(q[qs_all[s] + ql - n: qs_all[s] + ql, :heads])
    G = c["H"] // c["H_kv"]
    kvh = max(1, heads // G)
    kcs, vcs = bits(kc[:, :kvh].contiguous()), bits(vc[:, :kvh].contiguous())
    t0 = time.perf_counter()
    oracle.prefill_attention(rows, kcs, vcs, bt[s:s + 1].cpu().numpy(), np.array([ctx], np.int32),
                             np.array([0, n], np.int32), 1.0 / np.sqrt(D), c["B"], kvh, c["dtype"])
    dt = time.perf_counter() - t0
    flops = algorithmic_flops(np.array([ctx]), np.array([n]), heads, D)
    return {"value": round(flops / dt / 1e12, 6), "unit": "TFLOP/s", "cores": oracle.max_threads(), "kind": "oracle",
            "sample": f"last {n} query rows of the longest sequence (ctx {ctx}) x {heads} heads, {dt:.2f} s"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default=",".join(PREFILL_CONFIGS))
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--block-size", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--packed-all", action="store_true",
                    help="also time the packed entry on workloads without a shared prefix (shared = 0)")
    args = ap.parse_args()
    peak, peak_src = peaks()
    for name in args.configs.split(","):
        c = make_prefill(name, **({"B": args.block_size} if args.block_size else {}))
        q, kc, vc, bt, cl, qs = build(c)
        out = torch.empty_like(q)
        mql = int(c["qlen"].max())
        scale = 1.0 / np.sqrt(D)
        ws = torch.empty(16, dtype=torch.uint8, device="cuda")
        fn = lambda: pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, scale, max_query_len=mql,  # noqa: E731
                                                workspace=ws)
        pa.take_launch_count()
        t = time_it(fn, args.iters)
        launches = pa.take_launch_count() / (args.iters + 5)
        flops = algorithmic_flops(c["ctx"], c["qlen"], c["H"], D)
        tf = flops / t / 1e12
        res = {"config": name, "block_size": c["B"], "seqs": len(c["ctx"]), "query_tokens": int(c["qlen"].sum()),
               "mean_ctx": round(float(c["ctx"].mean()), 1), "ms": round(t * 1e3, 4),
               "tflops": round(tf, 1), "peak_tflops": peak, "peak_src": peak_src, "frac": round(tf / peak, 3),
               "query_tokens_per_s": round(c["qlen"].sum() / t, 0), "launches_per_call": launches}
        if c["kind"] == "prefix" or args.packed_all:  # the packed (cascade) entry on the same workload
            hqs = np.concatenate([[0], np.cumsum(c["qlen"])]).astype(np.int32)
            shared = c["shared"] if "shared" in c else np.zeros(len(c["ctx"]), np.int32)
            fnp = lambda: pa.paged_prefill_attention_packed(  # noqa: E731
                out, q, kc, vc, bt, cl, qs, scale, hqs, c["ctx"].astype(np.int32), shared.astype(np.int32),
                max_query_len=mql, workspace=ws)
            tp = time_it(fnp, args.iters)
            res["packed_ms"] = round(tp * 1e3, 4)
            res["packed_tflops"] = round(flops / tp / 1e12, 1)
            res["packed_frac"] = round(flops / tp / 1e12 / peak, 3)
        if name == "p_2k":  # library context: contiguous causal SDPA, same flops
            S, n = len(c["ctx"]), int(c["ctx"][0])
            qq = q.view(S, n, c["H"], D).transpose(1, 2).contiguous()
            kk = torch.rand_like(qq)
            vv = torch.rand_like(qq)
            ts = time_it(lambda: torch.nn.functional.scaled_dot_product_attention(qq, kk, vv, is_causal=True),
                         args.iters)
            res["sdpa_contiguous_ms"] = round(ts * 1e3, 4)
            res["sdpa_contiguous_tflops"] = round(flops / ts / 1e12, 1)
        if not args.no_cpu_baseline:
            res["cpu_baseline"] = oracle_baseline(c, q, kc, vc, bt, cl)
        print(json.dumps(res), flush=True)
        del q, kc, vc, out


if __name__ == "__main__":
    main()
