"""Context only (not a bench line, not the product path): the decode attention kernel of
this repo next to two library decode kernels on the SAME synthetic workloads.

  * vLLM `paged_attention_v1` / `paged_attention_v2` (vllm._C, precompiled for sm_100):
    the kernel of the paper's artifact (P:416-427 -- FasterTransformer-derived, a warp
    per block, v2 = 512-token partitions + reduce), i.e. the paper's own design
    recompiled for B200.  Its key cache layout is [NB][H_kv][D/x][B][x] and its value
    cache [NB][H_kv][D][B], so the caches are re-laid out once (outside the timing).
  * FlashInfer `trtllm_batch_decode_with_kv_cache` (prebuilt TRT-LLM-gen cubins for
    Blackwell): HND layout [NB][H_kv][B][D] with the same block tables, i.e. it runs on
    this repo's caches as they are.

Every kernel reads the same logical K/V bytes; GB/s = logical K/V bytes / mean time over
`--iters` back-to-back launches (CUDA events on the launching stream, after warm-up).
Each library output is compared with this repo's output (max-abs) so the timings are of
correct computations.  One JSON line per (config, kernel).

  python scripts/compare_libs.py c2_sharegpt c2_alpaca c4_long
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from synth import make_config, materialize_torch, tables_torch  # noqa: E402


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2_sharegpt", "c2_alpaca", "c4_long"])
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    for name in a.configs:
        wl = make_config(name)
        x = materialize_torch(wl, "cuda", poison=False)
        tb = tables_torch(wl, "cuda")
        q, kc, vc = x["query"], x["key_cache"], x["value_cache"]
        bt, cl = tb["block_tables"], tb["context_lens"]
        mcl = int(wl.max_context_len)
        kv = wl.logical_kv_bytes()
        base = {"config": name, "seqs": wl.S, "heads": wl.H, "kv_heads": wl.H_kv, "head_dim": wl.D,
                "block_size": wl.B, "dtype": wl.dtype, "kv_bytes": kv}

        def report(kernel, sec, out, ref, note=None):
            d = dict(base, kernel=kernel, us=round(sec * 1e6, 2), kv_GBps=round(kv / sec / 1e9, 1))
            if ref is not None:
                d["max_abs_vs_ours"] = float((out.float() - ref.float()).abs().max())
            if note:
                d["note"] = note
            print(json.dumps(d), flush=True)

        ours = torch.empty_like(q)
        ws = torch.zeros(max(16, pa.paged_attention_workspace_size(wl.S, wl.H, wl.D, mcl)), dtype=torch.uint8,
                         device="cuda")

        def run_ours():
            pa.paged_attention(ours, q, kc, vc, bt, cl, wl.scale, max_context_len=mcl, workspace=ws)

        report("ours: pa_paged_attention (coop, attention only)", time_it(run_ours, a.iters), ours, None)
        ref = ours.clone()

        # ---- vLLM (the paper's kernel) -------------------------------------------------
        try:
            import vllm._custom_ops as vops
            xv = 16 // q.element_size()
            NB, Hk, B, D = kc.shape
            vk = kc.view(NB, Hk, B, D // xv, xv).permute(0, 1, 3, 2, 4).contiguous()
            vv = vc.permute(0, 1, 3, 2).contiguous()
            one = torch.ones((), dtype=torch.float32, device="cuda")
            out = torch.empty_like(q)

            def v1():
                vops.paged_attention_v1(out, q, vk, vv, Hk, wl.scale, bt, cl, B, mcl, None, "auto", one, one)

            report("vllm paged_attention_v1 (paper's kernel)", time_it(v1, a.iters), out, ref)
            NPt = (mcl + 511) // 512
            es = torch.empty((wl.S, wl.H, NPt), dtype=torch.float32, device="cuda")
            ml = torch.empty_like(es)
            tmp = torch.empty((wl.S, wl.H, NPt, D), dtype=q.dtype, device="cuda")

            def v2():
                vops.paged_attention_v2(out, es, ml, tmp, q, vk, vv, Hk, wl.scale, bt, cl, B, mcl, None, "auto", one,
                                        one)

            report("vllm paged_attention_v2 (paper's kernel, 512-token partitions)", time_it(v2, a.iters), out, ref)
            del vk, vv
        except Exception as e:  # library missing or shape unsupported
            print(json.dumps(dict(base, kernel="vllm paged_attention", error=str(e)[:200])), flush=True)

        # ---- FlashInfer TRT-LLM-gen decode (Blackwell cubins) ---------------------------
        try:
            import flashinfer
            fws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            out = torch.empty_like(q)

            def fi():
                flashinfer.decode.trtllm_batch_decode_with_kv_cache(q, (kc, vc), fws, bt, cl, mcl,
                                                                    bmm1_scale=wl.scale, bmm2_scale=1.0, out=out,
                                                                    kv_layout="HND")

            report("flashinfer trtllm_batch_decode_with_kv_cache (TRT-LLM-gen)", time_it(fi, a.iters), out, ref)
        except Exception as e:
            print(json.dumps(dict(base, kernel="flashinfer trtllm decode", error=str(e)[:300])), flush=True)
        del x, q, kc, vc
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
