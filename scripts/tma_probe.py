"""Tensor-copy (cp.async.bulk.tensor, 128-B swizzle) vs plain bulk-copy throughput per SM on
a B200: boxes {64 cols x rows} of 2-byte elements at random box-aligned rows of a 4 GiB
tensor, 1-4 issuing warps per SM, several copies in flight each (pa_debug_tma_probe), and
pa_hbm_read_probe's plain 1-D bulk copies of the same sizes.  Prints GB/s per shape."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2309_06180_b200 as pa  # noqa: E402
from paper_2309_06180_b200 import _lib  # noqa: E402

L = _lib.raw()
f = L.pa_debug_tma_probe
f.restype = ctypes.c_int
f.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
              ctypes.c_void_p, ctypes.c_void_p]
dev = torch.device("cuda", 0)
sms = torch.cuda.get_device_properties(dev).multi_processor_count
buf = torch.ones(4 << 30, dtype=torch.uint8, device=dev)
nrows = buf.numel() // 256
sink = torch.zeros(8 * sms, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream().cuda_stream


def timed(fn, nbytes, reps=3):
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return round(best, 1)


if "--l2" in sys.argv:  # L2-resident source (32 MiB of the tensor), 16-row boxes, 1-8 issuing warps
    for rows in (16, 64):
        for warps in (1, 2, 4, 8):
            stages = max(2, min(16, (64 * 1024) // (rows * 128 * warps)))
            iters = max(64, (48 << 20) // (rows * 128 * warps * sms) * 4)
            nbytes = sms * warps * iters * rows * 128
            nr = (32 << 20) // 256

            def run():
                r = f(buf.data_ptr(), nr, rows, warps, stages, iters, sms, sink.data_ptr(), st)
                assert r == 0, r
            run()
            torch.cuda.synchronize()
            g = timed(run, nbytes)
            print(json.dumps({"kind": "tma_tensor_sw128_l2", "box_bytes": rows * 128, "warps_per_sm": warps,
                              "stages_per_warp": stages, "gbs": g, "per_sm_gbs": round(g / sms, 2)}), flush=True)
    sys.exit(0)
for rows in (16, 32, 64, 128):
    for warps in (1, 2, 4):
        stages = max(2, min(16, (64 * 1024) // (rows * 128 * warps)))
        iters = max(64, (48 << 20) // (rows * 128 * warps * sms) * 4)
        nbytes = sms * warps * iters * rows * 128

        def run():
            r = f(buf.data_ptr(), nrows, rows, warps, stages, iters, sms, sink.data_ptr(), st)
            assert r == 0, r
        run()
        torch.cuda.synchronize()
        print(json.dumps({"kind": "tma_tensor_sw128", "box_bytes": rows * 128, "warps_per_sm": warps,
                          "stages_per_warp": stages, "gbs": timed(run, nbytes),
                          "per_sm_B_per_clk": None}), flush=True)
for chunk in (2048, 4096, 8192, 16384, 32768):
    for cps in (1, 2, 4):
        stages = max(2, min(16, (64 * 1024) // chunk))
        if cps * stages * chunk > 200 * 1024:
            continue
        gbs = timed(lambda: pa.hbm_read_probe(buf, sink, chunk=chunk, stages=stages, ctas=cps * sms), buf.numel())
        print(json.dumps({"kind": "bulk_1d", "chunk_bytes": chunk, "ctas_per_sm": cps, "stages": stages, "gbs": gbs}),
              flush=True)
