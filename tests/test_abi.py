"""C-ABI checks that need no GPU: the library loads, exports every symbol include/pa.h
declares, rejects bad arguments on the host before any launch, and its host block
allocator matches the reference block manager (oracle/block_manager.py) and the
paper's worked examples (P:N = PAPER.md line N)."""
import ctypes
import os
import random
import re

import numpy as np
import pytest

from oracle.block_manager import BlockManager, OutOfBlocks

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pa = pytest.importorskip("paper_2309_06180_b200")
from paper_2309_06180_b200 import _lib  # noqa: E402

L = _lib.raw()
OK, INVALID, UNSUPPORTED, WORKSPACE, OOB = 0, 1, 2, 3, 5


def header_functions():
    txt = open(os.path.join(ROOT, "include", "pa.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pa_[a-z0-9_]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported():
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), f"{n} declared in pa.h but not exported"


def test_library_is_sm100a_only():
    """The shared library carries sm_100a SASS (no PTX JIT fallback for other archs)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in sass          # bulk async copies global -> shared
    assert "FHFMA" in sass           # mixed-precision FMA for q.k
    assert "FFMA2" in sass           # packed fp32x2 FMA for p*V
    assert "UTCHMMA" in sass         # tcgen05.mma kind::f16 (prefill attention, N4)
    assert "UTMALDG" in sass         # TMA tensor loads (prefill attention)
    assert "LDTM" in sass            # tcgen05.ld tensor memory -> registers


FAKE = 0x100000  # aligned, never dereferenced: every call below fails validation first


def attn(**kw):
    a = dict(out=FAKE, q=FAKE, kc=FAKE, vc=FAKE, bt=FAKE, cl=FAKE, scale=0.125, B=16, hkv=2, S=4, H=2, D=64, W=8,
             mcl=100, dt=0, pt=0, ws=None, wsb=0)
    a.update(kw)
    return L.pa_paged_attention_ex(a["out"], a["q"], a["kc"], a["vc"], a["bt"], a["cl"], a["scale"], a["B"], a["hkv"],
                                   a["S"], a["H"], a["D"], a["W"], a["mcl"], a["dt"], a["pt"], a.get("order"), a["ws"],
                                   a["wsb"], None)


@pytest.mark.parametrize("kw,status", [
    (dict(D=96), UNSUPPORTED),
    (dict(B=3), UNSUPPORTED),
    (dict(B=512), UNSUPPORTED),
    (dict(H=3, hkv=2), INVALID),
    (dict(hkv=0), INVALID),
    (dict(out=None), INVALID),
    (dict(q=FAKE + 8), INVALID),
    (dict(bt=FAKE + 2), INVALID),
    (dict(dt=7), INVALID),
    (dict(pt=24), INVALID),
    (dict(scale=float("nan")), INVALID),
    (dict(mcl=2048, W=128), WORKSPACE),
    (dict(mcl=2048, W=128, ws=FAKE, wsb=16), WORKSPACE),
])
def test_attention_argument_validation(kw, status):
    assert attn(**kw) == status
    assert _lib.last_error() != ""


def prefill(**kw):
    a = dict(out=FAKE, q=FAKE, kc=FAKE, vc=FAKE, bt=FAKE, cl=FAKE, qs=FAKE, scale=0.125, B=16, hkv=2, NB=64, S=4, H=2,
             D=128, W=8, T=100, mql=40, dt=2, ws=FAKE, wsb=16)
    a.update(kw)
    return L.pa_paged_prefill_attention(a["out"], a["q"], a["kc"], a["vc"], a["bt"], a["cl"], a["qs"], a["scale"],
                                        a["B"], a["hkv"], a["NB"], a["S"], a["H"], a["D"], a["W"], a["T"], a["mql"],
                                        a["dt"], a["ws"], a["wsb"], None)


@pytest.mark.parametrize("kw,status", [
    (dict(D=64), UNSUPPORTED),
    (dict(dt=0), UNSUPPORTED),
    (dict(B=3), UNSUPPORTED),
    (dict(H=3, hkv=2), INVALID),
    (dict(NB=0), INVALID),
    (dict(out=None), INVALID),
    (dict(q=FAKE + 8), INVALID),
    (dict(qs=FAKE + 2), INVALID),
    (dict(dt=7), INVALID),
    (dict(scale=float("inf")), INVALID),
    (dict(NB=1 << 28, hkv=8, H=8), INVALID),
    (dict(ws=None), WORKSPACE),
    (dict(wsb=8), WORKSPACE),
    (dict(ws=FAKE + 4), INVALID),
])
def test_prefill_argument_validation(kw, status):
    assert prefill(**kw) == status
    assert _lib.last_error() != ""


def test_prefill_empty_is_noop():
    assert prefill(T=0, out=None, q=None) == OK
    assert prefill(S=0, out=None) == OK


def test_attention_zero_seqs_is_noop():
    assert attn(S=0, out=None) == OK


def test_attention_requires_workspace():
    assert attn() == WORKSPACE


def test_workspace_size():
    """Counters + work list always; split partials only when a context needs > 1 partition."""
    f = L.pa_paged_attention_workspace_size
    assert 0 < f(4, 2, 64, 100, 0) < 1024
    assert f(4, 2, 64, 512, 0) == f(4, 2, 64, 100, 0)
    S, H, D = 256, 40, 128
    single = f(S, H, D, 512, 0)
    split = f(S, H, D, 2048, 0)
    assert split - single >= S * H * 4 * (D * 4 + 8)        # 4 partitions of o~ and (m, L)
    assert split - single < S * H * 4 * (D * 4 + 8) + S * 4 * 16 + 64
    assert f(S, H, D, 2048, 4096) == single


def test_cache_kernels_argument_validation():
    r = L.pa_reshape_and_cache
    assert r(FAKE, FAKE, FAKE, FAKE, FAKE, 4, 2, 96, 16, 1, None) == UNSUPPORTED
    assert r(FAKE, FAKE, FAKE, FAKE, FAKE + 4, 4, 2, 64, 16, 1, None) == INVALID
    assert r(None, FAKE, FAKE, FAKE, FAKE, 4, 2, 64, 16, 1, None) == INVALID
    assert r(None, None, None, None, None, 0, 2, 64, 16, 1, None) == OK
    c = L.pa_copy_blocks
    arr = (ctypes.c_void_p * 1)(FAKE)
    assert c(arr, arr, 0, FAKE, 1, 2, 16, 64, 1, None) == INVALID
    assert c(arr, arr, 300, FAKE, 1, 2, 16, 64, 1, None) == INVALID
    assert c(arr, arr, 1, None, 0, 2, 16, 64, 1, None) == OK
    bad = (ctypes.c_void_p * 1)(FAKE + 8)
    assert c(bad, arr, 1, FAKE, 1, 2, 16, 64, 1, None) == INVALID


def test_decode_step_staging_validation():
    need = L.pa_decode_step_staging_size(4, 2, 2, 64, 8, 0, 0)
    assert need > 0
    st = L.pa_decode_step
    r = st(FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None, 0, FAKE, FAKE, 0.1, 16, 2, 4, 2, 64, 8, 100, 0,
           FAKE, need - 1, None, 0, None)
    assert r == WORKSPACE


# ------------------------------------------------------------- host block allocator ----

def test_allocator_fig6_and_cow():
    """Fig.6 and the parallel-sampling copy-on-write."""
    a = pa.BlockAllocator(8, 4, [7, 1, 3, 0, 2, 4, 5, 6])
    h = a.allocate(7)
    bt, cl = a.export([h], 3)
    assert bt.tolist() == [[7, 1, -1]] and cl.tolist() == [7]
    c = a.fork(h)
    assert a.refcount(7) == 2 and a.refcount(1) == 2
    slot, cow = a.append_slot(h)
    assert cow == (1, 3) and slot == 3 * 4 + 3
    assert a.refcount(1) == 1
    assert a.append_slot(c) == (1 * 4 + 3, None)
    assert a.free(c) == 1 and a.free(h) == 2
    with pytest.raises(pa.PagedAttnError):
        a.free(h)
    with pytest.raises(ValueError):
        pa.BlockAllocator(4, 4, [0, 0, 1, 2])


def test_allocator_out_of_blocks():
    a = pa.BlockAllocator(2, 4)
    h = a.allocate(8)
    with pytest.raises(pa.PagedAttnError) as e:
        a.append_slot(h)
    assert e.value.status == OOB


def test_allocator_matches_reference_fuzz():
    """Same random op sequence on the C++ allocator and the reference block manager:
    identical handles, slots, copy-on-write pairs, refcounts and tables."""
    rs = random.Random(5)
    order = rs.sample(range(96), 96)
    a = pa.BlockAllocator(96, 4, order)
    m = BlockManager(96, 4, initial_order=order)
    live = []
    for step in range(6000):
        op = rs.random()
        if op < 0.15 or not live:
            n = rs.randint(1, 14)
            try:
                hm = m.allocate(n)
            except OutOfBlocks:
                with pytest.raises(pa.PagedAttnError):
                    a.allocate(n)
                h = live.pop(rs.randrange(len(live))) if live else None
                if h is not None:
                    assert a.free(h) == m.free(h)
                continue
            assert a.allocate(n) == hm
            live.append(hm)
        elif op < 0.7:
            h = rs.choice(live)
            try:
                kind, slot, cow = m.append_slot(h)
            except OutOfBlocks:
                with pytest.raises(pa.PagedAttnError):
                    a.append_slot(h)
                continue
            assert a.append_slot(h) == (slot, cow)
        elif op < 0.85:
            p = rs.choice(live)
            c = m.fork(p)
            assert a.fork(p) == c
            live.append(c)
        else:
            h = live.pop(rs.randrange(len(live)))
            assert a.free(h) == m.free(h)
        if step % 100 == 0:
            assert [a.refcount(b) for b in range(96)] == m.ref
            assert a.num_free() == m.num_free()
            if live:
                bt, cl = a.export(live, 64)
                rows, lens = m.export(live, 64)
                assert bt.tolist() == rows and cl.tolist() == lens


def test_tp_comm_validation():
    """N2 comm: invalid world / rank / head split / NULL buffers -> NULL with a message;
    the fused decode entry rejects a NULL comm and a head-count mismatch."""
    import ctypes as C
    arr = (C.c_void_p * 2)(FAKE, FAKE)
    GB = 4 * 8 * 128 * 2  # gather buffers for 4 sequences x 8 heads x 128 f16
    ok = L.pa_tp_comm_create(2, 0, 8, GB, arr, arr, arr, FAKE)
    assert ok
    L.pa_tp_comm_destroy(ok)
    assert not L.pa_tp_comm_create(0, 0, 8, GB, arr, arr, arr, FAKE)
    assert not L.pa_tp_comm_create(2, 2, 8, GB, arr, arr, arr, FAKE)
    assert not L.pa_tp_comm_create(2, 0, 7, GB, arr, arr, arr, FAKE)
    assert not L.pa_tp_comm_create(9, 0, 9, GB, arr, arr, arr, FAKE)
    bad = (C.c_void_p * 2)(FAKE, FAKE + 8)
    assert not L.pa_tp_comm_create(2, 0, 8, GB, bad, arr, arr, FAKE)
    assert _lib.last_error() != ""
    r = L.pa_paged_attention_decode_tp
    assert r(None, None, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0.1, 16, 4, 4, 4, 128, 8, 100, 1, None, FAKE, 4096,
             None) == INVALID
    comm = L.pa_tp_comm_create(2, 1, 8, GB, arr, arr, arr, FAKE)
    assert r(comm, None, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0.1, 16, 4, 4, 8, 128, 8, 100, 1, None, FAKE, 4096,
             None) == INVALID  # 8 local heads x 2 ranks != 8
    assert r(comm, None, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, 0.1, 16, 4, 5, 4, 128, 8, 100, 1, None, FAKE, 4096,
             None) == INVALID  # 5 sequences do not fit gather buffers sized for 4
    assert "gather buffers" in _lib.last_error()
    L.pa_tp_comm_destroy(comm)
    assert L.pa_ipc_handle_bytes() == 64


def test_decode_plan_longest_first_stable():
    """pa_decode_plan: indices sorted by context length, longest first, ties in index
    order (host only)."""
    import numpy as np
    import paper_2309_06180_b200 as pa
    ctx = np.array([5, 300, 17, 300, 0, 2048, 17], np.int32)
    assert pa.decode_plan(ctx).tolist() == [5, 1, 3, 2, 6, 0, 4]
    assert pa.decode_plan(np.zeros(0, np.int32)).tolist() == []


@pytest.mark.parametrize("order", [[0, 1, 2, 2], [0, 1, 2, 4], [3, 2, 1, -1]])
def test_seq_order_must_be_a_permutation(order):
    """A grid order that repeats or misses a sequence is rejected on the host, before any
    launch (it would compute one output twice and leave another unwritten)."""
    arr = (ctypes.c_int32 * 4)(*order)
    assert attn(order=arr, ws=FAKE, wsb=1 << 20) == INVALID
    assert "permutation" in _lib.last_error()


def grouped(**kw):
    a = dict(out=FAKE, q=FAKE, k=FAKE, v=FAKE, kc=FAKE, vc=FAKE, bt=FAKE, cl=FAKE, scale=0.125, B=16, hkv=8, NB=64,
             S=8, H=8, D=128, W=128, mcl=2048, gs=4, dt=1, ws=FAKE, wsb=1 << 30)
    a.update(kw)
    return L.pa_paged_attention_decode_grouped(a["out"], a["q"], a["k"], a["v"], a["kc"], a["vc"], a["bt"], a["cl"],
                                               a["scale"], a["B"], a["hkv"], a["NB"], a["S"], a["H"], a["D"], a["W"],
                                               a["mcl"], a["gs"], a["dt"], None, a["ws"], a["wsb"], None)


@pytest.mark.parametrize("kw,status", [
    (dict(dt=0), UNSUPPORTED),                 # f32: the tensor-core kernel is f16 / bf16
    (dict(D=64), UNSUPPORTED),
    (dict(B=8), UNSUPPORTED),                  # block_size >= 16
    (dict(gs=9), INVALID),                     # group_size in [1, 8]
    (dict(H=6, hkv=4), INVALID),               # H % H_kv
    (dict(k=None), INVALID),                   # the step's new token is required
    (dict(ws=None), WORKSPACE),
    (dict(wsb=16), WORKSPACE),                 # split context: counters + partial rows, not only the work counter
])
def test_grouped_argument_validation(kw, status):
    """pa_paged_attention_decode_grouped rejects bad arguments on the host (pa.h), incl. a
    workspace below pa_paged_attention_workspace_size for its split context."""
    assert grouped(**kw) == status
    assert _lib.last_error() != ""


def test_grouped_zero_seqs_is_noop():
    assert grouped(S=0, out=None) == OK
