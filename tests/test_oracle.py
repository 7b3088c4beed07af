"""Pins for the fp64 oracle (oracle/oracle.c) against what the paper and mathematics fix.

None of these re-types the oracle's formulas: each check is a closed form, an
invariant, a library routine, a 50-digit brute force, or a placement done here with
plain numpy indexing.  P:N = /root/reference/PAPER.md line N.
"""
import math

import numpy as np
import pytest

import oracle

mpmath = pytest.importorskip("mpmath")


def rng(seed):
    return np.random.default_rng(seed)


# ---------------------------------------------------------------- decoders (c8) ----

def test_fp16_decoder_exhaustive_vs_numpy():
    bits = np.arange(1 << 16, dtype=np.uint16)
    ours = oracle.decode(bits, "f16")
    ref = bits.view(np.float16).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan], ref[~nan])
    # signed zero preserved
    assert np.array_equal(np.signbit(ours[~nan]), np.signbit(ref[~nan]))


def test_bf16_decoder_exhaustive_vs_torch():
    torch = pytest.importorskip("torch")
    bits = np.arange(1 << 16, dtype=np.uint16)
    ours = oracle.decode(bits, "bf16")
    ref = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).double().numpy()
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(ours), nan)
    assert np.array_equal(ours[~nan], ref[~nan])


def test_fp32_decoder_vs_numpy():
    r = rng(1)
    bits = r.integers(0, 1 << 32, size=100000, dtype=np.uint64).astype(np.uint32)
    ours = oracle.decode(bits, "f32")
    ref = bits.view(np.float32).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(ours[~nan], ref[~nan])
    assert np.array_equal(np.isnan(ours), nan)


# ------------------------------------------------- Eq.3 closed forms ----

def test_single_token_returns_v():
    """n = 1: a = [1], o = v_1 exactly."""
    r = rng(2)
    q, K, V = r.uniform(-1, 1, 16), r.uniform(-1, 1, (1, 16)), r.uniform(-1, 1, (1, 16))
    assert np.array_equal(oracle.contiguous_attention(q, K, V, 0.25), V[0])


def test_equal_scores_give_mean():
    """q = 0: every score equal -> o = mean of the V rows."""
    r = rng(3)
    for n in (2, 7, 100):
        K, V = r.uniform(-1, 1, (n, 8)), r.uniform(-1, 1, (n, 8))
        out = oracle.contiguous_attention(np.zeros(8), K, V, 0.3)
        np.testing.assert_allclose(out, V.mean(axis=0), rtol=0, atol=1e-15)


def test_constant_values():
    r = rng(4)
    K = r.uniform(-1, 1, (33, 8))
    V = np.tile(r.uniform(-1, 1, 8), (33, 1))
    out = oracle.contiguous_attention(r.uniform(-1, 1, 8), K, V, 0.5)
    np.testing.assert_allclose(out, V[0], rtol=0, atol=1e-15)


def test_dominant_score():
    """One score larger than every other by > 60: o = that row (to e^-60)."""
    r = rng(5)
    K = r.uniform(-1, 1, (20, 4)) * 0.01
    K[13] = [100.0, 0, 0, 0]
    V = r.uniform(-1, 1, (20, 4))
    out = oracle.contiguous_attention(np.array([1.0, 0, 0, 0]), K, V, 1.0)
    np.testing.assert_allclose(out, V[13], rtol=0, atol=1e-20)


def test_convex_combination_bound():
    r = rng(6)
    for _ in range(50):
        n = int(r.integers(1, 64))
        K, V = r.uniform(-1, 1, (n, 8)), r.uniform(-1, 1, (n, 8))
        out = oracle.contiguous_attention(r.normal(0, 3, 8), K, V, 1.0)
        assert np.all(out <= V.max(axis=0) + 1e-15) and np.all(out >= V.min(axis=0) - 1e-15)


def test_empty_context_is_zero():
    """ctx = 0 -> out = 0 (reading c9)."""
    out = oracle.contiguous_attention(np.ones(4), np.zeros((0, 4)), np.zeros((0, 4)), 1.0)
    assert np.array_equal(out, np.zeros(4))


def test_brute_force_mpmath():
    """Eq.3 in 50-digit arithmetic on tiny inputs; the fp64 oracle within 1e-13 relative."""
    mpmath.mp.dps = 50
    r = rng(7)
    for _ in range(60):
        n, D = int(r.integers(1, 9)), int(r.integers(1, 7))
        q, K, V = r.uniform(-2, 2, D), r.uniform(-2, 2, (n, D)), r.uniform(-2, 2, (n, D))
        scale = 1.0 / math.sqrt(D)
        sc = [mpmath.mpf(scale) * mpmath.fsum(mpmath.mpf(q[d]) * mpmath.mpf(K[t, d]) for d in range(D))
              for t in range(n)]
        den = mpmath.fsum(mpmath.exp(s) for s in sc)
        ref = [mpmath.fsum(mpmath.exp(sc[t]) * mpmath.mpf(V[t, d]) for t in range(n)) / den
               for d in range(D)]
        out = oracle.contiguous_attention(q, K, V, scale)
        for d in range(D):
            assert abs(out[d] - float(ref[d])) <= 1e-13 * max(1.0, abs(float(ref[d])))


def test_score_spread_700_stays_finite():
    """Scores spanning +-700 stay finite: max subtraction in effect."""
    r = rng(8)
    K = np.zeros((10, 2))
    K[:, 0] = np.linspace(-700, 700, 10)
    V = r.uniform(-1, 1, (10, 2))
    out = oracle.contiguous_attention(np.array([1.0, 0.0]), K, V, 1.0)
    assert np.all(np.isfinite(out))
    np.testing.assert_allclose(out, V[-1], atol=1e-15)


# ------------------------------------------------------- Eq.4 == Eq.3 ----

def place(K, V, B, H_kv, kvh, rs, num_blocks=None, dtype=np.float32):
    """Place logical rows K[n][D], V[n][D] into a [NB][H_kv][B][D] cache with numpy
    indexing, on shuffled physical blocks; unused slots are NaN.  Returns caches + row."""
    n, D = K.shape
    nb = max(1, -(-n // B))
    NB = num_blocks or 2 * nb + 3
    phys = rs.permutation(NB)[:nb]
    kc = np.full((NB, H_kv, B, D), np.nan, dtype=dtype)
    vc = np.full((NB, H_kv, B, D), np.nan, dtype=dtype)
    for t in range(n):
        kc[phys[t // B], kvh, t % B, :] = K[t]
        vc[phys[t // B], kvh, t % B, :] = V[t]
    return kc, vc, phys.astype(np.int32)


def test_paged_equals_contiguous_bitwise_1000():
    """Paged (Eq.4) vs contiguous (Eq.3) on the same logical rows: bitwise identical over
    1000 seeded instances, B in {1,2,4,8,16,32} (S:309 asks only 1e-9)."""
    r = rng(9)
    for it in range(1000):
        n = int(r.integers(1, 129))
        D = int(r.integers(1, 17))
        B = int(r.choice([1, 2, 4, 8, 16, 32]))
        K = r.uniform(-1, 1, (n, D)).astype(np.float32)
        V = r.uniform(-1, 1, (n, D)).astype(np.float32)
        q = r.uniform(-1, 1, (1, 1, D)).astype(np.float32)
        kc, vc, phys = place(K, V, B, 1, 0, r)
        scale = 1.0 / math.sqrt(D)
        out = oracle.paged_attention(q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32),
                                     phys[None, :], np.array([n], np.int32), scale, B, 1, "f32")
        ref = oracle.contiguous_attention(q[0, 0].astype(np.float64), K.astype(np.float64),
                                          V.astype(np.float64), scale)
        assert np.array_equal(out[0, 0], ref), f"instance {it}"


def test_block_size_and_permutation_invariance_bitwise():
    r = rng(10)
    n, D = 77, 16
    K = r.uniform(-1, 1, (n, D)).astype(np.float32)
    V = r.uniform(-1, 1, (n, D)).astype(np.float32)
    q = r.uniform(-1, 1, (1, 1, D)).astype(np.float32).view(np.uint32)
    outs = []
    for B in (1, 8, 16, 32):
        for perm_seed in range(3):
            kc, vc, phys = place(K, V, B, 1, 0, np.random.default_rng(100 + perm_seed))
            outs.append(oracle.paged_attention(q, kc.view(np.uint32), vc.view(np.uint32), phys[None, :],
                                               np.array([n], np.int32), 0.25, B, 1, "f32"))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_gqa_head_mapping_and_multi_head():
    """Query head h reads kv head h / (H/H_kv) (reading c13); each head is Eq.3 on its own."""
    r = rng(11)
    n, D, B, H, H_kv = 40, 8, 4, 4, 2
    Ks = [r.uniform(-1, 1, (n, D)).astype(np.float32) for _ in range(H_kv)]
    Vs = [r.uniform(-1, 1, (n, D)).astype(np.float32) for _ in range(H_kv)]
    nb = n // B
    NB = 25
    phys = r.permutation(NB)[:nb].astype(np.int32)
    kc = np.full((NB, H_kv, B, D), np.nan, np.float32)
    vc = np.full((NB, H_kv, B, D), np.nan, np.float32)
    for h in range(H_kv):
        for t in range(n):
            kc[phys[t // B], h, t % B] = Ks[h][t]
            vc[phys[t // B], h, t % B] = Vs[h][t]
    q = r.uniform(-1, 1, (1, H, D)).astype(np.float32)
    out = oracle.paged_attention(q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32), phys[None, :],
                                 np.array([n], np.int32), 0.3, B, H_kv, "f32")
    for h in range(H):
        kvh = h // (H // H_kv)
        ref = oracle.contiguous_attention(q[0, h].astype(np.float64), Ks[kvh].astype(np.float64),
                                          Vs[kvh].astype(np.float64), 0.3)
        assert np.array_equal(out[0, h], ref)


def test_gather_matches_numpy_placement():
    r = rng(12)
    n, D, B = 50, 8, 8
    K = r.uniform(-1, 1, (n, D)).astype(np.float32)
    V = r.uniform(-1, 1, (n, D)).astype(np.float32)
    kc, vc, phys = place(K, V, B, 3, 2, r)
    kb, vb = oracle.gather_kv_bits(kc.view(np.uint32), vc.view(np.uint32), phys, n, 2, B, "f32")
    assert np.array_equal(kb, K.view(np.uint32)) and np.array_equal(vb, V.view(np.uint32))
    kd, vd = oracle.gather_kv(kc.view(np.uint32), vc.view(np.uint32), phys, n, 2, B, "f32")
    assert np.array_equal(kd, K.astype(np.float64)) and np.array_equal(vd, V.astype(np.float64))


@pytest.mark.parametrize("dtype,npdt", [("f16", np.float16)])
def test_paged_half_inputs_decode_exactly(dtype, npdt):
    r = rng(13)
    n, D, B = 30, 16, 16
    K = r.uniform(-1, 1, (n, D)).astype(npdt)
    V = r.uniform(-1, 1, (n, D)).astype(npdt)
    q = r.uniform(-1, 1, (1, 1, D)).astype(npdt)
    kc, vc, phys = place(K, V, B, 1, 0, r, dtype=npdt)
    out = oracle.paged_attention(q.view(np.uint16), kc.view(np.uint16), vc.view(np.uint16), phys[None, :],
                                 np.array([n], np.int32), 0.25, B, 1, dtype)
    ref = oracle.contiguous_attention(q[0, 0].astype(np.float64), K.astype(np.float64),
                                      V.astype(np.float64), 0.25)
    assert np.array_equal(out[0, 0], ref)


# ----------------------------------------------------- split-context merge (a6) ----

def test_split_merge_equals_unsplit():
    r = rng(14)
    S, H, D, B = 3, 2, 16, 16
    ctx = np.array([1, 300, 1000], np.int32)
    W = 64
    NB = 3 * W
    kc = r.uniform(-1, 1, (NB, H, B, D)).astype(np.float32)
    vc = r.uniform(-1, 1, (NB, H, B, D)).astype(np.float32)
    bt = r.permutation(NB)[: S * W].reshape(S, W).astype(np.int32)
    q = (r.uniform(-1, 1, (S, H, D)) * 4).astype(np.float32)
    args = (q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32), bt, ctx, 0.25, B, H, "f32")
    full = oracle.paged_attention(*args)
    for part in (16, 32, 512, 4096):
        sp = oracle.split_attention(*args, part)
        np.testing.assert_allclose(sp, full, rtol=0, atol=1e-13)


# ----------------------------------------- reshape_and_cache / copy_blocks oracles ----

def test_reshape_and_cache_fig6_slots():
    """Fig.6: 7-token prompt, B = 4, logical {0,1} -> physical {7,1}.
    Prompt slot_mapping = [28,29,30,31,4,5,6]; rows land at (7,0..3), (1,0..2)."""
    B, H_kv, D, NB = 4, 2, 4, 8
    r = rng(15)
    key = r.integers(0, 1 << 16, (7, H_kv, D), dtype=np.uint16)
    val = r.integers(0, 1 << 16, (7, H_kv, D), dtype=np.uint16)
    kc0 = r.integers(0, 1 << 16, (NB, H_kv, B, D), dtype=np.uint16)
    vc0 = r.integers(0, 1 << 16, (NB, H_kv, B, D), dtype=np.uint16)
    slots = np.array([28, 29, 30, 31, 4, 5, 6], np.int64)
    kc, vc = oracle.reshape_and_cache(key, val, kc0, vc0, slots, B, "f16")
    ek, ev = kc0.copy(), vc0.copy()
    for i, (b, o) in enumerate([(7, 0), (7, 1), (7, 2), (7, 3), (1, 0), (1, 1), (1, 2)]):
        ek[b, :, o, :] = key[i]
        ev[b, :, o, :] = val[i]
    assert np.array_equal(kc, ek) and np.array_equal(vc, ev)


def test_reshape_and_cache_skips_negative_slots():
    r = rng(16)
    key = r.integers(0, 1 << 16, (3, 1, 8), dtype=np.uint16)
    kc0 = r.integers(0, 1 << 16, (4, 1, 2, 8), dtype=np.uint16)
    kc, vc = oracle.reshape_and_cache(key, key, kc0, kc0, np.array([-1, 5, -7], np.int64), 2, "bf16")
    ek = kc0.copy()
    ek[2, 0, 1] = key[1, 0]
    assert np.array_equal(kc, ek) and np.array_equal(vc, ek)


def test_copy_blocks_paper_cow_and_snapshot_semantics():
    """CoW 1 -> 3 and repeated sources (beam fork)."""
    r = rng(17)
    layers = [r.integers(0, 1 << 32, (6, 2, 4, 4), dtype=np.uint64).astype(np.uint32) for _ in range(3)]
    vals = [r.integers(0, 1 << 32, (6, 2, 4, 4), dtype=np.uint64).astype(np.uint32) for _ in range(3)]
    kcs, vcs = oracle.copy_blocks(layers, vals, [[1, 3]], "f32")
    for l in range(3):
        e = layers[l].copy(); e[3] = layers[l][1]
        assert np.array_equal(kcs[l], e)
        e = vals[l].copy(); e[3] = vals[l][1]
        assert np.array_equal(vcs[l], e)
    kcs, vcs = oracle.copy_blocks(layers, vals, [[1, 3], [1, 4], [0, 5]], "f32")
    e = layers[0].copy(); e[3] = layers[0][1]; e[4] = layers[0][1]; e[5] = layers[0][0]
    assert np.array_equal(kcs[0], e)


def test_swap_blocks_round_trip_and_placement():
    """Swap-out then swap-in restores the GPU pool's live blocks; every
    destination block equals its source, every other block is untouched."""
    r = rng(18)
    gpu = [r.integers(0, 1 << 16, (10, 2, 4, 8), dtype=np.uint16) for _ in range(2)]
    gpuv = [r.integers(0, 1 << 16, (10, 2, 4, 8), dtype=np.uint16) for _ in range(2)]
    cpu = [np.zeros((6, 2, 4, 8), np.uint16) for _ in range(2)]
    cpuv = [np.zeros((6, 2, 4, 8), np.uint16) for _ in range(2)]
    out_pairs = [[3, 0], [7, 5], [1, 2]]
    ck, cv = oracle.swap_blocks(cpu, cpuv, gpu, gpuv, out_pairs)
    for l in range(2):
        e = cpu[l].copy(); e[0] = gpu[l][3]; e[5] = gpu[l][7]; e[2] = gpu[l][1]
        assert np.array_equal(ck[l], e)
    wiped = [np.zeros_like(g) for g in gpu]
    wipedv = [np.zeros_like(g) for g in gpuv]
    back = [[0, 4], [5, 9], [2, 6]]
    gk, gv = oracle.swap_blocks(wiped, wipedv, ck, cv, back)
    for l in range(2):
        assert np.array_equal(gk[l][4], gpu[l][3]) and np.array_equal(gk[l][9], gpu[l][7])
        assert np.array_equal(gv[l][6], gpuv[l][1])
        assert not gk[l][[0, 1, 2, 3, 5, 7, 8]].any()


# ------------------------------------ prompt phase / shared-prefix suffix (N4) --------

def _prefill_case(r, ctxs, qlens, H, H_kv, D, B):
    """Seeded fp32 case: per sequence a contiguous K/V [ctx][H_kv][D] placed on shuffled
    blocks (NaN elsewhere), query rows [T][H][D]."""
    S = len(ctxs)
    W = max(-(-c // B) for c in ctxs)
    NB = S * W + 5
    perm = r.permutation(NB)
    kc = np.full((NB, H_kv, B, D), np.nan, np.float32)
    vc = np.full((NB, H_kv, B, D), np.nan, np.float32)
    bt = np.zeros((S, W), np.int32)
    Ks, Vs = [], []
    for s, c in enumerate(ctxs):
        K = r.uniform(-1, 1, (c, H_kv, D)).astype(np.float32)
        V = r.uniform(-1, 1, (c, H_kv, D)).astype(np.float32)
        bt[s] = perm[s * W:(s + 1) * W]
        for t in range(c):
            kc[bt[s, t // B], :, t % B] = K[t]
            vc[bt[s, t // B], :, t % B] = V[t]
        Ks.append(K)
        Vs.append(V)
    qs = np.concatenate([[0], np.cumsum(qlens)]).astype(np.int32)
    Q = r.uniform(-1, 1, (int(qs[-1]), H, D)).astype(np.float32)
    return Q, kc, vc, bt, np.asarray(ctxs, np.int32), qs, Ks, Vs


def test_prefill_pure_prompt_equals_torch_causal_sdpa():
    """ctx == q_len (the prompt phase): the result is textbook causal
    self-attention -- pinned to torch's scaled_dot_product_attention(is_causal=True) in fp64
    (a library routine independent of the oracle's loops), GQA via repeat_interleave."""
    torch = pytest.importorskip("torch")
    r = rng(30)
    H, H_kv, D, B = 4, 2, 16, 8
    ctxs = [37, 1, 64]
    Q, kc, vc, bt, cl, qs, Ks, Vs = _prefill_case(r, ctxs, ctxs, H, H_kv, D, B)
    scale = 1.0 / math.sqrt(D)
    out = oracle.prefill_attention(Q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32), bt, cl, qs,
                                   scale, B, H_kv, "f32")
    for s, c in enumerate(ctxs):
        q = torch.from_numpy(Q[qs[s]:qs[s + 1]].astype(np.float64)).permute(1, 0, 2)  # [H][c][D]
        k = torch.from_numpy(Ks[s].astype(np.float64)).permute(1, 0, 2).repeat_interleave(H // H_kv, 0)
        v = torch.from_numpy(Vs[s].astype(np.float64)).permute(1, 0, 2).repeat_interleave(H // H_kv, 0)
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=scale)
        np.testing.assert_allclose(out[qs[s]:qs[s + 1]], ref.permute(1, 0, 2).numpy(), rtol=0, atol=1e-13)


def test_prefill_shared_prefix_suffix_rows_equal_decode():
    """ctx > q_len (suffix after a cached shared prefix): query row i equals the
    decode oracle (Eq.4) run with context length ctx - q_len + i + 1 -- bitwise, since a
    one-token step is the q_len == 1 case."""
    r = rng(31)
    H, H_kv, D, B = 4, 4, 8, 16
    ctxs, qlens = [50, 20, 33], [7, 20, 1]
    Q, kc, vc, bt, cl, qs, _, _ = _prefill_case(r, ctxs, qlens, H, H_kv, D, B)
    out = oracle.prefill_attention(Q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32), bt, cl, qs,
                                   0.3, B, H_kv, "f32")
    for s in range(len(ctxs)):
        for i in range(qlens[s]):
            row = qs[s] + i
            n = ctxs[s] - qlens[s] + i + 1
            ref = oracle.paged_attention(Q[row:row + 1].view(np.uint32), kc.view(np.uint32),
                                         vc.view(np.uint32), bt[s:s + 1], np.array([n], np.int32), 0.3, B,
                                         H_kv, "f32")
            assert np.array_equal(out[row], ref[0])


def test_prefill_suffix_rows_equal_torch_causal_sdpa_of_the_whole_sequence():
    """The suffix offset (reading c22: row i of a q_len-token suffix sits at position
    ctx - q_len + i) pinned to a library routine, not to the oracle's own formula: the
    suffix rows equal the LAST q_len rows of torch's causal scaled_dot_product_attention
    over the whole ctx-token sequence (in fp64), whose earlier query rows are arbitrary."""
    torch = pytest.importorskip("torch")
    r = rng(33)
    H, H_kv, D, B = 4, 2, 16, 8
    ctxs, qlens = [50, 21, 9], [7, 21, 1]
    Q, kc, vc, bt, cl, qs, Ks, Vs = _prefill_case(r, ctxs, qlens, H, H_kv, D, B)
    scale = 0.27
    out = oracle.prefill_attention(Q.view(np.uint32), kc.view(np.uint32), vc.view(np.uint32), bt, cl, qs,
                                   scale, B, H_kv, "f32")
    for s, (c, n) in enumerate(zip(ctxs, qlens)):
        qfull = np.concatenate([r.uniform(-1, 1, (c - n, H, D)), Q[qs[s]:qs[s + 1]].astype(np.float64)])
        q = torch.from_numpy(qfull).permute(1, 0, 2)  # [H][c][D]
        k = torch.from_numpy(Ks[s].astype(np.float64)).permute(1, 0, 2).repeat_interleave(H // H_kv, 0)
        v = torch.from_numpy(Vs[s].astype(np.float64)).permute(1, 0, 2).repeat_interleave(H // H_kv, 0)
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=scale)
        np.testing.assert_allclose(out[qs[s]:qs[s + 1]], ref.permute(1, 0, 2).numpy()[c - n:], rtol=0, atol=1e-13)


def test_prefill_first_prompt_row_is_v0_and_block_invariance():
    """Row 0 of a prompt attends to exactly one token: out = v_0 (closed form).  The
    result does not depend on block size or placement, bitwise."""
    H, H_kv, D = 2, 1, 8
    outs = []
    for B in (1, 4, 16):
        for seed in (40, 41):
            r = rng(32)  # same logical data
            Q, kc, vc, bt, cl, qs, Ks, Vs = _prefill_case(r, [29], [29], H, H_kv, D, 32)
            # re-place the same logical rows with block size B on a different permutation
            K, V = Ks[0], Vs[0]
            nb = -(-29 // B)
            NB = nb + 7
            phys = np.random.default_rng(seed).permutation(NB)[:nb].astype(np.int32)
            kc2 = np.full((NB, H_kv, B, D), np.nan, np.float32)
            vc2 = np.full((NB, H_kv, B, D), np.nan, np.float32)
            for t in range(29):
                kc2[phys[t // B], :, t % B] = K[t]
                vc2[phys[t // B], :, t % B] = V[t]
            out = oracle.prefill_attention(Q.view(np.uint32), kc2.view(np.uint32), vc2.view(np.uint32),
                                           phys[None, :], cl, qs, 0.35, B, H_kv, "f32")
            assert np.array_equal(out[0, 0], V[0, 0].astype(np.float64))
            assert np.array_equal(out[0, 1], V[0, 0].astype(np.float64))
            outs.append(out)
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
