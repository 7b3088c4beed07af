"""GPU parity of the multi-token (prompt / shared-prefix suffix) paged attention on the
tcgen05 tensor cores (pa_paged_prefill_attention) against the fp64
oracle (oracle.prefill_attention, pinned in tests/test_oracle.py).

Tolerance: the kernel rounds the softmax weights to the storage dtype
before P.V (each weight's relative error <= 2^-9 bf16 / 2^-11 f16, inputs |v| <= 1), plus
the output rounding -- inside TOL (bf16 1e-2, f16 2e-3)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_2309_06180_b200 as pa
from synth import rng as R
from synth.workload import place_private
from tests.pathutil import TOL, bits, max_abs

pytestmark = pytest.mark.gpu
D = 128


def prefill_problem(ctx, qlen, B, H, H_kv, dtype, place_seed=21, seed=88):
    """Logical K/V of every sequence's ctx tokens (drawn per (seq, kv head, token, dim),
    so independent of B and placement) on shuffled blocks, NaN elsewhere, plus the query
    rows [T][H][D] of each sequence's last qlen tokens."""
    ctx = np.asarray(ctx, np.int64)
    qlen = np.asarray(qlen, np.int64)
    bt, NB, _, _ = place_private(ctx, B, place_seed, pool_factor=1.5, min_extra=3)
    S, Tm = len(ctx), int(max(1, ctx.max()))
    dev = "cuda"
    s = torch.arange(S, device=dev).view(S, 1, 1, 1)
    h = torch.arange(H_kv, device=dev).view(1, H_kv, 1, 1)
    t = torch.arange(Tm, device=dev).view(1, 1, Tm, 1)
    d = torch.arange(D, device=dev).view(1, 1, 1, D)
    idx = ((s * H_kv + h) * Tm + t) * D + d
    K = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_KCACHE), idx), dtype)
    V = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_VCACHE), idx), dtype)
    kc = torch.full((NB, H_kv, B, D), float("nan"), dtype=K.dtype, device=dev)
    vc = torch.full_like(kc, float("nan"))
    btt = torch.as_tensor(bt, device=dev)
    for si in range(S):
        n = int(ctx[si])
        if n == 0:
            continue
        tt = torch.arange(n, device=dev)
        blocks = btt[si, tt // B].long()
        kc[blocks, :, tt % B, :] = K[si, :, :n, :].permute(1, 0, 2)
        vc[blocks, :, tt % B, :] = V[si, :, :n, :].permute(1, 0, 2)
    qs = np.concatenate([[0], np.cumsum(qlen)]).astype(np.int32)
    T = int(qs[-1])
    qi = torch.arange(T * H * D, device=dev).view(T, H, D)
    q = R.f32_to_dtype_t(R.uniform_f32_t(R.key(seed, R.STREAM_Q), qi), dtype).contiguous()
    return q, kc, vc, btt, torch.as_tensor(ctx.astype(np.int32), device=dev), torch.as_tensor(qs, device=dev)


def run(q, kc, vc, bt, cl, qs, scale):
    out = torch.full_like(q, float("nan"))
    pa.paged_prefill_attention(out, q, kc, vc, bt, cl, qs, scale)
    torch.cuda.synchronize()
    return out


def ref(q, kc, vc, bt, cl, qs, scale, B, H_kv, dtype):
    return oracle.prefill_attention(bits(q), bits(kc), bits(vc), bt.cpu().numpy(), cl.cpu().numpy(),
                                    qs.cpu().numpy(), scale, B, H_kv, dtype)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_prompt_phase_vs_oracle(dtype):
    """ctx == q_len: causal self-attention of whole prompts; lengths around the
    128-row query tile and 128-token KV tile boundaries, GQA 4:2."""
    ctx = [1, 5, 127, 128, 129, 255, 300, 700]
    H, H_kv, B = 4, 2, 16
    scale = 1.0 / np.sqrt(D)
    q, kc, vc, bt, cl, qs = prefill_problem(ctx, ctx, B, H, H_kv, dtype)
    out = run(q, kc, vc, bt, cl, qs, scale)
    assert torch.isfinite(out).all()
    assert max_abs(out, ref(q, kc, vc, bt, cl, qs, scale, B, H_kv, dtype)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_shared_prefix_suffix_vs_oracle(dtype):
    """ctx > q_len: the user-specific suffix after a cached shared prefix and
    chunked prompts; also q_len == 1 (a decode row) and q_len == ctx."""
    ctx = [600, 130, 1500, 64, 257, 1000]
    qlen = [64, 130, 1, 17, 200, 300]
    H, H_kv, B = 8, 8, 16
    scale = 0.09
    q, kc, vc, bt, cl, qs = prefill_problem(ctx, qlen, B, H, H_kv, dtype, seed=89)
    out = run(q, kc, vc, bt, cl, qs, scale)
    assert max_abs(out, ref(q, kc, vc, bt, cl, qs, scale, B, H_kv, dtype)) <= TOL[dtype]


def test_block_size_and_placement_invariance_bitwise():
    """The same logical problem with B in {1,2,4,8,16,32,64} and two placements gives
    bitwise identical outputs (KV tiles are logical 128-token tiles)."""
    ctx, qlen = [333, 140, 40], [333, 20, 40]
    outs = []
    for B in (1, 2, 4, 8, 16, 32, 64):
        for ps in (31, 32):
            q, kc, vc, bt, cl, qs = prefill_problem(ctx, qlen, B, 4, 1, "bf16", place_seed=ps)
            outs.append(run(q, kc, vc, bt, cl, qs, 0.1))
    for o in outs[1:]:
        assert torch.equal(o, outs[0])


@pytest.mark.parametrize("variant", ["2", "3"])
def test_chunked_prompt_equals_whole_prompt_bitwise(variant, tuning_env):
    """Prefilling a prompt in chunks (each chunk attends to the cached earlier chunks)
    gives the rows of the whole-prompt prefill bit for bit: with a given kernel, a row's
    result depends only on its position, never on which launch computes it."""
    tuning_env("PA_PREFILL", variant)
    n, B, H, H_kv = 700, 16, 4, 4
    q, kc, vc, bt, cl, qs = prefill_problem([n], [n], B, H, H_kv, "f16")
    whole = run(q, kc, vc, bt, cl, qs, 0.088)
    parts = []
    for a, b in ((0, 100), (100, 356), (356, 357), (357, 700)):
        cl_c = torch.tensor([b], dtype=torch.int32, device="cuda")
        qs_c = torch.tensor([0, b - a], dtype=torch.int32, device="cuda")
        parts.append(run(q[a:b].contiguous(), kc, vc, bt, cl_c, qs_c, 0.088))
    assert torch.equal(torch.cat(parts), whole)


def test_degenerate_cases():
    """q_len 0 sequences contribute nothing; ctx < q_len rows at negative positions are 0;
    a 1-token prompt returns its own V row exactly."""
    H, H_kv, B = 2, 1, 16
    q, kc, vc, bt, cl, qs = prefill_problem([50, 1, 30], [0, 1, 30], B, H, H_kv, "bf16")
    out = run(q, kc, vc, bt, cl, qs, 0.1)
    assert out.shape[0] == 31
    v0 = vc[bt[1, 0].long(), 0, 0]
    assert torch.equal(out[0, 0], v0) and torch.equal(out[0, 1], v0)
    # ctx < q_len: rows 0..4 of the 10-row query sit at positions -5..-1 -> 0
    q2, kc2, vc2, bt2, _, _ = prefill_problem([5], [10], B, H, H_kv, "bf16")
    cl2 = torch.tensor([5], dtype=torch.int32, device="cuda")
    qs2 = torch.tensor([0, 10], dtype=torch.int32, device="cuda")
    out2 = run(q2, kc2, vc2, bt2, cl2, qs2, 0.1)
    assert torch.count_nonzero(out2[:5]) == 0
    r2 = ref(q2, kc2, vc2, bt2, cl2, qs2, 0.1, B, H_kv, "bf16")
    assert max_abs(out2[5:], r2[5:]) <= TOL["bf16"]


def test_prefill_sharegpt_sized_sampled_rows():
    """A ShareGPT-sized prompt batch on the LLaMA-13B head shape (H = 40, D = 128,
    B = 16): sampled (row, head) outputs vs the oracle's Eq.4 row of length pos+1 (the
    decode oracle, pinned bitwise equal to the prefill oracle)."""
    from synth.workload import request_pool
    pool = request_pool(1001, "sharegpt", n=64)
    ctx = np.minimum(np.asarray(pool[0][:24], np.int64), 2048)
    ctx = np.maximum(ctx, 1)
    H = H_kv = 40
    B = 16
    q, kc, vc, bt, cl, qs = prefill_problem(ctx, ctx, B, H, H_kv, "f16", seed=90)
    scale = 1.0 / np.sqrt(D)
    out = run(q, kc, vc, bt, cl, qs, scale)
    assert torch.isfinite(out).all()
    rs = np.random.default_rng(5)
    qsn = qs.cpu().numpy()
    rows = rs.integers(0, int(qsn[-1]), 48)
    qb, kb, vb, btn, cln = bits(q), bits(kc), bits(vc), bt.cpu().numpy(), cl.cpu().numpy()
    for row in rows:
        s = int(np.searchsorted(qsn, row, side="right") - 1)
        pos = int(cln[s] - (qsn[s + 1] - qsn[s]) + (row - qsn[s]))
        r = oracle.paged_attention(qb[row:row + 1], kb, vb, btn[s:s + 1], np.array([pos + 1], np.int32), scale, B,
                                   H_kv, "f16")
        assert max_abs(out[row:row + 1], r) <= TOL["f16"]


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_kernel_variants_agree(dtype, tuning_env):
    """v2 (persistent, two query tiles per CTA) and v3 (persistent, one query tile, softmax
    split by key columns) each match the oracle
    and agree with one another to a few output ulps (the tensor cores' accumulation of
    the operand sources and the split row sums round differently)."""
    ctx = [600, 130, 1500, 64, 257, 1000, 300]
    qlen = [64, 130, 1, 17, 200, 300, 300]
    q, kc, vc, bt, cl, qs = prefill_problem(ctx, qlen, 16, 8, 2, dtype, seed=91)
    r = ref(q, kc, vc, bt, cl, qs, 0.09, 16, 2, dtype)
    outs = []
    for v in ("2", "3"):
        tuning_env("PA_PREFILL", v)
        outs.append(run(q, kc, vc, bt, cl, qs, 0.09))
        assert max_abs(outs[-1], r) <= TOL[dtype], f"variant {v}"
    ulp = 2.0 ** -10 if dtype == "f16" else 2.0 ** -7  # output ulp at |o| < 1
    for o in outs[1:]:
        diff = (o.float() - outs[0].float()).abs().max().item()
        assert diff <= 4 * ulp


# ------------------------------------------------------------- packed (cascade) -------

def shared_prefix_problem(groups, B, H, H_kv, dtype, seed=5):
    """groups: list of (prefix_len, [(own_len, q_len), ...]).  Each group's first
    prefix_len // B * B tokens sit in physical blocks SHARED by its members (the rest of a
    member's context -- the prefix tail, then its own tokens -- in private blocks); member
    ctx = prefix_len + own_len, its last q_len tokens are the query.  Returns the device
    tensors plus the host hints of pa_paged_prefill_attention_packed."""
    rs = np.random.default_rng(seed)
    ctxs, qlens, shared, rows = [], [], [], []
    blk = 0
    for P, members in groups:
        full = P // B
        shared_ids = list(range(blk, blk + full))
        blk += full
        for mi, (own, ql) in enumerate(members):
            c = P + own
            nb = -(-c // B)
            ids = shared_ids + list(range(blk, blk + nb - full))
            blk += nb - full
            ctxs.append(c)
            qlens.append(ql)
            shared.append(full * B if mi > 0 else 0)
            rows.append(ids)
    NB = blk + 3
    W = max(len(r) for r in rows)
    bt = np.full((len(rows), W), -1, np.int32)
    for s, r in enumerate(rows):
        bt[s, :len(r)] = r
    tdt = torch.float16 if dtype == "f16" else torch.bfloat16
    kc = torch.from_numpy(rs.uniform(-1, 1, (NB, H_kv, B, D)).astype(np.float32)).to(tdt).cuda()
    vc = torch.from_numpy(rs.uniform(-1, 1, (NB, H_kv, B, D)).astype(np.float32)).to(tdt).cuda()
    qs = np.concatenate([[0], np.cumsum(qlens)]).astype(np.int32)
    q = torch.from_numpy(rs.uniform(-1, 1, (int(qs[-1]), H, D)).astype(np.float32)).to(tdt).cuda()
    return (q, kc, vc, torch.as_tensor(bt).cuda(), torch.as_tensor(np.asarray(ctxs, np.int32)).cuda(),
            torch.as_tensor(qs).cuda(), qs, np.asarray(ctxs, np.int32), np.asarray(shared, np.int32))


def run_packed(q, kc, vc, bt, cl, qs, scale, hqs, hcl, hsp):
    out = torch.full_like(q, float("nan"))
    pa.paged_prefill_attention_packed(out, q, kc, vc, bt, cl, qs, scale, hqs, hcl, hsp)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("dtype,B,H,H_kv", [("f16", 16, 4, 4), ("bf16", 16, 4, 2), ("f16", 32, 2, 2)])
def test_packed_prefill_vs_oracle(dtype, B, H, H_kv):
    """Shared-prefix suffixes packed into 128-row tiles (cascade): groups with prefixes that
    are / are not block-aligned and longer / shorter than a key tile, members with 1..90
    query rows, q_len 0, a lone sequence without sharing, and a 300-row query that takes
    tiles of its own -- every row vs the fp64 oracle."""
    groups = [(341, [(30, 30), (5, 5), (60, 60), (1, 1), (33, 20), (90, 90)]),
              (80, [(40, 40), (20, 20), (31, 31), (0, 0), (16, 16)]),
              (0, [(300, 300)]),
              (200, [(10, 10)]),
              (130, [(7, 3), (9, 9), (64, 64), (12, 12)])]
    q, kc, vc, bt, cl, qs, hqs, hcl, hsp = shared_prefix_problem(groups, B, H, H_kv, dtype)
    out = run_packed(q, kc, vc, bt, cl, qs, 0.09, hqs, hcl, hsp)
    r = ref(q, kc, vc, bt, cl, qs, 0.09, B, H_kv, dtype)
    assert not torch.isnan(out).any()
    assert max_abs(out, r) <= TOL[dtype]


def test_packed_prefill_full_size_sampled():
    """The p_prefix5 / p_prefix1 workloads (256 requests after a 341 / 80-token shared
    prefix, LLaMA-13B attention shape): whole output finite, sampled rows x heads vs the
    oracle's Eq.4 row of length pos+1."""
    from synth.prefill import make_prefill
    for name in ("p_prefix5", "p_prefix1"):
        c = make_prefill(name)
        H, H_kv, B = c["H"], c["H_kv"], c["B"]
        dt = torch.float16
        g = torch.Generator(device="cuda")
        g.manual_seed(c["seed"])
        kc = (torch.rand((c["num_blocks"], H_kv, B, D), generator=g, device="cuda") * 2 - 1).to(dt)
        vc = (torch.rand(tuple(kc.shape), generator=g, device="cuda") * 2 - 1).to(dt)
        hqs = np.concatenate([[0], np.cumsum(c["qlen"])]).astype(np.int32)
        q = (torch.rand((int(hqs[-1]), H, D), generator=g, device="cuda") * 2 - 1).to(dt)
        bt = torch.as_tensor(c["block_tables"], device="cuda")
        cl = torch.as_tensor(c["ctx"].astype(np.int32), device="cuda")
        qs = torch.as_tensor(hqs, device="cuda")
        out = run_packed(q, kc, vc, bt, cl, qs, D ** -0.5, hqs, c["ctx"].astype(np.int32), c["shared"].astype(np.int32))
        assert torch.isfinite(out).all()
        rs = np.random.default_rng(11)
        qb, kb, vb, btn, cln = bits(q), bits(kc), bits(vc), bt.cpu().numpy(), cl.cpu().numpy()
        for row in rs.integers(0, int(hqs[-1]), 40):
            s = int(np.searchsorted(hqs, row, side="right") - 1)
            pos = int(cln[s] - (hqs[s + 1] - hqs[s]) + (row - hqs[s]))
            rr = oracle.paged_attention(qb[row:row + 1], kb, vb, btn[s:s + 1], np.array([pos + 1], np.int32),
                                        D ** -0.5, B, H_kv, "f16")
            assert max_abs(out[row:row + 1], rr) <= TOL["f16"], (name, row)


def _packed_fuzz(n=6, seed=6180):
    rs = np.random.default_rng(seed)
    out = []
    for i in range(n):
        groups = []
        for _ in range(int(rs.integers(1, 5))):
            P = int(rs.choice([0, 16, 64, 100, 128, 341, 600]))
            members = []
            for _ in range(int(rs.integers(1, 12))):
                own = int(rs.integers(0, 140))
                members.append((own, int(rs.integers(0, own + 1))))
            groups.append((P, members))
        out.append((groups, ["f16", "bf16"][i % 2], int(rs.choice([1, 2, 4])), int(rs.integers(1, 1 << 20))))
    return out


@pytest.mark.parametrize("groups,dtype,G,seed", _packed_fuzz())
def test_packed_prefill_fuzz_vs_oracle(groups, dtype, G, seed):
    """Seeded random shared-prefix problems through the packed (cascade) prompt kernel:
    prefixes 0..600 tokens (block-aligned or not), 1..11 members per group with 0..139 own
    tokens and 0..own query rows, GQA ratios 1/2/4 -- every row vs the fp64 oracle."""
    H_kv = 2
    q, kc, vc, bt, cl, qs, hqs, hcl, hsp = shared_prefix_problem(groups, 16, H_kv * G, H_kv, dtype, seed=seed)
    if q.shape[0] == 0:
        pytest.skip("no query rows drawn")
    out = run_packed(q, kc, vc, bt, cl, qs, 0.088, hqs, hcl, hsp)
    r = ref(q, kc, vc, bt, cl, qs, 0.088, 16, H_kv, dtype)
    assert not torch.isnan(out).any()
    assert max_abs(out, r) <= TOL[dtype]
