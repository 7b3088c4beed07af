// pa_prefill.cu -- multi-token (prefill / chunked-prefill / shared-prefix suffix) paged
// attention on the sm_100 tensor cores.
//
// Query token i of sequence s (i < q_len_s) sits at logical position
// ctx_s - q_len_s + i and attends causally to every cached token t <= that position,
// read through the block table (Eq.3/Eq.4; prompt phase P:145-147,
// shared prefix P:334-338: "the prompt phase computation only needs to execute on the
// user's task input").  The new tokens' K/V are already in the cache
// (pa_reshape_and_cache with a multi-token slot mapping, reading c5).
//
// Two persistent, warp-specialised kernels (one CTA per SM, TMA producer warp, tcgen05
// MMA-issuer warp, softmax warp groups; thread = query row = tensor-memory lane):
//   * Q tiles [128 x 128] and, per 128-token KV tile, K and V are brought into shared
//     memory by TMA tensor copies with the 128-byte swizzle (K and V gathered block by
//     block through the block table);
//   * S = Q K^T by 8 tcgen05.mma (M=128, N=128, K=16) into tensor memory (fp32);
//   * softmax threads read S rows back with tcgen05.ld, apply scale + causal mask, online
//     softmax in the exp2 domain, and write P (storage dtype) back into tensor memory;
//   * O += P V by 8 tcgen05.mma (P from tensor memory, V read MN-major).
// v2: two query tiles per work item share each K/V tile; v3: one query tile, its softmax
// split by key columns over two warp groups.
// P is rounded to the storage dtype before the second product (the FlashAttention
// convention); the parity tolerance covers it.
#include <cuda.h>

#include <algorithm>

#include "pa_common.cuh"
#include "pa_internal.h"
#include "pa_tc.cuh"


namespace pa {

using namespace tc;

namespace {

constexpr int kQ = 128;        // query rows per CTA
constexpr int kN = 128;        // KV tokens per tile
constexpr int kHalf = 128 * 128;  // bytes of one [128 rows][64 elements] swizzled half (2-byte elements)

}  // namespace


// ---- v2 (default): persistent, warp-specialised, two query tiles per CTA ------------------
// Warps 0-3 / 4-7: softmax of query tile 0 / 1 (thread = row = TMEM lane); warp 8: TMA
// producer; warp 9: tcgen05.mma issuer.  Tensor memory (512 columns): S_0, S_1, O_0, O_1
// (128 fp32 columns each); P_t (storage dtype, packed two per column) overwrites the first
// 64 columns of S_t and feeds O_t += P_t V as the tensor-memory A operand.  K and V are
// double-buffered separately; the MMA order PV_0(j), S_0(j+1), PV_1(j), S_1(j+1) keeps the
// tensor cores on one query tile while the other tile's softmax runs on the SM.  Softmax
// differences from v1: lazy rescaling (kLazy) and l summed from the fp32 weights.
#ifdef PA_PREFILL_TRACE  // timing experiments (variant build): clock64 events of CTA 0..63
__device__ long long g_pf_trace[64 * 256];
#define PF_T(slot)                                                                   \
    do {                                                                             \
        if (blockIdx.x < 64 && (slot) < 256) g_pf_trace[blockIdx.x * 256 + (slot)] = clock64(); \
    } while (0)
#else
#define PF_T(slot) \
    do {           \
    } while (0)
#endif

constexpr int kWarpsV2 = 10;
constexpr float kLazy = 8.f;  // P <= 2^8: no overflow in f16/bf16, same relative rounding
constexpr int kThreadsV2 = kWarpsV2 * 32;
// TMA producer warps of v2 / v3 / v6.  A warp issues its tensor copies one at a time (SASS: an
// ELECT loop around UTMALDG), and a 128-token tile of 16-token blocks is 32 copies of 2 KB
// (K and V, two 64-column halves); with one producer warp that issue rate, not the tensor
// cores, set the step time.  The extra producer warps split each tile's
// copies with warp 8; warp 8 alone arms the barriers (expect_tx) and loads Q.
#ifndef PA_PF_PROD
#define PA_PF_PROD 4
#endif
constexpr int kProd = PA_PF_PROD;
#ifndef PA_PF_PROD_V2
#define PA_PF_PROD_V2 2  // v2 holds 157 registers per thread: 4 producers would cap it at 152
#endif
constexpr int kProdV2 = PA_PF_PROD_V2;
constexpr int kThreadsV3 = kThreadsV2 + 32 * (kProd - 1);    // extra producers: warps 10..
constexpr int kThreadsWs = kThreadsV2 + 32 * (kProdV2 - 1);  // v2's

// Work item = (query-tile pair qp, head h, sequence s); items are dealt to persistent CTAs
// (one per SM) round-robin, longest pairs first.  The barrier phases run on across items,
// so a CTA's producer and MMA warps start the next item while its softmax warps are still
// writing the previous item's output.
struct PrefillItem {
    int h, s, qs, qlen, q0, base_pos, kv0, kv1, n0, n1, kv_len, n;
};
// Items in (sequence, head)-major order, query-tile pairs longest-first within a head: the
// items in flight at the same time on the SMs read the same K/V tiles, which then come
// from L2 (the pairs of one head re-read its K/V).  Longest-first over the whole grid
// instead left the working set of concurrent items far above L2 (ncu on p_2k: L2 hit rate
// 11%, 1.63 GB of DRAM reads for 0.35 GB of K/V).  CTAs draw items from a work counter,
// which balances the unequal causal lengths that this order mixes.
__device__ __forceinline__ bool prefill_item(const PrefillParams& p, int i, PrefillItem& it) {
    const int g = i / p.X;
    const int qp = p.X - 1 - i % p.X;
    it.h = g % p.H;
    it.s = g / p.H;
    it.qs = __ldg(p.query_start + it.s);
    it.qlen = __ldg(p.query_start + it.s + 1) - it.qs;
    it.q0 = qp * 2 * kQ;
    if (it.q0 >= it.qlen) return false;
    it.base_pos = __ldg(p.context_lens + it.s) - it.qlen;
    // tokens query tile t may attend to, and its number of 128-token KV tiles
    it.kv0 = it.base_pos + min(it.q0 + kQ, it.qlen);
    it.kv1 = it.q0 + kQ < it.qlen ? it.base_pos + min(it.q0 + 2 * kQ, it.qlen) : 0;
    it.n0 = it.kv0 > 0 ? (it.kv0 + kN - 1) / kN : 0;
    it.n1 = it.kv1 > 0 ? (it.kv1 + kN - 1) / kN : 0;
    it.kv_len = max(it.kv0, it.kv1);
    it.n = max(it.n0, it.n1);
    return true;
}

template <typename T>
__global__ void __launch_bounds__(kThreadsWs, 1) paged_prefill_ws_kernel(const __grid_constant__ PrefillParams p) {
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = tc::smem_align1024(smem_raw);
    unsigned char* sQ = smem;                // [2 tiles][2 halves][128][64]
    unsigned char* sK = smem + 4 * kHalf;    // [2 stages][2 halves][128][64]
    unsigned char* sV = sK + 4 * kHalf;      // [2 stages][2 halves][128][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 4 * kHalf);
    uint64_t* q_full = bars;         // 1
    uint64_t* q_empty = bars + 1;    // 1
    uint64_t* k_full = bars + 2;     // 2
    uint64_t* k_empty = bars + 4;    // 2
    uint64_t* v_full = bars + 6;     // 2
    uint64_t* v_empty = bars + 8;    // 2
    uint64_t* s_full = bars + 10;    // 2 (per query tile)
    uint64_t* p_full = bars + 12;    // 2
    uint64_t* o_done = bars + 14;    // 2
    uint64_t* o_free = bars + 16;    // 2
    uint64_t* sched_full = bars + 18;   // 4: work-item ring (producer -> MMA + softmax warps)
    uint64_t* sched_empty = bars + 22;  // 4
    int* sched_item = reinterpret_cast<int*>(bars + 26);  // 4
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sched_item + 4);
#ifdef PA_PREFILL_MUTEX
    int* mufu_owner = reinterpret_cast<int*>(tmem_slot + 1);  // softmax group in its exp phase, -1: none
    if (threadIdx.x == 0) *mufu_owner = -1;
#endif

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_items = p.X * p.H * p.S;
    pdl_wait();

    if (tid == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(&sched_full[i], 1);
            mbar_init(&sched_empty[i], kProdV2 + 2 * kQ);  // MMA warp + extra producers (one arrive each) + 256 softmax threads
        }
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], kQ);
            mbar_init(&o_done[i], 1);
            mbar_init(&o_free[i], kQ);
        }
        fence_mbar_init();
    }
    // V stages start zeroed: rows past kv_len of a last tile are never loaded and must not
    // hold NaN bit patterns (P = 0 there, but 0 * NaN = NaN in the MMA); later they hold
    // rows of earlier tiles (finite cache data)
    for (int i = tid; i < 4 * kHalf / 16; i += kThreadsWs)
        reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int B = 1 << p.log2B;

    if (warp == 8 || warp >= kWarpsV2) {
        // ---------------- TMA producers (pw 0 = warp 8) ----------------
        const int pw = warp == 8 ? 0 : warp - kWarpsV2 + 1;
        const int br = p.box_rows;
        uint32_t g = 0;    // KV tiles loaded by this CTA (stage = g & 1)
        uint32_t nq = 0;   // query tile pairs loaded
        for (uint32_t k = 0;; ++k) {
            // producer 0 draws the next work item and publishes it to the other warps
            const uint32_t slot = k & 3;
            int i = 0;
            if (pw == 0) {
                if (k >= 4) mbar_wait(&sched_empty[slot], ((k - 4) >> 2) & 1);
                if (lane == 0) {
                    i = atomicAdd(p.work_counter, 1);
                    sched_item[slot] = i;
                    mbar_arrive(&sched_full[slot]);
                }
                i = __shfl_sync(0xffffffffu, i, 0);
            } else {
                mbar_wait(&sched_full[slot], (k >> 2) & 1);
                i = *reinterpret_cast<volatile int*>(&sched_item[slot]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&sched_empty[slot]);
            }
            if (i >= n_items) break;
            PrefillItem it;
            if (!prefill_item(p, i, it)) continue;
            const int kvh = it.h / p.G;
            const int32_t* btrow = p.block_tables + (int64_t)it.s * p.W;
            // tile j = tokens [128j, min(kv_len, 128j+128)): nf boxes of br rows, then
            // single rows (never reading past kv_len).  Box b belongs to lane b % 32: the
            // lanes look up the block table in parallel and issue their own TMA copies.
            auto box_token = [&](int b, int nf) { return b < nf ? b * br : nf * br + (b - nf); };
            auto lookup = [&](int j, int (&rowv)[4]) {
                const int t0 = j * kN, len = min(it.kv_len, t0 + kN) - t0;
                const int nf = len / br, nb = nf + len % br;
#pragma unroll
                for (int u = 0; u < (4 + kProdV2 - 1) / kProdV2; ++u) {
                    const int b = pw + kProdV2 * (lane + 32 * u);  // boxes interleaved over the producers
                    if (b < nb) {
                        const int t = t0 + box_token(b, nf);
                        const int blk = __ldg(btrow + (t >> p.log2B));
                        rowv[u] = (blk * p.H_kv + kvh) * B + (t & (B - 1));
                    }
                }
            };
            auto issue = [&](unsigned char* dst0, const CUtensorMap* map, const CUtensorMap* map1, int j,
                             uint64_t* bar, const int (&rowv)[4]) {
                const int t0 = j * kN, len = min(it.kv_len, t0 + kN) - t0;
                const int nf = len / br, nb = nf + len % br;
                if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)len * 256u);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < (4 + kProdV2 - 1) / kProdV2; ++u) {
                    const int b = pw + kProdV2 * (lane + 32 * u);  // boxes interleaved over the producers
                    if (b < nb) {
                        const int off = box_token(b, nf) * 128;
                        const CUtensorMap* m = b < nf ? map : map1;
                        tma_load_2d(dst0 + off, m, 0, rowv[u], bar);
                        tma_load_2d(dst0 + kHalf + off, m, 64, rowv[u], bar);
                    }
                }
                __syncwarp();
            };
            int rowv[4] = {0, 0, 0, 0};
            if (it.n > 0) lookup(0, rowv);
            if (pw == 0 && nq > 0) mbar_wait(q_empty, (nq - 1) & 1);  // last S of the previous pair done
            if (pw == 0 && lane == 0) {
                mbar_arrive_expect_tx(q_full, 4u * kHalf);
                tma_load_3d(sQ, &p.tmap_q, 0, it.h, it.qs + it.q0, q_full);
                tma_load_3d(sQ + kHalf, &p.tmap_q, 64, it.h, it.qs + it.q0, q_full);
                tma_load_3d(sQ + 2 * kHalf, &p.tmap_q, 0, it.h, it.qs + it.q0 + kQ, q_full);
                tma_load_3d(sQ + 3 * kHalf, &p.tmap_q, 64, it.h, it.qs + it.q0 + kQ, q_full);
            }
            __syncwarp();
            ++nq;
            for (int j = 0; j < it.n; ++j, ++g) {
                const int st = g & 1;
                if (g >= 2) mbar_wait(&k_empty[st], ((g - 2) >> 1) & 1);
                issue(sK + st * 2 * kHalf, &p.tmap_k, &p.tmap_k1, j, &k_full[st], rowv);
                if (pw == 0 && lane == 0 && k == 0 && j < 16) PF_T(192 + 4 * j);
                if (g >= 2) mbar_wait(&v_empty[st], ((g - 2) >> 1) & 1);
                issue(sV + st * 2 * kHalf, &p.tmap_v, &p.tmap_v1, j, &v_full[st], rowv);
                if (pw == 0 && lane == 0 && k == 0 && j < 16) PF_T(192 + 4 * j + 1);
                if (j + 1 < it.n) lookup(j + 1, rowv);  // in flight while the next empty-wait spins
            }
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc_s = umma_idesc(kBF16, false), idesc_o = umma_idesc(kBF16, true);
        uint32_t g = 0, nq = 0;
        uint32_t np[2] = {0, 0};  // P tiles consumed per query tile (p_full phases)
        uint32_t nf[2] = {0, 0};  // pairs with tiles per query tile (o_free phases)
        auto issue_S = [&](int t, uint32_t gs) {  // S_t = Q_t K^T, K in stage gs & 1
            if (lane == 0) {
                const uint32_t q = smem_u32(sQ) + t * 2 * kHalf, k = smem_u32(sK) + (gs & 1) * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    umma_f16(tmem + t * 128, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(k + off, 16, 1024),
                             idesc_s, kk > 0);
                }
                umma_commit(&s_full[t]);
            }
            __syncwarp();
        };
        auto issue_PV = [&](int t, uint32_t gs, bool first) {  // O_t (+)= P_t V, P_t in tensor memory
            if (lane == 0) {
                const uint32_t v = smem_u32(sV) + (gs & 1) * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                                umma_desc_sw128(v + kk * 2048, kHalf, 1024), idesc_o, (!first) | (kk > 0));
                umma_commit(&o_done[t]);
            }
            __syncwarp();
        };
        for (uint32_t k = 0;; ++k) {
            const uint32_t slot = k & 3;
            mbar_wait(&sched_full[slot], (k >> 2) & 1);
            const int i = *reinterpret_cast<volatile int*>(&sched_item[slot]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sched_empty[slot]);
            if (i >= n_items) break;
            PrefillItem it;
            if (!prefill_item(p, i, it)) continue;
            mbar_wait(q_full, nq & 1);
            if (it.n > 0) {
                mbar_wait(&k_full[g & 1], (g >> 1) & 1);
                tc_fence_after();
                if (it.n0 > 0) issue_S(0, g);
                if (it.n1 > 0) issue_S(1, g);
                if (lane == 0) umma_commit(&k_empty[g & 1]);
                if (it.n == 1 && lane == 0) umma_commit(q_empty);
            } else if (lane == 0) {
                umma_commit(q_empty);
            }
            // O_t is overwritten by this pair's first P V: the softmax warp group must have
            // read O_t of its previous pair with tiles (o_free; a group with no tiles in a
            // pair neither arrives nor is waited for, so it can never run two phases ahead)
            if (it.n0 > 0 && nf[0]++ > 0) mbar_wait(&o_free[0], (nf[0] - 2) & 1);
            if (it.n1 > 0 && nf[1]++ > 0) mbar_wait(&o_free[1], (nf[1] - 2) & 1);
            ++nq;
            for (int j = 0; j < it.n; ++j, ++g) {
                const int st = g & 1;
                mbar_wait(&v_full[st], (g >> 1) & 1);
                if (lane == 0 && k == 0 && j < 16) PF_T(128 + 4 * j);
                if (j < it.n0) {
                    mbar_wait(&p_full[0], np[0]++ & 1);
                    tc_fence_after();
                    issue_PV(0, g, j == 0);
                }
                const bool more = j + 1 < it.n;
                if (more) {
                    if (lane == 0 && k == 0 && j < 16) PF_T(128 + 4 * j + 1);
                    mbar_wait(&k_full[st ^ 1], ((g + 1) >> 1) & 1);
                    if (lane == 0 && k == 0 && j < 16) PF_T(128 + 4 * j + 2);
                    tc_fence_after();
                    if (j + 1 < it.n0) issue_S(0, g + 1);
                }
                if (j < it.n1) {
                    mbar_wait(&p_full[1], np[1]++ & 1);
                    if (lane == 0 && k == 0 && j < 16) PF_T(128 + 4 * j + 3);
                    tc_fence_after();
                    issue_PV(1, g, j == 0);
                }
                if (lane == 0) umma_commit(&v_empty[st]);
                if (more) {
                    if (j + 1 < it.n1) issue_S(1, g + 1);
                    if (lane == 0) {
                        umma_commit(&k_empty[st ^ 1]);
                        if (j + 2 == it.n) umma_commit(q_empty);  // every S of this pair issued
                    }
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- softmax warp groups ----------------
        const int t = warp >> 2;
        const int r = tid & (kQ - 1);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 128 + lane_off, tO = tmem + 256 + t * 128 + lane_off;
        uint32_t ns = 0;  // S tiles consumed by this warp group (s_full / o_done phases)
        for (uint32_t k = 0;; ++k) {
            const uint32_t slot = k & 3;
            mbar_wait(&sched_full[slot], (k >> 2) & 1);
            const int i = *reinterpret_cast<volatile int*>(&sched_item[slot]);
            mbar_arrive(&sched_empty[slot]);
            if (i >= n_items) break;
            PrefillItem it;
            if (!prefill_item(p, i, it)) continue;
            const int nt = t == 0 ? it.n0 : it.n1;
            const int kvt = t == 0 ? it.kv0 : it.kv1;
            const int row = it.q0 + t * kQ + r;
            const bool row_valid = row < it.qlen;
            const int pos = row_valid ? it.base_pos + row : -1;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nt; ++j, ++ns) {
                mbar_wait(&s_full[t], ns & 1);
                tc_fence_after();
                if ((tid & 127) == 0 && k == 0 && j < 16) PF_T(t * 64 + 4 * j);
                float sa[32], sb[32], sc[32], sd[32];
                tmem_ld32_nw(tS + 0, sa);
                tmem_ld32_nw(tS + 32, sb);
                tmem_ld32_nw(tS + 64, sc);
                tmem_ld32_nw(tS + 96, sd);
                tmem_ld_wait();
                if ((tid & 127) == 0 && k == 0 && j < 16) PF_T(t * 64 + 4 * j + 1);
                const int lim = row_valid ? min(pos + 1, kvt) - j * kN : 0;
                // scale > 0: max(s) * c == max(s * c) exactly (rounding is monotonic)
                const bool full = __all_sync(0xffffffffu, lim >= kN);  // no masking in this tile
                float mt = -INFINITY;
                if (full) {
#pragma unroll
                    for (int u = 0; u < 32; ++u) mt = fmaxf(fmaxf(mt, sa[u]), fmaxf(sb[u], fmaxf(sc[u], sd[u])));
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        if (u < lim) mt = fmaxf(mt, sa[u]);
                        if (u + 32 < lim) mt = fmaxf(mt, sb[u]);
                        if (u + 64 < lim) mt = fmaxf(mt, sc[u]);
                        if (u + 96 < lim) mt = fmaxf(mt, sd[u]);
                    }
                }
                mt *= p.scale_log2;
                // lazy rescaling: the reference maximum m only moves when some row of the
                // warp sees a score more than kLazy (log2 units) above it, so O_t is rarely
                // rescaled; P = 2^(s*c - m) <= 2^kLazy and l use the same m
                const bool bump = __any_sync(0xffffffffu, mt > m + kLazy);
                const float mn = bump ? fmaxf(m, mt) : m;
                const float ms = (mn == -INFINITY) ? 0.f : mn;
                const float alpha = bump ? ex2(m - ms) : 1.f;
                // P rounded to the storage dtype (MMA operand); the row sum l accumulates
                // the fp32 values.  Full tiles take a select-free path.
                float2 rs2 = make_float2(0.f, 0.f);
                const float2 c2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-ms, -ms);
                auto emit = [&](const float (&x)[32], int c0) {
                    uint32_t pk[16];
                    if (full) {
#pragma unroll
                        for (int u = 0; u < 32; u += 2) {
                            const float2 e = ffma2(make_float2(x[u], x[u + 1]), c2, nm2);  // s*c - m
                            const float2 a = ex2_pair(e, u / 2);
                            rs2 = __fadd2_rn(rs2, a);
                            pk[u / 2] = pack2<T>(a.x, a.y);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < 32; u += 2) {
                            const float2 e = ffma2(make_float2(x[u], x[u + 1]), c2, nm2);
                            float2 a = make_float2(ex2(e.x), ex2(e.y));
                            a.x = (c0 + u < lim) ? a.x : 0.f;
                            a.y = (c0 + u + 1 < lim) ? a.y : 0.f;
                            rs2 = __fadd2_rn(rs2, a);
                            pk[u / 2] = pack2<T>(a.x, a.y);
                        }
                    }
                    tmem_st16(tS + c0 / 2, pk);
                };
#ifdef PA_PREFILL_MUTEX
                // one softmax group at a time in the MUFU-bound exp phase: the two groups
                // share every SM sub-partition's MUFU; alternating keeps each phase short
                if ((tid & 127) == 0)
                    while (atomicCAS(mufu_owner, -1, t) != -1) {
                    }
                asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
#endif
                emit(sa, 0);
                emit(sb, 32);
                emit(sc, 64);
                emit(sd, 96);
#ifdef PA_PREFILL_MUTEX
                asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
                if ((tid & 127) == 0) atomicExch(mufu_owner, -1);
#endif
                if ((tid & 127) == 0 && k == 0 && j < 16) PF_T(t * 64 + 4 * j + 2);
                // P_t is out; now O_t *= alpha.  PV_t of the previous tile has completed (this
                // S_t was issued after it), so this wait returns at once; it is not skipped
                // so that every o_done phase is waited on
                if (j > 0) {
                    mbar_wait(&o_done[t], (ns - 1) & 1);
                    tc_fence_after();
                }
                if (j > 0 && bump) {
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 32) {
                        float v[32];
                        tmem_ld32_nw(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) v[u] *= alpha;
                        tmem_st32(tO + c0, v);
                    }
                }
                l = l * alpha + (rs2.x + rs2.y);
                m = mn;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[t]);
                if ((tid & 127) == 0 && k == 0 && j < 16) PF_T(t * 64 + 4 * j + 3);
            }
            // epilogue: out row = O_t / l
            const float inv = l > 0.f ? 1.f / l : 0.f;
            T* orow = static_cast<T*>(p.out) + ((int64_t)(it.qs + row) * p.H + it.h) * 128;
            if (nt > 0) {
                mbar_wait(&o_done[t], (ns - 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                float v[32];
                if (nt > 0) {
                    tmem_ld32_nw(tO + c0, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) v[u] = 0.f;
                }
                if (row_valid) {
#pragma unroll
                    for (int c1 = 0; c1 < 32; c1 += 8) {
                        alignas(16) T w[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) w[u] = Elem<T>::from_f32(v[c1 + u] * inv);
                        *reinterpret_cast<uint4*>(orow + c0 + c1) = *reinterpret_cast<const uint4*>(w);
                    }
                }
            }
            if (nt > 0) {
                tc_fence_before();
                mbar_arrive(&o_free[t]);  // O_t may be overwritten by the next pair
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}



// ---- v3 (default): persistent, one query tile per item, softmax split by columns ----------
// The two softmax warp groups share the 128 rows of ONE query tile: group 0 takes key
// columns [0,64), group 1 [64,128) of every 128-key tile (warps w and w+4 address the same
// TMEM lanes).  Row maxima are exchanged through shared memory (named barrier, 256
// threads); each group keeps its own partial row sum with the same reference maximum, and
// the two sums are added in the epilogue.  Tensor memory: two S buffers (columns 0 and
// 128, P aliased in the first 64 columns of its buffer) and O (256..383), so the MMA warp
// computes S(j+1) = Q K_{j+1}^T while the softmax of tile j runs, and P V for tile j-1;
// the per-tile softmax is half as long as in v2 and off the tensor-core critical path.
// Shared memory: Q double-buffered (the next item's Q loads during this item), K and V in
// two stages each (192 KB).
constexpr int kKStages = 2, kVStages = 2;

struct PrefillItem1 {
    int h, s, qs, qlen, q0, base_pos, kv_len, n;
};
__device__ __forceinline__ bool prefill_item1(const PrefillParams& p, int i, PrefillItem1& it) {
    const int hs = p.H * p.S;
    const int qt = p.X - 1 - i / hs, rem = i % hs;  // longest query tiles first
    it.h = rem % p.H;
    it.s = rem / p.H;
    it.qs = __ldg(p.query_start + it.s);
    it.qlen = __ldg(p.query_start + it.s + 1) - it.qs;
    it.q0 = qt * kQ;
    if (it.q0 >= it.qlen) return false;
    it.base_pos = __ldg(p.context_lens + it.s) - it.qlen;
    it.kv_len = it.base_pos + min(it.q0 + kQ, it.qlen);
    it.n = it.kv_len > 0 ? (it.kv_len + kN - 1) / kN : 0;
    return true;
}

__device__ __forceinline__ void named_bar_sync_256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <typename T>
__global__ void __launch_bounds__(kThreadsV3, 1) paged_prefill_split_kernel(const __grid_constant__ PrefillParams p) {
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = tc::smem_align1024(smem_raw);
    unsigned char* sQ = smem;                          // [2 buffers][2 halves][128][64]
    unsigned char* sK = smem + 4 * kHalf;              // [3 stages][2 halves][128][64]
    unsigned char* sV = sK + 2 * kKStages * kHalf;     // [2 stages][2 halves][128][64]
    float* red = reinterpret_cast<float*>(sV + 2 * kVStages * kHalf);  // [2 parity][2 groups][128] row maxima
    float* lsum = red + 512;                                            // [2 groups][128] row sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(lsum + 256);
    uint64_t* q_full = bars;                 // 2
    uint64_t* q_empty = bars + 2;            // 2
    uint64_t* k_full = bars + 4;             // 3
    uint64_t* k_empty = bars + 7;            // 3
    uint64_t* v_full = bars + 10;            // 2
    uint64_t* v_empty = bars + 12;           // 2
    uint64_t* s_full = bars + 14;            // 2 (per S buffer)
    uint64_t* p_full = bars + 16;            // 1
    uint64_t* o_done = bars + 17;            // 1
    uint64_t* o_free = bars + 18;            // 1
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_items = p.X * p.H * p.S;
    pdl_wait();

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
        }
        for (int i = 0; i < kKStages; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
        }
        mbar_init(p_full, 2 * kQ);
        mbar_init(o_done, 1);
        mbar_init(o_free, 2 * kQ);
        fence_mbar_init();
    }
    // V stages start zeroed (see v2)
    for (int i = tid; i < 2 * kVStages * kHalf / 16; i += kThreadsV3)
        reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int B = 1 << p.log2B;

    if (warp == 8 || warp >= kWarpsV2) {
        // ---------------- TMA producers (pw 0 = warp 8) ----------------
        const int pw = warp == 8 ? 0 : warp - kWarpsV2 + 1;
        const int br = p.box_rows;
        uint32_t g = 0, nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
            PrefillItem1 it;
            if (!prefill_item1(p, i, it)) continue;
            const int kvh = it.h / p.G;
            const int32_t* btrow = p.block_tables + (int64_t)it.s * p.W;
            auto box_token = [&](int b, int nf) { return b < nf ? b * br : nf * br + (b - nf); };
            auto lookup = [&](int j, int (&rowv)[4]) {
                const int t0 = j * kN, len = min(it.kv_len, t0 + kN) - t0;
                const int nf = len / br, nb = nf + len % br;
#pragma unroll
                for (int u = 0; u < (4 + kProd - 1) / kProd; ++u) {
                    const int b = pw + kProd * (lane + 32 * u);  // boxes interleaved over the producers
                    if (b < nb) {
                        const int t = t0 + box_token(b, nf);
                        const int blk = __ldg(btrow + (t >> p.log2B));
                        rowv[u] = (blk * p.H_kv + kvh) * B + (t & (B - 1));
                    }
                }
            };
            auto issue = [&](unsigned char* dst0, const CUtensorMap* map, const CUtensorMap* map1, int j,
                             uint64_t* bar, const int (&rowv)[4]) {
                const int t0 = j * kN, len = min(it.kv_len, t0 + kN) - t0;
                const int nf = len / br, nb = nf + len % br;
                if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)len * 256u);
                __syncwarp();
#pragma unroll
                for (int u = 0; u < (4 + kProd - 1) / kProd; ++u) {
                    const int b = pw + kProd * (lane + 32 * u);  // boxes interleaved over the producers
                    if (b < nb) {
                        const int off = box_token(b, nf) * 128;
                        const CUtensorMap* m = b < nf ? map : map1;
                        tma_load_2d(dst0 + off, m, 0, rowv[u], bar);
                        tma_load_2d(dst0 + kHalf + off, m, 64, rowv[u], bar);
                    }
                }
                __syncwarp();
            };
            int rowv[4] = {0, 0, 0, 0};
            if (it.n > 0) lookup(0, rowv);
            const int qb = nq & 1;
            if (pw == 0 && nq >= 2) mbar_wait(&q_empty[qb], ((nq - 2) >> 1) & 1);
            if (pw == 0 && lane == 0) {
                mbar_arrive_expect_tx(&q_full[qb], 2u * kHalf);
                tma_load_3d(sQ + qb * 2 * kHalf, &p.tmap_q, 0, it.h, it.qs + it.q0, &q_full[qb]);
                tma_load_3d(sQ + qb * 2 * kHalf + kHalf, &p.tmap_q, 64, it.h, it.qs + it.q0, &q_full[qb]);
            }
            __syncwarp();
            ++nq;
            for (int j = 0; j < it.n; ++j, ++g) {
                const uint32_t ks = g % kKStages, vs = g & 1;
                if (g >= kKStages) mbar_wait(&k_empty[ks], ((g - kKStages) / kKStages) & 1);
                issue(sK + ks * 2 * kHalf, &p.tmap_k, &p.tmap_k1, j, &k_full[ks], rowv);
                if (g >= 2) mbar_wait(&v_empty[vs], ((g - 2) >> 1) & 1);
                issue(sV + vs * 2 * kHalf, &p.tmap_v, &p.tmap_v1, j, &v_full[vs], rowv);
                if (j + 1 < it.n) lookup(j + 1, rowv);
            }
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer ----------------
        const uint32_t idesc_s = umma_idesc(kBF16, false), idesc_o = umma_idesc(kBF16, true);
        uint32_t gk = 0, gv = 0, nq = 0, np = 0, nf = 0;
        auto issue_S = [&](uint32_t qb) {  // S(gk) = Q K(gk)^T into S buffer gk & 1
            const uint32_t ks = gk % kKStages;
            mbar_wait(&k_full[ks], (gk / kKStages) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t q = smem_u32(sQ) + qb * 2 * kHalf, k = smem_u32(sK) + ks * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    umma_f16(tmem + (gk & 1) * 128, umma_desc_sw128(q + off, 16, 1024),
                             umma_desc_sw128(k + off, 16, 1024), idesc_s, kk > 0);
                }
                umma_commit(&s_full[gk & 1]);
                umma_commit(&k_empty[ks]);
            }
            __syncwarp();
            ++gk;
        };
        for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
            PrefillItem1 it;
            if (!prefill_item1(p, i, it)) continue;
            const uint32_t qb = nq & 1;
            mbar_wait(&q_full[qb], (nq >> 1) & 1);
            ++nq;
            // S runs up to two tiles ahead of P V (two S buffers)
            for (int j = 0; j < min(it.n, 2); ++j) issue_S(qb);
            if (it.n <= 2 && lane == 0) umma_commit(&q_empty[qb]);  // every S of this item issued
            if (it.n > 0 && nf++ > 0) mbar_wait(o_free, (nf - 2) & 1);  // O read by the epilogue
            for (int j = 0; j < it.n; ++j) {
                mbar_wait(&v_full[gv & 1], (gv >> 1) & 1);
                mbar_wait(p_full, np++ & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t v = smem_u32(sV) + (gv & 1) * 2 * kHalf;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16_ts(tmem + 256, tmem + (gv & 1) * 128 + kk * 8,
                                    umma_desc_sw128(v + kk * 2048, kHalf, 1024), idesc_o, (j > 0) | (kk > 0));
                    umma_commit(o_done);
                    umma_commit(&v_empty[gv & 1]);
                }
                __syncwarp();
                ++gv;
                if (j + 2 < it.n) {
                    issue_S(qb);  // overwrites the P just consumed (in issue order)
                    if (j + 3 == it.n && lane == 0) umma_commit(&q_empty[qb]);
                }
            }
        }
    } else {
        // ---------------- softmax warp groups (column halves) ----------------
        const int hf = warp >> 2;              // key columns [64 hf, 64 hf + 64) of each tile
        const int r = tid & (kQ - 1);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tO = tmem + 256 + hf * 64 + lane_off;
        uint32_t ns = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
            PrefillItem1 it;
            if (!prefill_item1(p, i, it)) continue;
            const int row = it.q0 + r;
            const bool row_valid = row < it.qlen;
            const int pos = row_valid ? it.base_pos + row : -1;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < it.n; ++j, ++ns) {
                const uint32_t b = ns & 1;
                const uint32_t tS = tmem + b * 128 + lane_off;
                mbar_wait(&s_full[b], (ns >> 1) & 1);
                tc_fence_after();
                float sa[32], sb[32];
                tmem_ld32_nw(tS + hf * 64, sa);
                tmem_ld32_nw(tS + hf * 64 + 32, sb);
                tmem_ld_wait();
                const int lim = row_valid ? min(pos + 1, it.kv_len) - j * kN - hf * 64 : 0;
                const bool full = __all_sync(0xffffffffu, lim >= 64);
                float mo = -INFINITY;
                if (full) {
#pragma unroll
                    for (int u = 0; u < 32; u += 2)
                        mo = fmaxf(fmaxf(mo, fmaxf(sa[u], sa[u + 1])), fmaxf(sb[u], sb[u + 1]));
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        if (u < lim) mo = fmaxf(mo, sa[u]);
                        if (u + 32 < lim) mo = fmaxf(mo, sb[u]);
                    }
                }
                // row maximum over both halves (the S reads above complete before the other
                // group overwrites columns of this buffer with P)
                float* rd = red + (ns & 1) * 256;
                rd[hf * 128 + r] = mo;
                named_bar_sync_256();
                float mt = fmaxf(mo, rd[(hf ^ 1) * 128 + r]);
                mt *= p.scale_log2;
                // lazy rescaling, decided identically by both groups (same rows, same mt)
                const bool bump = __any_sync(0xffffffffu, mt > m + kLazy);
                const float mn = bump ? fmaxf(m, mt) : m;
                const float ms = (mn == -INFINITY) ? 0.f : mn;
                const float alpha = bump ? ex2(m - ms) : 1.f;
                float2 rs2 = make_float2(0.f, 0.f);
                const float2 c2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-ms, -ms);
                auto emit = [&](const float (&x)[32], int c0) {
                    uint32_t pk[16];
                    if (full) {
#pragma unroll
                        for (int u = 0; u < 32; u += 2) {
                            const float2 e = ffma2(make_float2(x[u], x[u + 1]), c2, nm2);
                            const float2 a = ex2_pair(e, u / 2);
                            rs2 = __fadd2_rn(rs2, a);
                            pk[u / 2] = pack2<T>(a.x, a.y);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < 32; u += 2) {
                            const float2 e = ffma2(make_float2(x[u], x[u + 1]), c2, nm2);
                            float2 a = make_float2(ex2(e.x), ex2(e.y));
                            a.x = (c0 + u < lim) ? a.x : 0.f;
                            a.y = (c0 + u + 1 < lim) ? a.y : 0.f;
                            rs2 = __fadd2_rn(rs2, a);
                            pk[u / 2] = pack2<T>(a.x, a.y);
                        }
                    }
                    tmem_st16(tS + hf * 32 + c0 / 2, pk);  // P columns of this half
                };
                emit(sa, 0);
                emit(sb, 32);
                if (j > 0) {  // P V of the previous tile done (never skipped: every phase is waited on)
                    mbar_wait(o_done, (ns - 1) & 1);
                    tc_fence_after();
                }
                if (j > 0 && bump) {  // O columns of this half *= alpha
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        float v[32];
                        tmem_ld32_nw(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) v[u] *= alpha;
                        tmem_st32(tO + c0, v);
                    }
                }
                l = l * alpha + (rs2.x + rs2.y);
                m = mn;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full);
            }
            // epilogue: both partial row sums, then this half's 64 output columns
            lsum[hf * 128 + r] = l;
            named_bar_sync_256();
            const float lt = l + lsum[(hf ^ 1) * 128 + r];
            named_bar_sync_256();  // lsum may be rewritten by the next item
            const float inv = lt > 0.f ? 1.f / lt : 0.f;
            T* orow = static_cast<T*>(p.out) + ((int64_t)(it.qs + row) * p.H + it.h) * 128 + hf * 64;
            if (it.n > 0) {
                mbar_wait(o_done, (ns - 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {
                float v[32];
                if (it.n > 0) {
                    tmem_ld32_nw(tO + c0, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) v[u] = 0.f;
                }
                if (row_valid) {
#pragma unroll
                    for (int c1 = 0; c1 < 32; c1 += 8) {
                        alignas(16) T w[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) w[u] = Elem<T>::from_f32(v[c1 + u] * inv);
                        *reinterpret_cast<uint4*>(orow + c0 + c1) = *reinterpret_cast<const uint4*>(w);
                    }
                }
            }
            if (it.n > 0) {
                tc_fence_before();
                mbar_arrive(o_free);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

size_t prefill_split_smem_bytes() {
    return 1024 + (4 + 2 * kKStages + 2 * kVStages) * (size_t)kHalf + (512 + 256) * 4 + 20 * 8;
}

size_t prefill_ws_smem_bytes() { return 1024 + 12 * (size_t)kHalf + 26 * 8 + 4 * 4 + 16; }

// ---- v6: packed shared-prefix suffixes (pa_paged_prefill_attention_packed) --------------
// Work item = (packed query tile t, head h), heads outermost so the CTAs running together
// read one head's shared prefix (it stays in L2).  The tile's 128 query rows are the rows
// of nm consecutive sequences (each <= 128 rows) that share their first P cached tokens,
// so the shared prefix is attended ONCE for all of them (cascade): K/V tiles 0..n_pre-1 are
// the prefix tokens [0, P) (every row sees every column), then n_suf tiles pack the
// members' own tokens [P, ctx_k) back to back (member k at packed columns [col_k, col_k +
// ctx_k - P)); a row of member k at position pos sees the contiguous packed columns
// [col_k, col_k + pos - P + 1) -- its causal range inside its own segment.
// Otherwise the v3 pipeline: one query tile, softmax split by key columns over two warp
// groups, S double-buffered in tensor memory, K / V in two stages each.  The producer
// publishes each item's member table (row offset, context, packed column offset, piece
// offset) in shared memory for the softmax warps.
constexpr int kMaxMem = 128;
constexpr int kMaxPre = 256;     // 16-token positions of the shared prefix (P <= 4096)
constexpr int kMaxPieces = 512;  // 16-token pieces of the members' own tokens per tile
constexpr int kThreadsV6 = kThreadsV2 + 32 * kProd;  // + scheduler warp 10, producers 11..
struct PackMem {
    int row_off, ctx, col_off, piece_off, qlen;
};
// One item's table, built by the scheduler warp one item ahead: the members, and the
// physical block of every 16-token position of the prefix and of every own-token piece,
// so the TMA producer issues copies without a global round trip of its own.
struct PackSlot {
    PackMem mem[kMaxMem + 1];
    int hdr[9];  // rows, packed columns seen, n_pre, n, nm, P, first query row, head, s0
    int pre_blk[kMaxPre];
    int piece_blk[kMaxPieces];
};

__device__ __forceinline__ void packed_item(const PackTable& t, const PrefillParams& p, int i, int& tile, int& h,
                                            int& s0, int& nm, int& P, int& r0) {
    tile = i % t.n_tiles;
    h = i / t.n_tiles;
    s0 = t.s0[tile];
    nm = t.nm[tile];
    P = t.P[tile];
    r0 = t.r0[tile];
}

template <typename T>
__global__ void __launch_bounds__(kThreadsV6, 1)
    paged_prefill_packed_kernel(const __grid_constant__ PrefillParams p, const __grid_constant__ PackTable pt) {
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = tc::smem_align1024(smem_raw);
    unsigned char* sQ = smem;                          // [2 buffers][2 halves][128][64]
    unsigned char* sK = smem + 4 * kHalf;              // [2 stages][2 halves][128][64]
    unsigned char* sV = sK + 2 * kKStages * kHalf;     // [2 stages][2 halves][128][64]
    unsigned char* stage = sV + 2 * kVStages * kHalf;  // [8 softmax warps][32 rows][64 B] output staging
    float* red = reinterpret_cast<float*>(stage + 8 * 2048);  // [2 parity][2 groups][128] row maxima
    float* lsum = red + 512;                                   // [2 groups][128] row sums
    PackSlot* slots = reinterpret_cast<PackSlot*>(lsum + 256);         // [2 parity]
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 2);
    uint64_t* q_full = bars;                 // 2
    uint64_t* q_empty = bars + 2;            // 2
    uint64_t* k_full = bars + 4;             // 2
    uint64_t* k_empty = bars + 6;            // 2
    uint64_t* v_full = bars + 8;             // 2
    uint64_t* v_empty = bars + 10;           // 2
    uint64_t* s_full = bars + 12;            // 2 (per S buffer)
    uint64_t* p_full = bars + 14;            // 1
    uint64_t* o_done = bars + 15;            // 1
    uint64_t* o_free = bars + 16;            // 1
    uint64_t* m_full = bars + 17;            // 2: item table published (scheduler warp)
    uint64_t* m_empty = bars + 19;           // 2: item table read (8 softmax warps, MMA, producers)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 21);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_items = pt.n_tiles * p.H;
    pdl_wait();

    if (tid == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&q_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&m_full[i], 1);
            mbar_init(&m_empty[i], 9 + kProd);
        }
        mbar_init(p_full, 2 * kQ);
        mbar_init(o_done, 1);
        mbar_init(o_free, 2 * kQ);
        fence_mbar_init();
    }
    // V stages start zeroed: columns of a last tile past its tokens are never loaded
    for (int i = tid; i < 2 * kVStages * kHalf / 16; i += kThreadsV6)
        reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int B = 1 << p.log2B;

    if (warp == 10) {
        // ---------------- scheduler: each item's table, one item ahead ----------------
        uint32_t nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            int tile, h, s0, nm, P, r0;
            packed_item(pt, p, i, tile, h, s0, nm, P, r0);
            const int qb = nq & 1;
            if (nq >= 2) mbar_wait(&m_empty[qb], ((nq - 2) >> 1) & 1);
            PackSlot& sl = slots[qb];
            PackMem* mt = sl.mem;
            const int qs0 = __ldg(p.query_start + s0) + r0;
            int col = 0, pcs = 0;
            for (int k0 = 0; k0 < nm; k0 += 32) {
                const int k = k0 + lane;
                int len = 0, np = 0, ro = 0, cx = 0, ql = 0;
                if (k < nm) {
                    const int a0 = __ldg(p.query_start + s0 + k);
                    ro = a0 - qs0;
                    ql = __ldg(p.query_start + s0 + k + 1) - a0;
                    cx = __ldg(p.context_lens + s0 + k);
                    len = cx - P;
                    np = (len + 15) >> 4;
                }
                int il = len, ip = np;  // inclusive scans over the lanes
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int a = __shfl_up_sync(0xffffffffu, il, off), b2 = __shfl_up_sync(0xffffffffu, ip, off);
                    if (lane >= off) {
                        il += a;
                        ip += b2;
                    }
                }
                if (k < nm) mt[k] = PackMem{ro, cx, col + il - len, pcs + ip - np, ql};
                col += __shfl_sync(0xffffffffu, il, 31);
                pcs += __shfl_sync(0xffffffffu, ip, 31);
            }
            const int rows = min(kQ, __ldg(p.query_start + s0 + nm) - qs0);
            __syncwarp();
            {   // packed columns the tile's rows can see: the last member's causal range ends
                // at its last row in this tile (a long query spans several tiles)
                const PackMem ml = mt[nm - 1];
                const int pos_max = ml.ctx - ml.qlen + (rows - 1 - ml.row_off);
                col = ml.col_off + min(ml.ctx - P, pos_max - P + 1);
            }
            // physical blocks: every 16-token position of the prefix (through s0's table) and
            // every own-token piece of every member
            const int32_t* bt0 = p.block_tables + (int64_t)s0 * p.W;
            for (int q = lane; q < ((P + 15) >> 4); q += 32) sl.pre_blk[q] = __ldg(bt0 + ((q << 4) >> p.log2B));
            for (int gp = lane; gp < pcs; gp += 32) {
                int lo = 0, hi = nm - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (mt[mid].piece_off <= gp) lo = mid; else hi = mid - 1;
                }
                const int tt0 = P + 16 * (gp - mt[lo].piece_off);
                sl.piece_blk[gp] = __ldg(p.block_tables + (int64_t)(s0 + lo) * p.W + (tt0 >> p.log2B));
            }
            const int n_pre = (P + kN - 1) / kN, n_suf = (col + kN - 1) / kN;
            if (lane == 0) {
                mt[nm] = PackMem{rows, 0, col, pcs, 0};
                sl.hdr[0] = rows;
                sl.hdr[1] = col;
                sl.hdr[2] = n_pre;
                sl.hdr[3] = n_pre + n_suf;
                sl.hdr[4] = nm;  // the item's fields for the other warps (no dynamically indexed
                sl.hdr[5] = P;   // parameter loads there)
                sl.hdr[6] = qs0;
                sl.hdr[7] = h;
                sl.hdr[8] = s0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_full[qb]);  // release: the table writes above
        }
    } else if (warp == 8 || warp > 10) {
        // ---------------- TMA producers (pw 0 = warp 8) ----------------
        const int pw = warp == 8 ? 0 : warp - 10;
        const int br = p.box_rows;
        uint32_t g = 0, nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            const int qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const PackSlot& sl = slots[qb];
            const PackMem* mt = sl.mem;
            const int col = sl.hdr[1], n_pre = sl.hdr[2], n = sl.hdr[3];
            const int nm = sl.hdr[4], P = sl.hdr[5], qs0 = sl.hdr[6], h = sl.hdr[7];
            const int kvh = h / p.G;
            const int pcs = mt[nm].piece_off;
            // ---- query tile
            if (pw == 0 && nq >= 2) mbar_wait(&q_empty[qb], ((nq - 2) >> 1) & 1);
            if (pw == 0 && lane == 0) {
                mbar_arrive_expect_tx(&q_full[qb], 2u * kHalf);
                tma_load_3d(sQ + qb * 2 * kHalf, &p.tmap_q, 0, h, qs0, &q_full[qb]);
                tma_load_3d(sQ + qb * 2 * kHalf + kHalf, &p.tmap_q, 64, h, qs0, &q_full[qb]);
            }
            __syncwarp();
            for (int j = 0; j < n; ++j, ++g) {
                const uint32_t ks = g % kKStages, vs = g & 1;
                for (int tsr = 0; tsr < 2; ++tsr) {  // K then V
                    uint64_t* bar = tsr ? &v_full[vs] : &k_full[ks];
                    if (tsr == 0 && g >= kKStages) mbar_wait(&k_empty[ks], ((g - kKStages) / kKStages) & 1);
                    if (tsr == 1 && g >= 2) mbar_wait(&v_empty[vs], ((g - 2) >> 1) & 1);
                    unsigned char* dst0 = tsr ? sV + vs * 2 * kHalf : sK + ks * 2 * kHalf;
                    const CUtensorMap* map = tsr ? &p.tmap_v : &p.tmap_k;
                    const CUtensorMap* map1 = tsr ? &p.tmap_v1 : &p.tmap_k1;
                    if (j < n_pre) {
                        // shared prefix tokens [128 j, min(P, 128 j + 128)) through s0's table
                        const int t0 = j * kN, len = min(P, t0 + kN) - t0;
                        const int nf = len / br, nb = nf + len % br;
                        if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)len * 256u);
                        __syncwarp();
                        for (int b2 = pw + kProd * lane; b2 < nb; b2 += 32 * kProd) {
                            const int tt = t0 + (b2 < nf ? b2 * br : nf * br + (b2 - nf));
                            const int blk = sl.pre_blk[tt >> 4];
                            const int row = (blk * p.H_kv + kvh) * B + (tt & (B - 1));
                            const int off = (tt - t0) * 128;
                            const CUtensorMap* m = b2 < nf ? map : map1;
                            tma_load_2d(dst0 + off, m, 0, row, bar);
                            tma_load_2d(dst0 + kHalf + off, m, 64, row, bar);
                        }
                    } else {
                        // packed members' own tokens: packed columns [c_lo, c_hi) of this tile;
                        // lane = one 16-token piece of one member (pieces are block-aligned
                        // because P is), split into single rows where it crosses the tile
                        const int c_lo = (j - n_pre) * kN, c_hi = min(col, c_lo + kN);
                        if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(c_hi - c_lo) * 256u);
                        __syncwarp();
                        for (int gp = pw + kProd * lane; gp < pcs; gp += 32 * kProd) {
                            int lo = 0, hi = nm - 1;  // member k of piece gp: last piece_off <= gp
                            while (lo < hi) {
                                const int mid = (lo + hi + 1) >> 1;
                                if (mt[mid].piece_off <= gp) lo = mid; else hi = mid - 1;
                            }
                            const PackMem mk = mt[lo];
                            const int q = gp - mk.piece_off;
                            const int len_k = mk.ctx - P;
                            const int pc0 = mk.col_off + 16 * q, pc1 = mk.col_off + min(16 * q + 16, len_k);
                            const int a = max(pc0, c_lo), b3 = min(pc1, c_hi);
                            if (a >= b3) continue;
                            const int tt0 = P + 16 * q;  // first token of the piece
                            const int blk = sl.piece_blk[gp];
                            const int row0 = (blk * p.H_kv + kvh) * B + (tt0 & (B - 1));
                            if (a == pc0 && b3 == pc1 && pc1 - pc0 == 16 && br == 16) {
                                tma_load_2d(dst0 + (a - c_lo) * 128, map, 0, row0, bar);
                                tma_load_2d(dst0 + kHalf + (a - c_lo) * 128, map, 64, row0, bar);
                            } else {
                                // rows [a, b3) of the piece as 8-row boxes, then 4/2/1
                                int c = a;
                                for (int rb = 8, mi = 0; rb >= 1; rb >>= 1, ++mi) {
                                    const CUtensorMap* mr = rb == 1 ? map1 : (tsr ? &p.tmap_vr[mi] : &p.tmap_kr[mi]);
                                    while (b3 - c >= rb && (rb == 8 || ((b3 - c) & rb))) {
                                        tma_load_2d(dst0 + (c - c_lo) * 128, mr, 0, row0 + (c - pc0), bar);
                                        tma_load_2d(dst0 + kHalf + (c - c_lo) * 128, mr, 64, row0 + (c - pc0), bar);
                                        c += rb;
                                    }
                                }
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (lane == 0) mbar_arrive(&m_empty[qb]);  // this item's table is no longer read here
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer (as v3) ----------------
        const uint32_t idesc_s = umma_idesc(kBF16, false), idesc_o = umma_idesc(kBF16, true);
        uint32_t gk = 0, gv = 0, nq = 0, np = 0, nf = 0;
        auto issue_S = [&](uint32_t qb) {  // S(gk) = Q K(gk)^T into S buffer gk & 1
            const uint32_t ks = gk % kKStages;
            mbar_wait(&k_full[ks], (gk / kKStages) & 1);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t q = smem_u32(sQ) + qb * 2 * kHalf, k = smem_u32(sK) + ks * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    umma_f16(tmem + (gk & 1) * 128, umma_desc_sw128(q + off, 16, 1024),
                             umma_desc_sw128(k + off, 16, 1024), idesc_s, kk > 0);
                }
                umma_commit(&s_full[gk & 1]);
                umma_commit(&k_empty[ks]);
            }
            __syncwarp();
            ++gk;
        };
        for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
            const uint32_t qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const int n = *reinterpret_cast<volatile int*>(&slots[qb].hdr[3]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_empty[qb]);
            mbar_wait(&q_full[qb], (nq >> 1) & 1);
            const int tb = min((int)nq, 17) * 14;  // trace slots of this item (PA_PREFILL_TRACE)
            if (lane == 0) PF_T(tb + 8);
            ++nq;
            for (int j = 0; j < min(n, 2); ++j) issue_S(qb);
            if (n <= 2 && lane == 0) umma_commit(&q_empty[qb]);
            if (n > 0 && nf++ > 0) mbar_wait(o_free, (nf - 2) & 1);
            if (lane == 0) PF_T(tb + 9);
            for (int j = 0; j < n; ++j) {
                mbar_wait(&v_full[gv & 1], (gv >> 1) & 1);
                mbar_wait(p_full, np++ & 1);
                if (lane == 0 && j < 4) PF_T(tb + 10 + j);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t v = smem_u32(sV) + (gv & 1) * 2 * kHalf;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16_ts(tmem + 256, tmem + (gv & 1) * 128 + kk * 8,
                                    umma_desc_sw128(v + kk * 2048, kHalf, 1024), idesc_o, (j > 0) | (kk > 0));
                    umma_commit(o_done);
                    umma_commit(&v_empty[gv & 1]);
                }
                __syncwarp();
                ++gv;
                if (j + 2 < n) {
                    issue_S(qb);
                    if (j + 3 == n && lane == 0) umma_commit(&q_empty[qb]);
                }
            }
        }
    } else {
        // ---------------- softmax warp groups (column halves) ----------------
        const int hf = warp >> 2;
        const int r = tid & (kQ - 1);
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tO = tmem + 256 + hf * 64 + lane_off;
        uint32_t ns = 0, nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            const uint32_t qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const int tb = min((int)nq, 17) * 14;  // trace slots of this item (PA_PREFILL_TRACE)
            if (tid == 0) PF_T(tb);
            const PackMem* mt = slots[qb].mem;
            const int rows = slots[qb].hdr[0], n_pre = slots[qb].hdr[2], n = slots[qb].hdr[3];
            const int nm = slots[qb].hdr[4], P = slots[qb].hdr[5], qs0 = slots[qb].hdr[6], h = slots[qb].hdr[7];
            // this row's member (last row_off <= r), its position and packed segment
            const bool row_valid = r < rows;
            int k = 0;
            {
                int lo = 0, hi = nm - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (mt[mid].row_off <= r) lo = mid; else hi = mid - 1;
                }
                k = lo;
            }
            const PackMem mk = mt[k];
            const int pos = mk.ctx - mk.qlen + (r - mk.row_off);
            const int seg_hi = mk.col_off + (pos - P) + 1;  // packed columns [col_off, seg_hi)
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_empty[qb]);  // the table is read (the item's values are in registers)
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < n; ++j, ++ns) {
                const uint32_t b = ns & 1;
                const uint32_t tS = tmem + b * 128 + lane_off;
                mbar_wait(&s_full[b], (ns >> 1) & 1);
                if (tid == 0 && j < 5) PF_T(tb + 1 + j);
                tc_fence_after();
                float sa[32], sb[32];
                tmem_ld32_nw(tS + hf * 64, sa);
                tmem_ld32_nw(tS + hf * 64 + 32, sb);
                tmem_ld_wait();
                // valid columns [lo, lim) of this half
                int lo, lim;
                if (!row_valid) {
                    lo = 0;
                    lim = 0;
                } else if (j < n_pre) {
                    lo = -hf * 64;
                    lim = min(P - j * kN, kN) - hf * 64;
                } else {
                    const int c0 = (j - n_pre) * kN + hf * 64;
                    lo = mk.col_off - c0;
                    lim = seg_hi - c0;
                }
                const bool partial = !__all_sync(0xffffffffu, lo <= 0 && lim >= 64);
                // a 32-column chunk no row of the warp sees takes no exponentials (P = 0): most
                // of a packed tile's own-token columns belong to the other members
                const bool live0 = !partial || __any_sync(0xffffffffu, lo < 32 && lim > 0 && lim > lo);
                const bool live1 = !partial || __any_sync(0xffffffffu, lo < 64 && lim > 32 && lim > lo);
                if (partial) {
                    // columns outside [lo, lim) become -inf: they drop out of the maximum and
                    // their weights are ex2(-inf) = 0 (also for NaN bit patterns in unused slots)
                    const uint32_t w = (uint32_t)max(lim - lo, 0);
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        sa[u] = (uint32_t)(u - lo) < w ? sa[u] : -INFINITY;
                        sb[u] = (uint32_t)(u + 32 - lo) < w ? sb[u] : -INFINITY;
                    }
                }
                float mo = -INFINITY;
#pragma unroll
                for (int u = 0; u < 32; u += 2)
                    mo = fmaxf(fmaxf(mo, fmaxf(sa[u], sa[u + 1])), fmaxf(sb[u], sb[u + 1]));
                float* rd = red + (ns & 1) * 256;
                rd[hf * 128 + r] = mo;
                named_bar_sync_256();
                float mt2 = fmaxf(mo, rd[(hf ^ 1) * 128 + r]);
                mt2 *= p.scale_log2;
                const bool bump = __any_sync(0xffffffffu, mt2 > m + kLazy);
                const float mn = bump ? fmaxf(m, mt2) : m;
                const float ms = (mn == -INFINITY) ? 0.f : mn;
                const float alpha = bump ? ex2(m - ms) : 1.f;
                float2 rs2 = make_float2(0.f, 0.f);
                const float2 c2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-ms, -ms);
                auto emit = [&](const float (&x)[32], int c0) {
                    uint32_t pk[16];
#pragma unroll
                    for (int u = 0; u < 32; u += 2) {
                        const float2 e = ffma2(make_float2(x[u], x[u + 1]), c2, nm2);
                        const float2 a = ex2_pair(e, u / 2);
                        rs2 = __fadd2_rn(rs2, a);
                        pk[u / 2] = pack2<T>(a.x, a.y);
                    }
                    tmem_st16(tS + hf * 32 + c0 / 2, pk);
                };
                const uint32_t zero[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
                if (live0) emit(sa, 0); else tmem_st16(tS + hf * 32, zero);
                if (live1) emit(sb, 32); else tmem_st16(tS + hf * 32 + 16, zero);
                if (j > 0) {
                    mbar_wait(o_done, (ns - 1) & 1);
                    tc_fence_after();
                }
                if (j > 0 && bump) {
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        float v[32];
                        tmem_ld32_nw(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) v[u] *= alpha;
                        tmem_st32(tO + c0, v);
                    }
                }
                l = l * alpha + (rs2.x + rs2.y);
                m = mn;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full);
            }
            lsum[hf * 128 + r] = l;
            named_bar_sync_256();
            const float lt = l + lsum[(hf ^ 1) * 128 + r];
            named_bar_sync_256();
            const float inv = lt > 0.f ? 1.f / lt : 0.f;
            if (n > 0) {
                mbar_wait(o_done, (ns - 1) & 1);
                tc_fence_after();
            }
            if (tid == 0) PF_T(tb + 6);
            // each warp writes its 32 rows x 64 columns in two 32-column chunks through its own
            // 2 KB of shared memory (16-B pieces XOR-swizzled by row), so that the global stores
            // cover 8 rows x 64 contiguous bytes per instruction instead of 32 rows x 16 bytes
            unsigned char* stg = stage + (warp & 7) * 2048;
            const int rw0 = (warp & 3) * 32;  // the warp's first row in the tile
#pragma unroll
            for (int c0 = 0; c0 < 64; c0 += 32) {
                float v[32];
                if (n > 0) {
                    tmem_ld32_nw(tO + c0, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) v[u] = 0.f;
                }
#pragma unroll
                for (int c1 = 0; c1 < 4; ++c1) {
                    alignas(16) T w[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) w[u] = Elem<T>::from_f32(v[c1 * 8 + u] * inv);
                    *reinterpret_cast<uint4*>(stg + lane * 64 + ((c1 ^ ((lane >> 1) & 3)) * 16)) =
                        *reinterpret_cast<const uint4*>(w);
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int rr = k * 8 + (lane >> 2), ch = lane & 3;
                    if (rw0 + rr < rows) {
                        const uint4 x = *reinterpret_cast<const uint4*>(stg + rr * 64 + ((ch ^ ((rr >> 1) & 3)) * 16));
                        T* dst = static_cast<T*>(p.out) + ((int64_t)(qs0 + rw0 + rr) * p.H + h) * 128 + hf * 64 + c0 +
                                 ch * 8;
                        *reinterpret_cast<uint4*>(dst) = x;
                    }
                }
                __syncwarp();
            }
            if (tid == 0) PF_T(tb + 7);
            if (n > 0) {
                tc_fence_before();
                mbar_arrive(o_free);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}


// ---- v7: packed shared-prefix suffixes, two query tiles per item (default packed kernel) ----
// As v6, but an item's packed rows fill TWO 128-row query tiles (<= 256 rows of members of one
// shared prefix), and both tiles walk the same key tiles (the prefix, then every member's own
// tokens packed back to back): v2's pipeline -- softmax warps 0-3 take tile 0, 4-7 tile 1
// (thread = row, all 128 columns, no cross-group exchange), S_t and O_t per tile in tensor
// memory, the MMA warp alternating P V_0(j), S_0(j+1), P V_1(j), S_1(j+1) so one tile's
// softmax overlaps the other tile's products -- and every key tile is copied once for both.
#ifndef PA_PF_PROD_V7
#define PA_PF_PROD_V7 2  // 128 S registers per softmax thread: 4 producers would cap registers at 144
#endif
constexpr int kProdV7 = PA_PF_PROD_V7;
constexpr int kThreadsV7 = kThreadsV2 + 32 * kProdV7;  // + scheduler warp 10, producers 11..

template <typename T>
__global__ void __launch_bounds__(kThreadsV7, 1)
    paged_prefill_packed2_kernel(const __grid_constant__ PrefillParams p, const __grid_constant__ PackTable pt) {
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = tc::smem_align1024(smem_raw);
    unsigned char* sQ = smem;                          // [2 tiles][2 halves][128][64]
    unsigned char* sK = smem + 4 * kHalf;              // [2 stages][2 halves][128][64]
    unsigned char* sV = sK + 2 * kKStages * kHalf;     // [2 stages][2 halves][128][64]
    unsigned char* stage = sV + 2 * kVStages * kHalf;  // [8 softmax warps][32 rows][64 B] output staging
    PackSlot* slots = reinterpret_cast<PackSlot*>(stage + 8 * 2048);  // [2 parity]
    uint64_t* bars = reinterpret_cast<uint64_t*>(slots + 2);
    uint64_t* q_full = bars;                 // 1
    uint64_t* q_empty = bars + 1;            // 1: every S of the item issued
    uint64_t* k_full = bars + 2;             // 2
    uint64_t* k_empty = bars + 4;            // 2
    uint64_t* v_full = bars + 6;             // 2
    uint64_t* v_empty = bars + 8;            // 2
    uint64_t* s_full = bars + 10;            // 2 (per query tile)
    uint64_t* p_full = bars + 12;            // 2 (per query tile)
    uint64_t* o_done = bars + 14;            // 2 (per query tile)
    uint64_t* o_free = bars + 16;            // 2 (per query tile)
    uint64_t* m_full = bars + 18;            // 2: item table published (scheduler warp)
    uint64_t* m_empty = bars + 20;           // 2: item table read (8 softmax warps, MMA, producers)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_items = pt.n_tiles * p.H;
    pdl_wait();

    if (tid == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], kQ);
            mbar_init(&o_done[i], 1);
            mbar_init(&o_free[i], kQ);
            mbar_init(&m_full[i], 1);
            mbar_init(&m_empty[i], 9 + kProdV7);
        }
        fence_mbar_init();
    }
    // V stages start zeroed: columns of a last tile past its tokens are never loaded
    for (int i = tid; i < 2 * kVStages * kHalf / 16; i += kThreadsV7)
        reinterpret_cast<uint4*>(sV)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int B = 1 << p.log2B;

    if (warp == 10) {
        // ---------------- scheduler: each item's table, one item ahead ----------------
        uint32_t nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            int tile, h, s0, nm, P, r0;
            packed_item(pt, p, i, tile, h, s0, nm, P, r0);
            const int qb = nq & 1;
            if (nq >= 2) mbar_wait(&m_empty[qb], ((nq - 2) >> 1) & 1);
            PackSlot& sl = slots[qb];
            PackMem* mt = sl.mem;
            const int qs0 = __ldg(p.query_start + s0) + r0;
            int col = 0, pcs = 0;
            for (int k0 = 0; k0 < nm; k0 += 32) {
                const int k = k0 + lane;
                int len = 0, np = 0, ro = 0, cx = 0, ql = 0;
                if (k < nm) {
                    const int a0 = __ldg(p.query_start + s0 + k);
                    ro = a0 - qs0;
                    ql = __ldg(p.query_start + s0 + k + 1) - a0;
                    cx = __ldg(p.context_lens + s0 + k);
                    len = cx - P;
                    np = (len + 15) >> 4;
                }
                int il = len, ip = np;  // inclusive scans over the lanes
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int a = __shfl_up_sync(0xffffffffu, il, off), b2 = __shfl_up_sync(0xffffffffu, ip, off);
                    if (lane >= off) {
                        il += a;
                        ip += b2;
                    }
                }
                if (k < nm) mt[k] = PackMem{ro, cx, col + il - len, pcs + ip - np, ql};
                col += __shfl_sync(0xffffffffu, il, 31);
                pcs += __shfl_sync(0xffffffffu, ip, 31);
            }
            const int rows = min(2 * kQ, __ldg(p.query_start + s0 + nm) - qs0);
            __syncwarp();
            {   // packed columns the tile's rows can see: the last member's causal range ends
                // at its last row in this tile (a long query spans several tiles)
                const PackMem ml = mt[nm - 1];
                const int pos_max = ml.ctx - ml.qlen + (rows - 1 - ml.row_off);
                col = ml.col_off + min(ml.ctx - P, pos_max - P + 1);
            }
            // physical blocks: every 16-token position of the prefix (through s0's table) and
            // every own-token piece of every member
            const int32_t* bt0 = p.block_tables + (int64_t)s0 * p.W;
            for (int q = lane; q < ((P + 15) >> 4); q += 32) sl.pre_blk[q] = __ldg(bt0 + ((q << 4) >> p.log2B));
            for (int gp = lane; gp < pcs; gp += 32) {
                int lo = 0, hi = nm - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (mt[mid].piece_off <= gp) lo = mid; else hi = mid - 1;
                }
                const int tt0 = P + 16 * (gp - mt[lo].piece_off);
                sl.piece_blk[gp] = __ldg(p.block_tables + (int64_t)(s0 + lo) * p.W + (tt0 >> p.log2B));
            }
            const int n_pre = (P + kN - 1) / kN, n_suf = (col + kN - 1) / kN;
            if (lane == 0) {
                mt[nm] = PackMem{rows, 0, col, pcs, 0};
                sl.hdr[0] = rows;
                sl.hdr[1] = col;
                sl.hdr[2] = n_pre;
                sl.hdr[3] = n_pre + n_suf;
                sl.hdr[4] = nm;  // the item's fields for the other warps (no dynamically indexed
                sl.hdr[5] = P;   // parameter loads there)
                sl.hdr[6] = qs0;
                sl.hdr[7] = h;
                sl.hdr[8] = s0;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_full[qb]);  // release: the table writes above
        }
    } else if (warp == 8 || warp > 10) {  // (v7: warps 8, 11..)
        // ---------------- TMA producers (pw 0 = warp 8) ----------------
        const int pw = warp == 8 ? 0 : warp - 10;
        const int br = p.box_rows;
        uint32_t g = 0, nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            const int qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const PackSlot& sl = slots[qb];
            const PackMem* mt = sl.mem;
            const int col = sl.hdr[1], n_pre = sl.hdr[2], n = sl.hdr[3];
            const int nm = sl.hdr[4], P = sl.hdr[5], qs0 = sl.hdr[6], h = sl.hdr[7];
            const int kvh = h / p.G;
            const int pcs = mt[nm].piece_off;
            // ---- the item's two query tiles (rows past the queries: zero fill / masked)
            if (pw == 0 && nq >= 1) mbar_wait(q_empty, (nq - 1) & 1);
            if (pw == 0 && lane == 0) {
                mbar_arrive_expect_tx(q_full, 4u * kHalf);
                tma_load_3d(sQ, &p.tmap_q, 0, h, qs0, q_full);
                tma_load_3d(sQ + kHalf, &p.tmap_q, 64, h, qs0, q_full);
                tma_load_3d(sQ + 2 * kHalf, &p.tmap_q, 0, h, qs0 + kQ, q_full);
                tma_load_3d(sQ + 3 * kHalf, &p.tmap_q, 64, h, qs0 + kQ, q_full);
            }
            __syncwarp();
            for (int j = 0; j < n; ++j, ++g) {
                const uint32_t ks = g % kKStages, vs = g & 1;
                for (int tsr = 0; tsr < 2; ++tsr) {  // K then V
                    uint64_t* bar = tsr ? &v_full[vs] : &k_full[ks];
                    if (tsr == 0 && g >= kKStages) mbar_wait(&k_empty[ks], ((g - kKStages) / kKStages) & 1);
                    if (tsr == 1 && g >= 2) mbar_wait(&v_empty[vs], ((g - 2) >> 1) & 1);
                    unsigned char* dst0 = tsr ? sV + vs * 2 * kHalf : sK + ks * 2 * kHalf;
                    const CUtensorMap* map = tsr ? &p.tmap_v : &p.tmap_k;
                    const CUtensorMap* map1 = tsr ? &p.tmap_v1 : &p.tmap_k1;
                    if (j < n_pre) {
                        // shared prefix tokens [128 j, min(P, 128 j + 128)) through s0's table
                        const int t0 = j * kN, len = min(P, t0 + kN) - t0;
                        const int nf = len / br, nb = nf + len % br;
                        if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)len * 256u);
                        __syncwarp();
                        for (int b2 = pw + kProdV7 * lane; b2 < nb; b2 += 32 * kProdV7) {
                            const int tt = t0 + (b2 < nf ? b2 * br : nf * br + (b2 - nf));
                            const int blk = sl.pre_blk[tt >> 4];
                            const int row = (blk * p.H_kv + kvh) * B + (tt & (B - 1));
                            const int off = (tt - t0) * 128;
                            const CUtensorMap* m = b2 < nf ? map : map1;
                            tma_load_2d(dst0 + off, m, 0, row, bar);
                            tma_load_2d(dst0 + kHalf + off, m, 64, row, bar);
                        }
                    } else {
                        // packed members' own tokens: packed columns [c_lo, c_hi) of this tile;
                        // lane = one 16-token piece of one member (pieces are block-aligned
                        // because P is), split into single rows where it crosses the tile
                        const int c_lo = (j - n_pre) * kN, c_hi = min(col, c_lo + kN);
                        if (pw == 0 && lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(c_hi - c_lo) * 256u);
                        __syncwarp();
                        for (int gp = pw + kProdV7 * lane; gp < pcs; gp += 32 * kProdV7) {
                            int lo = 0, hi = nm - 1;  // member k of piece gp: last piece_off <= gp
                            while (lo < hi) {
                                const int mid = (lo + hi + 1) >> 1;
                                if (mt[mid].piece_off <= gp) lo = mid; else hi = mid - 1;
                            }
                            const PackMem mk = mt[lo];
                            const int q = gp - mk.piece_off;
                            const int len_k = mk.ctx - P;
                            const int pc0 = mk.col_off + 16 * q, pc1 = mk.col_off + min(16 * q + 16, len_k);
                            const int a = max(pc0, c_lo), b3 = min(pc1, c_hi);
                            if (a >= b3) continue;
                            const int tt0 = P + 16 * q;  // first token of the piece
                            const int blk = sl.piece_blk[gp];
                            const int row0 = (blk * p.H_kv + kvh) * B + (tt0 & (B - 1));
                            if (a == pc0 && b3 == pc1 && pc1 - pc0 == 16 && br == 16) {
                                tma_load_2d(dst0 + (a - c_lo) * 128, map, 0, row0, bar);
                                tma_load_2d(dst0 + kHalf + (a - c_lo) * 128, map, 64, row0, bar);
                            } else {
                                // rows [a, b3) of the piece as 8-row boxes, then 4/2/1
                                int c = a;
                                for (int rb = 8, mi = 0; rb >= 1; rb >>= 1, ++mi) {
                                    const CUtensorMap* mr = rb == 1 ? map1 : (tsr ? &p.tmap_vr[mi] : &p.tmap_kr[mi]);
                                    while (b3 - c >= rb && (rb == 8 || ((b3 - c) & rb))) {
                                        tma_load_2d(dst0 + (c - c_lo) * 128, mr, 0, row0 + (c - pc0), bar);
                                        tma_load_2d(dst0 + kHalf + (c - c_lo) * 128, mr, 64, row0 + (c - pc0), bar);
                                        c += rb;
                                    }
                                }
                            }
                        }
                    }
                    __syncwarp();
                }
            }
            if (lane == 0) mbar_arrive(&m_empty[qb]);  // this item's table is no longer read here
        }
    } else if (warp == 9) {
        // ---------------- MMA issuer: v2's order over the two query tiles ----------------
        const uint32_t idesc_s = umma_idesc(kBF16, false), idesc_o = umma_idesc(kBF16, true);
        uint32_t g = 0, nq = 0, np[2] = {0u, 0u}, nf[2] = {0u, 0u};
        auto issue_S = [&](int t, uint32_t gg) {  // S_t = Q_t K(gg)^T
            if (lane == 0) {
                const uint32_t q = smem_u32(sQ) + t * 2 * kHalf, k = smem_u32(sK) + (gg % kKStages) * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    umma_f16(tmem + t * 128, umma_desc_sw128(q + off, 16, 1024), umma_desc_sw128(k + off, 16, 1024),
                             idesc_s, kk > 0);
                }
                umma_commit(&s_full[t]);
            }
            __syncwarp();
        };
        auto issue_PV = [&](int t, uint32_t gg, bool first) {  // O_t (+)= P_t V(gg)
            mbar_wait(&p_full[t], np[t]++ & 1);
            if (first && nf[t]++ > 0) mbar_wait(&o_free[t], (nf[t] - 2) & 1);  // the last item's O_t was read
            tc_fence_after();
            if (lane == 0) {
                const uint32_t v = smem_u32(sV) + (gg & 1) * 2 * kHalf;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    umma_f16_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8,
                                umma_desc_sw128(v + kk * 2048, kHalf, 1024), idesc_o, (first ? 0u : 1u) | (kk > 0));
                umma_commit(&o_done[t]);
            }
            __syncwarp();
        };
        for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
            const uint32_t qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const int rows = *reinterpret_cast<volatile int*>(&slots[qb].hdr[0]);
            const int n = *reinterpret_cast<volatile int*>(&slots[qb].hdr[3]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_empty[qb]);
            mbar_wait(q_full, nq & 1);
            ++nq;
            const bool two = rows > kQ;  // the second query tile has rows
            if (n == 0) {
                if (lane == 0) umma_commit(q_empty);
                __syncwarp();
                continue;
            }
            mbar_wait(&k_full[g % kKStages], (g / kKStages) & 1);
            tc_fence_after();
            issue_S(0, g);
            if (two) issue_S(1, g);
            if (lane == 0) {
                umma_commit(&k_empty[g % kKStages]);
                if (n == 1) umma_commit(q_empty);
            }
            __syncwarp();
            for (int j = 0; j < n; ++j, ++g) {
                mbar_wait(&v_full[g & 1], (g >> 1) & 1);
                issue_PV(0, g, j == 0);
                const bool more = j + 1 < n;
                if (more) {
                    mbar_wait(&k_full[(g + 1) % kKStages], ((g + 1) / kKStages) & 1);
                    tc_fence_after();
                    issue_S(0, g + 1);
                }
                if (two) issue_PV(1, g, j == 0);
                if (lane == 0) umma_commit(&v_empty[g & 1]);
                if (more) {
                    if (two) issue_S(1, g + 1);
                    if (lane == 0) {
                        umma_commit(&k_empty[(g + 1) % kKStages]);
                        if (j + 2 == n) umma_commit(q_empty);  // every S of this item issued
                    }
                }
                __syncwarp();
            }
        }
    } else {
        // ---------------- softmax: warps 0-3 query tile 0, 4-7 tile 1 (thread = row) ----------------
        const int t = warp >> 2;
        const int rt = tid & (kQ - 1);                    // row within the tile
        const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
        const uint32_t tS = tmem + t * 128 + lane_off, tO = tmem + 256 + t * 128 + lane_off;
        unsigned char* stg = stage + (warp & 7) * 2048;  // this warp's 32 rows x 32 columns staging
        const int rw0 = t * kQ + (warp & 3) * 32;         // the warp's first row in the item
        uint32_t ns = 0, nq = 0;
        for (int i = blockIdx.x; i < n_items; i += gridDim.x, ++nq) {
            const uint32_t qb = nq & 1;
            mbar_wait(&m_full[qb], (nq >> 1) & 1);
            const PackMem* mt = slots[qb].mem;
            const int rows = slots[qb].hdr[0], n_pre = slots[qb].hdr[2], n = slots[qb].hdr[3];
            const int nm = slots[qb].hdr[4], P = slots[qb].hdr[5], qs0 = slots[qb].hdr[6], h = slots[qb].hdr[7];
            const int r = t * kQ + rt;  // row within the item
            const bool row_valid = r < rows;
            int k = 0;
            {
                int lo = 0, hi = nm - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (mt[mid].row_off <= r) lo = mid; else hi = mid - 1;
                }
                k = lo;
            }
            const PackMem mk = mt[k];
            const int pos = mk.ctx - mk.qlen + (r - mk.row_off);
            const int seg_hi = mk.col_off + (pos - P) + 1;  // packed columns [col_off, seg_hi)
            __syncwarp();
            if (lane == 0) mbar_arrive(&m_empty[qb]);
            const bool active = t == 0 || rows > kQ;
            if (!active) continue;
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < n; ++j, ++ns) {
                mbar_wait(&s_full[t], ns & 1);
                tc_fence_after();
                float sv[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32_nw(tS + 32 * c, sv[c]);
                tmem_ld_wait();
                // valid columns [lo, lim) of this key tile
                int lo, lim;
                if (!row_valid) {
                    lo = 0;
                    lim = 0;
                } else if (j < n_pre) {
                    lo = 0;
                    lim = min(P - j * kN, kN);
                } else {
                    const int c0 = (j - n_pre) * kN;
                    lo = mk.col_off - c0;
                    lim = seg_hi - c0;
                }
                const bool partial = !__all_sync(0xffffffffu, lo <= 0 && lim >= kN);
                bool live[4];
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    live[c] = !partial || __any_sync(0xffffffffu, lo < 32 * c + 32 && lim > 32 * c && lim > lo);
                if (partial) {
                    const uint32_t w = (uint32_t)max(lim - lo, 0);
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int u = 0; u < 32; ++u) sv[c][u] = (uint32_t)(32 * c + u - lo) < w ? sv[c][u] : -INFINITY;
                }
                float mo = -INFINITY;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int u = 0; u < 32; u += 2) mo = fmaxf(mo, fmaxf(sv[c][u], sv[c][u + 1]));
                const float mt2 = mo * p.scale_log2;
                const bool bump = __any_sync(0xffffffffu, mt2 > m + kLazy);
                const float mn = bump ? fmaxf(m, mt2) : m;
                const float ms = (mn == -INFINITY) ? 0.f : mn;
                const float alpha = bump ? ex2(m - ms) : 1.f;
                float2 rs2 = make_float2(0.f, 0.f);
                const float2 c2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-ms, -ms);
                const uint32_t zero[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (live[c]) {
                        uint32_t pk[16];
#pragma unroll
                        for (int u = 0; u < 32; u += 2) {
                            const float2 e = ffma2(make_float2(sv[c][u], sv[c][u + 1]), c2, nm2);
                            const float2 a = ex2_pair(e, u / 2);
                            rs2 = __fadd2_rn(rs2, a);
                            pk[u / 2] = pack2<T>(a.x, a.y);
                        }
                        tmem_st16(tS + 16 * c, pk);
                    } else {
                        tmem_st16(tS + 16 * c, zero);
                    }
                }
                if (j > 0) {  // P V_t of the previous key tile completed (every o_done phase is waited)
                    mbar_wait(&o_done[t], (ns - 1) & 1);
                    tc_fence_after();
                }
                if (j > 0 && bump) {
#pragma unroll
                    for (int c0 = 0; c0 < 128; c0 += 32) {
                        float v[32];
                        tmem_ld32_nw(tO + c0, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int u = 0; u < 32; ++u) v[u] *= alpha;
                        tmem_st32(tO + c0, v);
                    }
                }
                l = l * alpha + (rs2.x + rs2.y);
                m = mn;
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&p_full[t]);
            }
            // epilogue: out rows = O_t / l through the warp's staging buffer (coalesced stores)
            const float inv = l > 0.f ? 1.f / l : 0.f;
            if (n > 0) {
                mbar_wait(&o_done[t], (ns - 1) & 1);
                tc_fence_after();
            }
#pragma unroll
            for (int c0 = 0; c0 < 128; c0 += 32) {
                float v[32];
                if (n > 0) {
                    tmem_ld32_nw(tO + c0, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int u = 0; u < 32; ++u) v[u] = 0.f;
                }
#pragma unroll
                for (int c1 = 0; c1 < 4; ++c1) {
                    alignas(16) T w[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) w[u] = Elem<T>::from_f32(v[c1 * 8 + u] * inv);
                    *reinterpret_cast<uint4*>(stg + lane * 64 + ((c1 ^ ((lane >> 1) & 3)) * 16)) =
                        *reinterpret_cast<const uint4*>(w);
                }
                __syncwarp();
#pragma unroll
                for (int kq = 0; kq < 4; ++kq) {
                    const int rr = kq * 8 + (lane >> 2), ch = lane & 3;
                    if (rw0 + rr < rows) {
                        const uint4 x = *reinterpret_cast<const uint4*>(stg + rr * 64 + ((ch ^ ((rr >> 1) & 3)) * 16));
                        T* dst = static_cast<T*>(p.out) + ((int64_t)(qs0 + rw0 + rr) * p.H + h) * 128 + c0 + ch * 8;
                        *reinterpret_cast<uint4*>(dst) = x;
                    }
                }
                __syncwarp();
            }
            if (n > 0) {
                tc_fence_before();
                mbar_arrive(&o_free[t]);  // O_t may take the next item
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

size_t prefill_packed2_smem_bytes() {
    return 1024 + (4 + 2 * kKStages + 2 * kVStages) * (size_t)kHalf + 8 * 2048 + 2 * sizeof(PackSlot) + 22 * 8 + 16;
}

cudaError_t launch_prefill_packed2(const PrefillParams& p, const PackTable& t, int dtype, cudaStream_t stream) {
    int dev = 0, num_sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
    const size_t smem = prefill_packed2_smem_bytes();
    const long long items = (long long)t.n_tiles * p.H;
    const dim3 grid((unsigned)std::min<long long>(items, num_sms));
    auto kern = dtype == 1 ? paged_prefill_packed2_kernel<__half> : paged_prefill_packed2_kernel<__nv_bfloat16>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    return launch_k(kern, grid, dim3(kThreadsV7), smem, stream, p, t);
}

size_t prefill_packed_smem_bytes() {
    return 1024 + (4 + 2 * kKStages + 2 * kVStages) * (size_t)kHalf + 8 * 2048 + (512 + 256) * 4 + 2 * sizeof(PackSlot) +
           21 * 8 + 16;
}

cudaError_t launch_prefill_packed(const PrefillParams& p, const PackTable& t, int dtype, cudaStream_t stream) {
    int dev = 0, num_sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
    const size_t smem = prefill_packed_smem_bytes();
    const long long items = (long long)t.n_tiles * p.H;
    const dim3 grid((unsigned)std::min<long long>(items, num_sms));
    auto kern = dtype == 1 ? paged_prefill_packed_kernel<__half> : paged_prefill_packed_kernel<__nv_bfloat16>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    return launch_k(kern, grid, dim3(kThreadsV6), smem, stream, p, t);
}

// variant: 2 / 3 forces a kernel (PA_PREFILL, read once by pa_api.cpp); 0 = default: v3 when
// no query needs more than 1.5 tiles of 128 rows (v2's pairs would mostly leave the second
// softmax group idle), else v2, whose two query tiles share each K/V tile (measured,
// DESIGN.md §8c).  (v1: one tile per CTA, v4: 64-token K/V tiles, v5: four softmax warp
// groups -- measured slower and removed; their numbers stay in DESIGN §8c.)
cudaError_t launch_prefill(const PrefillParams& p, int dtype, int num_seqs, int max_query_len, int variant,
                           cudaStream_t stream) {
    if (variant != 2 && variant != 3) variant = max_query_len <= kQ + kQ / 2 ? 3 : 2;
    int dev = 0, num_sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
    PrefillParams q = p;
    q.S = num_seqs;
    if (variant == 2) {
        const size_t smem = prefill_ws_smem_bytes();
        q.X = (max_query_len + 2 * kQ - 1) / (2 * kQ);
        cudaError_t me = cudaMemsetAsync(q.work_counter, 0, sizeof(int), stream);
        if (me != cudaSuccess) return me;
        const long long items = (long long)q.X * q.H * q.S;
        const dim3 grid((unsigned)std::min<long long>(items, num_sms));
        auto kern = dtype == 1 ? paged_prefill_ws_kernel<__half> : paged_prefill_ws_kernel<__nv_bfloat16>;
        cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
        if (e != cudaSuccess) return e;
        return launch_k(kern, grid, dim3(kThreadsWs), smem, stream, q);
    }
    const size_t smem = prefill_split_smem_bytes();
    q.X = (max_query_len + kQ - 1) / kQ;
    const long long items = (long long)q.X * q.H * q.S;
    const dim3 grid((unsigned)std::min<long long>(items, num_sms));
    auto kern = dtype == 1 ? paged_prefill_split_kernel<__half> : paged_prefill_split_kernel<__nv_bfloat16>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    return launch_k(kern, grid, dim3(kThreadsV3), smem, stream, q);
}

}  // namespace pa

#ifdef PA_PREFILL_TRACE
extern "C" int pa_debug_prefill_trace_read(long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, pa::g_pf_trace, sizeof(long long) * (size_t)n);
}
#endif
