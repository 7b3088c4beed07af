// pa_attention.cu -- PagedAttention decode kernels for B200 (sm_100a).
//
// Eq.4 of the paper: for every (sequence s, query head h) the kernel walks
// the sequence's logical tokens through its block table, computes
// l_t = scale * q.K_t, a numerically stable softmax and sum_t softmax_t * V_t.
//
// B200 design:
//  * Work unit = (sequence, query head, partition of <= PT logical tokens); one WARP
//    walks the unit's 16-token LOGICAL tiles in order, so the arithmetic never depends
//    on block_size, physical placement, head grouping, scheduling or grid shape ->
//    bitwise invariance (BJ:north_star's permutation / block-size properties).
//  * Scheduler ("coop", the only one shipped): one CTA per (partition, group of 4 query
//    heads, sequence); a producer warp stages the group's K/V tiles into shared memory
//    with 1-D bulk async copies (cp.async.bulk, SASS UBLKCP) completing on per-stage
//    mbarriers, 4 consumer warps compute.  For block_size < 16 a tile is several pieces.
//    (Grid, persistent-warp, persistent-CTA and work-list schedulers were measured and
//    removed; DESIGN §7 keeps their numbers.)
//  * Lane mapping: a K/V row of RB = D*e bytes is covered by LT = RB/32 lanes, each
//    owning two 16-byte chunks (c and c+LT: conflict-free 128-byte phases); a warp
//    handles TG = 32/LT tokens at once.  q.k uses the sm_100 mixed-precision FMA
//    (FHFMA, f16/bf16 x f16/bf16 + f32) straight from the packed storage dtype; the
//    dot product is reduced with warp shuffles across the LT lanes.  Each token group
//    keeps its own online-softmax state (m, l, acc[]) in the exp2 domain, and p*V is
//    accumulated with packed FMAs.  No tensor cores: a one-query decode step is a
//    memory-bound GEMV (BJ:north_star).
//  * End of a unit: token groups merge by shuffles (log-sum-exp, fixed order).  A
//    context that fits one partition writes `out` directly (16-byte stores); otherwise
//    each partition publishes (m, L, o~) and the LAST partition of the (sequence,
//    head) to finish -- an epoch-tagged atomic counter, see split_arrive -- merges them
//    in partition order (split-context variant, BJ:north_star).
//  * Fused decode entry (pa_paged_attention_decode): the step's new token (logical
//    position ctx-1) is bulk-copied from the key/value inputs straight into its tile
//    row, and one warp per (sequence, kv head) stores it to its cache slot
//    (reshape_and_cache) -- no separate launch.
#include "pa_common.cuh"
#include "pa_internal.h"

#include <algorithm>
#include <cfloat>
#include <cstdio>

namespace pa {

template <typename T, int D>
struct AttnCfg {
    static constexpr int E = Elem<T>::kBytes;
    static constexpr int RB = D * E;         // bytes per K/V row
    static constexpr int NCH = RB / 16;      // 16-byte chunks per row
    static constexpr int LT = NCH / 2;       // lanes per token (2 chunks each)
    static constexpr int TG = 32 / LT;       // tokens per warp step (token groups)
    static constexpr int TPL = kTile / TG;   // tokens per lane per tile
    static constexpr int EPC = 16 / E;       // elements per chunk
    static constexpr int STAGE_BYTES = 2 * kTile * RB;
    static_assert(LT >= 1 && LT <= 16 && TG * LT == 32, "row must span 2..32 lanes");
    static_assert(TPL >= 1 && TPL * TG == kTile, "tile must split evenly over token groups");
};

// ===================================================================== per-tile math ===

// Online-softmax update of one 16-token tile (nv valid rows) for the calling lane's
// token group g and chunks (c, c+LT).  State in the exp2 domain.
template <typename T, int D>
__device__ __forceinline__ void tile_update(const char* sK, const char* sV, int nv, const uint4& q0, const uint4& q1,
                                            float scale_log2, int g, int c, float& m, float& l,
                                            float2 (&acc)[AttnCfg<T, D>::EPC]) {
    using C = AttnCfg<T, D>;
    constexpr int RB = C::RB, LT = C::LT, TG = C::TG, TPL = C::TPL, EPC = C::EPC;
    float sc[TPL];
#pragma unroll
    for (int jj = 0; jj < TPL; ++jj) {
        const char* row = sK + (jj * TG + g) * RB;
        const uint4 k0 = lds128(row + c * 16), k1 = lds128(row + (c + LT) * 16);
        float x = dot16<T>(q0, k0, 0.f) + dot16<T>(q1, k1, 0.f);
#pragma unroll
        for (int off = LT / 2; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        sc[jj] = x * scale_log2;
    }
    if (nv < kTile) {
#pragma unroll
        for (int jj = 0; jj < TPL; ++jj)
            if (jj * TG + g >= nv) sc[jj] = -INFINITY;
    }
    float mt = sc[0];
#pragma unroll
    for (int jj = 1; jj < TPL; ++jj) mt = fmaxf(mt, sc[jj]);
    const float mn = fmaxf(m, mt);
    const float ms = (mn == -INFINITY) ? 0.f : mn;
    const float alpha = ex2(m - ms);
    float ps[TPL], psum = 0.f;
#pragma unroll
    for (int jj = 0; jj < TPL; ++jj) {
        ps[jj] = ex2(sc[jj] - ms);
        psum += ps[jj];
    }
    l = l * alpha + psum;
    const float2 aa = make_float2(alpha, alpha);
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = fmul2(acc[e], aa);
    if (nv == kTile) {
#pragma unroll
        for (int jj = 0; jj < TPL; ++jj) {
            const char* row = sV + (jj * TG + g) * RB;
            const uint4 v0 = lds128(row + c * 16), v1 = lds128(row + (c + LT) * 16);
            axpy16<T>(acc, ps[jj], v0);
            axpy16<T>(acc + EPC / 2, ps[jj], v1);
        }
    } else {
#pragma unroll
        for (int jj = 0; jj < TPL; ++jj) {
            if (jj * TG + g < nv) {  // rows past the context were never loaded (reading c3)
                const char* row = sV + (jj * TG + g) * RB;
                const uint4 v0 = lds128(row + c * 16), v1 = lds128(row + (c + LT) * 16);
                axpy16<T>(acc, ps[jj], v0);
                axpy16<T>(acc + EPC / 2, ps[jj], v1);
            }
        }
    }
    m = mn;
}

// Merge the warp's token groups (log-sum-exp, fixed butterfly order).
template <typename T, int D>
__device__ __forceinline__ void merge_token_groups(float& m, float& l, float2 (&acc)[AttnCfg<T, D>::EPC]) {
    using C = AttnCfg<T, D>;
    constexpr int LT = C::LT, EPC = C::EPC;
#pragma unroll
    for (int off = LT; off < 32; off <<= 1) {
        const float mo = __shfl_xor_sync(0xffffffffu, m, off);
        const float lo = __shfl_xor_sync(0xffffffffu, l, off);
        const float mn = fmaxf(m, mo);
        const float ms = (mn == -INFINITY) ? 0.f : mn;
        const float a = ex2(m - ms), b = ex2(mo - ms);
        l = l * a + lo * b;
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
            const float ox = __shfl_xor_sync(0xffffffffu, acc[e].x, off);
            const float oy = __shfl_xor_sync(0xffffffffu, acc[e].y, off);
            acc[e] = make_float2(acc[e].x * a + ox * b, acc[e].y * a + oy * b);
        }
        m = mn;
    }
}

// Lanes of token group 0: out row = acc / l (0 for an empty context), 16-byte stores.
template <typename T, int D>
__device__ __forceinline__ void store_out(T* o, float l, const float2 (&acc)[AttnCfg<T, D>::EPC], int c) {
    using C = AttnCfg<T, D>;
    constexpr int LT = C::LT, EPC = C::EPC;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        alignas(16) T v[EPC];
#pragma unroll
        for (int e = 0; e < EPC / 2; ++e) {
            v[2 * e] = Elem<T>::from_f32(l > 0.f ? acc[half * EPC / 2 + e].x / l : 0.f);
            v[2 * e + 1] = Elem<T>::from_f32(l > 0.f ? acc[half * EPC / 2 + e].y / l : 0.f);
        }
        *reinterpret_cast<uint4*>(o + (c + half * LT) * EPC) = *reinterpret_cast<const uint4*>(v);
    }
}

// store_out to this (sequence, head)'s output row: `out`, or with the fused TP all-gather
// (N2) the row of global head out_h0 + h in every rank's gather buffer.
template <typename T, int D>
__device__ __forceinline__ void store_out_p(const AttnParams& p, int64_t sh, float l,
                                            const float2 (&acc)[AttnCfg<T, D>::EPC], int c) {
    if (p.n_out_peers == 0) {
        store_out<T, D>(static_cast<T*>(p.out) + sh * D, l, acc, c);
        return;
    }
    const int64_t s = sh / p.H, h = sh - s * p.H;
    const int64_t off = (s * p.out_H + p.out_h0 + h) * D;
    for (int k = 0; k < p.n_out_peers; ++k) store_out<T, D>(static_cast<T*>(p.out_peers[k]) + off, l, acc, c);
    // order this thread's peer stores before the completion flag at system scope: the flag
    // kernel's st.release.sys then covers them without relying on kernel-boundary
    // semantics for memory written to ANOTHER GPU (pa_tp.cu)
    __threadfence_system();
}

// Lanes of token group 0: normalised partial o~ = acc / l (fp32).
template <typename T, int D>
__device__ __forceinline__ void store_partial(float* o, float l, const float2 (&acc)[AttnCfg<T, D>::EPC], int c) {
    using C = AttnCfg<T, D>;
    constexpr int LT = C::LT, EPC = C::EPC;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int e = 0; e < EPC / 2; e += 2) {
            const float2 a0 = acc[half * EPC / 2 + e], a1 = acc[half * EPC / 2 + e + 1];
            *reinterpret_cast<float4*>(o + (c + half * LT) * EPC + 2 * e) =
                make_float4(a0.x / l, a0.y / l, a1.x / l, a1.y / l);
        }
    }
}

// Split-context merge of (sequence, head) sh over its np partitions, in partition order:
//   M = max m_p;  out = sum_p 2^(m_p - M) L_p o~_p / sum_p 2^(m_p - M) L_p
// ml[p] = (m_p, L_p), po[p*D + d] = o~_p[d]: the global workspace (written by other CTAs,
// read through L2) or this CTA's shared memory -- the arithmetic is the same either way.
template <typename T, int D, bool kGlobal>
__device__ __forceinline__ void merge_partitions_from(const AttnParams& p, int64_t sh, const float2* ml,
                                                      const float* po, int np, int lane) {
    auto ld2 = [](const float2* a) { return kGlobal ? __ldcg(a) : *a; };
    auto ld1 = [](const float* a) { return kGlobal ? __ldcg(a) : *a; };
    float M = -INFINITY;
    for (int i = 0; i < np; ++i) M = fmaxf(M, ld2(&ml[i]).x);
    float L = 0.f;
    constexpr int DPL = D / 32;  // dims per lane
    float o[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[e] = 0.f;
    for (int i = 0; i < np; ++i) {
        const float2 mi = ld2(&ml[i]);
        const float w = mi.y * ex2(mi.x - M);
        L += w;
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] += w * ld1(po + (int64_t)i * D + lane * DPL + e);
    }
    auto store_row = [&](T* out_row) {
#pragma unroll
        for (int e = 0; e < DPL; ++e) out_row[lane * DPL + e] = Elem<T>::from_f32(o[e] / L);
    };
    if (p.n_out_peers == 0) {
        store_row(static_cast<T*>(p.out) + sh * D);
    } else {
        const int64_t s = sh / p.H, h = sh - s * p.H;
        const int64_t off = (s * p.out_H + p.out_h0 + h) * D;
        for (int k = 0; k < p.n_out_peers; ++k) store_row(static_cast<T*>(p.out_peers[k]) + off);
        __threadfence_system();  // see store_out_p
    }
}

template <typename T, int D>
__device__ __forceinline__ void merge_partitions(const AttnParams& p, int64_t sh, int np, int lane) {
    merge_partitions_from<T, D, true>(p, sh, p.part_ml + sh * p.NP, p.part_o + sh * p.NP * D, np, lane);
}

// Split-context completion count of (sequence, head) sh, called once per partition by
// lane 0 after its (m, L, o~) is published; true for the partition that completes the
// set of n.  The counter word is (epoch << 32 | partitions done): a word carrying another
// launch's epoch counts as 0, and the completing partition stores 0 back (nobody else
// touches the word again in this launch).  So the host never zeroes the counters -- no
// memset node between decode steps, which keeps the programmatic-dependent-launch chain
// intact -- and a workspace region that held partials of an earlier call with another
// layout is still a valid counter array (epochs are scrambled 32-bit tags, pa_api.cpp).
// The first CAS guesses the common state 0 (no extra load).
__device__ __forceinline__ bool split_arrive(const AttnParams& p, int64_t sh, int n) {
    unsigned long long* ctr = p.counters + sh;
    const unsigned long long E = (unsigned long long)p.epoch << 32;
    unsigned long long cur = 0ull;
    for (;;) {
        const unsigned long long want = ((cur & 0xffffffff00000000ull) == E ? cur : E) + 1ull;
        const unsigned long long prev = atomicCAS(ctr, cur, want);
        if (prev == cur) {
            if ((int)(want & 0xffffffffull) < n) return false;
            atomicExch(ctr, 0ull);
            return true;
        }
        cur = prev;
    }
}

// Publish this partition's (m, L, o~); the last partition to finish merges.  Whole warp.
template <typename T, int D>
__device__ __forceinline__ void finish_split(const AttnParams& p, int64_t sh, int part, int nparts, float m, float l,
                                             const float2 (&acc)[AttnCfg<T, D>::EPC], int g, int c, int lane) {
    if (g == 0) store_partial<T, D>(p.part_o + (sh * p.NP + part) * D, l, acc, c);
    if (lane == 0) p.part_ml[sh * p.NP + part] = make_float2(m, l);
    __syncwarp();
    int last = 0;
    if (lane == 0) {
        __threadfence();
        last = split_arrive(p, sh, min(nparts, p.NP));
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
        __threadfence();
        merge_partitions<T, D>(p, sh, min(nparts, p.NP), lane);
    }
}

// ===================================================================== tile loaders ===

// Grid scheduler: block ids of the partition prefetched in shared memory (sbt, from
// logical block jb0).  Copies rows [tok0, tok0 + nv) (nv may be 0) of kv head `head_off`.
__device__ __forceinline__ void issue_tile(char* sK, char* sV, uint64_t* bar, const char* kc, const char* vc,
                                           const int* sbt, int jb0, int tok0, int nv, int p1, int log2B,
                                           int64_t blk_stride, int64_t head_off, int RB, int lane) {
    const int B = 1 << log2B;
    if (B >= kTile) {
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)(nv * RB);
            mbar_arrive_expect_tx(bar, 2 * bytes);
            if (bytes) {
                const int blk = sbt[(tok0 >> log2B) - jb0];
                const int64_t off = (int64_t)blk * blk_stride + head_off + (int64_t)(tok0 & (B - 1)) * RB;
                bulk_g2s(sK, kc + off, bytes, bar);
                bulk_g2s(sV, vc + off, bytes, bar);
            }
        }
    } else {
        if (lane == 0) mbar_arrive_expect_tx(bar, (uint32_t)(2 * nv * RB));
        __syncwarp();
        const int pieces = kTile >> log2B;
        if (lane < pieces) {
            const int tk = tok0 + (lane << log2B);
            if (tk < p1) {
                const int blk = sbt[(tk >> log2B) - jb0];
                const int nvp = min(B, p1 - tk);
                const int64_t off = (int64_t)blk * blk_stride + head_off;
                const uint32_t bytes = (uint32_t)(nvp * RB);
                bulk_g2s(sK + (lane << log2B) * RB, kc + off, bytes, bar);
                bulk_g2s(sV + (lane << log2B) * RB, vc + off, bytes, bar);
            }
        }
    }
    __syncwarp();
}

// Store the new token's row (already in shared memory) to its cache slot: lanes of
// token group 0, two 16-byte chunks of K and of V each.
template <typename T, int D>
__device__ __forceinline__ void write_new_token(const AttnParams& p, const char* sKrow, const char* sVrow, int s,
                                                int kvh, int t_new, int c) {
    using C = AttnCfg<T, D>;
    constexpr int RB = C::RB, LT = C::LT;
    const int blk = __ldg(p.block_tables + (int64_t)s * p.W + (t_new >> p.log2B));
    const int64_t off = (int64_t)blk * (((int64_t)p.H_kv << p.log2B) * RB) + (((int64_t)kvh << p.log2B) * RB) +
                        (int64_t)(t_new & ((1 << p.log2B) - 1)) * RB;
    uint4* dk = reinterpret_cast<uint4*>(static_cast<char*>(p.key_cache_w) + off);
    uint4* dv = reinterpret_cast<uint4*>(static_cast<char*>(p.value_cache_w) + off);
    dk[c] = lds128(sKrow + c * 16);
    dk[c + LT] = lds128(sKrow + (c + LT) * 16);
    dv[c] = lds128(sVrow + c * 16);
    dv[c + LT] = lds128(sVrow + (c + LT) * 16);
}

// ================================================================== coop scheduler ===
//
// One CTA = (partition, group of HPC query heads, sequence) with HPC consumer warps (one
// query head each) and one producer warp.  A tile stage holds the K and V rows of the
// group's NKV kv heads for 16 logical tokens: with block_size 16 the NKV head slabs of
// a block are contiguous, so a full tile is ONE bulk copy of NKV*B*D*e bytes for K and
// one for V (16 KB each for 4 fp16 heads of D=128).  Consumers wait on full[k], compute
// their head, and release the stage with one arrive per warp on empty[k]; the producer
// waits on empty[k] before refilling it.  The CTA's warps therefore stay in lockstep on
// the same blocks (contiguous DRAM reads), and no consumer ever issues a copy.
#ifdef PA_DECODE_TRACE  // timing experiments (variant build): per-CTA globaltimer events
__device__ unsigned long long g_dec_trace[(1 << 17) * 4];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DEC_T(slot, v)                                                                              \
    do {                                                                                          \
        const unsigned cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);      \
        if (cta < (1u << 17)) g_dec_trace[cta * 4 + (slot)] = (v);                                  \
    } while (0)
#else
#define DEC_T(slot, v) \
    do {               \
    } while (0)
#endif

template <typename T, int D>
#ifndef PA_COOP_MINB
#define PA_COOP_MINB 1
#endif
__global__ void __launch_bounds__(288, PA_COOP_MINB) paged_attention_coop_kernel(const AttnParams p) {
    using C = AttnCfg<T, D>;
    constexpr int RB = C::RB, LT = C::LT, EPC = C::EPC;
    extern __shared__ __align__(128) unsigned char smem[];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HPC = p.HPC, STG = p.STG, G = p.G, PT = p.PT;
    const int NKVmax = HPC % G == 0 ? HPC / G : (HPC + G - 1) / G + 1;  // stage layout stride (host-sized)
    const int slab = kTile * RB;                   // one kv head x 16 rows
    const int stage_bytes = 2 * NKVmax * slab;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STG * stage_bytes);
    uint64_t* empty = full + STG;
    int* sbt = reinterpret_cast<int*>(empty + STG);
    pdl_wait();
#ifdef PA_DECODE_TRACE
    if (threadIdx.x == 0) DEC_T(0, gtimer());
#endif
    int bt_pref = 0;  // producer lane i: block id jb0 + i, loaded while ctx is in flight
    const int hg = p.pz ? blockIdx.x : blockIdx.y;
    const int zs = p.pz ? blockIdx.y : blockIdx.z;
    const int s = zs < p.n_order ? (int)p.seq_order[zs] : zs;  // longest-first plan (scheduling only)
    // this CTA walks the arithmetic partitions [c0, c0 + PPC) of the context back to
    // back; each is finished exactly as if it had its own CTA (bitwise identical)
    const int c0 = (p.pz ? blockIdx.z : blockIdx.x) * p.PPC;
    int ctx;
    {
        // the partition's first 32 block ids depend only on (s, c0): the producer loads
        // them (in-row entries past the context are read, never used) in parallel with
        // context_lens[s] instead of after it -- one dependent global round trip less
        const int jb = (c0 * PT) >> p.log2B;
        if (warp == HPC && jb + lane < p.W) bt_pref = __ldg(p.block_tables + (int64_t)s * p.W + jb + lane);
        ctx = p.context_lens[s];
    }
    // consumer warps' query rows, also in flight across the barrier below
    uint4 q0 = make_uint4(0u, 0u, 0u, 0u), q1 = q0;
    if (warp < HPC && hg * HPC + warp < p.H) {
        const uint4* qrow = reinterpret_cast<const uint4*>(static_cast<const char*>(p.query) +
                                                           ((int64_t)s * p.H + hg * HPC + warp) * RB);
        q0 = __ldg(qrow + lane % LT);
        q1 = __ldg(qrow + lane % LT + LT);
    }
    if (threadIdx.x < STG) {
        mbar_init(&full[threadIdx.x], 1);
        mbar_init(&empty[threadIdx.x], min(HPC, p.H - hg * HPC));
    }
    fence_mbar_init();
    __syncthreads();
    pdl_launch_dependents();  // the next kernel may become resident during our last wave
    const int h0 = hg * HPC;
    const int nh = min(HPC, p.H - h0);          // consumer warps with a head
    const int kvh0 = h0 / G;
    const int NKV = (h0 + nh - 1) / G - kvh0 + 1;  // kv heads the group reads
    const int nparts = ctx > 0 ? (ctx + PT - 1) / PT : 1;
    if (c0 > 0 && c0 >= nparts) return;  // this sequence has fewer partitions (CTA-uniform)
    const int p0 = c0 * PT;
    const int p1 = min(ctx, p0 + p.PPC * PT);
    const int ntiles = p1 > p0 ? (p1 - p0 + kTile - 1) / kTile : 0;
    const int t_new = (p.new_key != nullptr && ctx > 0 && p1 == ctx) ? ctx - 1 : -1;
    const int pc = t_new >= 0 ? t_new : p1;

    if (warp == HPC) {  // ------------------------------------------------ producer warp
        // the partition's block ids into shared memory (producer-only: no CTA barrier)
        const int jb0 = p0 >> p.log2B;
        const int nb = p1 > p0 ? ((p1 - 1) >> p.log2B) - jb0 + 1 : 0;
        const int32_t* btrow = p.block_tables + (int64_t)s * p.W;
        if (lane < nb) sbt[lane] = bt_pref;
        for (int i = 32 + lane; i < nb; i += 32) sbt[i] = __ldg(btrow + jb0 + i);
        __syncwarp();
        const int B = 1 << p.log2B;
        const char* kc = static_cast<const char*>(p.key_cache);
        const char* vc = static_cast<const char*>(p.value_cache);
        const int64_t blk_bytes = ((int64_t)p.H_kv << p.log2B) * RB;
        const int pieces = B >= kTile ? 1 : kTile / B;
        // stage cursor and phases kept incrementally (no per-tile integer division)
        int k = 0;
        uint32_t ephase = 0;
        char* sK = reinterpret_cast<char*>(smem);
        for (int j = 0, tok0 = p0; j < ntiles; ++j, tok0 += kTile) {
            if (j >= STG) mbar_wait(&empty[k], ephase);
            char* sV = sK + NKVmax * slab;
            const int nvc = max(0, min(kTile, pc - tok0));
            const bool has_new = t_new >= tok0 && t_new < tok0 + kTile;
            if (lane == 0)
                mbar_arrive_expect_tx(&full[k], (uint32_t)(2 * NKV * (nvc + (has_new ? 1 : 0)) * RB));
            __syncwarp();
            if (B >= kTile && nvc == kTile && B == kTile) {
                // whole tile of the group = NKV contiguous head slabs of one block
                if (lane == 0) {
                    const int blk = sbt[(tok0 >> p.log2B) - jb0];
                    const int64_t off = (int64_t)blk * blk_bytes + (int64_t)kvh0 * slab;
                    bulk_g2s(sK, kc + off, (uint32_t)(NKV * slab), &full[k]);
                    bulk_g2s(sV, vc + off, (uint32_t)(NKV * slab), &full[k]);
                }
            } else if (nvc > 0) {
                for (int it = lane; it < NKV * pieces; it += 32) {
                    const int kh = it / pieces, pi = it - kh * pieces;
                    const int tk = tok0 + pi * min(B, kTile);
                    if (tk >= pc) continue;
                    const int blk = sbt[(tk >> p.log2B) - jb0];
                    const int rows = min(min(B, kTile), pc - tk);
                    const int64_t off = (int64_t)blk * blk_bytes + ((int64_t)(kvh0 + kh) << p.log2B) * RB +
                                        (int64_t)(tk & (B - 1)) * RB;
                    const int dst = kh * slab + (tk - tok0) * RB;
                    bulk_g2s(sK + dst, kc + off, (uint32_t)(rows * RB), &full[k]);
                    bulk_g2s(sV + dst, vc + off, (uint32_t)(rows * RB), &full[k]);
                }
            }
            if (has_new && lane < NKV) {  // the new token's rows come from the step's inputs
                const int64_t src = ((int64_t)s * p.H_kv + kvh0 + lane) * RB;
                const int dst = lane * slab + (t_new - tok0) * RB;
                bulk_g2s(sK + dst, static_cast<const char*>(p.new_key) + src, RB, &full[k]);
                bulk_g2s(sV + dst, static_cast<const char*>(p.new_value) + src, RB, &full[k]);
            }
            __syncwarp();
            if (++k == STG) {
                k = 0;
                sK = reinterpret_cast<char*>(smem);
                if (j >= STG) ephase ^= 1u;  // wrapped past a round that waited on empty
            } else {
                sK += stage_bytes;
            }
        }
        return;
    }
    if (warp >= nh) return;  // ragged last head group

    // ------------------------------------------------------------------ consumer warps
    const int h = h0 + warp;
    const int kh = h / G - kvh0;
    const int g = lane / LT, c = lane % LT;
    const int64_t sh = (int64_t)s * p.H + h;
    // a CTA that owns every partition of a split context merges them itself, in shared
    // memory (same arithmetic as the workspace path, no counters, no global round trip)
    const bool whole = nparts > 1 && c0 == 0 && p1 == ctx;
    float* my_po = reinterpret_cast<float*>(
                       smem + (((size_t)STG * stage_bytes + 16 * STG + 4 * (size_t)(p.PPC * PT / (1 << p.log2B) + 2) +
                                15) & ~(size_t)15)) +
                   (size_t)warp * p.PPC * D;
    float2* my_ml = reinterpret_cast<float2*>(
                        smem + (((size_t)STG * stage_bytes + 16 * STG + 4 * (size_t)(p.PPC * PT / (1 << p.log2B) + 2) +
                                 15) & ~(size_t)15) + (size_t)HPC * p.PPC * D * 4) +
                    (size_t)warp * p.PPC;
    float m = -INFINITY, l = 0.f;
    float2 acc[EPC];
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = make_float2(0.f, 0.f);
    // incremental cursors: stage k / phase, stage pointer, current partition and its end,
    // the tile holding the new token (-1: none or not written by this warp)
    int k = 0, part = c0, part_end = min(p1, (c0 + 1) * PT);
    uint32_t fphase = 0;
    const char* sKb = reinterpret_cast<const char*>(smem) + kh * slab;
    const int j_new = (t_new >= 0 && h % G == 0) ? (t_new - p0) / kTile : -1;
    for (int j = 0, tok0 = p0; j < ntiles; ++j, tok0 += kTile) {
        mbar_wait(&full[k], fphase);
#ifdef PA_DECODE_TRACE
        if (j == 0 && threadIdx.x == 0) DEC_T(1, gtimer());
#endif
        const char* sK = sKb;
        const char* sV = sK + NKVmax * slab;
        if (j == j_new && g == 0)
            write_new_token<T, D>(p, sK + (t_new - tok0) * RB, sV + (t_new - tok0) * RB, s, h / G, t_new, c);
        tile_update<T, D>(sK, sV, min(kTile, p1 - tok0), q0, q1, p.scale_log2, g, c, m, l, acc);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[k]);
        if (++k == STG) {
            k = 0;
            fphase ^= 1u;
            sKb = reinterpret_cast<const char*>(smem) + kh * slab;
        } else {
            sKb += stage_bytes;
        }
        if (tok0 + kTile >= part_end) {  // last tile of this partition
            merge_token_groups<T, D>(m, l, acc);
            if (nparts == 1) {
                if (g == 0) store_out_p<T, D>(p, sh, l, acc, c);
            } else if (whole) {  // keep (m, L, o~) in shared memory; merged below
                if (g == 0) store_partial<T, D>(my_po + (part - c0) * D, l, acc, c);
                if (lane == 0) my_ml[part - c0] = make_float2(m, l);
            } else {
                finish_split<T, D>(p, sh, part, nparts, m, l, acc, g, c, lane);
            }
            m = -INFINITY;
            l = 0.f;
#pragma unroll
            for (int e = 0; e < EPC; ++e) acc[e] = make_float2(0.f, 0.f);
            ++part;
            part_end = min(p1, part_end + PT);
        }
    }
    if (ntiles == 0 && g == 0)  // empty context
        store_out_p<T, D>(p, sh, 0.f, acc, c);
    if (whole) {
        __syncwarp();
        merge_partitions_from<T, D, false>(p, sh, my_ml, my_po, nparts, lane);
    }
#ifdef PA_DECODE_TRACE
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        DEC_T(2, gtimer());
        DEC_T(3, (unsigned long long)smid | ((unsigned long long)ntiles << 16) | ((unsigned long long)s << 32));
    }
#endif
}

// ========================================= sharing-aware scheduler ===
//
// Sequences of one sequence group (the n samples of a request, the k beams of a beam
// search) share physical blocks.  One CTA = (partition, group of HPC query
// heads, group of M consecutive sequences); consumer warp (member m, head i) runs the
// standard per-(sequence, head) tile arithmetic, so outputs are bit-identical to the
// other schedulers.  The producer warp looks up the M members' physical blocks for each
// 16-token logical tile, copies every DISTINCT block once into a slot of the stage and
// publishes the member -> slot map with the stage: a block shared by the whole group
// crosses L2 -> SM once instead of M times.  Tiles holding a member's new token are
// never shared (copy-on-write made that block private).
#ifndef PA_SHARED_MINB
#define PA_SHARED_MINB 4  // register cap for 4 CTAs/SM (56 regs): c5 470-476 vs 475-486 us at 72 regs
                          // (no cap: 102 regs, 2 CTAs/SM, 930 us)
#endif
template <typename T, int D>
__global__ void __launch_bounds__(288, PA_SHARED_MINB) paged_attention_shared_kernel(const AttnParams p) {
    using C = AttnCfg<T, D>;
    constexpr int RB = C::RB, LT = C::LT, EPC = C::EPC;
    extern __shared__ __align__(128) unsigned char smem[];

    const int hg = blockIdx.y, grp = blockIdx.z, part = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HPC = p.HPC, STG = p.STG, G = p.G, PT = p.PT, M = p.GM;
    const int NC = M * HPC;                               // consumer warps
    const int h0 = hg * HPC, nh = min(HPC, p.H - h0);
    const int kvh0 = h0 / G, NKV = (h0 + nh - 1) / G - kvh0 + 1;
    const int NKVmax = HPC % G == 0 ? HPC / G : (HPC + G - 1) / G + 1;
    const int slab = kTile * RB;                          // one kv head x 16 rows
    const int slot_bytes = 2 * NKVmax * slab;             // K | V of the head group
    const int NSL = p.GSL;                                // distinct-block slots per stage
    // stage = NSL slots | header: member -> slot map [M], then the logical tile index
    // (-1 = end of the partition's stream)
    const int stage_bytes = NSL * slot_bytes + 16 * ((M + 16) / 16) * 4;
    const int s0 = grp * M, nm = min(M, p.S - s0);        // members of this group
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)STG * stage_bytes);
    uint64_t* empty = full + STG;
    if (threadIdx.x < STG) {
        mbar_init(&full[threadIdx.x], 1);
        mbar_init(&empty[threadIdx.x], NC);
    }
    fence_mbar_init();
    __syncthreads();
    pdl_wait();
    // the group's partition: tiles [part*PT, part*PT + PT) of every member still active
    int gmax = 0;  // longest member context
    for (int m = 0; m < nm; ++m) gmax = max(gmax, __ldg(p.context_lens + s0 + m));
    const int p0 = part * PT;
    if (part > 0 && p0 >= gmax) return;  // no member reaches this partition (CTA-uniform)
    const int ntiles = (min(gmax, p0 + PT) - p0 + kTile - 1) / kTile;
    auto slot_map = [&](int k) { return reinterpret_cast<int*>(smem + (size_t)k * stage_bytes + NSL * slot_bytes); };

    if (warp == NC) {  // ================================================ producer warp
        const int B = 1 << p.log2B;
        const char* kc = static_cast<const char*>(p.key_cache);
        const char* vc = static_cast<const char*>(p.value_cache);
        const int64_t blk_bytes = ((int64_t)p.H_kv << p.log2B) * RB;
        // lane m < nm: member m's context, copy limit and new-token position
        const int my_s = s0 + min(lane, nm - 1);
        const int my_ctx = lane < nm ? __ldg(p.context_lens + my_s) : 0;
        const int my_p1 = min(my_ctx, p0 + PT);
        const int my_tnew = (p.new_key != nullptr && lane < nm && my_ctx > 0 && my_p1 == my_ctx) ? my_ctx - 1 : -1;
        const int my_pc = my_tnew >= 0 ? my_tnew : my_p1;
        const int32_t* btrow = p.block_tables + (int64_t)my_s * p.W;
        int n = 0;  // stages emitted so far
        // block id of the member's next tile, loaded one tile ahead (its L2 round trip
        // overlaps this tile's stage wait and copy issue)
        int blk_next = (lane < nm && B >= kTile && p0 < my_p1) ? __ldg(btrow + (p0 >> p.log2B)) : -1;
        for (int j = 0; j < ntiles; ++j) {
            const int tok0 = p0 + j * kTile;
            const int blk_cur = blk_next;
            if (lane < nm && B >= kTile && tok0 + kTile < my_p1) blk_next = __ldg(btrow + ((tok0 + kTile) >> p.log2B));
            // per member: block id, rows needed, whether the tile holds its new token
            const bool act = lane < nm && tok0 < my_p1;
            const int rows = act ? max(0, min(kTile, my_pc - tok0)) : 0;
            const bool has_new = act && my_tnew >= tok0 && my_tnew < tok0 + kTile;
            // B >= 16: one block per tile; B < 16: a tile spans several blocks -> no sharing
            const int blk = (act && rows > 0 && B >= kTile) ? blk_cur : -1;
            const bool shareable = act && !has_new && B >= kTile && rows > 0;
            // leader = first member with the same block (shareable tiles only)
            int leader = lane;
            for (int m = 0; m < nm; ++m) {
                const int bm = __shfl_sync(0xffffffffu, blk, m);
                const bool sm = __shfl_sync(0xffffffffu, shareable, m);
                if (shareable && sm && bm == blk && m < leader) leader = m;
            }
            const bool is_leader = act && leader == lane;
            const unsigned leaders = __ballot_sync(0xffffffffu, is_leader);
            const int my_slot_if_leader = __popc(leaders & ((1u << lane) - 1u));
            const int slot = __shfl_sync(0xffffffffu, my_slot_if_leader, leader);
            // rows a shared slot must hold: the largest need among its members
            // (a match.any / redux.sync version of this leader search measured 60% slower)
            int need = rows;
            for (int m = 0; m < nm; ++m) {
                const int lm = __shfl_sync(0xffffffffu, leader, m);
                const int rm = __shfl_sync(0xffffffffu, rows, m);
                if (is_leader && lm == lane) need = max(need, rm);
            }
            const int nd = __popc(leaders);  // distinct slots the tile needs
            for (int r0 = 0; r0 < nd; r0 += NSL) {  // one stage per NSL distinct blocks
                const int k = n % STG;
                if (n >= STG) mbar_wait(&empty[k], ((n / STG) - 1) & 1);
                char* st = reinterpret_cast<char*>(smem) + (size_t)k * stage_bytes;
                const bool mine = is_leader && my_slot_if_leader >= r0 && my_slot_if_leader < r0 + NSL;
                const uint32_t my_tx = mine ? (uint32_t)(2 * NKV * (need + (has_new ? 1 : 0)) * RB) : 0u;
                uint32_t tx = my_tx;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) tx += __shfl_xor_sync(0xffffffffu, tx, off);
                if (lane < M) slot_map(k)[lane] = (act && slot >= r0 && slot < r0 + NSL) ? slot - r0 : -1;
                if (lane == 0) slot_map(k)[M] = j;
                __syncwarp();
                if (lane == 0) mbar_arrive_expect_tx(&full[k], tx);  // also publishes the header
                __syncwarp();
                if (mine) {
                    char* sK = st + (size_t)(my_slot_if_leader - r0) * slot_bytes;
                    char* sV = sK + NKVmax * slab;
                    if (need > 0) {
                        if (B >= kTile) {
                            if (B == kTile && need == kTile) {  // NKV contiguous head slabs of one block
                                const int64_t off = (int64_t)blk * blk_bytes + (int64_t)kvh0 * slab;
                                bulk_g2s(sK, kc + off, (uint32_t)(NKV * slab), &full[k]);
                                bulk_g2s(sV, vc + off, (uint32_t)(NKV * slab), &full[k]);
                            } else {
                                for (int kh = 0; kh < NKV; ++kh) {
                                    const int64_t off = (int64_t)blk * blk_bytes +
                                                        ((int64_t)(kvh0 + kh) << p.log2B) * RB +
                                                        (int64_t)(tok0 & (B - 1)) * RB;
                                    bulk_g2s(sK + kh * slab, kc + off, (uint32_t)(need * RB), &full[k]);
                                    bulk_g2s(sV + kh * slab, vc + off, (uint32_t)(need * RB), &full[k]);
                                }
                            }
                        } else {
                            for (int kh = 0; kh < NKV; ++kh)
                                for (int tk = tok0; tk < tok0 + need; tk += B) {
                                    const int b2 = __ldg(btrow + (tk >> p.log2B));
                                    const int r2 = min(B, tok0 + need - tk);
                                    const int64_t off =
                                        (int64_t)b2 * blk_bytes + ((int64_t)(kvh0 + kh) << p.log2B) * RB;
                                    bulk_g2s(sK + kh * slab + (tk - tok0) * RB, kc + off, (uint32_t)(r2 * RB),
                                             &full[k]);
                                    bulk_g2s(sV + kh * slab + (tk - tok0) * RB, vc + off, (uint32_t)(r2 * RB),
                                             &full[k]);
                                }
                        }
                    }
                    if (has_new)
                        for (int kh = 0; kh < NKV; ++kh) {
                            const int64_t src = ((int64_t)my_s * p.H_kv + kvh0 + kh) * RB;
                            const int dst = kh * slab + (my_tnew - tok0) * RB;
                            bulk_g2s(sK + dst, static_cast<const char*>(p.new_key) + src, RB, &full[k]);
                            bulk_g2s(sV + dst, static_cast<const char*>(p.new_value) + src, RB, &full[k]);
                        }
                }
                __syncwarp();
                ++n;
            }
        }
        {  // end-of-stream stage: header only
            const int k = n % STG;
            if (n >= STG) mbar_wait(&empty[k], ((n / STG) - 1) & 1);
            if (lane == 0) {
                slot_map(k)[M] = -1;
                mbar_arrive_expect_tx(&full[k], 0u);
            }
        }
        return;
    }

    // ============================================================== consumer warps
    const int mem = warp / HPC, hi = warp - mem * HPC;
    const bool active = mem < nm && hi < nh;
    const int s = s0 + min(mem, nm - 1), h = h0 + min(hi, nh - 1);
    const int ctx = __ldg(p.context_lens + s);
    const int nparts = ctx > 0 ? (ctx + PT - 1) / PT : 1;
    const int p1 = min(ctx, p0 + PT);
    const int t_new = (p.new_key != nullptr && ctx > 0 && p1 == ctx) ? ctx - 1 : -1;
    const int kh = h / G - kvh0;
    const int g = lane / LT, c = lane % LT;
    const int64_t sh = (int64_t)s * p.H + h;
    const uint4* qrow = reinterpret_cast<const uint4*>(static_cast<const char*>(p.query) + sh * RB);
    const uint4 q0 = __ldg(qrow + c), q1 = __ldg(qrow + c + LT);
    const int my_ntiles = p1 > p0 ? (p1 - p0 + kTile - 1) / kTile : 0;
    float m = -INFINITY, l = 0.f;
    float2 acc[EPC];
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = make_float2(0.f, 0.f);
    for (int n = 0;; ++n) {  // the producer's stage stream, ended by tile index -1
        const int k = n % STG;
        mbar_wait(&full[k], (n / STG) & 1);
        const int j = slot_map(k)[M];
        if (j < 0) break;
        const int slot = slot_map(k)[mem];
        if (active && j < my_ntiles && slot >= 0) {
            const char* sK = reinterpret_cast<const char*>(smem) + (size_t)k * stage_bytes + (size_t)slot * slot_bytes +
                             kh * slab;
            const char* sV = sK + NKVmax * slab;
            const int tok0 = p0 + j * kTile;
            if (t_new >= tok0 && t_new < tok0 + kTile && h % G == 0 && g == 0)
                write_new_token<T, D>(p, sK + (t_new - tok0) * RB, sV + (t_new - tok0) * RB, s, h / G, t_new, c);
            tile_update<T, D>(sK, sV, min(kTile, p1 - tok0), q0, q1, p.scale_log2, g, c, m, l, acc);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[k]);
    }
    if (!active) return;
    if (part > 0 && p0 >= ctx) return;  // this member has no tokens in the partition
    merge_token_groups<T, D>(m, l, acc);
    if (nparts == 1) {
        if (g == 0) store_out_p<T, D>(p, sh, l, acc, c);
    } else {
        finish_split<T, D>(p, sh, part, nparts, m, l, acc, g, c, lane);
    }
}

// ==================================================================== debug gather ===

// Test-only: copy the logical K/V rows of (s, kvh) through the grid scheduler's loader.
template <typename T, int D>
__global__ void __launch_bounds__(32) debug_gather_kernel(GatherParams p) {
    constexpr int RB = D * Elem<T>::kBytes;
    constexpr int PT = 512;
    __shared__ __align__(128) char stage[2 * kTile * RB];
    __shared__ uint64_t bar;
    __shared__ int sbt[PT + 2];
    const int s = blockIdx.x, kvh = blockIdx.y, lane = threadIdx.x;
    const int ctx = p.context_lens[s];
    if (lane == 0) mbar_init(&bar, 1);
    fence_mbar_init();
    __syncwarp();
    const char* kc = static_cast<const char*>(p.key_cache);
    const char* vc = static_cast<const char*>(p.value_cache);
    const int64_t blk_stride = ((int64_t)p.H_kv << p.log2B) * RB;
    const int64_t head_off = ((int64_t)kvh << p.log2B) * RB;
    uint32_t phase = 0;
    for (int p0 = 0; p0 < ctx; p0 += PT) {
        const int p1 = min(ctx, p0 + PT);
        const int jb0 = p0 >> p.log2B;
        const int nb = ((p1 - 1) >> p.log2B) - jb0 + 1;
        for (int i = lane; i < nb; i += 32) sbt[i] = p.block_tables[(int64_t)s * p.W + jb0 + i];
        __syncwarp();
        for (int tok0 = p0; tok0 < p1; tok0 += kTile) {
            const int nv = min(kTile, p1 - tok0);
            issue_tile(stage, stage + kTile * RB, &bar, kc, vc, sbt, jb0, tok0, nv, p1, p.log2B, blk_stride, head_off,
                       RB, lane);
            mbar_wait(&bar, phase);
            phase ^= 1u;
            for (int t = 0; t < nv; ++t) {
                char* ko = static_cast<char*>(p.k_out) + (((int64_t)s * p.H_kv + kvh) * p.max_ctx + tok0 + t) * RB;
                char* vo = static_cast<char*>(p.v_out) + (((int64_t)s * p.H_kv + kvh) * p.max_ctx + tok0 + t) * RB;
                for (int i = lane; i < RB / 16; i += 32) {
                    reinterpret_cast<uint4*>(ko)[i] = reinterpret_cast<const uint4*>(stage + t * RB)[i];
                    reinterpret_cast<uint4*>(vo)[i] = reinterpret_cast<const uint4*>(stage + kTile * RB + t * RB)[i];
                }
            }
            __syncwarp();
        }
    }
}

// ================================================================== host launchers ===

int attention_row_bytes(int dtype, int head_dim) { return head_dim * (dtype == 0 ? 4 : 2); }

size_t attention_smem_bytes_coop(int row_bytes, int hpc, int G, int stg, int partition_tokens, int block_size,
                                 int ppc, int head_dim) {
    // partition_tokens here = tokens one CTA walks (PPC partitions)
    const int nkv_max = hpc % G == 0 ? hpc / G : (hpc + G - 1) / G + 1;
    const size_t tbl = 4 * (size_t)(partition_tokens / block_size + 2);
    const size_t head = (((size_t)stg * 2 * nkv_max * kTile * (size_t)row_bytes + 16 * (size_t)stg + tbl) + 15) & ~(size_t)15;
    return head + (size_t)hpc * ppc * ((size_t)head_dim * 4 + 8);  // in-CTA partials
}

size_t attention_smem_bytes_shared(int row_bytes, int hpc, int G, int stg, int gm, int nsl) {
    const int nkv_max = hpc % G == 0 ? hpc / G : (hpc + G - 1) / G + 1;
    const size_t stage = (size_t)nsl * 2 * nkv_max * kTile * row_bytes + 16 * (size_t)((gm + 16) / 16) * 4;
    return (size_t)stg * stage + 16 * (size_t)stg;
}

template <typename T, int D>
static cudaError_t launch_attention_t(const AttnParams& p, int num_seqs, int sched, size_t smem,
                                      cudaStream_t stream) {
    if (sched == 4) {  // sharing-aware: groups of GM consecutive sequences
        auto kern = paged_attention_shared_kernel<T, D>;
        cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
        if (e != cudaSuccess) return e;
        const int groups = (p.H + p.HPC - 1) / p.HPC;
        const int sgroups = (num_seqs + p.GM - 1) / p.GM;
        return launch_k(kern, dim3(p.NP, groups, sgroups), dim3((p.GM * p.HPC + 1) * 32), smem, stream, p);
    }
    // coop: HPC consumer warps + 1 producer warp per CTA
    auto kern = paged_attention_coop_kernel<T, D>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    const int groups = (p.H + p.HPC - 1) / p.HPC;
    if (p.pz)  // partition index slowest: partitions >= 1 (and the empty ones) launch last
        return launch_k(kern, dim3(groups, num_seqs, (p.NP + p.PPC - 1) / p.PPC), dim3((p.HPC + 1) * 32), smem,
                        stream, p);
    return launch_k(kern, dim3((p.NP + p.PPC - 1) / p.PPC, groups, num_seqs), dim3((p.HPC + 1) * 32), smem, stream,
                    p);
}

cudaError_t launch_attention(const AttnParams& p, int dtype, int head_dim, int num_seqs, int sched, size_t smem,
                             cudaStream_t stream) {
    if (dtype == 0) {
        return head_dim == 64 ? launch_attention_t<float, 64>(p, num_seqs, sched, smem, stream)
                              : launch_attention_t<float, 128>(p, num_seqs, sched, smem, stream);
    } else if (dtype == 1) {
        return head_dim == 64 ? launch_attention_t<__half, 64>(p, num_seqs, sched, smem, stream)
                              : launch_attention_t<__half, 128>(p, num_seqs, sched, smem, stream);
    }
    return head_dim == 64 ? launch_attention_t<__nv_bfloat16, 64>(p, num_seqs, sched, smem, stream)
                          : launch_attention_t<__nv_bfloat16, 128>(p, num_seqs, sched, smem, stream);
}

cudaError_t launch_debug_gather(const GatherParams& p, int dtype, int head_dim, int num_seqs, cudaStream_t stream) {
    dim3 grid(num_seqs, p.H_kv);
    if (dtype == 0) {
        if (head_dim == 64) debug_gather_kernel<float, 64><<<grid, 32, 0, stream>>>(p);
        else debug_gather_kernel<float, 128><<<grid, 32, 0, stream>>>(p);
    } else if (dtype == 1) {
        if (head_dim == 64) debug_gather_kernel<__half, 64><<<grid, 32, 0, stream>>>(p);
        else debug_gather_kernel<__half, 128><<<grid, 32, 0, stream>>>(p);
    } else {
        if (head_dim == 64) debug_gather_kernel<__nv_bfloat16, 64><<<grid, 32, 0, stream>>>(p);
        else debug_gather_kernel<__nv_bfloat16, 128><<<grid, 32, 0, stream>>>(p);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace pa

#ifdef PA_DECODE_TRACE
extern "C" int pa_debug_decode_trace_read(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, pa::g_dec_trace, sizeof(unsigned long long) * (size_t)n);
}
#endif
