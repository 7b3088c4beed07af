// pa_attention.cu -- PagedAttention decode kernels for B200 (sm_100a).
//
// Eq.4 of the paper: for every (sequence s, query head h) the kernel walks
// the sequence's logical tokens through its block table, computes
// l_t = scale * q.K_t, a numerically stable softmax and sum_t softmax_t * V_t.
//
// B200 design:
//  * One CTA per (partition, group of HPC query heads, sequence); warp w owns one query
//    head and walks the partition's 16-token LOGICAL tiles in order (the arithmetic
//    never depends on block_size, physical placement, head grouping or grid shape ->
//    bitwise invariance).  The partition's block ids are prefetched into shared memory
//    once per CTA (shared by its heads), so no copy waits on a dependent global load
//    (the paper's "extra overhead of accessing the block table").
//  * Tiles are staged into shared memory by 1-D bulk async copies (cp.async.bulk,
//    SASS UBLKCP) completing on a per-stage mbarrier; each warp keeps STG tiles in flight
//    (lane 0 issues; for block_size < 16 lanes issue one piece each).
//  * Lane mapping: a K/V row of RB = D*e bytes is covered by LT = RB/32 lanes, each
//    owning two 16-byte chunks (c and c+LT: conflict-free 128-byte phases); a warp
//    handles TG = 32/LT tokens at once.  q.k uses the sm_100 mixed-precision FMA
//    (FHFMA, f16/bf16 x f16/bf16 + f32) straight from the packed storage dtype; the
//    dot product is reduced with warp shuffles across the LT lanes.  Each token group
//    keeps its own online-softmax state (m, l, acc[]) in the exp2 domain, and p*V is
//    accumulated with packed fp32x2 FMAs (FFMA2).  No tensor cores: a one-query decode
//    step is a memory-bound GEMV (BJ:north_star).
//  * End: token groups merge by shuffles (log-sum-exp, fixed order).  A sequence whose
//    context fits one partition writes `out` directly (16-byte stores); otherwise each
//    partition writes (m, L, o~) and paged_attention_reduce merges them (split-context
//    variant, BJ:north_star).
#include "pa_common.cuh"
#include "pa_internal.h"

#include <cfloat>

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

// Issue the bulk copies of logical tile `tok0` (nv valid tokens, nv <= 16) of kv head
// `kvh` into (sK, sV).  sbt holds the block ids of logical blocks jb0, jb0+1, ...
// Called by a whole warp (lanes 0..pieces-1 issue).  Only rows t < p1 are copied, so
// slots past the context are never read (reading c3).
__device__ __forceinline__ void issue_tile(char* sK, char* sV, uint64_t* bar, const char* kc, const char* vc,
                                           const int* sbt, int jb0, int tok0, int nv, int p1, int log2B,
                                           int64_t blk_stride, int64_t head_off, int RB, int lane) {
    const int B = 1 << log2B;
    if (B >= kTile) {
        if (lane == 0) {
            const int blk = nv > 0 ? sbt[(tok0 >> log2B) - jb0] : 0;
            const int64_t off = (int64_t)blk * blk_stride + head_off + (int64_t)(tok0 & (B - 1)) * RB;
            const uint32_t bytes = (uint32_t)(nv * RB);
            mbar_arrive_expect_tx(bar, 2 * bytes);
            if (bytes) {
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

// One warp walks the logical tiles [p0, p1) of (sequence s, query head h) and leaves
// the online-softmax state of its token groups merged: every lane ends with (m, l) of
// the whole range (exp2 domain) and acc[] = unnormalised sum p*V for its two chunks.
//
// Fused cache write (decode entry point): when t_new >= 0 the token at logical position
// t_new (= ctx - 1, the last row of this partition) is this step's new token.  Its K/V
// row comes from new_key/new_value in registers; one warp per (sequence, kv head)
// stores it into the cache slot (reshape_and_cache), and the tile loader
// copies only the rows before it, the row itself being written into shared memory.
template <typename T, int D>
__device__ __forceinline__ void walk_partition(const AttnParams& p, int s, int h, int p0, int p1, int t_new,
                                               const int* sbt, int jb0, char* stage0, uint64_t* wbars, int lane,
                                               float& m_out, float& l_out, float2 (&acc)[AttnCfg<T, D>::EPC]) {
    using C = AttnCfg<T, D>;
    constexpr int RB = C::RB, LT = C::LT, TG = C::TG, TPL = C::TPL, EPC = C::EPC;
    const int STG = p.STG;
    const int ntiles = p1 > p0 ? (p1 - p0 + kTile - 1) / kTile : 0;
    const int kvh = h / p.G;
    const int g = lane / LT, c = lane % LT;
    const uint4* qrow = reinterpret_cast<const uint4*>(static_cast<const char*>(p.query) +
                                                        ((int64_t)s * p.H + h) * RB);
    const uint4 q0 = __ldg(qrow + c), q1 = __ldg(qrow + c + LT);

    const char* kc = static_cast<const char*>(p.key_cache);
    const char* vc = static_cast<const char*>(p.value_cache);
    const int64_t blk_bytes = ((int64_t)p.H_kv << p.log2B) * RB;
    const int64_t head_off = ((int64_t)kvh << p.log2B) * RB;

    // rows copied from the cache end at pc (the new token's row is supplied directly)
    const int pc = t_new >= 0 ? t_new : p1;
    uint4 nk0 = make_uint4(0, 0, 0, 0), nk1 = nk0, nv0 = nk0, nv1 = nk0;
    if (t_new >= 0) {
        const uint4* kr = reinterpret_cast<const uint4*>(static_cast<const char*>(p.new_key) +
                                                          ((int64_t)s * p.H_kv + kvh) * RB);
        const uint4* vr = reinterpret_cast<const uint4*>(static_cast<const char*>(p.new_value) +
                                                          ((int64_t)s * p.H_kv + kvh) * RB);
        nk0 = __ldg(kr + c);
        nk1 = __ldg(kr + c + LT);
        nv0 = __ldg(vr + c);
        nv1 = __ldg(vr + c + LT);
        if (g == 0 && h % p.G == 0) {  // the one writer of (s, kvh)
            const int blk = sbt[(t_new >> p.log2B) - jb0];
            const int64_t off = (int64_t)blk * blk_bytes + head_off + (int64_t)(t_new & ((1 << p.log2B) - 1)) * RB;
            uint4* dk = reinterpret_cast<uint4*>(static_cast<char*>(p.key_cache_w) + off);
            uint4* dv = reinterpret_cast<uint4*>(static_cast<char*>(p.value_cache_w) + off);
            dk[c] = nk0;
            dk[c + LT] = nk1;
            dv[c] = nv0;
            dv[c + LT] = nv1;
        }
    }

    for (int j = 0; j < STG && j < ntiles; ++j) {
        const int tok0 = p0 + j * kTile;
        issue_tile(stage0 + j * C::STAGE_BYTES, stage0 + j * C::STAGE_BYTES + kTile * RB, &wbars[j], kc, vc, sbt,
                   jb0, tok0, max(0, min(kTile, pc - tok0)), pc, p.log2B, blk_bytes, head_off, RB, lane);
    }

    float m = -INFINITY, l = 0.f;
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = make_float2(0.f, 0.f);

    int k = 0;
    uint32_t phase = 0;
    for (int j = 0; j < ntiles; ++j) {
        const int tok0 = p0 + j * kTile;
        const int nv = min(kTile, p1 - tok0);
        const char* sK = stage0 + k * C::STAGE_BYTES;
        const char* sV = sK + kTile * RB;
        mbar_wait(&wbars[k], phase);
        if (t_new >= tok0 && t_new < tok0 + kTile) {  // place the new token's row (last tile)
            if (g == 0) {
                char* rk = const_cast<char*>(sK) + (t_new - tok0) * RB;
                char* rv = const_cast<char*>(sV) + (t_new - tok0) * RB;
                reinterpret_cast<uint4*>(rk)[c] = nk0;
                reinterpret_cast<uint4*>(rk)[c + LT] = nk1;
                reinterpret_cast<uint4*>(rv)[c] = nv0;
                reinterpret_cast<uint4*>(rv)[c + LT] = nv1;
            }
            __syncwarp();
        }

        float sc[TPL];
#pragma unroll
        for (int jj = 0; jj < TPL; ++jj) {
            const char* row = sK + (jj * TG + g) * RB;
            const uint4 k0 = lds128(row + c * 16), k1 = lds128(row + (c + LT) * 16);
            float x = dot16<T>(q0, k0, 0.f) + dot16<T>(q1, k1, 0.f);
#pragma unroll
            for (int off = LT / 2; off >= 1; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
            sc[jj] = x * p.scale_log2;
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
                if (jj * TG + g < nv) {  // rows past the context were never loaded
                    const char* row = sV + (jj * TG + g) * RB;
                    const uint4 v0 = lds128(row + c * 16), v1 = lds128(row + (c + LT) * 16);
                    axpy16<T>(acc, ps[jj], v0);
                    axpy16<T>(acc + EPC / 2, ps[jj], v1);
                }
            }
        }
        m = mn;
        __syncwarp();
        if (j + STG < ntiles) {
            const int t2 = p0 + (j + STG) * kTile;
            issue_tile(stage0 + k * C::STAGE_BYTES, stage0 + k * C::STAGE_BYTES + kTile * RB, &wbars[k], kc, vc, sbt,
                       jb0, t2, max(0, min(kTile, pc - t2)), pc, p.log2B, blk_bytes, head_off, RB, lane);
        }
        if (++k == STG) {
            k = 0;
            phase ^= 1u;
        }
    }

    // merge the token groups of the warp (log-sum-exp, fixed order)
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
    m_out = m;
    l_out = l;
}

// One CTA = (partition, group of HPC query heads, sequence); warp w owns query head
// hg*HPC + w for the whole partition and keeps STG tiles in flight; warps do not
// synchronise with each other between the prologue and the epilogue.
//
// Split-context epilogue (BJ:north_star): every partition writes its (m_p, L_p, o~_p);
// the LAST partition CTA of the (sequence, head group) to finish -- detected with an
// atomic counter in the workspace -- merges them in partition order:
//   M = max m_p;  out = sum_p 2^(m_p - M) L_p o~_p / sum_p 2^(m_p - M) L_p
// (the counters are zeroed on the stream right before the launch).
template <typename T, int D>
__global__ void __launch_bounds__(256)
paged_attention_kernel(const AttnParams p) {
    using C = AttnCfg<T, D>;
    constexpr int LT = C::LT, EPC = C::EPC;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_last;

    const int part = blockIdx.x, hg = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int HPC = p.HPC, STG = p.STG;
    const int h = hg * HPC + warp;
    const bool active = h < p.H;  // ragged last head group
    pdl_wait();  // the step's copy_blocks / reshape_and_cache have landed
    const int ctx = p.context_lens[s];
    const int p0 = part * p.PT;
    if (part > 0 && p0 >= ctx) return;  // this sequence has fewer partitions (CTA-uniform)
    const int p1 = min(ctx, p0 + p.PT);
    const int nparts = ctx > 0 ? (ctx + p.PT - 1) / p.PT : 1;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)HPC * STG * C::STAGE_BYTES);
    int* sbt = reinterpret_cast<int*>(bars + HPC * STG);

    // ---- prologue: block ids of this partition (shared by the CTA's heads), barriers -
    const int jb0 = p0 >> p.log2B;
    const int nb = p1 > p0 ? ((p1 - 1) >> p.log2B) - jb0 + 1 : 0;
    const int32_t* btrow = p.block_tables + (int64_t)s * p.W;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sbt[i] = __ldg(btrow + jb0 + i);
    if (threadIdx.x < HPC * STG) mbar_init(&bars[threadIdx.x], 1);
    fence_mbar_init();
    __syncthreads();

    float m = -INFINITY, l = 0.f;
    float2 acc[EPC];
    const int t_new = (p.new_key != nullptr && ctx > 0 && p1 == ctx) ? ctx - 1 : -1;
    if (active)
        walk_partition<T, D>(p, s, h, p0, p1, t_new, sbt, jb0,
                             reinterpret_cast<char*>(smem) + (size_t)warp * STG * C::STAGE_BYTES, bars + warp * STG,
                             lane, m, l, acc);
    pdl_launch_dependents();  // the next kernel may be scheduled during our last wave
    const int g = lane / LT, c = lane % LT;
    const int64_t sh = (int64_t)s * p.H + h;

    if (nparts == 1) {  // whole context in this CTA: write the output directly
        if (!active || g != 0) return;
        T* o = static_cast<T*>(p.out) + sh * D;
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
        return;
    }

    // ---- split: publish this partition's (m, L, o~) --------------------------------
    if (active && g == 0) {
        float* o = p.part_o + (sh * p.NP + part) * D;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
#pragma unroll
            for (int e = 0; e < EPC / 2; e += 2) {
                const float2 a0 = acc[half * EPC / 2 + e], a1 = acc[half * EPC / 2 + e + 1];
                *reinterpret_cast<float4*>(o + (c + half * LT) * EPC + 2 * e) =
                    make_float4(a0.x / l, a0.y / l, a1.x / l, a1.y / l);
            }
        }
        if (lane == 0) p.part_ml[sh * p.NP + part] = make_float2(m, l);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        int* cnt = p.counters + (int64_t)s * gridDim.y + hg;
        const int old = atomicAdd(cnt, 1);
        s_last = (old == min(nparts, p.NP) - 1);
    }
    __syncthreads();
    if (!s_last || !active) return;
    __threadfence();

    // ---- last partition: merge all partitions of this head, in partition order -----
    const int np = min(nparts, p.NP);
    const float2* ml = p.part_ml + sh * p.NP;
    float M = -INFINITY;
    for (int i = 0; i < np; ++i) M = fmaxf(M, __ldcg(&ml[i]).x);
    float L = 0.f;
    constexpr int DPL = D / 32;  // dims per lane
    float o[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) o[e] = 0.f;
    const float* po = p.part_o + sh * p.NP * D;
    for (int i = 0; i < np; ++i) {
        const float2 mi = __ldcg(&ml[i]);
        const float w = mi.y * ex2(mi.x - M);
        L += w;
#pragma unroll
        for (int e = 0; e < DPL; ++e) o[e] += w * __ldcg(po + (int64_t)i * D + lane * DPL + e);
    }
    T* out = static_cast<T*>(p.out) + sh * D + lane * DPL;
#pragma unroll
    for (int e = 0; e < DPL; ++e) out[e] = Elem<T>::from_f32(o[e] / L);
}

// Test-only: copy the logical K/V rows of (s, kvh) through the same tile loader.
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

// ---------------------------------------------------------------- host launchers -----

int attention_stage_bytes(int dtype, int head_dim) { return 2 * kTile * head_dim * (dtype == 0 ? 4 : 2); }

size_t attention_smem_bytes(int stage_bytes, int hpc, int stg, int partition_tokens, int block_size) {
    const size_t tbl = 4 * (size_t)(partition_tokens / block_size + 2);
    return (size_t)hpc * stg * stage_bytes + 8 * (size_t)hpc * stg + tbl;
}

template <typename T, int D>
static cudaError_t launch_attention_t(const AttnParams& p, int num_seqs, size_t smem, cudaStream_t stream) {
    auto kern = paged_attention_kernel<T, D>;
    static size_t configured = 0;  // per instantiation; only grows
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const int groups = (p.H + p.HPC - 1) / p.HPC;
    if (p.NP > 1) {
        cudaError_t e = cudaMemsetAsync(p.counters, 0, sizeof(int) * (size_t)num_seqs * groups, stream);
        if (e != cudaSuccess) return e;
    }
    return launch_k(kern, dim3(p.NP, groups, num_seqs), dim3(p.HPC * 32), smem, stream, p);
}

cudaError_t launch_attention(const AttnParams& p, int dtype, int head_dim, int num_seqs, size_t smem,
                             cudaStream_t stream) {
    if (dtype == 0) {
        return head_dim == 64 ? launch_attention_t<float, 64>(p, num_seqs, smem, stream)
                              : launch_attention_t<float, 128>(p, num_seqs, smem, stream);
    } else if (dtype == 1) {
        return head_dim == 64 ? launch_attention_t<__half, 64>(p, num_seqs, smem, stream)
                              : launch_attention_t<__half, 128>(p, num_seqs, smem, stream);
    }
    return head_dim == 64 ? launch_attention_t<__nv_bfloat16, 64>(p, num_seqs, smem, stream)
                          : launch_attention_t<__nv_bfloat16, 128>(p, num_seqs, smem, stream);
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
