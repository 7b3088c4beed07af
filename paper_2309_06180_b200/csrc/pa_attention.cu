// pa_attention.cu -- PagedAttention decode kernels for B200 (sm_100a).
//
// Eq.4 of the paper: for every (sequence s, query head h) the kernel walks
// the sequence's logical tokens through its block table, computes
// l_t = scale * q.K_t, a numerically stable softmax and sum_t softmax_t * V_t.
//
// B200 design:
//  * One CTA per (partition, head, sequence); NW warps, each an independent consumer of
//    16-token LOGICAL tiles i = warp, warp+NW, ... of the partition (the compute never
//    depends on block_size, physical placement or grid shape -> bitwise invariance).
//  * Tiles are staged into shared memory by 1-D bulk async copies (cp.async.bulk,
//    SASS UBLKCP) completing on a per-stage mbarrier; each warp keeps STG tiles in flight
//    (lane 0 issues; for block_size < 16 lanes issue one piece each).  The partition's
//    block ids are prefetched into shared memory first, so no copy waits on a dependent
//    global load (the paper's "extra overhead of accessing the block table").
//  * Lane mapping: a K/V row of RB = D*e bytes is covered by LT = RB/32 lanes, each
//    owning two 16-byte chunks (c and c+LT: conflict-free 128-byte phases); a warp
//    handles TG = 32/LT tokens at once.  q.k uses the sm_100 mixed-precision FMA
//    (FHFMA, f16/bf16 x f16/bf16 + f32) straight from the packed storage dtype; the
//    dot product is reduced with warp shuffles across the LT lanes.  Each token group
//    keeps its own online-softmax state (m, l, acc[]) in the exp2 domain, and p*V is
//    accumulated with packed fp32x2 FMAs (FFMA2).  No tensor cores: a one-query decode
//    step is a memory-bound GEMV (BJ:north_star).
//  * End of CTA: token groups merge by shuffles, warps through shared memory (log-sum-
//    exp, fixed order).  A sequence whose context fits one partition writes `out`
//    directly; otherwise each partition writes (m, L, o~) and paged_attention_reduce
//    merges them (split-context variant, BJ:north_star).
#include "pa_common.cuh"
#include "pa_internal.h"

#include <cfloat>

namespace pa {

template <typename T, int D, int NW, int STG>
struct AttnCfg {
    static constexpr int E = Elem<T>::kBytes;
    static constexpr int RB = D * E;         // bytes per K/V row
    static constexpr int NCH = RB / 16;      // 16-byte chunks per row
    static constexpr int LT = NCH / 2;       // lanes per token (2 chunks each)
    static constexpr int TG = 32 / LT;       // tokens per warp step (token groups)
    static constexpr int TPL = kTile / TG;   // tokens per lane per tile
    static constexpr int EPC = 16 / E;       // elements per chunk
    static constexpr int STAGE_BYTES = 2 * kTile * RB;
    static constexpr int STAGES_BYTES = NW * STG * STAGE_BYTES;
    static_assert(LT >= 1 && LT <= 16 && TG * LT == 32, "row must span 2..32 lanes");
    static_assert(TPL >= 1 && TPL * TG == kTile, "tile must split evenly over token groups");
};

// Shared-memory footprint of the attention kernel (host + device).
template <typename T, int D, int NW, int STG>
__host__ __device__ constexpr size_t attn_fixed_smem() {
    using C = AttnCfg<T, D, NW, STG>;
    // stages | mbarriers | reduction scratch (NW*D acc + NW m + NW l)
    return (size_t)C::STAGES_BYTES + 8 * NW * STG + 4 * (NW * D + 2 * NW);
}

// Issue the bulk copies of logical tile `tok0` (nv valid tokens, nv <= 16) of kv head
// `kvh` into (sK, sV).  sbt holds the block ids of logical blocks jb0, jb0+1, ...
// Called by a whole warp (lanes 0..pieces-1 issue).
__device__ __forceinline__ void issue_tile(char* sK, char* sV, uint64_t* bar, const char* kc, const char* vc,
                                           const int* sbt, int jb0, int tok0, int nv, int p1, int log2B,
                                           int64_t blk_stride, int64_t head_off, int RB, int lane) {
    const int B = 1 << log2B;
    if (B >= kTile) {
        if (lane == 0) {
            const int blk = sbt[(tok0 >> log2B) - jb0];
            const int64_t off = (int64_t)blk * blk_stride + head_off + (int64_t)(tok0 & (B - 1)) * RB;
            const uint32_t bytes = (uint32_t)(nv * RB);
            mbar_arrive_expect_tx(bar, 2 * bytes);
            bulk_g2s(sK, kc + off, bytes, bar);
            bulk_g2s(sV, vc + off, bytes, bar);
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
}

template <typename T, int D, int NW, int STG>
__global__ void __launch_bounds__(NW * 32)
paged_attention_kernel(const AttnParams p) {
    using C = AttnCfg<T, D, NW, STG>;
    constexpr int RB = C::RB, LT = C::LT, TG = C::TG, TPL = C::TPL, EPC = C::EPC;
    extern __shared__ __align__(128) unsigned char smem[];

    const int part = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ctx = p.context_lens[s];
    const int p0 = part * p.PT;
    if (part > 0 && p0 >= ctx) return;  // this sequence has fewer partitions
    const int p1 = min(ctx, p0 + p.PT);
    const int ntiles = p1 > p0 ? (p1 - p0 + kTile - 1) / kTile : 0;
    const int nparts = ctx > 0 ? (ctx + p.PT - 1) / p.PT : 1;
    const int kvh = h / p.G;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES_BYTES);
    float* red = reinterpret_cast<float*>(bars + NW * STG);  // [NW][D] acc, [NW] m, [NW] l
    float* red_m = red + NW * D;
    float* red_l = red_m + NW;
    int* sbt = reinterpret_cast<int*>(red_l + NW);

    // ---- prologue: block ids of this partition, barriers ---------------------------
    const int jb0 = p0 >> p.log2B;
    const int nb = ntiles ? ((p1 - 1) >> p.log2B) - jb0 + 1 : 0;
    const int32_t* btrow = p.block_tables + (int64_t)s * p.W;
    for (int i = threadIdx.x; i < nb; i += NW * 32) sbt[i] = __ldg(btrow + jb0 + i);
    if (threadIdx.x < NW * STG) mbar_init(&bars[threadIdx.x], 1);
    fence_mbar_init();

    // q chunks of this lane (storage dtype, registers)
    const int g = lane / LT, c = lane % LT;
    const uint4* qrow = reinterpret_cast<const uint4*>(static_cast<const char*>(p.query) +
                                                        ((int64_t)s * p.H + h) * RB);
    const uint4 q0 = __ldg(qrow + c), q1 = __ldg(qrow + c + LT);
    __syncthreads();

    const char* kc = static_cast<const char*>(p.key_cache);
    const char* vc = static_cast<const char*>(p.value_cache);
    const int64_t blk_stride = (int64_t)p.H_kv << p.log2B;  // rows per physical block
    const int64_t head_off = ((int64_t)kvh << p.log2B) * RB;
    char* stage0 = reinterpret_cast<char*>(smem) + warp * STG * C::STAGE_BYTES;
    uint64_t* wbars = bars + warp * STG;

    const int my_n = ntiles > warp ? (ntiles - warp + NW - 1) / NW : 0;
#pragma unroll
    for (int j = 0; j < STG; ++j) {
        if (j < my_n) {
            const int tok0 = p0 + (warp + j * NW) * kTile;
            issue_tile(stage0 + j * C::STAGE_BYTES, stage0 + j * C::STAGE_BYTES + kTile * RB, &wbars[j], kc, vc,
                       sbt, jb0, tok0, min(kTile, p1 - tok0), p1, p.log2B, blk_stride * RB, head_off, RB, lane);
        }
    }

    float m = -INFINITY, l = 0.f;
    float2 acc[EPC];
#pragma unroll
    for (int e = 0; e < EPC; ++e) acc[e] = make_float2(0.f, 0.f);

    int k = 0;
    uint32_t phase = 0;
    for (int j = 0; j < my_n; ++j) {
        const int tok0 = p0 + (warp + j * NW) * kTile;
        const int nv = min(kTile, p1 - tok0);
        const char* sK = stage0 + k * C::STAGE_BYTES;
        const char* sV = sK + kTile * RB;
        mbar_wait(&wbars[k], phase);

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
                if (jj * TG + g < nv) {  // never touch rows past the context (reading c3)
                    const char* row = sV + (jj * TG + g) * RB;
                    const uint4 v0 = lds128(row + c * 16), v1 = lds128(row + (c + LT) * 16);
                    axpy16<T>(acc, ps[jj], v0);
                    axpy16<T>(acc + EPC / 2, ps[jj], v1);
                }
            }
        }
        m = mn;
        __syncwarp();
        if (j + STG < my_n) {
            const int t2 = p0 + (warp + (j + STG) * NW) * kTile;
            issue_tile(stage0 + k * C::STAGE_BYTES, stage0 + k * C::STAGE_BYTES + kTile * RB, &wbars[k], kc, vc, sbt,
                       jb0, t2, min(kTile, p1 - t2), p1, p.log2B, blk_stride * RB, head_off, RB, lane);
        }
        if (++k == STG) {
            k = 0;
            phase ^= 1u;
        }
    }

    // ---- merge token groups inside the warp (log-sum-exp, fixed order) -------------
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
    if (g == 0) {
        float* dst = red + warp * D;
#pragma unroll
        for (int e = 0; e < EPC / 2; ++e) {
            dst[c * EPC + 2 * e] = acc[e].x;
            dst[c * EPC + 2 * e + 1] = acc[e].y;
            dst[(c + LT) * EPC + 2 * e] = acc[EPC / 2 + e].x;
            dst[(c + LT) * EPC + 2 * e + 1] = acc[EPC / 2 + e].y;
        }
        if (lane == 0) {
            red_m[warp] = m;
            red_l[warp] = l;
        }
    }
    __syncthreads();

    // ---- merge warps, write the output or this partition's (m, L, o~) --------------
    float M = red_m[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) M = fmaxf(M, red_m[w]);
    const float Ms = (M == -INFINITY) ? 0.f : M;
    float wgt[NW];
    float L = 0.f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        wgt[w] = ex2(red_m[w] - Ms);
        L += red_l[w] * wgt[w];
    }
    const int64_t sh = (int64_t)s * p.H + h;
    for (int d = threadIdx.x; d < D; d += NW * 32) {
        float o = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) o += red[w * D + d] * wgt[w];
        if (nparts == 1) {
            static_cast<T*>(p.out)[sh * D + d] = Elem<T>::from_f32(L > 0.f ? o / L : 0.f);
        } else {
            p.part_o[(sh * p.NP + part) * D + d] = o / L;
        }
    }
    if (nparts > 1 && threadIdx.x == 0) p.part_ml[sh * p.NP + part] = make_float2(M, L);
}

// Log-sum-exp merge of the partitions (split-context variant):
//   M = max m_p;  out = sum_p 2^(m_p - M) L_p o~_p / sum_p 2^(m_p - M) L_p
template <typename T, int D>
__global__ void __launch_bounds__(128) paged_attention_reduce_kernel(const AttnParams p) {
    const int h = blockIdx.x, s = blockIdx.y;
    const int ctx = p.context_lens[s];
    int nparts = ctx > 0 ? (ctx + p.PT - 1) / p.PT : 1;
    if (nparts <= 1) return;
    nparts = min(nparts, p.NP);
    const int64_t sh = (int64_t)s * p.H + h;
    const float2* ml = p.part_ml + sh * p.NP;
    __shared__ float w_s[64];
    __shared__ float invL_s;
    float M = -INFINITY;
    for (int i = 0; i < nparts; ++i) M = fmaxf(M, ml[i].x);
    if (threadIdx.x == 0) {
        float L = 0.f;
        for (int i = 0; i < nparts; ++i) L += ml[i].y * ex2(ml[i].x - M);
        invL_s = L;
    }
    for (int i = threadIdx.x; i < nparts && i < 64; i += blockDim.x) w_s[i] = ml[i].y * ex2(ml[i].x - M);
    __syncthreads();
    const float L = invL_s;
    const float* po = p.part_o + sh * p.NP * D;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        float o = 0.f;
        for (int i = 0; i < nparts; ++i) o += (i < 64 ? w_s[i] : ml[i].y * ex2(ml[i].x - M)) * po[(int64_t)i * D + d];
        static_cast<T*>(p.out)[sh * D + d] = Elem<T>::from_f32(o / L);
    }
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

template <typename T, int D>
struct AttnVariant {
    static constexpr int NW = 4;
    static constexpr int RB = D * Elem<T>::kBytes;
    static constexpr int STG = RB <= 128 ? 6 : (RB <= 256 ? 3 : 2);
};

size_t attention_smem_bytes(int dtype, int head_dim, int partition_tokens, int block_size) {
    size_t fixed = 0;
#define PA_SMEM_CASE(TT, DD)                                                                   \
    fixed = attn_fixed_smem<TT, DD, AttnVariant<TT, DD>::NW, AttnVariant<TT, DD>::STG>();
    if (dtype == 0 && head_dim == 64) { PA_SMEM_CASE(float, 64) }
    else if (dtype == 0) { PA_SMEM_CASE(float, 128) }
    else if (dtype == 1 && head_dim == 64) { PA_SMEM_CASE(__half, 64) }
    else if (dtype == 1) { PA_SMEM_CASE(__half, 128) }
    else if (head_dim == 64) { PA_SMEM_CASE(__nv_bfloat16, 64) }
    else { PA_SMEM_CASE(__nv_bfloat16, 128) }
#undef PA_SMEM_CASE
    const size_t tbl = 4 * (size_t)(partition_tokens / block_size + 2);
    return fixed + tbl;
}

template <typename T, int D>
static cudaError_t launch_attention_t(const AttnParams& p, int num_seqs, int num_heads, size_t smem,
                                      cudaStream_t stream) {
    using V = AttnVariant<T, D>;
    auto kern = paged_attention_kernel<T, D, V::NW, V::STG>;
    static size_t configured = 0;  // per instantiation; smem size only grows
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    dim3 grid(p.NP, num_heads, num_seqs);
    kern<<<grid, V::NW * 32, smem, stream>>>(p);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || p.NP <= 1) return e;
    paged_attention_reduce_kernel<T, D><<<dim3(num_heads, num_seqs), 128, 0, stream>>>(p);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_attention(const AttnParams& p, int dtype, int head_dim, int num_seqs, int num_heads,
                             cudaStream_t stream) {
    const size_t smem = attention_smem_bytes(dtype, head_dim, p.PT, 1 << p.log2B);
    if (dtype == 0) {
        return head_dim == 64 ? launch_attention_t<float, 64>(p, num_seqs, num_heads, smem, stream)
                              : launch_attention_t<float, 128>(p, num_seqs, num_heads, smem, stream);
    } else if (dtype == 1) {
        return head_dim == 64 ? launch_attention_t<__half, 64>(p, num_seqs, num_heads, smem, stream)
                              : launch_attention_t<__half, 128>(p, num_seqs, num_heads, smem, stream);
    }
    return head_dim == 64 ? launch_attention_t<__nv_bfloat16, 64>(p, num_seqs, num_heads, smem, stream)
                          : launch_attention_t<__nv_bfloat16, 128>(p, num_seqs, num_heads, smem, stream);
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
