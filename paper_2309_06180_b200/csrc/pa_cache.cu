// pa_cache.cu -- the two kernels that maintain the paged KV cache (sm_100a).
//
//  reshape_and_cache  fused reshape + block write: each new token's K/V row
//                     per kv head goes to (slot / B, head, slot % B) of the
//                     [NB][H_kv][B][D] cache; 16-byte vector copies, bit-exact.
//  copy_blocks        fused block copy: every copy-on-write (src, dst) pair
//                     of every layer in ONE launch instead of many cudaMemcpyAsync calls.
//  swap_blocks        block transfers between pools (GPU <-> pinned CPU memory),
//                     one launch for every pair and layer; host memory is read/written
//                     over the host link directly (mapped pinned memory).
//  validate_tables    test helper: block ids in range, ctx <= W*B.
#include "pa_common.cuh"
#include "pa_internal.h"

namespace pa {

// One CTA per token; 256 threads issue all of the token's 16-byte loads (K and V, every
// kv head) before any store so each thread has several requests in flight.
__global__ void __launch_bounds__(256) reshape_and_cache_kernel(const CacheWriteParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const int i = blockIdx.x;
    const int64_t slot = p.slot_mapping[i];
    if (slot < 0) return;  // padding token (reading c11)
    const int64_t b = slot >> p.log2B;
    const int o = (int)(slot & ((1 << p.log2B) - 1));
    const int cpr = p.row_bytes >> 4;  // 16-byte chunks per row
    const int nvec = p.H_kv * cpr;
    const uint4* ks = static_cast<const uint4*>(p.key) + (int64_t)i * nvec;
    const uint4* vs = static_cast<const uint4*>(p.value) + (int64_t)i * nvec;
    uint4* kc = static_cast<uint4*>(p.key_cache);
    uint4* vc = static_cast<uint4*>(p.value_cache);
    constexpr int U = 4;
    for (int v0 = threadIdx.x; v0 < nvec; v0 += U * 256) {
        uint4 kr[U], vr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * 256;
            if (v < nvec) {
                kr[u] = __ldg(ks + v);
                vr[u] = __ldg(vs + v);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + u * 256;
            if (v < nvec) {
                const int h = v / cpr, cc = v - h * cpr;
                const int64_t dst = ((((b * p.H_kv + h) << p.log2B) + o) * cpr) + cc;
                kc[dst] = kr[u];
                vc[dst] = vr[u];
            }
        }
    }
}

__global__ void __launch_bounds__(256) copy_blocks_kernel(const __grid_constant__ CopyBlocksParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const int pair = blockIdx.x, layer = blockIdx.y, which = blockIdx.z;
    const int64_t src = p.block_mapping[2 * pair], dst = p.block_mapping[2 * pair + 1];
    char* base = static_cast<char*>(which == 0 ? p.key_caches[layer] : p.value_caches[layer]);
    const uint4* s = reinterpret_cast<const uint4*>(base + src * p.block_bytes);
    uint4* d = reinterpret_cast<uint4*>(base + dst * p.block_bytes);
    const int n = (int)(p.block_bytes >> 4);
    constexpr int U = 4;
    int i = threadIdx.x;
    for (; i + (U - 1) * 256 < n; i += U * 256) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = s[i + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u) d[i + u * 256] = r[u];
    }
    for (; i < n; i += 256) d[i] = s[i];
}

// Codes are row-major over (row s, position 0 = ctx, 1 + j = entry j) so atomicMin
// yields the first problem in row order; entries of a row with a bad ctx are skipped.
__global__ void __launch_bounds__(256) swap_blocks_kernel(const __grid_constant__ SwapBlocksParams p) {
    pdl_launch_dependents();
    pdl_wait();
    const int pair = blockIdx.x, layer = blockIdx.y, which = blockIdx.z;
    const int64_t src = p.block_mapping[2 * pair], dst = p.block_mapping[2 * pair + 1];
    const char* sb = static_cast<const char*>(which == 0 ? p.src_key[layer] : p.src_value[layer]);
    char* db = static_cast<char*>(which == 0 ? p.dst_key[layer] : p.dst_value[layer]);
    const uint4* s = reinterpret_cast<const uint4*>(sb + src * p.block_bytes);
    uint4* d = reinterpret_cast<uint4*>(db + dst * p.block_bytes);
    const int n = (int)(p.block_bytes >> 4);
    constexpr int U = 8;  // host-link latency is long: more 16-byte requests in flight per thread
    int i = threadIdx.x;
    for (; i + (U - 1) * 256 < n; i += U * 256) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = s[i + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u) d[i + u * 256] = r[u];
    }
    for (; i < n; i += 256) d[i] = s[i];
}

__global__ void validate_tables_kernel(const int32_t* bt, const int32_t* ctx, int S, int W, int B, int NB,
                                       unsigned long long* first_bad) {
    const int64_t total = (int64_t)S * W;
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < total; f += (int64_t)gridDim.x * blockDim.x) {
        const int s = (int)(f / W), j = (int)(f % W);
        const int n = ctx[s];
        const bool bad_ctx = n < 0 || (int64_t)n > (int64_t)W * B;
        unsigned long long code = ~0ull;
        if (bad_ctx) {
            if (j == 0) code = (unsigned long long)s * (W + 1);
        } else if ((int64_t)j * B < n) {
            const int b = bt[f];
            if (b < 0 || b >= NB) code = (unsigned long long)s * (W + 1) + 1 + j;
        }
        if (code != ~0ull) atomicMin(first_bad, code);
    }
}

cudaError_t launch_reshape_and_cache(const CacheWriteParams& p, cudaStream_t stream) {
    return launch_k(reshape_and_cache_kernel, dim3(p.num_tokens), dim3(256), 0, stream, p);
}

cudaError_t launch_copy_blocks(const CopyBlocksParams& p, int num_layers, int num_pairs, cudaStream_t stream) {
    return launch_k(copy_blocks_kernel, dim3(num_pairs, num_layers, 2), dim3(256), 0, stream, p);
}

cudaError_t launch_swap_blocks(const SwapBlocksParams& p, int num_layers, int num_pairs, cudaStream_t stream) {
    return launch_k(swap_blocks_kernel, dim3(num_pairs, num_layers, 2), dim3(256), 0, stream, p);
}

cudaError_t launch_validate_tables(const int32_t* bt, const int32_t* ctx, int S, int W, int B, int NB,
                                   unsigned long long* d_first_bad, cudaStream_t stream) {
    validate_tables_kernel<<<148, 256, 0, stream>>>(bt, ctx, S, W, B, NB, d_first_bad);
    count_launch();
    return cudaGetLastError();
}

}  // namespace pa
