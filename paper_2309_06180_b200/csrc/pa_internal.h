// pa_internal.h -- host/device interface between the C ABI layer and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace pa {

struct AttnParams {
    void* out;                  // [S][H][D]
    const void* query;          // [S][H][D]
    const void* key_cache;      // [NB][H_kv][B][D]
    const void* value_cache;    // [NB][H_kv][B][D]
    const int32_t* block_tables;  // [S][W]
    const int32_t* context_lens;  // [S]
    float2* part_ml;            // [S][H][NP] (m, L) in the exp2 domain (split only)
    float* part_o;              // [S][H][NP][D] normalised partial outputs (split only)
    float scale_log2;           // scale * log2(e)
    int log2B;                  // block_size = 1 << log2B
    int H, H_kv, G;             // query heads, kv heads, H / H_kv
    int W;                      // block table row stride
    int PT;                     // partition size in tokens (multiple of 16)
    int NP;                     // partitions in the grid = ceil(max_ctx / PT)
};

struct GatherParams {
    void* k_out;
    void* v_out;
    const void* key_cache;
    const void* value_cache;
    const int32_t* block_tables;
    const int32_t* context_lens;
    int log2B, H_kv, W, max_ctx;
};

struct CacheWriteParams {
    const void* key;
    const void* value;
    void* key_cache;
    void* value_cache;
    const int64_t* slot_mapping;
    int num_tokens, H_kv, row_bytes, log2B;
};

constexpr int kMaxLayers = 256;
struct CopyBlocksParams {
    void* key_caches[kMaxLayers];
    void* value_caches[kMaxLayers];
    const int64_t* block_mapping;
    int64_t block_bytes;
};

void count_launch();

size_t attention_smem_bytes(int dtype, int head_dim, int partition_tokens, int block_size);
cudaError_t launch_attention(const AttnParams& p, int dtype, int head_dim, int num_seqs, int num_heads,
                             cudaStream_t stream);
cudaError_t launch_debug_gather(const GatherParams& p, int dtype, int head_dim, int num_seqs, cudaStream_t stream);
cudaError_t launch_reshape_and_cache(const CacheWriteParams& p, cudaStream_t stream);
cudaError_t launch_copy_blocks(const CopyBlocksParams& p, int num_layers, int num_pairs, cudaStream_t stream);
cudaError_t launch_validate_tables(const int32_t* bt, const int32_t* ctx, int S, int W, int B, int NB,
                                   unsigned long long* d_first_bad, cudaStream_t stream);

}  // namespace pa
