// pa_internal.h -- host/device interface between the C ABI layer and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <utility>

#include "../../include/pa.h"

namespace pa {

// Multi-token causal attention over the paged cache (pa_prefill.cu, N4).  TMA tensor maps
// are built by the host for every call (they hold the tensors' base addresses).
struct PrefillParams {
    CUtensorMap tmap_q;           // query [T][H][D], box {64, 1, 128}, 128-byte swizzle
    CUtensorMap tmap_k;           // key cache as [NB*H_kv*B][D], box {64, box_rows}
    CUtensorMap tmap_v;           // value cache, same
    CUtensorMap tmap_k1;          // key cache, box {64, 1} (tails shorter than box_rows)
    CUtensorMap tmap_v1;          // value cache, box {64, 1}
    CUtensorMap tmap_kr[3];       // key cache, boxes {64, 8 >> i} (packed kernel: partial pieces)
    CUtensorMap tmap_vr[3];       // value cache, same
    void* out;                    // [T][H][D]
    const int32_t* block_tables;  // [S][W]
    const int32_t* context_lens;  // [S]
    const int32_t* query_start;   // [S+1]
    float scale_log2;
    int log2B, H, H_kv, G, W;
    int box_rows;                 // min(block_size, 128) tokens per TMA box
    int X, S;                     // query-tile pairs per sequence (grid of work items), sequences
    int* work_counter;            // v2: dynamic work-item counter (zeroed on the stream by the launcher)
};

// Packed prompt-phase work (N4, pa_paged_prefill_attention_packed): query tile t holds <= 128
// query rows of sequences s0[t] .. s0[t] + nm[t] - 1 (consecutive), starting at row r0[t] of
// the first (r0 > 0 only when one long query spans several tiles), which share their first
// P[t] cached tokens (the same physical blocks; P a multiple of the block size, at most
// every member's first query position).
constexpr int kMaxPackTiles = 1024;
struct PackTable {
    int n_tiles;
    int s0[kMaxPackTiles];
    int P[kMaxPackTiles];
    uint16_t nm[kMaxPackTiles];
    uint16_t r0[kMaxPackTiles];
};

constexpr int kMaxTpPeers = 8;
constexpr int kMaxSeqOrder = PA_MAX_SEQ_ORDER;  // longest-first grid order carried in the kernel parameters

struct AttnParams {
    void* out;                  // [S][H][D]
    const void* query;          // [S][H][D]
    const void* key_cache;      // [NB][H_kv][B][D]
    const void* value_cache;    // [NB][H_kv][B][D]
    const int32_t* block_tables;  // [S][W]
    const int32_t* context_lens;  // [S]
    const void* new_key;        // [S][H_kv][D] this step's token (fused decode entry) or NULL
    const void* new_value;
    void* key_cache_w;          // writable aliases of the caches (fused decode entry)
    void* value_cache_w;
    float2* part_ml;            // [S][H][NP] (m, L) in the exp2 domain (split only)
    float* part_o;              // [S][H][NP][D] normalised partial outputs (split only)
    unsigned long long* counters;  // [S][H] split completion words (epoch << 32 | partitions done);
                                   // never zeroed by the host: see split_arrive (pa_attention.cu)
    uint32_t epoch;             // this launch's nonzero 32-bit tag for the completion words
    float scale_log2;           // scale * log2(e)
    int log2B;                  // block_size = 1 << log2B
    int H, H_kv, G;             // query heads, kv heads, H / H_kv
    int W;                      // block table row stride
    int PT;                     // partition size in tokens (multiple of 16)
    int NP;                     // partitions in the grid = ceil(max_ctx / PT)
    int HPC;                    // warps per CTA
    int PPC;                    // coop scheduler: partitions walked by one CTA (scheduling only)
    int GM;                     // sharing-aware scheduler: sequences per group
    int S;                      // number of sequences
    int pz;                     // coop: grid (head group, sequence, partition), partitions slowest
    int STG;                    // tiles in flight per warp (shared-memory stages)
    int GSL;                    // grouped / shared decode: block slots per stage (a tile with more distinct
                                // blocks than GSL takes several stages)
    // fused tensor-parallel all-gather (N2): when n_out_peers > 0 every output row of local
    // head h is stored to out_peers[k] + ((s * out_H) + out_h0 + h) * D for every rank k
    // (peer memory over NVLink) instead of `out`
    int n_out_peers;
    int out_H, out_h0;
    void* out_peers[kMaxTpPeers];
    // grid order (scheduling only, pa_decode_plan): the CTAs of grid sequence slot z work on
    // sequence seq_order[z] when z < n_order (longest contexts first, so the long CTAs do
    // not start in the last wave); kernel parameters, so no extra memory round trip
    int n_order;
    uint16_t seq_order[kMaxSeqOrder];
};

// Sharing-aware decode on the tcgen05 tensor cores (N1, pa_paged_attention_decode_grouped,
// pa_decode_tc.cu).  TMA tensor maps are built by the host for every call.
struct GroupTcParams {
    CUtensorMap tmap_kq;     // key cache as [NB*H_kv*B rows][D], box {64 cols, 64 rows}: a 16-row
                             // piece of four adjacent kv heads (consecutive in a B = 16 block), one half
    CUtensorMap tmap_vq;     // value cache, same
    CUtensorMap tmap_k[5];   // key cache as [NB*H_kv*B rows][D], boxes {64 cols, 16 >> i rows}, 128-B swizzle
    CUtensorMap tmap_v[5];   // value cache, same
    CUtensorMap tmap_nk;     // the step's new key as [S*H_kv rows][D], box {64, 1}
    CUtensorMap tmap_nv;     // new value, same
    void* out;               // [S][H][D]
    const void* query;       // [S][H][D] (rows copied into tensor memory by the softmax warps)
    void* key_cache;         // writable cache bases (the new token's row is stored by the kernel)
    void* value_cache;
    const void* new_key;     // [S][H_kv][D]
    const void* new_value;
    const int32_t* block_tables;  // [S][W]
    const int32_t* context_lens;  // [S]
    unsigned long long* work_counter;  // 8 bytes of workspace: (epoch << 32 | items handed out)
    unsigned long long* counters;      // [S*H] split-context completion words (epoch-tagged)
    float* part_o;                     // [S][H][NPt][128] O / L of each part
    float2* part_ml;                   // [S][H][NPt] (m, L) of each part, exp2 domain
    int NPt;                           // parts per group (split context; the last part to the end)
    int part_log;                      // a part = 1 << part_log 16-token positions (4: 256 tokens, 5: 512)
    uint32_t epoch;
    float scale_log2;
    int log2B, H, H_kv, G, W, S;
    int GM;                  // sequences per group (<= 8)
    int n_hp, n_items;       // head quads per group, work items = groups x head quads
    int n_gorder;            // > 0: work items walk the groups in gorder (pa_decode_plan's order,
    uint16_t gorder[kMaxSeqOrder];  // by each group's first appearance; scheduling only)
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

struct SwapBlocksParams {
    void* dst_key[kMaxLayers];
    void* dst_value[kMaxLayers];
    const void* src_key[kMaxLayers];
    const void* src_value[kMaxLayers];
    const int64_t* block_mapping;
    int64_t block_bytes;
};

void count_launch();
bool pdl_enabled();  // PA_PDL=0 (read once at load) disables programmatic dependent launch
uint32_t next_epoch();  // nonzero, scrambled per-launch tag for split completion words
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device), thread-safe
cudaError_t ensure_smem_attr(const void* kern, size_t smem);

// Launch `kern` on `stream`, with programmatic stream serialisation when enabled.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                     Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int attention_row_bytes(int dtype, int head_dim);
size_t attention_smem_bytes_coop(int row_bytes, int hpc, int G, int stg, int partition_tokens, int block_size,
                                 int ppc, int head_dim);
size_t attention_smem_bytes_shared(int row_bytes, int hpc, int G, int stg, int gm, int nsl);
// sched: 2 = coop (default), 4 = sharing-aware groups of GM sequences
cudaError_t launch_attention(const AttnParams& p, int dtype, int head_dim, int num_seqs, int sched, size_t smem,
                             cudaStream_t stream);
size_t group_tc_smem_bytes();
cudaError_t launch_group_tc(const GroupTcParams& p, int dtype, cudaStream_t stream);
// variant: 0 = by max_query_len (default), 2 / 3 = force (PA_PREFILL ablation)
cudaError_t launch_prefill(const PrefillParams& p, int dtype, int num_seqs, int max_query_len, int variant,
                           cudaStream_t stream);
cudaError_t launch_prefill_packed(const PrefillParams& p, const PackTable& t, int dtype, cudaStream_t stream);
// v7: two 128-row query tiles per item (tables packed with <= 256 rows per tile)
cudaError_t launch_prefill_packed2(const PrefillParams& p, const PackTable& t, int dtype, cudaStream_t stream);
// N2: rank `rank` publishes `epoch` to every peer's flag array, then waits (bounded) until
// every peer has published it to this rank; status = 1 on timeout
cudaError_t launch_tp_signal_wait(int32_t* const* flag_peers, int world, int rank, int32_t epoch, int32_t* status,
                                  long long timeout_ns, cudaStream_t stream);
cudaError_t launch_debug_gather(const GatherParams& p, int dtype, int head_dim, int num_seqs, cudaStream_t stream);
cudaError_t launch_reshape_and_cache(const CacheWriteParams& p, cudaStream_t stream);
cudaError_t launch_copy_blocks(const CopyBlocksParams& p, int num_layers, int num_pairs, cudaStream_t stream);
cudaError_t launch_swap_blocks(const SwapBlocksParams& p, int num_layers, int num_pairs, cudaStream_t stream);
cudaError_t launch_hbm_read_probe(const void* buf, int64_t nchunks, int chunk, int stages, int grid, uint32_t* sink,
                                  cudaStream_t stream);
cudaError_t launch_validate_tables(const int32_t* bt, const int32_t* ctx, int S, int W, int B, int NB,
                                   unsigned long long* d_first_bad, cudaStream_t stream);

}  // namespace pa
