/*
 * pa.h -- C ABI of libpagedattn.so, the B200 (sm_100a) PagedAttention decode hot path.
 *
 * Paper: Kwon et al., "Efficient Memory Management for Large Language Model Serving
 * with PagedAttention", SOSP'23 (arXiv 2309.06180).  P:N = PAPER.md line N.
 *
 * Conventions for every entry point
 *  - Tensor pointers are DEVICE pointers owned by the caller unless a parameter says
 *    HOST.  The library never allocates or frees device memory on these calls and
 *    never synchronises the stream (except the pa_debug_* / pa_validate_* helpers and
 *    pa_decode_step's documented D2H copy, which is stream-ordered).
 *  - Element type of query/out/key/value/caches is `dtype` (fp32, fp16 or bf16);
 *    arithmetic is fp32 with round-to-nearest-even output.
 *  - KV cache layout ("optimized for block read"; reading c7):
 *        key_cache, value_cache: [num_blocks][num_kv_heads][block_size][head_dim]
 *    so one (block, kv head) chunk is block_size*head_dim contiguous elements.
 *  - block_tables: int32 [num_seqs][max_blocks_per_seq] row-major (row stride W);
 *    entry j < ceil(ctx/B) of row s is the physical block of logical block j
 *    (P:254-256).  Entries beyond are never read.  context_lens: int32 [num_seqs],
 *    the number of tokens INCLUDING the current one (written before attention).
 *  - Errors are detected on the host before any launch and returned as a status;
 *    pa_last_error() gives a thread-local message.  Checked: null pointers, 16-byte
 *    alignment of every tensor pointer, dims <= 0, num_heads % num_kv_heads,
 *    head_dim in {64, 128}, block_size a power of two in [1, 256], workspace size.
 *    Device-side contract violations (a block id outside [0, num_blocks), ctx >
 *    W*block_size, repeated slots) are undefined behaviour; pa_validate_tables()
 *    checks them in tests.  A failed launch returns PA_ERR_CUDA.
 */
#ifndef PAGED_ATTN_PA_H_
#define PAGED_ATTN_PA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pa_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum { PA_F32 = 0, PA_F16 = 1, PA_BF16 = 2 } pa_dtype_t;

typedef enum {
    PA_OK = 0,
    PA_ERR_INVALID_ARG = 1,
    PA_ERR_UNSUPPORTED = 2,
    PA_ERR_WORKSPACE = 3,
    PA_ERR_CUDA = 4,
    PA_ERR_OUT_OF_BLOCKS = 5
} pa_status_t;

/* Library default partition size (tokens) of the split-context variant. */
#define PA_DEFAULT_PARTITION_TOKENS 512

/* ------------------------------------------------------------------------------------
 * pa_paged_attention -- single-query decode attention over the paged KV cache.
 *
 * Eq.4: for every sequence s and query head h, with kv head
 * kvh = h / (num_heads / num_kv_heads) and n = context_lens[s]:
 *     l_t = scale * q[s][h] . K[t],   t = 0..n-1, K[t] = key_cache[bt[s][t/B]][kvh][t%B]
 *     out[s][h] = sum_t softmax(l)_t * V[t]                 (n == 0 -> out = 0)
 * out, query: [num_seqs][num_heads][head_dim].  `scale` is the caller's (1/sqrt(D)
 * in every config, reading c1).
 *
 * Contexts longer than PA_DEFAULT_PARTITION_TOKENS use the split-context variant
 * (BJ:north_star): partitions of that many logical tokens each produce (m, L, o~)
 * into `workspace`; the last partition of each (sequence, head group) to finish
 * merges them by log-sum-exp in partition order (one kernel launch per call).  The
 * partition size depends on nothing but the context length, so results are bitwise
 * identical for any batch composition, block size, physical placement or head
 * sharding.  max_context_len: host upper bound of context_lens (<= 0 -> W *
 * block_size); it only sizes the grid.  PRECONDITION: every context_lens[s] <=
 * max_context_len (a longer context is undefined behaviour: only its first
 * ceil(max_context_len / PT) partitions are attended; pass <= 0 when unsure).
 * workspace: device, >= pa_paged_attention_workspace_size(), 16-byte aligned, any
 * content, never zeroed by the call: the split-completion words carry a per-launch
 * 32-bit tag and the completing partition resets its word, so no memset node sits
 * between decode steps (that keeps the programmatic-dependent-launch chain of
 * consecutive steps intact).  Do not share one workspace between calls running
 * concurrently on different streams.  May be NULL when that size is 0.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_paged_attention(void* out, const void* query, const void* key_cache,
                               const void* value_cache, const int32_t* block_tables,
                               const int32_t* context_lens, float scale, int block_size,
                               int num_kv_heads, int num_seqs, int num_heads, int head_dim,
                               int max_blocks_per_seq, int max_context_len, pa_dtype_t dtype,
                               void* workspace, size_t workspace_bytes, pa_stream_t stream);

/* Same, with an explicit partition size in tokens (a positive multiple of 16;
 * 0 -> PA_DEFAULT_PARTITION_TOKENS; a partition size >= max_context_len runs the
 * single-pass kernel only) and an optional grid order host_seq_order (HOST int32
 * [num_seqs], a permutation of 0..num_seqs-1, e.g. from pa_decode_plan; NULL = natural
 * order; honoured when num_seqs <= PA_MAX_SEQ_ORDER, ignored above).  The order is
 * scheduling only -- which sequence's CTAs the hardware dispatches first -- and never
 * changes a result bit.  Not a permutation -> PA_ERR_INVALID_ARG. */
#define PA_MAX_SEQ_ORDER 2048
pa_status_t pa_paged_attention_ex(void* out, const void* query, const void* key_cache,
                                  const void* value_cache, const int32_t* block_tables,
                                  const int32_t* context_lens, float scale, int block_size,
                                  int num_kv_heads, int num_seqs, int num_heads, int head_dim,
                                  int max_blocks_per_seq, int max_context_len, pa_dtype_t dtype,
                                  int partition_tokens, const int32_t* host_seq_order,
                                  void* workspace, size_t workspace_bytes, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_decode_plan -- the longest-first grid order of a decode batch (scheduling only).
 * host_context_lens: HOST int32 [num_seqs]; order_out: HOST int32 [num_seqs] receives
 * the sequence indices sorted by context length, longest first (ties in index order).
 * With the natural order the CTAs of a long sequence that happens to sit at the end of
 * the batch start in the last wave and run alone (the kernel's tail); longest first they
 * start in the first wave and short sequences fill the end.  O(S log S) on the host,
 * once per decode iteration: every layer of the iteration reuses it, as it reuses the
 * block tables (the paper's scheduler already holds the lengths on the CPU).
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_decode_plan(const int32_t* host_context_lens, int num_seqs, int32_t* order_out);

/* ------------------------------------------------------------------------------------
 * pa_paged_attention_decode -- the decode step's cache write fused into the attention
 * kernel ("saves the newly generated KV cache" and attends in one pass).
 * key, value: [num_seqs][num_kv_heads][head_dim], the new token of every sequence,
 * whose logical position is context_lens[s] - 1 (so its slot is
 * block_tables[s][(ctx-1)/B]*B + (ctx-1)%B).  Equivalent to pa_reshape_and_cache with
 * that slot_mapping followed by pa_paged_attention, bit for bit: the cache receives the
 * same bytes and the output is identical.  Sequences with ctx == 0 write nothing and
 * output 0.  Default partitioning; workspace as for pa_paged_attention; host_seq_order
 * as for pa_paged_attention_ex (NULL = natural order).
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_paged_attention_decode(void* out, const void* query, const void* key,
                                      const void* value, void* key_cache, void* value_cache,
                                      const int32_t* block_tables, const int32_t* context_lens,
                                      float scale, int block_size, int num_kv_heads, int num_seqs,
                                      int num_heads, int head_dim, int max_blocks_per_seq,
                                      int max_context_len, pa_dtype_t dtype,
                                      const int32_t* host_seq_order, void* workspace,
                                      size_t workspace_bytes, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_paged_attention_decode_shared -- pa_paged_attention_decode for batches whose
 * sequences come in groups that share physical blocks (parallel sampling, beam search,
 * P:295-332).  Sequences [g*group_size, (g+1)*group_size) form group
 * g (the last group may be smaller); each distinct physical block a group reads at a
 * logical position is brought into shared memory once and used by every member.
 * Outputs and cache bytes are bit-identical to pa_paged_attention_decode; only the
 * traffic changes.  group_size in [1, 8] (larger values are processed in groups of 8;
 * 1 is the plain decode entry).  Other arguments as pa_paged_attention_decode.
 * A CTA (partition, 8/group_size query heads, one group) streams ONE distinct block per
 * shared-memory stage, so a logical tile costs one stage when the members share its
 * block and d stages when they read d different blocks: faster than the plain entry when
 * the members share most blocks (beam search, C5: 498 vs 561 us), slower when they
 * diverge (parallel samples after the fork, C3) -- the caller chooses per batch.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_paged_attention_decode_shared(void* out, const void* query, const void* key,
                                             const void* value, void* key_cache, void* value_cache,
                                             const int32_t* block_tables,
                                             const int32_t* context_lens, float scale,
                                             int block_size, int num_kv_heads, int num_seqs,
                                             int num_heads, int head_dim, int max_blocks_per_seq,
                                             int max_context_len, int group_size, pa_dtype_t dtype,
                                             void* workspace, size_t workspace_bytes,
                                             pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_paged_attention_decode_grouped -- the sharing-aware decode step
 * on the tcgen05 tensor cores.  Same grouping and arguments as
 * pa_paged_attention_decode_shared plus num_blocks (NB, rows of the caches, for the TMA
 * tensor maps) and host_seq_order (as pa_paged_attention_ex: the groups are walked in the
 * order of their first sequence in it, e.g. pa_decode_plan's longest first; NULL =
 * natural order; scheduling only).  Persistent CTAs (one per SM) take work items =
 * (group, split-context part, 4 query heads): a scheduler warp looks up the members'
 * physical blocks, keeps every DISTINCT 16-row block piece once (its owner set), and two
 * producer warps TMA-load K and V of each piece for the 4 heads (one 64-row box per tensor
 * half); S = Q K^T and O += P V run as tcgen05.mma with Q, S,
 * P and O in tensor memory -- one set of products for the 4 heads, block-diagonal by
 * lane quadrant -- each member's scores masked to the pieces it owns and its context
 * (Eq.4; sharing P:295-332).  The new token's K/V is written to its
 * cache slot before the pieces are read, as pa_paged_attention_decode leaves the cache.
 * P is rounded to the storage dtype before P V (results match the oracle within the
 * stated tolerance; not bit-identical to the CUDA-core kernels).  Supports f16/bf16,
 * head_dim 128, power-of-two block_size >= 16, group_size in [1, 8]
 * (PA_ERR_UNSUPPORTED otherwise); NB*H_kv*B < 2^31.  Split context (a6, BJ:north_star):
 * when the (group, head quad) items alone give fewer than 4 per SM, each group's context
 * is cut into parts of 512 tokens (from max_context_len, <= 0: W * B; the last part takes
 * every position past it, so a low bound costs balance, never tokens), a row with more
 * than one part is merged in part order by the part that completes it (deterministic).
 * workspace: >= pa_paged_attention_workspace_size(num_seqs, num_heads, head_dim,
 * max_context_len, 0) bytes (PA_ERR_WORKSPACE otherwise), any content: an epoch-tagged
 * work counter, epoch-tagged merge counters and the parts' partial rows; never reset by
 * the host.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_paged_attention_decode_grouped(void* out, const void* query, const void* key,
                                              const void* value, void* key_cache, void* value_cache,
                                              const int32_t* block_tables,
                                              const int32_t* context_lens, float scale,
                                              int block_size, int num_kv_heads, int num_blocks,
                                              int num_seqs, int num_heads, int head_dim,
                                              int max_blocks_per_seq, int max_context_len,
                                              int group_size, pa_dtype_t dtype,
                                              const int32_t* host_seq_order, void* workspace,
                                              size_t workspace_bytes, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_paged_prefill_attention -- multi-token causal attention over the paged cache: the
 * prompt phase, a chunk of a long prompt, or the user-specific suffix after
 * a cached shared prefix ("the prompt phase computation only needs to execute
 * on the user's task input").  SURVEY §8(f) N4; runs on the tcgen05 tensor cores.
 *
 * Sequence s owns query rows [query_start[s], query_start[s+1]) of query [T][H][D]
 * (T = num_query_tokens); its q_len new tokens are the LAST q_len of its context_lens[s]
 * cached tokens (they must already be in the cache -- pa_reshape_and_cache with the
 * multi-token slot mapping, reading c5/c22).  Row i (position p = ctx - q_len + i)
 * attends causally to tokens 0..p through block_tables (Eq.4 with n = p + 1, the
 * autoregressive mask of P:140-142):
 *     out[row][h][:] = sum_{t<=p} softmax_t(scale * q . k_t) v_t
 * Rows with p < 0 (ctx < q_len) are 0.
 *
 * out, query: [T][H][D] (16-byte aligned); caches [num_blocks][H_kv][B][D];
 * block_tables [S][max_blocks_per_seq]; context_lens [S]; query_start [S+1] int32 with
 * query_start[0] = 0, non-decreasing, query_start[S] = T; max_query_len >= every q_len
 * (sizes the grid).  All device pointers; the caller owns every buffer.  f16/bf16,
 * head_dim 128 only (PA_ERR_UNSUPPORTED otherwise).  Softmax weights are rounded to the
 * storage dtype before the P.V product.  T == 0 or S == 0 is a no-op.
 * workspace: device, >= PA_PREFILL_WORKSPACE_BYTES, 16-byte aligned, any content: the
 * call zeroes its work-item counter on `stream` (calls sharing a workspace must be
 * ordered on one stream).  Asynchronous on `stream`.
 * ---------------------------------------------------------------------------------- */
#define PA_PREFILL_WORKSPACE_BYTES 16
pa_status_t pa_paged_prefill_attention(void* out, const void* query, const void* key_cache,
                                       const void* value_cache, const int32_t* block_tables,
                                       const int32_t* context_lens, const int32_t* query_start,
                                       float scale, int block_size, int num_kv_heads,
                                       int num_blocks, int num_seqs, int num_heads, int head_dim,
                                       int max_blocks_per_seq, int num_query_tokens,
                                       int max_query_len, pa_dtype_t dtype, void* workspace,
                                       size_t workspace_bytes, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_paged_prefill_attention_packed -- pa_paged_prefill_attention for batches whose
 * requests share a cached prefix (the shared-prefix workload of P:334-338):
 * the query rows of consecutive sequences that share their first P cached tokens are
 * packed into one item of up to 256 rows (two 128-row query tiles on the tensor cores that
 * walk the same key tiles), the shared prefix is attended ONCE for all of them
 * and each row's own tokens [P, ctx) are attended causally in packed key tiles (cascade
 * attention; same results as pa_paged_prefill_attention within the tolerance, different
 * accumulation order).  Extra HOST arrays, which the scheduler already holds:
 * host_query_start [S+1] and host_context_lens [S] (copies of the device arrays), and
 * host_shared_prefix [S]: the number of leading cached tokens sequence s shares -- the
 * same physical blocks -- with sequence s-1 (0 when none; only its multiple of the block
 * size is used).  The library packs greedily in order: an item grows while it stays <= 256
 * rows and its members' own tokens past the shared prefix P (P a multiple of the block
 * size, at most every member's first query position) stay <= 256 packed key columns; a
 * query longer than 256 rows takes items of its own.  A batch whose items would each hold
 * one sequence (nothing packs) runs pa_paged_prefill_attention's kernels.  Falls back to
 * pa_paged_prefill_attention's kernels when block_size < 16 or more than 1024 tiles would
 * be needed.  Other arguments, layouts and errors as pa_paged_prefill_attention.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_paged_prefill_attention_packed(
    void* out, const void* query, const void* key_cache, const void* value_cache,
    const int32_t* block_tables, const int32_t* context_lens, const int32_t* query_start,
    const int32_t* host_query_start, const int32_t* host_context_lens,
    const int32_t* host_shared_prefix, float scale, int block_size, int num_kv_heads,
    int num_blocks, int num_seqs, int num_heads, int head_dim, int max_blocks_per_seq,
    int num_query_tokens, int max_query_len, pa_dtype_t dtype, void* workspace,
    size_t workspace_bytes, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * Fused tensor-parallel all-gather.  Rank r of `world`
 * computes heads [r*H_loc, (r+1)*H_loc) of the decode step (its own kv-head slice of the
 * caches, the same block tables on every rank) and the attention kernel stores
 * every output row straight into EVERY rank's gather buffer [S][H_total][D] (peer memory
 * over NVLink; pointers opened with pa_ipc_open_handle), then a one-warp kernel exchanges
 * completion flags: no NCCL call, no permute.
 *
 * pa_tp_comm_create: gather_a/gather_b/flags are HOST arrays of `world` DEVICE pointers
 * as seen from this process (index k = rank k's buffer: gather buffers of
 * gather_bytes >= S*H_total*D*e bytes each, 16-byte aligned; flag arrays int32[world],
 * zero-initialised before first use);
 * status: this rank's device int32, set to 1 if a flag wait times out (PA_TP_TIMEOUT_MS,
 * default 10000) instead of hanging.  Returns NULL on invalid arguments (pa_last_error).
 * The comm does not own any buffer.
 *
 * pa_paged_attention_decode_tp: arguments as pa_paged_attention_decode with the LOCAL
 * head counts (num_heads * world == num_heads_total).  Calls alternate between the two
 * gather buffers; *buffer_out (0 = gather_a, 1 = gather_b) names the one holding this
 * call's full [S][H_total][D] output once the stream reaches the end of the call.  A
 * result is valid until this rank issues its NEXT call: reads of it must be enqueued on
 * `stream` before that call (a peer's call after next may overwrite the buffer as soon
 * as this rank's next call has published its flags).  Every rank must make the same
 * sequence of calls.  Output bits equal the single-GPU decode's.  Returns
 * PA_ERR_INVALID_ARG if num_seqs*H_total*head_dim*e exceeds gather_bytes or the local
 * head count does not match.  The attention kernel issues a system-scope fence after
 * its peer stores, before the flag kernel's st.release.sys.  host_seq_order as for
 * pa_paged_attention_ex.
 * ---------------------------------------------------------------------------------- */
typedef struct pa_tp_comm pa_tp_comm_t;
pa_tp_comm_t* pa_tp_comm_create(int world, int rank, int num_heads_total, size_t gather_bytes,
                                void* const* gather_a, void* const* gather_b,
                                int32_t* const* flags, int32_t* status);
void pa_tp_comm_destroy(pa_tp_comm_t* comm);
pa_status_t pa_paged_attention_decode_tp(pa_tp_comm_t* comm, int* buffer_out, const void* query,
                                         const void* key, const void* value, void* key_cache,
                                         void* value_cache, const int32_t* block_tables,
                                         const int32_t* context_lens, float scale, int block_size,
                                         int num_kv_heads, int num_seqs, int num_heads,
                                         int head_dim, int max_blocks_per_seq,
                                         int max_context_len, pa_dtype_t dtype,
                                         const int32_t* host_seq_order, void* workspace,
                                         size_t workspace_bytes, pa_stream_t stream);

/* CUDA IPC of device allocations between the ranks' processes (for the gather buffers and
 * flags above).  Handles are pa_ipc_handle_bytes() opaque bytes; pa_device_alloc /
 * pa_device_free give whole allocations whose handle maps to offset 0. */
size_t pa_ipc_handle_bytes(void);
pa_status_t pa_ipc_get_handle(const void* dev_ptr, void* handle_out);
pa_status_t pa_ipc_open_handle(const void* handle, void** dev_ptr_out);
pa_status_t pa_ipc_close_handle(void* dev_ptr);
pa_status_t pa_device_alloc(size_t bytes, void** dev_ptr_out);
pa_status_t pa_device_free(void* dev_ptr);

/* Bytes of workspace pa_paged_attention(_ex) needs: 8 bytes of split-completion word
 * per (sequence, head) plus, when a context is split, the partials.
 * partition_tokens as in pa_paged_attention_ex. */
size_t pa_paged_attention_workspace_size(int num_seqs, int num_heads, int head_dim,
                                         int max_context_len, int partition_tokens);

/* ------------------------------------------------------------------------------------
 * pa_reshape_and_cache -- fused reshape + block write.
 * For token i with slot = slot_mapping[i] >= 0: b = slot / B, o = slot % B and
 *     key_cache[b][h][o][:] = key[i][h][:],  value_cache[b][h][o][:] = value[i][h][:]
 * for every kv head h.  slot < 0 skips the token (reading c11).  Bit-exact copy.
 * key, value: [num_tokens][num_kv_heads][head_dim]; slot_mapping: int64 [num_tokens].
 * Slots must be distinct and < num_blocks * block_size.  num_tokens == 0 is a no-op.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_reshape_and_cache(const void* key, const void* value, void* key_cache,
                                 void* value_cache, const int64_t* slot_mapping, int num_tokens,
                                 int num_kv_heads, int head_dim, int block_size, pa_dtype_t dtype,
                                 pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_copy_blocks -- fused block copy for copy-on-write.
 * For every layer l < num_layers and pair p: key_caches[l][dst] <- key_caches[l][src]
 * and the same for value_caches, whole blocks (num_kv_heads*block_size*head_dim
 * elements), in ONE launch.  key_caches / value_caches: HOST arrays of num_layers
 * device pointers.  block_mapping: device int64 [num_pairs][2] = (src, dst).
 * Precondition (reading c12): dst ids distinct and disjoint from every src id (a CoW
 * destination is always a fresh block); src ids may repeat.  num_pairs == 0
 * is a no-op.  num_layers <= 256.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_copy_blocks(void* const* key_caches, void* const* value_caches, int num_layers,
                           const int64_t* block_mapping, int num_pairs, int num_kv_heads,
                           int block_size, int head_dim, pa_dtype_t dtype, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_swap_blocks -- block transfers between two block pools: swapping evicted KV blocks
 * to CPU memory and back.  For every layer l < num_layers
 * and pair p = (src, dst): dst_key_caches[l][dst] <- src_key_caches[l][src] and the same
 * for values, whole blocks (num_kv_heads*block_size*head_dim elements), in ONE launch.
 * Each cache pointer may be device memory or pinned, mapped host memory (cudaHostAlloc /
 * torch pin_memory; with unified addressing the GPU reads and writes it over the host
 * link directly), so a GPU->CPU swap-out and a CPU->GPU swap-in are both one kernel
 * instead of one cudaMemcpyAsync per block (the small-transfer penalty of P:708-710).
 * The four cache arrays are HOST arrays of num_layers pointers.  block_mapping:
 * int64 [num_pairs][2], device or mapped host memory.  dst ids distinct; a pool is
 * never both source and destination of one call.  num_pairs == 0 is a no-op.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_swap_blocks(void* const* dst_key_caches, void* const* dst_value_caches,
                           const void* const* src_key_caches, const void* const* src_value_caches,
                           int num_layers, const int64_t* block_mapping, int num_pairs,
                           int num_kv_heads, int block_size, int head_dim, pa_dtype_t dtype,
                           pa_stream_t stream);
/* Benchmark baseline only: the same transfer as one cudaMemcpyAsync per (pair, layer,
 * K/V) -- what a per-block swap costs (Fig.19 analogue, scripts/swap_bench.py). */
pa_status_t pa_swap_blocks_memcpy(void* const* dst_key_caches, void* const* dst_value_caches,
                                  const void* const* src_key_caches,
                                  const void* const* src_value_caches, int num_layers,
                                  const int64_t* host_block_mapping, int num_pairs,
                                  int num_kv_heads, int block_size, int head_dim,
                                  pa_dtype_t dtype, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * pa_decode_step -- one decode step of one attention layer from HOST inputs: the
 * end-to-end call of bench.py's "e2e" number.  Stream-ordered:
 *   H2D  query/key/value/block_tables/context_lens/block_mapping
 *        (HOST, ideally pinned) into the device staging buffer `staging`
 *   pa_copy_blocks (if num_pairs > 0) on (key_cache, value_cache)
 *   pa_paged_attention_decode (cache write + attention).  host_slot_mapping may be
 *   NULL and is not read: a decode token's slot follows from its block table row.
 *   D2H  out -> host_out (HOST)
 * key_cache/value_cache/workspace/staging: DEVICE.  staging must hold
 * pa_decode_step_staging_size() bytes.  The call returns after enqueueing; the
 * caller synchronises the stream before reading host_out.
 * Transfer modes.  Default: the batch is processed in C chunks of sequences (default 4,
 * PA_E2E_CHUNKS; at most 16): chunk c's kernel overlaps the H2D of chunk c+1 and the
 * D2H of chunk c-1 on two internal copy streams, and consecutive chunk kernels run on
 * two internal compute streams (each with half of `workspace`, which must then hold
 * 2 x the workspace of ceil(S/C) sequences, else one stream is used; PA_E2E_STREAMS=1
 * forces one) so one chunk's CTAs fill the SMs while the previous chunk's tail drains.
 * PA_E2E_SPLIT="w0,w1,..." sets relative chunk sizes (first to last) instead of equal
 * ones.  PA_E2E_GRAPH=1 captures the enqueued step once into a CUDA graph (internal
 * capture stream; cache of 8 per device, keyed on every pointer, size and tuning
 * variable of the call) and replays it with one launch on `stream`; host buffer
 * CONTENTS are read when the graph runs, so they may change between calls.
 * PA_E2E_MODE=zerocopy (ablation, measured slower): only block_tables, context_lens and
 * block_mapping are copied; the kernel reads q / new k / new v straight from pinned,
 * device-mapped host memory and stores out straight into host_out (PA_ERR_INVALID_ARG
 * if a buffer is not mapped).  In every mode (internal streams: one set per device)
 * every step still orders after the previous work of `stream` and joins back into `stream`, so
 * the synchronisation rule above is unchanged.  Results equal the unchunked step bit
 * for bit (sequences are independent).  Enqueueing is serialised per device.
 * ---------------------------------------------------------------------------------- */
size_t pa_decode_step_staging_size(int num_seqs, int num_heads, int num_kv_heads, int head_dim,
                                   int max_blocks_per_seq, int num_pairs, pa_dtype_t dtype);
pa_status_t pa_decode_step(void* host_out, const void* host_query, const void* host_key,
                           const void* host_value, const int64_t* host_slot_mapping,
                           const int32_t* host_block_tables, const int32_t* host_context_lens,
                           const int64_t* host_block_mapping, int num_pairs,
                           void* key_cache, void* value_cache, float scale, int block_size,
                           int num_kv_heads, int num_seqs, int num_heads, int head_dim,
                           int max_blocks_per_seq, int max_context_len, pa_dtype_t dtype,
                           void* staging, size_t staging_bytes, void* workspace,
                           size_t workspace_bytes, pa_stream_t stream);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* pa_last_error(void);

/* Number of kernel launches the library issued on this thread since the last call
 * (bench.py's gpu_launches evidence).  Resets the counter. */
long long pa_take_launch_count(void);

/* ------------------------------------------------------------------------------------
 * Test-only helpers (synchronising).
 * pa_debug_gather_kv: k_out/v_out [num_seqs][num_kv_heads][max_ctx][head_dim] (DEVICE)
 * receive the K/V rows of logical tokens t < context_lens[s] through the SAME tile
 * loader the attention kernel uses (block-table lookup + bulk copy into shared memory),
 * rows t >= ctx untouched.  For the bitwise block-table indexing check.
 * pa_validate_tables: every live entry bt[s][j], j < ceil(ctx[s]/B), in [0,NB);
 * 0 <= ctx[s] <= W*B.  *first_bad_out (HOST) = first bad flat index s*W+j (or
 * -(s+1) for a bad ctx) or -1 when all valid.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_debug_gather_kv(void* k_out, void* v_out, const void* key_cache,
                               const void* value_cache, const int32_t* block_tables,
                               const int32_t* context_lens, int block_size, int num_kv_heads,
                               int num_seqs, int head_dim, int max_blocks_per_seq, int max_ctx,
                               pa_dtype_t dtype, pa_stream_t stream);
pa_status_t pa_validate_tables(const int32_t* block_tables, const int32_t* context_lens,
                               int num_seqs, int max_blocks_per_seq, int block_size,
                               int num_blocks, int64_t* first_bad_out, pa_stream_t stream);

/* ------------------------------------------------------------------------------------
 * Host block allocator -- the paper's KV block manager (P:249-256, P:295-332,
 * P:451-458), used only on the host to generate block tables, slot mappings and
 * copy-on-write pairs.  Single-threaded per allocator object.
 *  - physical blocks 0..num_blocks-1, handed out in `initial_order` (HOST int32
 *    [num_blocks], a permutation; NULL = 0,1,2,...); freed blocks join the BACK of
 *    the FIFO free list (Fig.9: after freeing 2,4,5,8 the next blocks are 9-12).
 *  - allocate(n): ceil(n/B) fresh blocks, filled left to right.
 *  - append_slot: the slot (block*B + offset) of one new token; a new block when the
 *    last is full; copy-on-write when the last block is partial and shared
 *    (refcount > 1): cow_src_out / cow_dst_out receive (old, new), else -1.
 *  - fork: a child sharing every block (refcount + 1).
 *  - free: drop the sequence; blocks whose refcount reaches 0 are freed.
 * Errors: PA_ERR_OUT_OF_BLOCKS (free list empty), PA_ERR_INVALID_ARG (unknown or
 * freed handle = double free, bad sizes).
 * ---------------------------------------------------------------------------------- */
typedef struct pa_alloc pa_alloc_t;
pa_alloc_t* pa_alloc_create(int num_blocks, int block_size, const int32_t* initial_order);
void pa_alloc_destroy(pa_alloc_t* a);
pa_status_t pa_alloc_allocate(pa_alloc_t* a, int num_tokens, int* seq_out);
pa_status_t pa_alloc_append_slot(pa_alloc_t* a, int seq, int64_t* slot_out, int* cow_src_out,
                                 int* cow_dst_out);
pa_status_t pa_alloc_fork(pa_alloc_t* a, int parent, int* child_out);
pa_status_t pa_alloc_free(pa_alloc_t* a, int seq, int* freed_out);
/* Rows of the given sequences into block_tables_out (HOST int32 [n][W], padded -1)
 * and their token counts into context_lens_out (HOST int32 [n]). */
pa_status_t pa_alloc_export(const pa_alloc_t* a, const int* seqs, int n, int W,
                            int32_t* block_tables_out, int32_t* context_lens_out);
int pa_alloc_refcount(const pa_alloc_t* a, int block);
int pa_alloc_num_free(const pa_alloc_t* a);
int pa_alloc_num_blocks_of(const pa_alloc_t* a, int seq); /* -1 if unknown */

/* ------------------------------------------------------------------------------------
 * pa_hbm_read_probe -- measurement helper (not on the hot path): the same-run read-only
 * HBM ceiling for the roofline (SURVEY §8(d) asks for a read-only probe beside the copy
 * peak; the decode kernel is a read stream).  Persistent CTAs (grid = `ctas`,
 * <= 0 -> 2 per SM) stream the buffer `buf` (DEVICE, `bytes` a multiple of `chunk`, 16-B
 * aligned) into shared memory with 1-D bulk copies of `chunk` bytes (multiple of 16,
 * <= 64 KiB), `stages` in flight per CTA (stages * chunk <= 200 KiB), the attention
 * kernel's own load mechanism.  Nothing is written to global memory except one 32-bit
 * word per CTA into `sink` (DEVICE, >= grid words).  Asynchronous on `stream`; time it
 * with events.  Errors: PA_ERR_INVALID_ARG on bad sizes / pointers.
 * ---------------------------------------------------------------------------------- */
pa_status_t pa_hbm_read_probe(const void* buf, size_t bytes, int chunk, int stages, int ctas,
                              uint32_t* sink, pa_stream_t stream);

/* Tests / A-B scripts only: re-read the PA_* tuning environment variables (read once,
 * at the first call, otherwise; never on the launch path).  Not thread-safe with
 * concurrent launches. */
void pa_reload_tuning(void);

#ifdef __cplusplus
}
#endif
#endif /* PAGED_ATTN_PA_H_ */
