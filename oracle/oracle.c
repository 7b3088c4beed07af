/*
 * oracle.c -- plain, slow, fp64 CPU oracle for the PagedAttention decode hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares
 * no code, header, table or helper with the CUDA path (paper_2309_06180_b200/csrc)
 * and never includes include/pa.h.
 *
 * Citations: P:N = /root/reference/PAPER.md line N (the vLLM paper, arXiv 2309.06180).
 *
 *   Eq.3  a_ij = exp(q_i.k_j/sqrt(d)) / sum_{t<=i} exp(q_i.k_t/sqrt(d)),
 *                     o_i = sum_j a_ij v_j
 *   Eq.4  the same result computed block by block, K_j/V_j fetched through
 *                     the block table; blocks need not be contiguous.
 *   P:418-419         fused reshape + block write  -> oracle_reshape_and_cache
 *   P:424-427         fused block copy (CoW) -> oracle_copy_blocks
 *   P:363-366         swapping blocks to the CPU pool and back -> oracle_swap_blocks
 *   P:140-147,334-338 prompt-phase / shared-prefix-suffix causal attention over the
 *                     paged cache -> oracle_prefill_attention
 *
 * Readings of the paper: the caller passes `scale` (c1); the
 * Eq.4 denominator is the sum of element-wise exponentials (c2); only t < ctx is read
 * (c3); ctx includes the current token, written before attention (c5); one block table
 * per sequence shared by all heads (c6); cache layout [NB][H_kv][B][D] (c7); ctx == 0
 * gives a zero output (c9); slot < 0 is skipped (c11); GQA head h reads kv head
 * h / (H / H_kv) (c13).
 *
 * Everything is computed in IEEE fp64 with sequential loops, no blocking, no fusion,
 * no reordering.  Softmax is two-pass with max subtraction (the SPEC's allowed
 * evaluation): pass 1 the max, pass 2 the exponentials, their sum and the
 * weighted V sum, then one division.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_F32 0
#define ORACLE_F16 1
#define ORACLE_BF16 2

/* ---- element decoding: the storage dtype -> fp64, bit-exactly ------------------ */

/* IEEE 754 binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits. */
static double dec_f16(uint16_t h) {
    int sign = h >> 15;
    int e = (h >> 10) & 0x1f;
    int m = h & 0x3ff;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24);               /* subnormal: m * 2^(1-15-10) */
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(m | 0x400), e - 25);  /* (1.m) * 2^(e-15), scaled by 2^10 */
    return sign ? -v : v;
}

/* bfloat16 is by definition the upper 16 bits of an IEEE binary32. */
static double dec_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static double dec_f32(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static int elem_bytes(int dtype) { return dtype == ORACLE_F32 ? 4 : 2; }

/* Decode element `idx` of a raw array of the given dtype. */
static double load(const void* base, int64_t idx, int dtype) {
    if (dtype == ORACLE_F32) return dec_f32(((const uint32_t*)base)[idx]);
    if (dtype == ORACLE_F16) return dec_f16(((const uint16_t*)base)[idx]);
    return dec_bf16(((const uint16_t*)base)[idx]);
}

double oracle_decode(uint32_t bits, int dtype) {
    if (dtype == ORACLE_F32) return dec_f32(bits);
    if (dtype == ORACLE_F16) return dec_f16((uint16_t)bits);
    return dec_bf16((uint16_t)bits);
}

/* Decode n elements into an fp64 array (used by tests to compare against numpy). */
void oracle_decode_array(const void* src, int64_t n, int dtype, double* dst) {
    for (int64_t i = 0; i < n; ++i) dst[i] = load(src, i, dtype);
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- Eq.3: contiguous attention for one query ---------------------------------- */

/* q[D], K[n][D], V[n][D] already in fp64.  n == 0 gives out = 0 (c9). */
void oracle_contiguous_attention(double* out, const double* q, const double* K,
                                 const double* V, int n, int D, double scale) {
    for (int d = 0; d < D; ++d) out[d] = 0.0;
    if (n <= 0) return;
    double* l = (double*)malloc(sizeof(double) * (size_t)n);
    /* scores l_t = scale * sum_d q_d K_td, sequential d */
    for (int t = 0; t < n; ++t) {
        double dot = 0.0;
        for (int d = 0; d < D; ++d) dot += q[d] * K[(int64_t)t * D + d];
        l[t] = scale * dot;
    }
    double m = -INFINITY;
    for (int t = 0; t < n; ++t)
        if (l[t] > m) m = l[t];
    double L = 0.0;
    for (int t = 0; t < n; ++t) {
        double w = exp(l[t] - m);
        L += w;
        for (int d = 0; d < D; ++d) out[d] += w * V[(int64_t)t * D + d];
    }
    for (int d = 0; d < D; ++d) out[d] /= L;
    free(l);
}

/* ---- Eq.4: paged attention -------------------------------------------------------- */

/* Physical element index of (block b, kv head h, slot o, dim d) in [NB][H_kv][B][D]
 * (reading c7). */
static int64_t cache_index(int64_t b, int h, int o, int d, int H_kv, int B, int D) {
    return ((b * H_kv + h) * (int64_t)B + o) * (int64_t)D + d;
}

/* One (sequence, head) of Eq.4.  Tokens are visited in logical order t = 0..n-1; the
 * block table translates logical block t/B to a physical block (Fig.6). */
static void paged_one(double* out, const void* query, const void* kc, const void* vc,
                      const int32_t* bt_row, int n, int s, int h, double scale, int B,
                      int H_kv, int H, int D, int dtype) {
    const int kvh = h / (H / H_kv);
    const int64_t qoff = ((int64_t)s * H + h) * D;
    for (int d = 0; d < D; ++d) out[d] = 0.0;
    if (n <= 0) return;
    double* l = (double*)malloc(sizeof(double) * (size_t)n);
    for (int t = 0; t < n; ++t) {
        int64_t b = bt_row[t / B];
        int o = t % B;
        double dot = 0.0;
        for (int d = 0; d < D; ++d)
            dot += load(query, qoff + d, dtype) * load(kc, cache_index(b, kvh, o, d, H_kv, B, D), dtype);
        l[t] = scale * dot;
    }
    double m = -INFINITY;
    for (int t = 0; t < n; ++t)
        if (l[t] > m) m = l[t];
    double L = 0.0;
    for (int t = 0; t < n; ++t) {
        int64_t b = bt_row[t / B];
        int o = t % B;
        double w = exp(l[t] - m);
        L += w;
        for (int d = 0; d < D; ++d) out[d] += w * load(vc, cache_index(b, kvh, o, d, H_kv, B, D), dtype);
    }
    for (int d = 0; d < D; ++d) out[d] /= L;
    free(l);
}

/* out: fp64 [S][H][D].  query: [S][H][D]; caches: [NB][H_kv][B][D]; block_tables:
 * [S][W]; context_lens: [S].  All inputs in the storage dtype. */
void oracle_paged_attention(double* out, const void* query, const void* key_cache,
                            const void* value_cache, const int32_t* block_tables,
                            const int32_t* context_lens, double scale, int block_size,
                            int num_kv_heads, int num_seqs, int num_heads, int head_dim,
                            int W, int dtype) {
    int64_t total = (int64_t)num_seqs * num_heads;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < total; ++i) {
        int s = (int)(i / num_heads), h = (int)(i % num_heads);
        paged_one(out + i * head_dim, query, key_cache, value_cache,
                  block_tables + (int64_t)s * W, context_lens[s], s, h, scale, block_size,
                  num_kv_heads, num_heads, head_dim, dtype);
    }
}

/* Multi-token (prompt / chunked-prompt / shared-prefix suffix) attention, P:145-147,
 * P:334-338 with Eq.4.  Sequence s owns query rows [query_start[s], query_start[s+1])
 * of query [T][H][D]; its q_len = query_start[s+1]-query_start[s] new tokens are the LAST
 * q_len of its context_lens[s] cached tokens (reading c22), so query row i sits at
 * position p = ctx - q_len + i and attends causally to tokens 0..p (the autoregressive
 * mask of P:140-142).  That is Eq.4 with n = p + 1 -- computed here by the same per-row
 * routine as decode.  out: fp64 [T][H][D]. */
void oracle_prefill_attention(double* out, const void* query, const void* key_cache,
                              const void* value_cache, const int32_t* block_tables,
                              const int32_t* context_lens, const int32_t* query_start,
                              double scale, int block_size, int num_kv_heads, int num_seqs,
                              int num_heads, int head_dim, int W, int dtype) {
    int64_t T = query_start[num_seqs];
    int64_t total = T * num_heads;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < total; ++i) {
        int64_t row = i / num_heads;
        int h = (int)(i % num_heads);
        int s = 0;
        while (query_start[s + 1] <= row) ++s;
        int q_len = query_start[s + 1] - query_start[s];
        int pos = context_lens[s] - q_len + (int)(row - query_start[s]);
        paged_one(out + i * head_dim, query, key_cache, value_cache,
                  block_tables + (int64_t)s * W, pos + 1, (int)row, h, scale, block_size,
                  num_kv_heads, num_heads, head_dim, dtype);
    }
}

/* Gather the logical K and V rows of (seq s, kv head kvh) into contiguous fp64 arrays
 * K[n][D], V[n][D] -- the "contiguous cache" that Eq.3 assumes. */
void oracle_gather_kv(double* K, double* V, const void* key_cache, const void* value_cache,
                      const int32_t* bt_row, int n, int kvh, int block_size,
                      int num_kv_heads, int head_dim, int dtype) {
    for (int t = 0; t < n; ++t) {
        int64_t b = bt_row[t / block_size];
        int o = t % block_size;
        for (int d = 0; d < head_dim; ++d) {
            int64_t idx = cache_index(b, kvh, o, d, num_kv_heads, block_size, head_dim);
            K[(int64_t)t * head_dim + d] = load(key_cache, idx, dtype);
            V[(int64_t)t * head_dim + d] = load(value_cache, idx, dtype);
        }
    }
}

/* Raw-bits gather (for the bitwise block-table indexing check): out[n][D] elements of
 * the storage dtype, copied from the physical slots of logical tokens 0..n-1. */
void oracle_gather_kv_bits(void* k_out, void* v_out, const void* key_cache,
                           const void* value_cache, const int32_t* bt_row, int n, int kvh,
                           int block_size, int num_kv_heads, int head_dim, int dtype) {
    int e = elem_bytes(dtype);
    for (int t = 0; t < n; ++t) {
        int64_t b = bt_row[t / block_size];
        int o = t % block_size;
        int64_t src = cache_index(b, kvh, o, 0, num_kv_heads, block_size, head_dim);
        memcpy((char*)k_out + (int64_t)t * head_dim * e, (const char*)key_cache + src * e,
               (size_t)head_dim * e);
        memcpy((char*)v_out + (int64_t)t * head_dim * e, (const char*)value_cache + src * e,
               (size_t)head_dim * e);
    }
}

/* ---- split-context: per-partition (m_p, L_p, o~_p) and the log-sum-exp merge ------ */

/* Partition the logical context [0, n) into consecutive pieces of `part` tokens.  For
 * piece p: m_p = max l_t, L_p = sum exp(l_t - m_p), o~_p = sum exp(l_t - m_p) v_t / L_p.
 * Merge: M = max m_p;  o = sum_p e^{m_p - M} L_p o~_p / sum_p e^{m_p - M} L_p.
 * (not in the paper -- BJ:north_star's split-context variant.)
 * Writes out[S][H][D] like oracle_paged_attention. */
void oracle_split_attention(double* out, const void* query, const void* key_cache,
                            const void* value_cache, const int32_t* block_tables,
                            const int32_t* context_lens, double scale, int block_size,
                            int num_kv_heads, int num_seqs, int num_heads, int head_dim,
                            int W, int dtype, int part) {
    int64_t total = (int64_t)num_seqs * num_heads;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < total; ++i) {
        int s = (int)(i / num_heads), h = (int)(i % num_heads);
        int n = context_lens[s];
        int D = head_dim;
        double* o = out + i * D;
        for (int d = 0; d < D; ++d) o[d] = 0.0;
        if (n <= 0) continue;
        int kvh = h / (num_heads / num_kv_heads);
        const int32_t* bt_row = block_tables + (int64_t)s * W;
        int np = (n + part - 1) / part;
        double* mp = (double*)malloc(sizeof(double) * np);
        double* Lp = (double*)malloc(sizeof(double) * np);
        double* op = (double*)calloc((size_t)np * D, sizeof(double));
        double* K = (double*)malloc(sizeof(double) * (size_t)part * D);
        double* V = (double*)malloc(sizeof(double) * (size_t)part * D);
        double* q = (double*)malloc(sizeof(double) * D);
        for (int d = 0; d < D; ++d) q[d] = load(query, ((int64_t)s * num_heads + h) * D + d, dtype);
        for (int p = 0; p < np; ++p) {
            int t0 = p * part, t1 = t0 + part < n ? t0 + part : n;
            int len = t1 - t0;
            for (int t = 0; t < len; ++t) {
                int tt = t0 + t;
                int64_t b = bt_row[tt / block_size];
                for (int d = 0; d < D; ++d) {
                    int64_t idx = cache_index(b, kvh, tt % block_size, d, num_kv_heads, block_size, D);
                    K[(int64_t)t * D + d] = load(key_cache, idx, dtype);
                    V[(int64_t)t * D + d] = load(value_cache, idx, dtype);
                }
            }
            double m = -INFINITY;
            double* l = (double*)malloc(sizeof(double) * len);
            for (int t = 0; t < len; ++t) {
                double dot = 0.0;
                for (int d = 0; d < D; ++d) dot += q[d] * K[(int64_t)t * D + d];
                l[t] = scale * dot;
                if (l[t] > m) m = l[t];
            }
            double L = 0.0;
            for (int t = 0; t < len; ++t) {
                double w = exp(l[t] - m);
                L += w;
                for (int d = 0; d < D; ++d) op[(int64_t)p * D + d] += w * V[(int64_t)t * D + d];
            }
            for (int d = 0; d < D; ++d) op[(int64_t)p * D + d] /= L;
            mp[p] = m;
            Lp[p] = L;
            free(l);
        }
        double M = -INFINITY;
        for (int p = 0; p < np; ++p)
            if (mp[p] > M) M = mp[p];
        double den = 0.0;
        for (int p = 0; p < np; ++p) {
            double w = exp(mp[p] - M) * Lp[p];
            den += w;
            for (int d = 0; d < D; ++d) o[d] += w * op[(int64_t)p * D + d];
        }
        for (int d = 0; d < D; ++d) o[d] /= den;
        free(mp); free(Lp); free(op); free(K); free(V); free(q);
    }
}

/* ---- fused reshape + block write ------------------------------------- */

/* For token i with slot s = slot_mapping[i] >= 0: block b = s / B, offset o = s % B;
 * key_cache[b][h][o][:] = key[i][h][:] for every kv head h, and the same for V.
 * Operates on raw bit patterns; every other element is left unchanged (c11: s < 0 is
 * skipped).  Tokens are applied in order i = 0..T-1 (a later token wins on a repeated
 * slot; the product contract forbids repeats). */
void oracle_reshape_and_cache(const void* key, const void* value, void* key_cache,
                              void* value_cache, const int64_t* slot_mapping, int num_tokens,
                              int num_kv_heads, int head_dim, int block_size, int dtype) {
    int e = elem_bytes(dtype);
    size_t row = (size_t)head_dim * e;
    for (int i = 0; i < num_tokens; ++i) {
        int64_t s = slot_mapping[i];
        if (s < 0) continue;
        int64_t b = s / block_size;
        int o = (int)(s % block_size);
        for (int h = 0; h < num_kv_heads; ++h) {
            int64_t src = ((int64_t)i * num_kv_heads + h) * head_dim;
            int64_t dst = cache_index(b, h, o, 0, num_kv_heads, block_size, head_dim);
            memcpy((char*)key_cache + dst * e, (const char*)key + src * e, row);
            memcpy((char*)value_cache + dst * e, (const char*)value + src * e, row);
        }
    }
}

/* ---- fused block copy -------------------------------------------------- */

/* For every layer l and pair (src, dst): cache_l[dst] <- cache_l[src] (whole block:
 * all kv heads, all B slots), for K and V.  Simultaneous semantics: every source is
 * read from a snapshot taken before any destination is written (reading c12). */
void oracle_copy_blocks(void** key_caches, void** value_caches, int num_layers,
                        const int64_t* block_mapping, int num_pairs, int num_kv_heads,
                        int block_size, int head_dim, int num_blocks, int dtype) {
    size_t blk = (size_t)num_kv_heads * block_size * head_dim * elem_bytes(dtype);
    size_t total = blk * (size_t)num_blocks;
    char* snap = (char*)malloc(total);
    for (int l = 0; l < num_layers; ++l) {
        for (int kv = 0; kv < 2; ++kv) {
            char* cache = (char*)(kv == 0 ? key_caches[l] : value_caches[l]);
            memcpy(snap, cache, total);
            for (int p = 0; p < num_pairs; ++p) {
                int64_t src = block_mapping[2 * p], dst = block_mapping[2 * p + 1];
                memcpy(cache + dst * blk, snap + src * blk, blk);
            }
        }
    }
    free(snap);
}

/* ---- swapping between block pools -------------------------------------- */

/* For every layer l and pair (src, dst): dst_cache_l[dst] <- src_cache_l[src] (whole
 * blocks of block_bytes), for K and V.  The two pools are distinct arrays (GPU pool and
 * CPU swap pool), so there is no aliasing between sources and destinations. */
void oracle_swap_blocks(void** dst_key, void** dst_value, void** src_key, void** src_value, int num_layers,
                        const int64_t* block_mapping, int num_pairs, int64_t block_bytes) {
    for (int l = 0; l < num_layers; ++l)
        for (int p = 0; p < num_pairs; ++p) {
            int64_t src = block_mapping[2 * p], dst = block_mapping[2 * p + 1];
            memcpy((char*)dst_key[l] + dst * block_bytes, (const char*)src_key[l] + src * block_bytes,
                   (size_t)block_bytes);
            memcpy((char*)dst_value[l] + dst * block_bytes, (const char*)src_value[l] + src * block_bytes,
                   (size_t)block_bytes);
        }
}
