// pa_decode_tc.cu -- sharing-aware decode attention on the tcgen05 tensor cores (SURVEY
// §8(f) N1, pa_paged_attention_decode_grouped).
//
// Sequences of one sequence group (the n samples of a request, the k beams of a beam search,
// P:295-332) share physical blocks.  Eq.4 for every member of the group and every
// query head, with each DISTINCT 16-row block piece read from HBM once for the whole group:
//
//   * work item = (group of GM consecutive sequences, pair of query heads); persistent CTAs
//     (one per SM) draw items from an epoch-tagged counter;
//   * producer warp: looks up the members' block ids 32 logical 16-token positions at a
//     time, keeps one "slot" per distinct piece (owner mask = the members that read it at
//     that position) and TMA-loads its K and V rows for both heads into a tile of 4 slots
//     (128-byte swizzle; a partial piece in 16/8/4/2/1-row boxes so nothing past the context
//     is read; a member's new token row comes from the step's key/value input);
//   * MMA warp: S_h = Q_h K_h^T for the tile's 4 slots at once (M = 128 rows: the members'
//     query rows, replicated by a zero row stride in the descriptor; N = 64 tokens; K = 128)
//     into tensor memory, then O_h += P_h V_h (P from tensor memory, one K=16 step per slot);
//   * softmax warps (one per head, TMEM lane quadrant = head): lane m = member m reads its S
//     row, masks columns it does not own or that lie past its context, online softmax in the
//     exp2 domain with lazy rescaling, writes P (storage dtype) back into tensor memory;
//     epilogue O / l to `out` and the member's new K/V row to its cache slot (the fused
//     reshape_and_cache of the decode step).
// So the per-(member, token) CUDA-core work of the coop/shared kernels (a 128-wide dot
// product and axpy each) becomes two tensor-core MMAs per shared piece; a shared piece costs
// the same MMA work whether one or eight members own it.
#include "pa_common.cuh"
#include "pa_internal.h"
#include "pa_tc.cuh"

#include <type_traits>

namespace pa {
using namespace tc;

namespace {
constexpr int kNH = 4;                      // query heads per work item (one TMEM lane quadrant each)
#ifndef PA_TC_SLOTS
#define PA_TC_SLOTS 2
#endif
#ifndef PA_TC_KBUF
#define PA_TC_KBUF 2
#endif
#ifndef PA_TC_VBUF
#define PA_TC_VBUF 4
#endif
constexpr int kSlots = PA_TC_SLOTS;         // 16-row block pieces per MMA tile
constexpr int kBK = PA_TC_KBUF;             // K tile buffers (free once S = Q K^T has completed)
constexpr int kBV = PA_TC_VBUF;             // V tile buffers (free once P V has completed)
constexpr int kPiece = 16 * 128;            // [16 rows][64 cols] swizzled, 2-byte elements
constexpr int kQuad = kNH * kPiece;         // one piece, the item's kv heads stacked: [64 rows][128 B] = 8 KB
constexpr int kHalfReg = kSlots * kQuad;    // one 64-column half of the tile: 16 KB
constexpr int kTensor = 2 * kHalfReg;       // K (or V) of a tile: 32 KB [half][piece][head][16 rows][128 B]
constexpr int kMaxGM = 8;
constexpr int kListCap = 32 * kMaxGM;       // pieces of one 32-position chunk
constexpr float kLazyTc = 8.f;              // P <= 2^8 between rescales
constexpr int kNCh = 4;                     // piece-list chunks in flight (scheduler -> producer)
constexpr int kThreadsTc = 384;             // warps: 0-3 softmax (head w = lane quadrant w), 4 K producer,
                                            // 5 MMA, 6 scheduler, 7 V producer, 8-11 epilogue (head w - 8)
// tensor memory columns: Q0 | Q1 (16-bit pairs, by item parity) | S0 | S1 | O; lanes
// 32w..32w+31 = head w's members
constexpr int kTmQ = 0, kTmS = 128, kSCols = 16 * kNH * kSlots, kTmO = kTmS + 2 * kSCols;
constexpr int kNumBars = 2 * kBK + 2 * kBV + 2 + 2 + 2 + 1 + 1 + 4 + 4 + 2 + 2 * kNCh + 4;

struct TileMeta {
    int ns, last;
    int p[kSlots], own[kSlots], nrows[kSlots];
};

struct TcItem {
    int s0, gmv, h[kNH], kvh[kNH];
    int part;     // split-context part: piece positions [part << part_log, (part + 1) << part_log) (the last: to the end)
    unsigned st;  // bit w: head w of the quad exists (H % 4 tail: duplicates are not stored)
    bool quad;    // the 4 kv heads are consecutive (one 64-row box per piece half when B == 16)
};

__device__ __forceinline__ TcItem tc_item(const GroupTcParams& p, int i) {
    TcItem it;
    // item = (group, part, head quad), group-major: a group's parts and quads are consecutive
    const int per_g = p.n_hp * p.NPt;
    const int gi = i / per_g, r = i - gi * per_g;
    it.part = r / p.n_hp;
    const int hq = r - it.part * p.n_hp;
    const int g = gi < p.n_gorder ? (int)p.gorder[gi] : gi;  // longest-first plan (scheduling only)
    it.s0 = g * p.GM;
    it.gmv = min(p.GM, p.S - it.s0);
    it.st = 0;
    it.quad = true;
#pragma unroll
    for (int w = 0; w < kNH; ++w) {
        it.h[w] = min(kNH * hq + w, p.H - 1);
        if (kNH * hq + w < p.H) it.st |= 1u << w;
        it.kvh[w] = it.h[w] / p.G;
        if (it.kvh[w] != it.kvh[0] + w) it.quad = false;
    }
    return it;
}

// Next dynamic work item of this launch: the counter word is (epoch << 32 | items handed
// out).  One atomic add per fetch; a word still carrying another launch's epoch is claimed
// with a compare-and-swap that starts this launch's count (so the host never resets it).
__device__ __forceinline__ int fetch_item(unsigned long long* ctr, uint32_t epoch) {
    const unsigned long long E = (unsigned long long)epoch << 32;
    for (;;) {
        const unsigned long long old = atomicAdd(ctr, 1ull);
        if ((old & 0xffffffff00000000ull) == E) return (int)(old & 0xffffffffull);
        // stale word: install (E, 1) -- this call's item 0 -- unless another caller converts
        // it first; CAS against the latest stale value, so concurrent adds cannot livelock it
        unsigned long long cur = old + 1ull;
        for (;;) {
            const unsigned long long prev = atomicCAS(ctr, cur, E | 1ull);
            if (prev == cur) return 0;
            if ((prev & 0xffffffff00000000ull) == E) break;  // converted by another caller: add again
            cur = prev;
        }
    }
}

// Split-context completion count of row sh (one call per part holding its tokens, after the
// part's (m, L, O / L) is published): true for the part that completes the set of n.  The
// word is (epoch << 32 | parts done); another launch's epoch counts as 0 and the completing
// part stores 0 back, so the host never resets the counters (as the coop kernel's).
__device__ __forceinline__ bool split_done(const GroupTcParams& p, int64_t sh, int n) {
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
}  // namespace

#ifdef PA_TC_TRACE  // timing experiments (variant build): clock64 per tile of CTAs 0..7
constexpr int kTrTiles = 1024;
__device__ long long g_tc_trace[8 * kTrTiles * 8];
__device__ unsigned long long g_tc_span[1024 * 8];
__device__ long long g_tc_ep[8 * 64 * 8];  // CTAs 0..7, items 0..63: epilogue start, o_last seen, O stored, done
#define TC_EP(item, ev)                                                                                      \
    do {                                                                                                     \
        if (blockIdx.x < 8 && (item) < 64 && lane == 0 && hh == 0) g_tc_ep[(blockIdx.x * 64 + (item)) * 8 + (ev)] = clock64(); \
    } while (0)  // per CTA: globaltimer at entry, after pdl_wait, at exit; items
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TC_SPAN(ev, v)                                                     \
    do {                                                                   \
        if (blockIdx.x < 1024) g_tc_span[blockIdx.x * 8 + (ev)] = (v);    \
    } while (0)
#define TC_T(tile, ev)                                                                               \
    do {                                                                                             \
        if (blockIdx.x < 8 && (tile) < kTrTiles) g_tc_trace[(blockIdx.x * kTrTiles + (tile)) * 8 + (ev)] = clock64(); \
    } while (0)
#else
#define TC_T(tile, ev) \
    do {               \
    } while (0)
#define TC_SPAN(ev, v) \
    do {               \
    } while (0)
#define TC_EP(item, ev) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ int sel4(const int (&a)[kNH], int w) {
    return w == 0 ? a[0] : w == 1 ? a[1] : w == 2 ? a[2] : a[3];
}

template <typename T>
__global__ void __launch_bounds__(kThreadsTc, 1)
    paged_attention_group_tc_kernel(const __grid_constant__ GroupTcParams p) {
    constexpr bool kBF16 = std::is_same<T, __nv_bfloat16>::value;
    constexpr int kProd = kNH, kMma = kNH + 1, kSched = kNH + 2, kVProd = kNH + 3, kEpi0 = kNH + 4;  // 0..kNH-1: softmax
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem =
        tc::smem_align1024(smem_raw);
    unsigned char* sK = smem;                         // kBK x K [half][piece][head][16][128 B]
    unsigned char* sV = sK + kBK * kTensor;           // kBV x V, same
    TileMeta* meta = reinterpret_cast<TileMeta*>(sV + kBV * kTensor);  // [kBV], written with V
    int2* kmeta = reinterpret_cast<int2*>(meta + kBV);                   // [kBK] (pieces, last), written with K
    int2* clist = kmeta + kBK;                        // kNCh x kListCap distinct pieces
    int4* chdr = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(clist + kNCh * kListCap) + 15) &
                                         ~uintptr_t(15));  // kNCh: (item, pieces, last list of the item)
    uint64_t* bars = reinterpret_cast<uint64_t*>(chdr + kNCh);
    uint64_t* k_full = bars;                    // kBK: K bytes + K producer arrive
    uint64_t* k_empty = k_full + kBK;           // kBK: MMA commit after S
    uint64_t* v_full = k_empty + kBK;           // kBV: V bytes + V producer arrive (meta written)
    uint64_t* v_empty = v_full + kBV;           // kBV: MMA commit after P V + kNH softmax warps
    uint64_t* q_full = v_empty + kBV;           // 2 (by item parity): the softmax lanes wrote Q
    uint64_t* s_full = q_full + 2;              // [S buffer]
    uint64_t* p_full = s_full + 2;              // [S buffer]: the softmax lanes
    uint64_t* o_last = p_full + 2;              // 1: an item's last P V has completed
    uint64_t* o_free = o_last + 1;              // 1: the softmax lanes read O
    uint64_t* item_full = o_free + 1;           // 4: producer -> MMA + softmax
    uint64_t* item_empty = item_full + 4;       // 4: MMA + kNH softmax warps
    uint64_t* o_step = item_empty + 4;          // 2: P V number k on o_step[k & 1] (MMA warp only)
    uint64_t* chunk_full = o_step + 2;          // kNCh: scheduler -> producer (a piece list is written)
    uint64_t* chunk_empty = chunk_full + kNCh;  // kNCh: producer -> scheduler (the list has been issued)
    uint64_t* st_full = chunk_empty + kNCh;     // 2: the softmax warps handed an item's (m, L) rows over
    uint64_t* st_empty = st_full + 2;           // 2: the epilogue warps read them
    int* item_ring = reinterpret_cast<int*>(bars + kNumBars);
    int* st_item = item_ring + 4;               // 2 item indices handed to the epilogue warps (-1: done)
    float4* stats = reinterpret_cast<float4*>(st_item + 4);  // [2][kNH][32] (m, L, P V count, ctx) per row
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stats + 2 * kNH * 32);
    volatile int* pv_done = reinterpret_cast<volatile int*>(tmem_slot + 1);  // last completed P V (tile index)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef PA_TC_TRACE
    if (tid == 0) TC_SPAN(6, gtimer());  // kernel entry
#endif
    if (tid == 0) {
        for (int i = 0; i < kBK; ++i) {
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
        }
        for (int i = 0; i < kBV; ++i) {
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1 + kNH);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 32 * kNH);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 32 * kNH);
        }
        mbar_init(o_last, 1);
        mbar_init(&o_step[0], 1);
        mbar_init(&o_step[1], 1);
        mbar_init(o_free, 32 * kNH);
        *pv_done = -1;
        for (int i = 0; i < 4; ++i) {
            mbar_init(&item_full[i], 1);
            mbar_init(&item_empty[i], 1 + kNH);
        }
        for (int i = 0; i < kNCh; ++i) {
            mbar_init(&chunk_full[i], 1);
            mbar_init(&chunk_empty[i], 2);  // K and V producers
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&st_full[i], kNH);
            mbar_init(&st_empty[i], kNH);
        }
        fence_mbar_init();
    }
    if (warp == kMma) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
#ifdef PA_TC_TRACE
    if (tid == 0) TC_SPAN(0, gtimer());
#endif
    pdl_wait();  // inputs of the preceding kernel on the stream are visible from here on
#ifdef PA_TC_TRACE
    if (tid == 0) TC_SPAN(1, gtimer());
#endif
    pdl_launch_dependents();
    const int ppb_log = p.log2B - 4;  // 16-row pieces per block (log2)

    if (warp == kSched) {
        // ================================================================ scheduler ===
        // Runs one item ahead of the MMA / softmax warps (and up to kNCh piece lists ahead of
        // the producer): claims work items, writes each member's new K/V row to its cache
        // slot, and turns the members' block tables into lists of distinct pieces, so the
        // producer only issues copies and no item boundary waits on a global round trip.
        // An item is claimed only once the previous one has started, so no CTA hoards work
        // that an idle one could take at the end of the launch.
        uint32_t ccount = 0;
        auto take_chunk = [&]() -> int {
            const int c = (int)(ccount % kNCh);
            if (ccount >= (uint32_t)kNCh) mbar_wait(&chunk_empty[c], ((ccount / kNCh) - 1) & 1);
            return c;
        };
        for (uint32_t k = 0;; ++k) {
            const uint32_t slot = k & 3;
            if (k >= 1) mbar_wait(&item_empty[(k - 1) & 3], ((k - 1) >> 2) & 1);  // item k-1 has started
            int i = 0, myctx = 0, maxp = 0;
            TcItem it;
            for (bool first = k == 0;; first = false) {
                // first item by CTA index, later ones from the shared counter
                i = (int)blockIdx.x;
                if (!first) {
                    if (lane == 0) i = (int)gridDim.x + fetch_item(p.work_counter, p.epoch);
                    i = __shfl_sync(0xffffffffu, i, 0);
                }
                if (i >= p.n_items) break;
                it = tc_item(p, i);
                myctx = lane < it.gmv ? max(0, __ldg(p.context_lens + it.s0 + lane)) : 0;
                maxp = 0;
#pragma unroll
                for (int m = 0; m < kMaxGM; ++m) maxp = max(maxp, (__shfl_sync(0xffffffffu, myctx, m) + 15) >> 4);
                if (it.part == 0 || (it.part << p.part_log) < maxp) break;
                // a part past the group's longest context: so are the group's remaining items
                // (parts are consecutive), which a counter-claimed item may skip for everyone
                if (!first && lane == 0) {
                    const long long gend = (long long)(i / (p.n_hp * p.NPt) + 1) * (p.n_hp * p.NPt) - gridDim.x;
                    atomicMax(p.work_counter, ((unsigned long long)p.epoch << 32) | (unsigned long long)gend);
                }
            }
            if (lane == 0) {
                item_ring[slot] = i;
                mbar_arrive(&item_full[slot]);
            }
            if (i >= p.n_items) {  // terminal list: the producer stops
#ifdef PA_TC_TRACE
                if (lane == 0) TC_SPAN(3, k);
#endif
                const int c = take_chunk();
                if (lane == 0) {
                    chdr[c] = make_int4(i, 0, 1, 0);
                    mbar_arrive(&chunk_full[c]);
                }
                break;
            }
            // member's new token: written by the item of the part holding its last piece
            const int mypart = myctx > 0 ? min(((myctx - 1) >> 4) >> p.part_log, p.NPt - 1) : -1;
            const int myblk = mypart == it.part
                                  ? __ldg(p.block_tables + (int64_t)(it.s0 + lane) * p.W + ((myctx - 1) >> p.log2B))
                                  : 0;
            int ctxs[kMaxGM];
#pragma unroll
            for (int m = 0; m < kMaxGM; ++m) ctxs[m] = __shfl_sync(0xffffffffu, myctx, m);
            // reshape_and_cache of the step, first: member m's new K/V rows of the
            // quad's kv heads to slot ctx_m - 1, so that every piece below is read whole from
            // the cache (one box per tensor and half); lane = row (member, head w, K|V)
            for (int r0 = 0; r0 < it.gmv * 2 * kNH; r0 += 32) {
                const int r = r0 + lane, m = min(r >> 3, kMaxGM - 1), w = (r >> 1) & 3, t = r & 1;
                const int cm = __shfl_sync(0xffffffffu, myctx, m);
                const int blk = __shfl_sync(0xffffffffu, myblk, m);
                const int mp = __shfl_sync(0xffffffffu, mypart, m);
                if (r < it.gmv * 2 * kNH && cm > 0 && mp == it.part && ((it.st >> w) & 1u)) {
                    const int tp = cm - 1, kvw = sel4(it.kvh, w);
                    const int64_t dst = ((((int64_t)blk * p.H_kv + kvw) << p.log2B) + (tp & ((1 << p.log2B) - 1))) * 128;
                    const int64_t src = ((int64_t)(it.s0 + m) * p.H_kv + kvw) * 128;
                    const uint4* sp = reinterpret_cast<const uint4*>(static_cast<const T*>(t ? p.new_value : p.new_key) + src);
                    uint4* dp = reinterpret_cast<uint4*>(static_cast<T*>(t ? p.value_cache : p.key_cache) + dst);
                    uint4 v[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) v[u] = __ldg(sp + u);
#pragma unroll
                    for (int u = 0; u < 16; ++u) dp[u] = v[u];
                }
            }
            fence_proxy_async_global();  // the rows above are read by the producer's TMA copies
            __syncwarp();
            const int pbeg = it.part << p.part_log, pend = it.part == p.NPt - 1 ? maxp : min(maxp, pbeg + (1 << p.part_log));
            for (int p0 = pbeg; p0 < max(pend, pbeg + 1); p0 += 32) {
                // distinct pieces of 32 logical positions: lane = position
                const int c = take_chunk();
                int2* list = clist + c * kListCap;
                const int pp = p0 + lane;
                int id[kMaxGM];
#pragma unroll
                for (int m = 0; m < kMaxGM; ++m) {
                    id[m] = -1;
                    if (m < it.gmv && pp < pend && pp < ((ctxs[m] + 15) >> 4)) {
                        const int blk =
                            __ldg(p.block_tables + (int64_t)(it.s0 + m) * p.W + ((pp << 4) >> p.log2B));
                        id[m] = (blk << ppb_log) | (pp & ((1 << ppb_log) - 1));
                    }
                }
                unsigned lead = 0;
#pragma unroll
                for (int m = 0; m < kMaxGM; ++m) {
                    bool first = id[m] >= 0;
#pragma unroll
                    for (int m2 = 0; m2 < m; ++m2) first = first && id[m2] != id[m];
                    if (first) lead |= 1u << m;
                }
                const int n = __popc(lead);
                int incl = n;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += v;
                }
                const int total = __shfl_sync(0xffffffffu, incl, 31);
                int e = incl - n;
#pragma unroll
                for (int m = 0; m < kMaxGM; ++m) {
                    if ((lead >> m) & 1u) {
                        int own = 0, nrows = 0;
#pragma unroll
                        for (int m2 = 0; m2 < kMaxGM; ++m2) {
                            if (id[m2] == id[m]) {
                                own |= 1 << m2;
                                nrows = max(nrows, min(16, ctxs[m2] - 16 * pp));
                            }
                        }
                        list[e++] = make_int2(id[m], (pp << 18) | (own << 10) | (nrows << 4));
                    }
                }
                __syncwarp();
                if (lane == 0) {
#ifdef PA_TC_TRACE
                    if (ccount == 0) TC_SPAN(7, gtimer());
#endif
                    chdr[c] = make_int4(i, total, p0 + 32 >= pend ? 1 : 0, 0);
                    mbar_arrive(&chunk_full[c]);
                }
                ++ccount;
            }
        }
    } else if (warp == kProd || warp == kVProd) {
        // ================================================================ producers ===
        // Two warps issue the TMA copies of the scheduler's piece lists, kSlots pieces per
        // tile: K into the K ring (a buffer is free again once S has completed) and V into
        // the deeper V ring (free once P V has completed), so K of later tiles is not held
        // back by the softmax -> P V chain.  Both walk the same lists with the same tiling.
        const bool isv = warp == kVProd;
        const int nbuf = isv ? kBV : kBK;
        uint64_t* fullb = isv ? v_full : k_full;
        uint64_t* emptyb = isv ? v_empty : k_empty;
        unsigned char* base = isv ? sV : sK;
        const CUtensorMap* mq = isv ? &p.tmap_vq : &p.tmap_kq;
        const CUtensorMap* m1 = isv ? &p.tmap_v[0] : &p.tmap_k[0];
        uint32_t tcount = 0, ccount = 0;
        int fill = 0, b = 0;
        unsigned char* tb = base;
        auto acquire = [&]() {
            b = (int)(tcount % nbuf);
            if (tcount >= (uint32_t)nbuf) mbar_wait(&emptyb[b], ((tcount / nbuf) - 1) & 1);
            tb = base + b * kTensor;
        };
        auto publish = [&](int ns, int last) {  // lane 0
#ifdef PA_TC_TRACE
            if (!isv && tcount == 0) TC_SPAN(5, gtimer());
#endif
            if (isv) {
                meta[b].ns = ns;
                meta[b].last = last;
            } else {
                kmeta[b] = make_int2(ns, last);
                TC_T(tcount, 1);
            }
            mbar_arrive(&fullb[b]);
        };
        for (;;) {
            const int c = (int)(ccount % kNCh);
            mbar_wait(&chunk_full[c], (ccount / kNCh) & 1);
            const volatile int* hv = reinterpret_cast<const volatile int*>(&chdr[c]);
            const int i = hv[0], total = hv[1], last_chunk = hv[2];
            if (i >= p.n_items) {
#ifdef PA_TC_TRACE
                if (!isv && lane == 0) TC_SPAN(4, tcount);
#endif
                break;
            }
            const TcItem it = tc_item(p, i);
            const int2* list = clist + c * kListCap;
            const bool quad_box = it.quad && p.log2B == 4;  // the 4 kv heads' pieces are 64 adjacent rows
            for (int q = 0; q < total;) {
                if (fill == 0) {
                    acquire();
                    if (lane == 0 && !isv) TC_T(tcount, 0);
                }
                // the next k2 pieces of the open tile are issued together
                const int k2 = min(kSlots - fill, total - q);
                uint64_t* bar = &fullb[b];
                if (lane == 0) {
                    if (isv) {
                        for (int jj = 0; jj < k2; ++jj) {
                            const int y = list[q + jj].y;
                            meta[b].p[fill + jj] = y >> 18;
                            meta[b].own[fill + jj] = (y >> 10) & 0xff;
                            meta[b].nrows[fill + jj] = (y >> 4) & 31;
                        }
                    }
                    mbar_expect_tx(bar, (uint32_t)k2 * (uint32_t)kQuad * 2u);  // whole pieces, 2 halves
                }
                __syncwarp();
                {   // whole pieces (rows past a context are read but never used; V's are zeroed
                    // in shared memory by the softmax warps).  quad: lane = (piece, half), the 4
                    // kv heads' rows in ONE 64-row box; otherwise lane = (piece, half, head)
                    const int jj = quad_box ? (lane >> 1) : (lane >> 3);
                    const int cc = quad_box ? (lane & 1) : ((lane >> 2) & 1), w = lane & 3;
                    if (jj < k2) {
                        const int2 ent = list[q + jj];
                        const int blk = ent.x >> ppb_log, pc = ent.x & ((1 << ppb_log) - 1);
                        unsigned char* dst = tb + cc * kHalfReg + (fill + jj) * kQuad;
                        if (quad_box) {
                            tma_load_2d(dst, mq, cc * 64, (blk * p.H_kv + it.kvh[0]) << 4, bar);
                        } else {
                            tma_load_2d(dst + w * kPiece, m1, cc * 64,
                                        ((blk * p.H_kv + sel4(it.kvh, w)) << p.log2B) | (pc << 4), bar);
                        }
                    }
                }
                __syncwarp();
                fill += k2;
                q += k2;
                // the item's last piece closes its tile (last = 1: no empty tile takes a buffer)
                const bool item_end = last_chunk && q == total;
                if (fill == kSlots || item_end) {
                    if (lane == 0) publish(fill, item_end ? 1 : 0);
                    ++tcount;
                    fill = 0;
                }
            }
            __syncwarp();  // every lane has read the list before the scheduler rewrites it
            if (lane == 0) mbar_arrive(&chunk_empty[c]);
            ++ccount;
            if (last_chunk && total == 0) {  // an item without pieces (every context 0): an empty tile closes it
                if (fill == 0) acquire();
                if (lane == 0) publish(fill, 1);
                ++tcount;
                fill = 0;
                __syncwarp();
            }
        }
    } else if (warp == kMma) {
        // ================================================================ MMA issuer ===
        // One set of products covers the item's kNH heads: A rows (tensor-memory lanes)
        // 32w..32w+31 hold head w's members, and the B rows of each piece are head 0's 16 K
        // rows, then head 1's, ...  S (N = 16 kNH per piece) is then block-diagonal -- the
        // off-diagonal products are computed and ignored -- and P carries zeros off the
        // diagonal, so O = P V accumulates each head's rows from its own V rows only.
        // One thread issues everything (tcgen05.mma is single-thread); descriptors are
        // built once and stepped by constant offsets (address field = bytes >> 4).
        if (lane == 0) {
            const uint32_t idesc_o = umma_idesc(kBF16, true, 128);
            const uint64_t kdesc0 = umma_desc_sw128(smem_u32(sK), 16, 1024);
            const uint64_t vdesc0 = umma_desc_sw128(smem_u32(sV), kHalfReg, 1024);
            uint32_t tcount = 0, nitem = 0, scount = 0, pvitems = 0, pv_issued = 0, pv_pub = 0;
            // the completion of every issued P V, in order, published to the softmax warps as
            // a tile index in shared memory (they wait on it only to rescale O -- rarely).
            // P V k commits to o_step[k & 1]; at most two are unpublished, so no barrier ever
            // runs two phases ahead of this thread's waits
            auto publish_one = [&](bool block) -> bool {
                if (pv_pub >= pv_issued) return false;
                uint64_t* bar = &o_step[pv_pub & 1];
                const uint32_t par = (pv_pub >> 1) & 1;
                if (block) {
                    mbar_wait(bar, par);
                } else if (!mbar_test(bar, par)) {
                    return false;
                }
                tc_fence_after();
                *pv_done = (int)pv_pub;
                ++pv_pub;
                return true;
            };
            auto issue_pv = [&](uint32_t ptile, uint32_t pt, int pns, bool started, bool last_pv) {
                const uint32_t sb = pt & 1;
                const int vb = (int)(ptile % kBV);
                while (pv_pub + 2 <= pv_issued) publish_one(true);
                while (publish_one(false)) {
                }
                mbar_wait(&p_full[sb], (pt >> 1) & 1);
                TC_T(pt, 3);
                if (!started) {  // the item's first P V overwrites O: the previous epilogue must be done
                    if (pvitems > 0) mbar_wait(o_free, (pvitems - 1) & 1);
                    ++pvitems;
                }
                mbar_wait(&v_full[vb], (ptile / kBV) & 1);  // V landed (the softmax saw it too, before P)
                tc_fence_after();
                const uint64_t vd = vdesc0 + (uint64_t)((vb * kTensor) >> 4);
                const uint32_t pa = tmem + kTmS + sb * kSCols;
                for (int j = 0; j < pns; ++j)
#pragma unroll
                    for (int w = 0; w < kNH; ++w)  // k-step = one head's 16 rows of piece j
                        umma_f16_ts(tmem + kTmO, pa + 8 * kNH * j + 8 * w,
                                    vd + (uint64_t)((j * kQuad + w * kPiece) >> 4), idesc_o,
                                    (started || j > 0 || w > 0) ? 1u : 0u);
                umma_commit(&o_step[pv_issued & 1]);
                if (last_pv) umma_commit(o_last);
                umma_commit(&v_empty[vb]);
                ++pv_issued;
            };
            for (uint32_t k = 0;; ++k) {
                const uint32_t slot = k & 3;
                mbar_wait(&item_full[slot], (k >> 2) & 1);
                const int i = *reinterpret_cast<volatile int*>(&item_ring[slot]);
                mbar_arrive(&item_empty[slot]);
                if (i >= p.n_items) break;
                const uint32_t qb = nitem & 1;
                bool q_seen = false, started = false;
                int pend_ns = 0;
                bool pend = false;
                uint32_t pend_t = 0, pend_tile = 0;
                for (;;) {
                    const uint32_t tile = tcount;
                    const int kb = (int)(tile % kBK);
                    mbar_wait(&k_full[kb], (tile / kBK) & 1);
                    TC_T(tcount, 2);
                    ++tcount;
                    const int ns = *reinterpret_cast<volatile int*>(&kmeta[kb].x);
                    const int last = *reinterpret_cast<volatile int*>(&kmeta[kb].y);
                    uint32_t t = 0;
                    if (ns > 0) {
                        if (!q_seen) {  // the softmax warps have put this item's queries in tensor memory
                            mbar_wait(&q_full[qb], (nitem >> 1) & 1);
                            q_seen = true;
                        }
                        t = scount++;
                        const uint32_t sb = t & 1;
                        tc_fence_after();
                        const uint32_t idesc_s = umma_idesc(kBF16, false, 16 * kNH * ns);
                        const uint64_t kd = kdesc0 + (uint64_t)((kb * kTensor) >> 4);
                        const uint32_t d = tmem + kTmS + sb * kSCols, qa = tmem + kTmQ + 64 * qb;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)  // S = Q (tensor memory) x K^T (all pieces, all heads)
                            umma_f16_ts(d, qa + 8 * kk, kd + (uint64_t)(((kk >> 2) * kHalfReg + (kk & 3) * 32) >> 4),
                                        idesc_s, kk > 0 ? 1u : 0u);
                        umma_commit(&s_full[sb]);
                        TC_T(tcount - 1, 7);
                    }
                    umma_commit(&k_empty[kb]);  // K is free once S has completed
                    if (pend) {
                        issue_pv(pend_tile, pend_t, pend_ns, started, last && ns == 0);
                        started = true;
                        pend = false;
                    }
                    if (ns > 0) {
                        pend = true;
                        pend_tile = tile;
                        pend_t = t;
                        pend_ns = ns;
                    } else {  // an empty tile: its V slot is released once it is this tile's
                        const int vb = (int)(tile % kBV);
                        mbar_wait(&v_full[vb], (tile / kBV) & 1);
                        umma_commit(&v_empty[vb]);
                    }
                    if (last) break;
                }
                if (pend) issue_pv(pend_tile, pend_t, pend_ns, started, true);
                if (!q_seen) mbar_wait(&q_full[qb], (nitem >> 1) & 1);  // keep the q_full phases in step
                ++nitem;
            }
        }
        __syncwarp();
    } else if (warp >= kEpi0) {
        // ================================================================ epilogue ===
        // Per item, after its last P V: O (this warp's lane quadrant = head hh) / L to `out`
        // -- or, for rows with a split context, O / L and (m, L), merged by the last part -- so the
        // softmax warps go straight on to the next item's scores
        const int hh = warp - kEpi0;
        const uint32_t tO = tmem + ((uint32_t)(32 * hh) << 16) + kTmO;
        uint32_t ocount = 0;
        for (uint32_t e = 0;; ++e) {
            const uint32_t es = e & 1;
            mbar_wait(&st_full[es], (e >> 1) & 1);
            const int i_cur = *reinterpret_cast<volatile int*>(&st_item[es]);
            const volatile float* sv4 = reinterpret_cast<const volatile float*>(&stats[(es * kNH + hh) * 32 + lane]);
            const float4 stv = make_float4(sv4[0], sv4[1], sv4[2], sv4[3]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&st_empty[es]);
            if (i_cur < 0) break;
            const TcItem it = tc_item(p, i_cur);
            const bool member = lane < it.gmv;
            const float mref = stv.x, l = stv.y;
            const int npv = __float_as_int(stv.z), ctx = __float_as_int(stv.w);
            TC_EP(e, 0);
            if (npv > 0) {
                mbar_wait(o_last, ocount & 1);  // one phase per item with tiles
                ++ocount;
                tc_fence_after();
            }
            TC_EP(e, 1);
            const float inv = l > 0.f ? 1.f / l : 0.f;
            // split context (a6): parts holding this member's tokens; with more than one,
            // each part publishes (m, L, O / L) and the last to finish merges
            const int nps = max(1, min((ctx + (16 << p.part_log) - 1) >> (4 + p.part_log), p.NPt));
            const bool mine = member && ((it.st >> hh) & 1u) && it.part < nps;
            const bool split = mine && nps > 1;
            const bool store = mine && !split;
            const int64_t sh = (int64_t)(it.s0 + lane) * p.H + sel4(it.h, hh);
            T* orow = static_cast<T*>(p.out) + sh * 128;
            float* prow = p.part_o + (sh * p.NPt + it.part) * 128;
            // O in two 64-column halves (one wait each); tensor memory is released to the next
            // item's P V once both are in registers, before the second half's stores
            auto emit = [&](const float (&v)[32], int c0) {
                if (split) {
#pragma unroll
                    for (int c1 = 0; c1 < 32; c1 += 4)
                        *reinterpret_cast<float4*>(prow + c0 + c1) =
                            make_float4(v[c1] * inv, v[c1 + 1] * inv, v[c1 + 2] * inv, v[c1 + 3] * inv);
                }
                if (store) {
#pragma unroll
                    for (int c1 = 0; c1 < 32; c1 += 8) {
                        uint4 w;
                        w.x = pack2<T>(v[c1] * inv, v[c1 + 1] * inv);
                        w.y = pack2<T>(v[c1 + 2] * inv, v[c1 + 3] * inv);
                        w.z = pack2<T>(v[c1 + 4] * inv, v[c1 + 5] * inv);
                        w.w = pack2<T>(v[c1 + 6] * inv, v[c1 + 7] * inv);
                        *reinterpret_cast<uint4*>(orow + c0 + c1) = w;
                    }
                }
            };
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                float ov[2][32];
                if (npv > 0) {
                    tmem_ld32_nw(tO + 64 * hf, ov[0]);
                    tmem_ld32_nw(tO + 64 * hf + 32, ov[1]);
                    tmem_ld_wait();
                    if (hf == 1) {
                        TC_EP(e, 4);
                        tc_fence_before();
                        mbar_arrive(o_free);
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int u = 0; u < 32; ++u) ov[c][u] = 0.f;
                }
                emit(ov[0], 64 * hf);
                emit(ov[1], 64 * hf + 32);
            }
            TC_EP(e, 2);
            // split rows (a6): (m, L) next to O / L, counted in; the part that completes a row's
            // set merges it: o = sum_j L_j 2^(m_j - M) o~_j / sum_j L_j 2^(m_j - M), in part
            // order (deterministic whichever CTA merges)
            if (__any_sync(0xffffffffu, split)) {
                bool done = false;
                if (split) {
                    p.part_ml[sh * p.NPt + it.part] = make_float2(mref, l);
                    __threadfence();
                    done = split_done(p, sh, nps);
                }
                unsigned todo = __ballot_sync(0xffffffffu, done);
                if (todo) __threadfence();
            while (todo) {  // whole warp merges row r: lane = 4 dims
                const int r = __ffs(todo) - 1;
                todo &= todo - 1;
                const int np = __shfl_sync(0xffffffffu, nps, r);
                const int64_t shr = __shfl_sync(0xffffffffu, sh, r);
                const float2* ml = p.part_ml + shr * p.NPt;
                const float4* po = reinterpret_cast<const float4*>(p.part_o + shr * p.NPt * 128) + lane;
                float M = -INFINITY, L = 0.f;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int j0 = 0; j0 < np; j0 += 4) {
                    float2 mv[4];
                    float4 pv[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (j0 + u < np) {
                            mv[u] = __ldcg(&ml[j0 + u]);
                            pv[u] = __ldcg(po + (j0 + u) * 32);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (j0 + u < np) {
                            const float Mn = fmaxf(M, mv[u].x);
                            const float sc = ex2(M - Mn), wj = mv[u].y * ex2(mv[u].x - Mn);
                            o.x = o.x * sc + wj * pv[u].x;
                            o.y = o.y * sc + wj * pv[u].y;
                            o.z = o.z * sc + wj * pv[u].z;
                            o.w = o.w * sc + wj * pv[u].w;
                            L = L * sc + wj;
                            M = Mn;
                        }
                    }
                }
                const float il = 1.f / L;
                uint2 st;
                st.x = pack2<T>(o.x * il, o.y * il);
                st.y = pack2<T>(o.z * il, o.w * il);
                *reinterpret_cast<uint2*>(static_cast<T*>(p.out) + shr * 128 + 4 * lane) = st;
            }
            }
            TC_EP(e, 3);
        }
    } else {
        // ================================================================ softmax ===
        const int hh = warp;  // head w of the quad = TMEM lane quadrant w
        const uint32_t lane_base = (uint32_t)(32 * hh) << 16;
        const uint32_t tO = tmem + lane_base + kTmO;
        const float c2 = p.scale_log2;
        uint32_t tcount = 0, scount = 0, ocount = 0, nq = 0;
        // the members' query rows of this head into tensor memory (the A operand of S = Q K^T):
        // lane m = member m's row (16-bit pairs), signalled on q_full[nq & 1]
        int ctx_next = 0;  // the next item's context length of this lane's member, loaded with its queries
        auto put_q = [&](const TcItem& q_it) {
            const bool mem = lane < q_it.gmv;  // tcgen05.st is warp-collective: other lanes store zeros
            ctx_next = mem ? max(0, __ldg(p.context_lens + q_it.s0 + lane)) : 0;
            const uint4* src = reinterpret_cast<const uint4*>(static_cast<const T*>(p.query) +
                                                              ((int64_t)(q_it.s0 + (mem ? lane : 0)) * p.H +
                                                               sel4(q_it.h, hh)) * 128);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t w0[16], w1[16];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint4 v0 = mem ? __ldg(src + 8 * half + c) : make_uint4(0u, 0u, 0u, 0u);
                    const uint4 v1 = mem ? __ldg(src + 8 * half + 4 + c) : make_uint4(0u, 0u, 0u, 0u);
                    w0[4 * c] = v0.x;
                    w0[4 * c + 1] = v0.y;
                    w0[4 * c + 2] = v0.z;
                    w0[4 * c + 3] = v0.w;
                    w1[4 * c] = v1.x;
                    w1[4 * c + 1] = v1.y;
                    w1[4 * c + 2] = v1.z;
                    w1[4 * c + 3] = v1.w;
                }
                tmem_st16(tmem + lane_base + kTmQ + 64 * (nq & 1) + 32 * half, w0);
                tmem_st16(tmem + lane_base + kTmQ + 64 * (nq & 1) + 32 * half + 16, w1);
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&q_full[nq & 1]);
            ++nq;
        };
        uint32_t nep = 0;  // items handed to the epilogue warps
        int i = 0;
        {
            mbar_wait(&item_full[0], 0);
            i = *reinterpret_cast<volatile int*>(&item_ring[0]);
            if (i < p.n_items) put_q(tc_item(p, i));
        }
        for (uint32_t k = 0;; ++k) {
            const uint32_t slot = k & 3;
            if (k > 0) {
                mbar_wait(&item_full[slot], (k >> 2) & 1);
                i = *reinterpret_cast<volatile int*>(&item_ring[slot]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&item_empty[slot]);
            if (i >= p.n_items) break;
            const int i_cur = i;
            const TcItem it = tc_item(p, i);
            const bool member = lane < it.gmv;
            const int ctx = ctx_next;  // loaded when this item's queries were (off the item boundary)
            float mref = -INFINITY, l = 0.f;
            int npv = 0;
            bool qnext = false;  // the next item's queries are in the other Q buffer already
            const uint32_t nslot = (k + 1) & 3, npar = ((k + 1) >> 2) & 1;
            for (;;) {
                if (!qnext) {  // as soon as the producer has published the next item
                    int ready = lane == 0 ? (int)mbar_test(&item_full[nslot], npar) : 0;
                    ready = __shfl_sync(0xffffffffu, ready, 0);
                    if (ready) {
                        const int i2 = *reinterpret_cast<volatile int*>(&item_ring[nslot]);
                        if (i2 < p.n_items) put_q(tc_item(p, i2));
                        qnext = true;
                    }
                }
                const int b = (int)(tcount % kBV);
                mbar_wait(&v_full[b], (tcount / kBV) & 1);  // V landed and the tile's meta written
                ++tcount;
                const int ns = *reinterpret_cast<volatile int*>(&meta[b].ns);
                const int last = *reinterpret_cast<volatile int*>(&meta[b].last);
                int vm[kSlots], nr[kSlots];
#pragma unroll
                for (int j = 0; j < kSlots; ++j) {
                    const int own = *reinterpret_cast<volatile int*>(&meta[b].own[j]);
                    const int pj = *reinterpret_cast<volatile int*>(&meta[b].p[j]);
                    nr[j] = j < ns ? *reinterpret_cast<volatile int*>(&meta[b].nrows[j]) : 16;
                    vm[j] = (j < ns && member && ((own >> lane) & 1)) ? min(16, ctx - 16 * pj) : 0;
                }
                // V rows past the last context in a piece were loaded from unused cache slots:
                // zero this head's (P = 0 there, but 0 x NaN = NaN in the product)
#pragma unroll
                for (int j = 0; j < kSlots; ++j) {
                    if (nr[j] < 16) {
                        unsigned char* vb = sV + b * kTensor + j * kQuad + hh * kPiece;
                        for (int u = lane; u < (16 - nr[j]) * 16; u += 32) {
                            const int row = nr[j] + (u >> 4), half = (u >> 3) & 1, ch = u & 7;
                            *reinterpret_cast<uint4*>(vb + half * kHalfReg + row * 128 + ch * 16) =
                                make_uint4(0u, 0u, 0u, 0u);
                        }
                    }
                }
                fence_proxy_async_smem();  // before the P V product reads them (after p_full)
                __syncwarp();
                if (lane == 0) mbar_arrive(&v_empty[b]);
                if (ns > 0) {
                    const uint32_t t = scount++, sb = t & 1;
                    mbar_wait(&s_full[sb], (t >> 1) & 1);
                    if (lane == 0 && hh == 0) TC_T(t, 4);
                    tc_fence_after();
                    const uint32_t tS = tmem + lane_base + kTmS + sb * kSCols;
                    // this head's 16 columns of every piece (the diagonal block)
                    float sv[kSlots][16];
#pragma unroll
                    for (int j = 0; j < kSlots; ++j) tmem_ld16_nw(tS + 16 * kNH * j + 16 * hh, sv[j]);
                    tmem_ld_wait();
                    float mt = -INFINITY;
#pragma unroll
                    for (int j = 0; j < kSlots; ++j)
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            sv[j][u] *= c2;
                            if (u < vm[j]) mt = fmaxf(mt, sv[j][u]);
                        }
                    const bool bump = __any_sync(0xffffffffu, mt > mref + kLazyTc);
                    const float mn = bump ? fmaxf(mref, mt) : mref;
                    const float ms = (mn == -INFINITY) ? 0.f : mn;
                    const float alpha = bump ? ex2(mref - ms) : 1.f;
                    float rs = 0.f;
#pragma unroll
                    for (int j = 0; j < kSlots; ++j) {
                        // packed P of piece j (8 kNH columns): this head's 8, zeros elsewhere
                        uint32_t pk[8 * kNH];
#pragma unroll
                        for (int u = 0; u < 16; u += 2) {
                            const float a0 = u < vm[j] ? ex2(sv[j][u] - ms) : 0.f;
                            const float a1 = u + 1 < vm[j] ? ex2(sv[j][u + 1] - ms) : 0.f;
                            rs += a0 + a1;
                            const uint32_t pv = pack2<T>(a0, a1);
#pragma unroll
                            for (int w = 0; w < kNH; ++w) pk[8 * w + u / 2] = hh == w ? pv : 0u;
                        }
                        uint32_t pa[16], pb2[16];
#pragma unroll
                        for (int u = 0; u < 16; ++u) {
                            pa[u] = pk[u];
                            pb2[u] = pk[16 + u];
                        }
                        tmem_st16(tS + 8 * kNH * j, pa);
                        tmem_st16(tS + 8 * kNH * j + 16, pb2);
                    }
                    if (lane == 0 && hh == 0) TC_T(t, 5);
                    if (npv > 0 && bump) {  // O is rescaled once P V of the previous tile has completed
                        while (*pv_done < (int)t - 1) {
                        }
                        tc_fence_after();
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
                    l = l * alpha + rs;
                    mref = mn;
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(&p_full[sb]);
                    if (lane == 0 && hh == 0) TC_T(t, 6);
                    ++npv;
                }
                if (last) break;
            }
            // every S of this item has been read: the next item's queries may replace Q now,
            // so the MMA warp can start it while this epilogue runs
            {
                mbar_wait(&item_full[nslot], npar);
                const int i2 = *reinterpret_cast<volatile int*>(&item_ring[nslot]);
                if (!qnext && i2 < p.n_items) put_q(tc_item(p, i2));
                i = i2;
            }
            // ---- hand the item's epilogue (O / L to out) to the epilogue warps
            {
                const uint32_t es = nep & 1;
                if (nep >= 2) mbar_wait(&st_empty[es], ((nep >> 1) - 1) & 1);
                stats[(es * kNH + hh) * 32 + lane] = make_float4(mref, l, __int_as_float(npv), __int_as_float(ctx));
                if (hh == 0 && lane == 0) st_item[es] = i_cur;
                __syncwarp();
                if (lane == 0) mbar_arrive(&st_full[es]);
                ++nep;
            }
        }
        {   // no more items
            const uint32_t es = nep & 1;
            if (nep >= 2) mbar_wait(&st_empty[es], ((nep >> 1) - 1) & 1);
            if (hh == 0 && lane == 0) st_item[es] = -1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&st_full[es]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
#ifdef PA_TC_TRACE
    if (tid == 0) TC_SPAN(2, gtimer());
#endif
}

#ifdef PA_TC_TRACE
extern "C" int pa_debug_tc_trace_reset(void) {
    void* a = nullptr;
    void* b = nullptr;
    cudaGetSymbolAddress(&a, g_tc_trace);
    cudaGetSymbolAddress(&b, g_tc_span);
    cudaMemset(a, 0, sizeof(g_tc_trace));
    cudaGetSymbolAddress(&a, g_tc_ep);
    cudaMemset(a, 0, sizeof(g_tc_ep));
    return (int)cudaMemset(b, 0, sizeof(g_tc_span));
}
extern "C" int pa_debug_tc_ep(void* host_out, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host_out, g_tc_ep, bytes < sizeof(g_tc_ep) ? bytes : sizeof(g_tc_ep));
}
extern "C" int pa_debug_tc_span(void* host_out, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host_out, g_tc_span, bytes < sizeof(g_tc_span) ? bytes : sizeof(g_tc_span));
}
extern "C" int pa_debug_tc_trace(void* host_out, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host_out, g_tc_trace, bytes < sizeof(g_tc_trace) ? bytes : sizeof(g_tc_trace));
}
#endif

size_t group_tc_smem_bytes() {
    return 1024 + (size_t)(kBK + kBV) * kTensor + kBV * sizeof(TileMeta) + kBK * sizeof(int2) +
           kNCh * kListCap * sizeof(int2) + 16 +
           kNCh * sizeof(int4) + kNumBars * 8 + 12 * 4 + 16 + 2 * kNH * 32 * sizeof(float4) + 16;
}

cudaError_t launch_group_tc(const GroupTcParams& p, int dtype, cudaStream_t stream) {
    const size_t smem = group_tc_smem_bytes();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::max(1, std::min(sms, p.n_items));
    if (dtype == 2) {
        cudaError_t e = ensure_smem_attr((const void*)paged_attention_group_tc_kernel<__nv_bfloat16>, smem);
        if (e != cudaSuccess) return e;
        return launch_k(paged_attention_group_tc_kernel<__nv_bfloat16>, dim3(grid), dim3(kThreadsTc), smem, stream, p);
    }
    cudaError_t e = ensure_smem_attr((const void*)paged_attention_group_tc_kernel<__half>, smem);
    if (e != cudaSuccess) return e;
    return launch_k(paged_attention_group_tc_kernel<__half>, dim3(grid), dim3(kThreadsTc), smem, stream, p);
}

}  // namespace pa
