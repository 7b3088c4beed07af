// pa_probe.cu -- read-only HBM streaming probe (measurement helper, not on the hot path).
//
// The attention kernel's roofline is a READ stream (K/V in, a few MB out), while the
// driver's MEASURED_PEAKS hbm_gbs is a device-to-device copy (read + write).  This probe
// gives the same-run read-only ceiling with the attention kernel's own load mechanism:
// persistent CTAs stream disjoint chunks of a buffer into shared memory with 1-D bulk
// copies (cp.async.bulk, SASS UBLKCP) completing on mbarriers, and never write to global
// memory except one 4-byte word per CTA (so the loads are observable).  Bytes read / time
// = the highest read bandwidth this mechanism reaches.
#include "pa_common.cuh"
#include "pa_internal.h"

namespace pa {

// One elected thread per CTA keeps `stages` bulk copies of `chunk` bytes in flight:
// wait stage s, fold one word of it into the checksum, refill it with the CTA's next chunk.
__global__ void __launch_bounds__(32) hbm_read_probe_kernel(const char* __restrict__ buf, int64_t nchunks,
                                                            int chunk, int stages, uint32_t* __restrict__ sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);
    unsigned char* data = smem + 128;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
    const uint64_t pol = policy_evict_first();
    int64_t c = blockIdx.x;
    int issued = 0;
    for (; issued < stages && c < nchunks; ++issued, c += gridDim.x) {
        mbar_arrive_expect_tx(&bar[issued], chunk);
        bulk_g2s_hint(data + (size_t)issued * chunk, buf + c * chunk, chunk, &bar[issued], pol);
    }
    uint32_t acc = 0;
    int64_t done = 0;
    const int64_t mine = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    for (; done < mine; ++done) {
        const int s = (int)(done % stages);
        const uint32_t par = (uint32_t)((done / stages) & 1);
        mbar_wait(&bar[s], par);
        acc ^= *reinterpret_cast<const uint32_t*>(data + (size_t)s * chunk + ((done * 64) % chunk));
        if (c < nchunks) {
            mbar_arrive_expect_tx(&bar[s], chunk);
            bulk_g2s_hint(data + (size_t)s * chunk, buf + c * chunk, chunk, &bar[s], pol);
            c += gridDim.x;
        }
    }
    sink[blockIdx.x] = acc;
}

cudaError_t launch_hbm_read_probe(const void* buf, int64_t nchunks, int chunk, int stages, int grid, uint32_t* sink,
                                  cudaStream_t stream) {
    const size_t smem = 128 + (size_t)stages * chunk;
    cudaError_t e = ensure_smem_attr((const void*)hbm_read_probe_kernel, smem);
    if (e != cudaSuccess) return e;
    count_launch();
    hbm_read_probe_kernel<<<grid, 32, smem, stream>>>(static_cast<const char*>(buf), nchunks, chunk, stages, sink);
    return cudaGetLastError();
}

}  // namespace pa

// ---- TMA tensor-copy throughput probe (test-only) ---------------------------
// `warps` issuing warps per CTA (one elected lane each) stream 128-byte-swizzled 2-D boxes
// {64 cols, rows} of a [nrows][128] 2-byte tensor into `stages` shared-memory slots per warp,
// at pseudo-random row offsets (box-aligned), `iters` boxes per warp.  Bytes / time = the
// tensor-copy ceiling of one SM for that box shape.
#include "pa_tc.cuh"
namespace pa {
__global__ void __launch_bounds__(256) tma_probe_kernel(const __grid_constant__ CUtensorMap map, int nrows, int rows,
                                                        int stages, int iters, uint32_t* sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem =
        tc::smem_align1024(smem_raw);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int box = rows * 128;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nw * stages * box);
    if (threadIdx.x < nw * stages) mbar_init(&bars[threadIdx.x], 1);
    fence_mbar_init();
    __syncthreads();
    if (lane != 0) return;
    uint64_t* wb = bars + warp * stages;
    unsigned char* ws = smem + (size_t)warp * stages * box;
    uint32_t x = 2654435761u * (blockIdx.x * nw + warp + 1);
    const int nbox = nrows / rows;
    for (int it = 0; it < iters; ++it) {
        const int s = it % stages;
        if (it >= stages) mbar_wait(&wb[s], ((it / stages) - 1) & 1);
        x = x * 1664525u + 1013904223u;
        const int r = (int)((x >> 8) % (uint32_t)nbox) * rows;
        mbar_arrive_expect_tx(&wb[s], (uint32_t)box);
        tc::tma_load_2d(ws + (size_t)s * box, &map, (it & 1) * 64, r, &wb[s]);
    }
    for (int it = iters - stages; it < iters; ++it)
        if (it >= 0) mbar_wait(&wb[it % stages], (it / stages) & 1);
    sink[blockIdx.x * nw + warp] = x;
}
}  // namespace pa

extern "C" int pa_debug_tma_probe(const void* buf, long long nrows, int rows, int warps, int stages, int iters,
                                  int grid, uint32_t* sink, void* stream) {
    CUtensorMap map;
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return -1;
    auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                             CUtensorMapFloatOOBfill)>(fn);
    const cuuint64_t dims[2] = {128, (cuuint64_t)nrows};
    const cuuint64_t str[1] = {256};
    const cuuint32_t box[2] = {64, (cuuint32_t)rows};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(buf), dims, str, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return -2;
    const size_t smem = 1024 + (size_t)warps * stages * rows * 128 + 8 * warps * stages;
    if (cudaFuncSetAttribute(pa::tma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return -3;
    pa::tma_probe_kernel<<<grid, 32 * warps, smem, (cudaStream_t)stream>>>(map, (int)nrows, rows, stages, iters, sink);
    return (int)cudaGetLastError();
}
