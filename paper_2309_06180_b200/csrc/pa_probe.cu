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
