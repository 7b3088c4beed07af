// pa_tp.cu -- completion handshake of the fused tensor-parallel all-gather.
//
// each GPU worker computes the attention of its subset of heads with the same
// block tables; the head slices are then gathered.  In the fused path the attention
// kernel itself stores every output row into every rank's gather buffer (peer memory over
// NVLink, pointers opened with CUDA IPC), so the only collective work left is this
// handshake: rank r publishes `epoch` in slot r of every rank's flag array (system-scope
// release, after the stream-ordered attention kernel), then waits until every rank has
// published `epoch` in its own array (system-scope acquire).  The wait is bounded: after
// timeout_ns it sets *status = 1 and returns instead of hanging the GPU.
#include "pa_common.cuh"
#include "pa_internal.h"

namespace pa {

namespace {

struct TpSignalParams {
    int32_t* flags[kMaxTpPeers];  // flags[k] = rank k's flag array [world] (peer memory)
    int32_t* status;
    long long timeout_ns;
    int world, rank;
    int32_t epoch;
};

__device__ __forceinline__ void st_release_sys(int32_t* p, int32_t v) {
    asm volatile("st.release.sys.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_acquire_sys(const int32_t* p) {
    int32_t v;
    asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void tp_signal_wait_kernel(const __grid_constant__ TpSignalParams p) {
    pdl_wait();  // the attention kernel (and its peer stores) has completed
    const int k = threadIdx.x;
    if (k < p.world) {
        __threadfence_system();
        st_release_sys(p.flags[k] + p.rank, p.epoch);
    }
    __syncwarp();
    if (k < p.world) {
        const int32_t* mine = p.flags[p.rank] + k;
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(mine) - p.epoch < 0) {  // wrap-safe epoch compare
            __nanosleep(64);
            if ((long long)(globaltimer() - t0) > p.timeout_ns) {
                atomicExch(p.status, 1);
                break;
            }
        }
    }
}

}  // namespace

cudaError_t launch_tp_signal_wait(int32_t* const* flag_peers, int world, int rank, int32_t epoch, int32_t* status,
                                  long long timeout_ns, cudaStream_t stream) {
    TpSignalParams p{};
    for (int k = 0; k < world; ++k) p.flags[k] = flag_peers[k];
    p.status = status;
    p.timeout_ns = timeout_ns;
    p.world = world;
    p.rank = rank;
    p.epoch = epoch;
    return launch_k(tp_signal_wait_kernel, dim3(1), dim3(32), 0, stream, p);
}

}  // namespace pa
