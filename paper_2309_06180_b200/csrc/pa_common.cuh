// pa_common.cuh -- device helpers shared by the libpagedattn kernels (sm_100a only).
//
// PTX wrappers for the Blackwell async-copy path (1-D bulk copies completing on an
// mbarrier, SASS UBLKCP / SYNCS), the mixed-precision FMA (FHFMA: f16/bf16 x f16/bf16
// + f32 -> f32) and the packed fp32x2 FMA (FFMA2) that sm_100 adds.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libpagedattn is written for sm_100a (B200) only"
#endif

namespace pa {

constexpr int kTile = 16;  // logical tokens per attention tile, independent of block_size

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier ------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive (count 1) and raise the expected transaction bytes of the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// plain arrive (count 1, no transaction bytes): consumer releases a stage
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Spin until the phase with the given parity has completed.  The retry loop lives
// inside the asm so the compiler keeps the warp converged around the shuffles that follow.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "PA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra PA_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ---- 1-D bulk copy global -> shared, completion counted on an mbarrier ----------------
// bytes: multiple of 16; both addresses 16-byte aligned.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(smem_dst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ---- programmatic dependent launch (PDL) -----------------------------------------------
// Kernels of this library are launched with programmatic stream serialisation: a kernel
// may be scheduled while its predecessor drains, and blocks in pdl_wait() until the
// predecessor grid has completed and its memory is visible.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Plain global atomic add returning the old value.  Written in PTX so the compiler does
// not wrap it in its warp-aggregation sequence, whose shuffle of the returned value
// would expose the atomic's round trip at the call site instead of at first use.
__device__ __forceinline__ int atom_add_global(int* addr, int v) {
    int old;
    asm volatile("atom.relaxed.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(addr), "r"(v) : "memory");
    return old;
}

// ---- math -----------------------------------------------------------------------------
__device__ __forceinline__ float ex2(float x) {  // 2^x, ex2.approx (MUFU.EX2); ex2(-inf) = +0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// acc += lo(a)*lo(b) + hi(a)*hi(b) for packed 16-bit pairs, fp32 accumulation (FHFMA).
__device__ __forceinline__ float fhfma2_f16(uint32_t a, uint32_t b, float c) {
    asm("{\n\t.reg .f16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
        "fma.rn.f32.f16 %0, al, bl, %0;\n\tfma.rn.f32.f16 %0, ah, bh, %0;\n\t}"
        : "+f"(c)
        : "r"(a), "r"(b));
    return c;
}
__device__ __forceinline__ float fhfma2_bf16(uint32_t a, uint32_t b, float c) {
    asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
        "fma.rn.f32.bf16 %0, al, bl, %0;\n\tfma.rn.f32.bf16 %0, ah, bh, %0;\n\t}"
        : "+f"(c)
        : "r"(a), "r"(b));
    return c;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

__device__ __forceinline__ float2 unpack_f16(uint32_t u) {
    return __half22float2(*reinterpret_cast<const __half2*>(&u));
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}

// ---- element traits -------------------------------------------------------------------
template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static constexpr int kBytes = 4;
    __device__ static float to_f32(float x) { return x; }
    __device__ static float from_f32(float x) { return x; }
};
template <>
struct Elem<__half> {
    static constexpr int kBytes = 2;
    __device__ static float to_f32(__half x) { return __half2float(x); }
    __device__ static __half from_f32(float x) { return __float2half_rn(x); }
};
template <>
struct Elem<__nv_bfloat16> {
    static constexpr int kBytes = 2;
    __device__ static float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
    __device__ static __nv_bfloat16 from_f32(float x) { return __float2bfloat16_rn(x); }
};

// Dot product of one 16-byte chunk of q (registers, storage dtype) with one 16-byte
// chunk of K (shared memory), fp32 accumulate.
template <typename T>
__device__ __forceinline__ float dot16(const uint4& q, const uint4& k, float acc);
template <>
__device__ __forceinline__ float dot16<__half>(const uint4& q, const uint4& k, float acc) {
    acc = fhfma2_f16(q.x, k.x, acc);
    acc = fhfma2_f16(q.y, k.y, acc);
    acc = fhfma2_f16(q.z, k.z, acc);
    acc = fhfma2_f16(q.w, k.w, acc);
    return acc;
}
template <>
__device__ __forceinline__ float dot16<__nv_bfloat16>(const uint4& q, const uint4& k, float acc) {
    acc = fhfma2_bf16(q.x, k.x, acc);
    acc = fhfma2_bf16(q.y, k.y, acc);
    acc = fhfma2_bf16(q.z, k.z, acc);
    acc = fhfma2_bf16(q.w, k.w, acc);
    return acc;
}
template <>
__device__ __forceinline__ float dot16<float>(const uint4& q, const uint4& k, float acc) {
    float2 a = make_float2(0.f, 0.f);
    a = ffma2(make_float2(__uint_as_float(q.x), __uint_as_float(q.y)),
              make_float2(__uint_as_float(k.x), __uint_as_float(k.y)), a);
    a = ffma2(make_float2(__uint_as_float(q.z), __uint_as_float(q.w)),
              make_float2(__uint_as_float(k.z), __uint_as_float(k.w)), a);
    return acc + (a.x + a.y);
}

// acc += p * (lo(v), hi(v)) for one packed 16-bit pair, p already in the storage dtype:
// two mixed-precision FMAs (FHFMA: 16-bit operands, fp32 accumulator), no unpacking.
__device__ __forceinline__ void fhfma_pv_f16(float2& acc, uint32_t v, unsigned short p) {
    asm("{\n\t.reg .f16 vl, vh, pp;\n\tmov.b32 {vl, vh}, %2;\n\tmov.b16 pp, %3;\n\t"
        "fma.rn.f32.f16 %0, vl, pp, %0;\n\tfma.rn.f32.f16 %1, vh, pp, %1;\n\t}"
        : "+f"(acc.x), "+f"(acc.y)
        : "r"(v), "h"(p));
}
__device__ __forceinline__ void fhfma_pv_bf16(float2& acc, uint32_t v, unsigned short p) {
    asm("{\n\t.reg .b16 vl, vh;\n\tmov.b32 {vl, vh}, %2;\n\t"
        "fma.rn.f32.bf16 %0, vl, %3, %0;\n\tfma.rn.f32.bf16 %1, vh, %3, %1;\n\t}"
        : "+f"(acc.x), "+f"(acc.y)
        : "r"(v), "h"(p));
}

// acc[0..EPC/2) += p * v  for one 16-byte chunk of V (EPC elements), fp32 accumulators.
// 16-bit caches: the softmax weight p is rounded once to the storage dtype (RN) and
// multiplied in FHFMA (as FlashAttention rounds P for its P.V product, DESIGN c25):
// 8 instructions per chunk instead of 4 unpacks (8 HADD2.F32) + 4 FFMA2.  -DPA_PV_F32
// restores the fp32-weight path (unpack + FFMA2) for A/B.
template <typename T>
__device__ __forceinline__ void axpy16(float2* acc, float p, const uint4& v);
#ifndef PA_PV_F32
template <>
__device__ __forceinline__ void axpy16<__half>(float2* acc, float p, const uint4& v) {
    const unsigned short ph = __half_as_ushort(__float2half_rn(p));
    fhfma_pv_f16(acc[0], v.x, ph);
    fhfma_pv_f16(acc[1], v.y, ph);
    fhfma_pv_f16(acc[2], v.z, ph);
    fhfma_pv_f16(acc[3], v.w, ph);
}
template <>
__device__ __forceinline__ void axpy16<__nv_bfloat16>(float2* acc, float p, const uint4& v) {
    const unsigned short pb = __bfloat16_as_ushort(__float2bfloat16_rn(p));
    fhfma_pv_bf16(acc[0], v.x, pb);
    fhfma_pv_bf16(acc[1], v.y, pb);
    fhfma_pv_bf16(acc[2], v.z, pb);
    fhfma_pv_bf16(acc[3], v.w, pb);
}
#else
template <>
__device__ __forceinline__ void axpy16<__half>(float2* acc, float p, const uint4& v) {
    const float2 pp = make_float2(p, p);
    acc[0] = ffma2(pp, unpack_f16(v.x), acc[0]);
    acc[1] = ffma2(pp, unpack_f16(v.y), acc[1]);
    acc[2] = ffma2(pp, unpack_f16(v.z), acc[2]);
    acc[3] = ffma2(pp, unpack_f16(v.w), acc[3]);
}
template <>
__device__ __forceinline__ void axpy16<__nv_bfloat16>(float2* acc, float p, const uint4& v) {
    const float2 pp = make_float2(p, p);
    acc[0] = ffma2(pp, unpack_bf16(v.x), acc[0]);
    acc[1] = ffma2(pp, unpack_bf16(v.y), acc[1]);
    acc[2] = ffma2(pp, unpack_bf16(v.z), acc[2]);
    acc[3] = ffma2(pp, unpack_bf16(v.w), acc[3]);
}
#endif
template <>
__device__ __forceinline__ void axpy16<float>(float2* acc, float p, const uint4& v) {
    const float2 pp = make_float2(p, p);
    acc[0] = ffma2(pp, make_float2(__uint_as_float(v.x), __uint_as_float(v.y)), acc[0]);
    acc[1] = ffma2(pp, make_float2(__uint_as_float(v.z), __uint_as_float(v.w)), acc[1]);
}

__device__ __forceinline__ uint4 lds128(const void* p) { return *reinterpret_cast<const uint4*>(p); }

}  // namespace pa
