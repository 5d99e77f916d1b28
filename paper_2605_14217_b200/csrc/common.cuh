// Shared device helpers for libpreft (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "preft.h"

namespace preft {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- vectors
//
// Vec<T, VEC> moves W elements of T per memory instruction:
//   bf16, VEC: 8 x bf16 = one 128-bit access
//   f32,  VEC: 4 x f32  = one 128-bit access
//   f64,  VEC: 2 x f64  = one 128-bit access (float64 drop-in mode)
//   any,  !VEC: one element (unaligned / odd-width fallback)
// Loads come in three flavours:
//   ld_stream  read-once activations (x): L1::no_allocate, non-coherent path
//   ld_weight  adapter weights reused by neighbouring warps: L1-cached __ldg
//   ld_rw      rows that are read then written by the same warp (y, h)

template <typename T, bool VEC>
struct Vec;

__device__ __forceinline__ void bf16x2_to_acc(uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
}

__device__ __forceinline__ uint32_t f32x2_to_bf16(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&p);
}

template <>
struct Vec<__nv_bfloat16, true> {
    static constexpr int W = 8;
    using acc_t = float;
    using raw_t = uint4;
    __device__ __forceinline__ static raw_t zero() { return make_uint4(0, 0, 0, 0); }
    __device__ __forceinline__ static raw_t ld_stream(const __nv_bfloat16* p) {
        raw_t r;
        asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
            : "l"(p));
        return r;
    }
    __device__ __forceinline__ static raw_t ld_weight(const __nv_bfloat16* p) {
        return __ldg(reinterpret_cast<const uint4*>(p));
    }
    __device__ __forceinline__ static raw_t ld_rw(const __nv_bfloat16* p) {
        return *reinterpret_cast<const uint4*>(p);
    }
    __device__ __forceinline__ static void st(__nv_bfloat16* p, const float (&f)[W]) {
        uint4 r;
        r.x = f32x2_to_bf16(f[0], f[1]);
        r.y = f32x2_to_bf16(f[2], f[3]);
        r.z = f32x2_to_bf16(f[4], f[5]);
        r.w = f32x2_to_bf16(f[6], f[7]);
        *reinterpret_cast<uint4*>(p) = r;
    }
    __device__ __forceinline__ static void to_acc(const raw_t& r, float (&f)[W]) {
        bf16x2_to_acc(r.x, f[0], f[1]);
        bf16x2_to_acc(r.y, f[2], f[3]);
        bf16x2_to_acc(r.z, f[4], f[5]);
        bf16x2_to_acc(r.w, f[6], f[7]);
    }
};

template <>
struct Vec<float, true> {
    static constexpr int W = 4;
    using acc_t = float;
    using raw_t = float4;
    __device__ __forceinline__ static raw_t zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ static raw_t ld_stream(const float* p) {
        raw_t r;
        asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
            : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
            : "l"(p));
        return r;
    }
    __device__ __forceinline__ static raw_t ld_weight(const float* p) {
        return __ldg(reinterpret_cast<const float4*>(p));
    }
    __device__ __forceinline__ static raw_t ld_rw(const float* p) {
        return *reinterpret_cast<const float4*>(p);
    }
    __device__ __forceinline__ static void st(float* p, const float (&f)[W]) {
        *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    }
    __device__ __forceinline__ static void to_acc(const raw_t& r, float (&f)[W]) {
        f[0] = r.x;
        f[1] = r.y;
        f[2] = r.z;
        f[3] = r.w;
    }
};

template <>
struct Vec<__nv_bfloat16, false> {
    static constexpr int W = 1;
    using acc_t = float;
    using raw_t = unsigned short;
    __device__ __forceinline__ static raw_t zero() { return 0; }
    __device__ __forceinline__ static raw_t ld_stream(const __nv_bfloat16* p) {
        return __ldg(reinterpret_cast<const unsigned short*>(p));
    }
    __device__ __forceinline__ static raw_t ld_weight(const __nv_bfloat16* p) {
        return __ldg(reinterpret_cast<const unsigned short*>(p));
    }
    __device__ __forceinline__ static raw_t ld_rw(const __nv_bfloat16* p) {
        return *reinterpret_cast<const unsigned short*>(p);
    }
    __device__ __forceinline__ static void st(__nv_bfloat16* p, const float (&f)[W]) {
        *p = __float2bfloat16_rn(f[0]);
    }
    __device__ __forceinline__ static void to_acc(const raw_t& r, float (&f)[W]) {
        f[0] = __uint_as_float(static_cast<uint32_t>(r) << 16);
    }
};

template <>
struct Vec<float, false> {
    static constexpr int W = 1;
    using acc_t = float;
    using raw_t = float;
    __device__ __forceinline__ static raw_t zero() { return 0.f; }
    __device__ __forceinline__ static raw_t ld_stream(const float* p) { return __ldg(p); }
    __device__ __forceinline__ static raw_t ld_weight(const float* p) { return __ldg(p); }
    __device__ __forceinline__ static raw_t ld_rw(const float* p) { return *p; }
    __device__ __forceinline__ static void st(float* p, const float (&f)[W]) { *p = f[0]; }
    __device__ __forceinline__ static void to_acc(const raw_t& r, float (&f)[W]) { f[0] = r; }
};

// f64 mode: the reference computes in float64 (adapters.py:280); B200 keeps
// FP64 SIMT, so the drop-in float64 API runs the same kernels in double.
template <>
struct Vec<double, true> {
    static constexpr int W = 2;
    using acc_t = double;
    using raw_t = double2;
    __device__ __forceinline__ static raw_t zero() { return make_double2(0.0, 0.0); }
    __device__ __forceinline__ static raw_t ld_stream(const double* p) {
        raw_t r;
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
        return r;
    }
    __device__ __forceinline__ static raw_t ld_weight(const double* p) {
        return __ldg(reinterpret_cast<const double2*>(p));
    }
    __device__ __forceinline__ static raw_t ld_rw(const double* p) { return *reinterpret_cast<const double2*>(p); }
    __device__ __forceinline__ static void st(double* p, const double (&f)[W]) {
        *reinterpret_cast<double2*>(p) = make_double2(f[0], f[1]);
    }
    __device__ __forceinline__ static void to_acc(const raw_t& r, double (&f)[W]) {
        f[0] = r.x;
        f[1] = r.y;
    }
};

template <>
struct Vec<double, false> {
    static constexpr int W = 1;
    using acc_t = double;
    using raw_t = double;
    __device__ __forceinline__ static raw_t zero() { return 0.0; }
    __device__ __forceinline__ static raw_t ld_stream(const double* p) { return __ldg(p); }
    __device__ __forceinline__ static raw_t ld_weight(const double* p) { return __ldg(p); }
    __device__ __forceinline__ static raw_t ld_rw(const double* p) { return *p; }
    __device__ __forceinline__ static void st(double* p, const double (&f)[W]) { *p = f[0]; }
    __device__ __forceinline__ static void to_acc(const raw_t& r, double (&f)[W]) { f[0] = r; }
};

// ---------------------------------------------------------------- arithmetic

__device__ __forceinline__ float macc(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double macc(double a, double b, double c) { return fma(a, b, c); }

template <typename A>
__device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Programmatic dependent launch (sm_90+): let the next kernel in the stream
// launch now, then wait until the previous kernel's writes are visible.  Both
// are no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Contiguous share [lo, hi) of n items for worker w of nw (balanced to +-1).
__device__ __forceinline__ void even_share(int n, int w, int nw, int& lo, int& hi) {
    lo = static_cast<int>((static_cast<long long>(w) * n) / nw);
    hi = static_cast<int>((static_cast<long long>(w + 1) * n) / nw);
}

}  // namespace preft
