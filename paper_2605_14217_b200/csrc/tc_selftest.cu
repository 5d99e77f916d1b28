// Self-test of the tcgen05 building blocks (tc.cuh): one CTA computes
// D[128 x N] = A[128 x K] . B[N x K]^T from bf16 global operands with the
// K-major no-swizzle staging, UMMA issue, commit -> mbarrier, and a TMEM ->
// register epilogue.  Exposed as preft_tc_selftest so the GPU test suite
// pins the descriptor / TMEM mechanics independently of the ReFT kernel.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace preft {

__global__ void __launch_bounds__(128, 1) tc_selftest_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B,
                                                             float* D, int K, int N, uint32_t ncols) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    unsigned char* sA = smem;
    unsigned char* sB = smem + 128 * K * 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kc = K / 8;
    for (int idx = tid; idx < 128 * kc; idx += blockDim.x) {
        const int r = idx / kc, c8 = idx % kc;
        const uint4 v = reinterpret_cast<const uint4*>(A + static_cast<long long>(r) * K)[c8];
        *reinterpret_cast<uint4*>(sA + tc::kmajor_offset(r, c8 * 8, K)) = v;
    }
    for (int idx = tid; idx < N * kc; idx += blockDim.x) {
        const int r = idx / kc, c8 = idx % kc;
        const uint4 v = reinterpret_cast<const uint4*>(B + static_cast<long long>(r) * K)[c8];
        *reinterpret_cast<uint4*>(sB + tc::kmajor_offset(r, c8 * 8, K)) = v;
    }
    if (warp == 0) tc::tmem_alloc(&tslot, ncols);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t taddr = tslot;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_bf16_f32(128, N);
        for (int k = 0; k < K / 16; ++k) {
            const uint64_t ad = tc::desc_kmajor(tc::smem_u32(sA) + k * 256, 128, K * 16);
            const uint64_t bd = tc::desc_kmajor(tc::smem_u32(sB) + k * 256, 128, K * 16);
            tc::mma_bf16(taddr, ad, bd, idesc, k > 0 ? 1u : 0u);
        }
        tc::mma_commit(&mbar);
    }
    __syncwarp();
    tc::mbar_wait(&mbar, 0);
    tc::fence_after_sync();
    const int row = warp * 32 + lane;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        tc::tmem_ld16(taddr + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) D[static_cast<long long>(row) * N + c0 + j] = __uint_as_float(v[j]);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(taddr, ncols);
}

int tc_selftest(const void* A, const void* B, float* D, int K, int N, cudaStream_t s) {
    if (!A || !B || !D || K < 16 || K % 16 || N < 16 || N > 256 || N % 16) return PREFT_ERR_SHAPE;
    uint32_t ncols = 32;
    while (ncols < static_cast<uint32_t>(N)) ncols <<= 1;
    const size_t smem = static_cast<size_t>(128 + N) * K * 2;
    if (smem > 200 * 1024) return PREFT_ERR_SHAPE;
    cudaError_t e = cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return -static_cast<int>(e);
    tc_selftest_kernel<<<1, 128, smem, s>>>(static_cast<const __nv_bfloat16*>(A), static_cast<const __nv_bfloat16*>(B),
                                            D, K, N, ncols);
    e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
