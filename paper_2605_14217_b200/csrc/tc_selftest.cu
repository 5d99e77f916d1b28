// Self-test of the tcgen05 building blocks (tc.cuh): one CTA computes
// D[128 x N] = A[128 x K] . B[N x K]^T from bf16 global operands, with A
// staged one of three ways:
//   mode 0  threads, K-major SWIZZLE_NONE (core-matrix) layout
//   mode 1  threads, K-major SWIZZLE_128B layout
//   mode 2  TMA (cp.async.bulk.tensor, 64 x 128 boxes, 128 B swizzle)
// B is always thread-staged SWIZZLE_NONE.  Then UMMA issue, commit ->
// mbarrier and a TMEM -> register epilogue.  Exposed as preft_tc_selftest so
// the GPU suite pins descriptors, swizzle and TMA independently of the ReFT
// kernel that is built from them.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

__global__ void __launch_bounds__(128, 1) tc_selftest_kernel(const __grid_constant__ CUtensorMap tmap,
                                                             const __nv_bfloat16* A, const __nv_bfloat16* B, float* D,
                                                             int K, int N, uint32_t ncols, int mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ __align__(8) uint64_t tbar;
    __shared__ uint32_t tslot;
    unsigned char* sA = smem;                  // 128 x K (1024 B aligned)
    unsigned char* sB = smem + 128 * K * 2;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int kc = K / 8;
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_init(&tbar, 1);
        tc::fence_mbar_init();
    }
    __syncthreads();
    if (mode == 2) {
        if (tid == 0) {
            tc::mbar_expect_tx(&tbar, 128 * K * 2);
            for (int p = 0; p < K / 64; ++p) tc::tma_load_2d(tc::smem_u32(sA) + p * 128 * 128, &tmap, p * 64, 0, &tbar);
        }
    } else {
        for (int idx = tid; idx < 128 * kc; idx += blockDim.x) {
            const int r = idx / kc, c8 = idx % kc;
            const uint4 v = reinterpret_cast<const uint4*>(A + static_cast<long long>(r) * K)[c8];
            const uint32_t off = mode == 1 ? tc::sw128_offset(r, c8 * 8, 128) : tc::kmajor_offset(r, c8 * 8, K);
            *reinterpret_cast<uint4*>(sA + off) = v;
        }
    }
    for (int idx = tid; idx < N * kc; idx += blockDim.x) {
        const int r = idx / kc, c8 = idx % kc;
        const uint4 v = reinterpret_cast<const uint4*>(B + static_cast<long long>(r) * K)[c8];
        *reinterpret_cast<uint4*>(sB + tc::kmajor_offset(r, c8 * 8, K)) = v;
    }
    if (warp == 0) tc::tmem_alloc(&tslot, ncols);
    if (mode == 2) tc::mbar_wait(&tbar, 0);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t taddr = tslot;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_bf16_f32(128, N);
        for (int k = 0; k < K / 16; ++k) {
            const uint64_t ad = mode == 0 ? tc::desc_kmajor(tc::smem_u32(sA) + k * 256, 128, K * 16)
                                          : tc::desc_kmajor_sw128(tc::smem_u32(sA) + (k >> 2) * 128 * 128 + (k & 3) * 32);
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

int tc_selftest(const void* A, const void* B, float* D, int K, int N, int mode, cudaStream_t s) {
    if (!A || !B || !D || K < 16 || K % 16 || N < 16 || N > 256 || N % 16 || mode < 0 || mode > 2)
        return PREFT_ERR_SHAPE;
    if (mode > 0 && K % 64) return PREFT_ERR_SHAPE;
    uint32_t ncols = 32;
    while (ncols < static_cast<uint32_t>(N)) ncols <<= 1;
    const size_t smem = static_cast<size_t>(128 + N) * K * 2;
    if (smem > 200 * 1024) return PREFT_ERR_SHAPE;
    CUtensorMap tmap{};
    if (mode == 2 && !make_tmap_bf16_sw128(&tmap, A, 128, K, K, 64, 128)) return PREFT_ERR_CONFIG;
    cudaError_t e = cudaFuncSetAttribute(tc_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return -static_cast<int>(e);
    tc_selftest_kernel<<<1, 128, smem, s>>>(tmap, static_cast<const __nv_bfloat16*>(A),
                                            static_cast<const __nv_bfloat16*>(B), D, K, N, ncols, mode);
    e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
