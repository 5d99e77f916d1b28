// K3-TC — tensor-core ReFT^P for sm_100a (bf16, rank 16 or 32, d = C x 512).
//
//     h[t, :] += s_a * ((h[t, :] . A_a^T + b_a) . B_a)      (adapters.py:292-295)
//
// At r >= 16 the residual edit is a real contraction (4*r*d FLOP against
// 4*d bytes per token: 105-315 TFLOP/s at the HBM roofline, beyond SIMT
// FP32), so both products run on tcgen05 with fp32 accumulators in TMEM.
//
// Work unit: one K1 tile = up to 128 slot-sorted tokens of ONE adapter
// (UMMA M = 128).  A thread-block cluster of C = d/512 CTAs owns a tile; CTA
// c owns the 512 columns [512c, 512c + 512) of d:
//   1. cp.async gathers the tile's h rows (its 512-column slice, 128 KB) and,
//      when the adapter changes, its slices of A (r x 512) and Bt (512 x r)
//      into shared memory (K-major no-swizzle UMMA layout, tc.cuh);
//   2. shrink: TMEM[128 x r] = H_slice . A_slice^T   (32 UMMAs, K = 512);
//   3. the C partial rank-r rows are reduced through distributed shared
//      memory: CTA c sums rows [128c/C, 128(c+1)/C) over the cluster, adds
//      bias, scales, splits v = hi + lo into two bf16 operands (so the expand
//      keeps ~fp32 accuracy) and pushes them into every CTA's smem;
//   4. expand: TMEM[128 x 512] = V_hi . Bt_slice^T + V_lo . Bt_slice^T (N = 256 x 2);
//   5. epilogue: TMEM -> registers, h_slice += delta in shared memory, then
//      the updated rows go back to global memory with coalesced 16 B stores.
// h therefore crosses HBM exactly once in and once out (the algorithmic
// minimum); weights are re-staged only when the tile's adapter changes.
// Tiles of LoRA-class slots (slot < slot_split) are skipped.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace preft {

constexpr int kTcSlice = 512;
constexpr int kTcRows = 128;
constexpr int kTcThreads = 256;

struct ReftTcArgs {
    __nv_bfloat16* h;
    long long ldh;
    int d;
    int slot_base;
    const __nv_bfloat16* A;   // [S][R][d]
    const __nv_bfloat16* Bt;  // [S][d][R]
    const float* bias;        // [S][R]
    const float* scale;       // [S]
    const int2* tokens;
    const int4* tiles;
    const int* counters;
};

template <int R>
struct TcSmem {
    static constexpr int H = 0;                               // 128 x 512 bf16
    static constexpr int A = H + kTcRows * kTcSlice * 2;      // R x 512 bf16
    static constexpr int BT = A + R * kTcSlice * 2;           // 512 x R bf16
    static constexpr int VHI = BT + kTcSlice * R * 2;         // 128 x R bf16
    static constexpr int VLO = VHI + kTcRows * R * 2;         // 128 x R bf16
    static constexpr int P = VLO + kTcRows * R * 2;           // 128 x R f32 partials
    static constexpr int TOTAL = P + kTcRows * R * 4;
};

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_dsmem_u16(uint32_t addr, unsigned short v) {
    asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

template <int R>
__global__ void __launch_bounds__(kTcThreads, 1) reft_tc_kernel(const ReftTcArgs a) {
    using L = TcSmem<R>;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ int s_rows[kTcRows];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = static_cast<int>(tc::cluster_nctarank());
    const int crank = static_cast<int>(tc::cluster_ctarank());
    const int cluster_id = blockIdx.x / C, nclusters = gridDim.x / C;
    const int col0 = crank * kTcSlice;
    const int ntiles = a.counters[PREFT_CTR_TILES];
    const uint32_t sbase = tc::smem_u32(sm);
    const uint32_t sH = sbase + L::H, sA = sbase + L::A, sBt = sbase + L::BT;
    const uint32_t sVhi = sbase + L::VHI, sVlo = sbase + L::VLO, sP = sbase + L::P;

    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    uint32_t phase = 0;
    int cur_slot = -1;
    const int rows_per = kTcRows / C;

    for (int t = cluster_id; t < ntiles; t += nclusters) {
        const int4 tile = a.tiles[t];  // (slot, first sorted position, n tokens, segment)
        if (tile.x < a.slot_base) continue;  // LoRA-class tile: same decision in every CTA of the cluster
        const int slot = tile.x - a.slot_base;
        const int ntok = tile.z;
        if (tid < kTcRows) s_rows[tid] = tid < ntok ? a.tokens[tile.y + tid].x : -1;
        __syncthreads();

        // ---- 1. stage h rows (and weights when the adapter changes)
        {
            const __nv_bfloat16* hb = a.h + col0;
            for (int i = tid; i < kTcRows * (kTcSlice / 8); i += kTcThreads) {
                const int r8 = i & 7, c8 = (i >> 3) & 63, row = (i >> 9) * 8 + r8;
                const int tok = s_rows[row];
                if (tok >= 0)
                    cp_async16(sH + tc::kmajor_offset(row, c8 * 8, kTcSlice),
                               hb + static_cast<long long>(tok) * a.ldh + c8 * 8);
            }
            if (slot != cur_slot) {
                const __nv_bfloat16* Ab = a.A + static_cast<long long>(slot) * R * a.d + col0;
                for (int i = tid; i < R * (kTcSlice / 8); i += kTcThreads) {
                    const int r8 = i & 7, c8 = (i >> 3) & 63, k = (i >> 9) * 8 + r8;
                    cp_async16(sA + tc::kmajor_offset(k, c8 * 8, kTcSlice), Ab + static_cast<long long>(k) * a.d + c8 * 8);
                }
                const __nv_bfloat16* Bb = a.Bt + (static_cast<long long>(slot) * a.d + col0) * R;
                for (int i = tid; i < kTcSlice * (R / 8); i += kTcThreads) {
                    const int n = i / (R / 8), c8 = i % (R / 8);
                    cp_async16(sBt + tc::kmajor_offset(n, c8 * 8, R), Bb + static_cast<long long>(n) * R + c8 * 8);
                }
                cur_slot = slot;
            }
            cp_async_wait_all();
            tc::fence_proxy_async();
            __syncthreads();
        }

        // ---- 2. shrink: TMEM[0:R] = H . A^T
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t id = tc::idesc_bf16_f32(kTcRows, R);
#pragma unroll 4
            for (int k = 0; k < kTcSlice / 16; ++k)
                tc::mma_bf16(tmem, tc::desc_kmajor(sH + k * 256, 128, kTcSlice * 16),
                             tc::desc_kmajor(sA + k * 256, 128, kTcSlice * 16), id, k > 0 ? 1u : 0u);
            tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();
        if (warp < 4) {
            const int row = warp * 32 + lane;
            float* P = reinterpret_cast<float*>(sm + L::P);
#pragma unroll
            for (int c0 = 0; c0 < R; c0 += 16) {
                uint32_t v[16];
                tc::tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) P[row * R + c0 + j] = __uint_as_float(v[j]);
            }
        }
        tc::fence_before_sync();
        tc::cluster_sync();  // every CTA's partial rows are visible cluster-wide

        // ---- 3. reduce-scatter the partials, push bf16 hi/lo V to every CTA
        for (int idx = tid; idx < rows_per * R; idx += kTcThreads) {
            const int j = crank * rows_per + idx / R, k = idx % R;
            const uint32_t off = static_cast<uint32_t>((j * R + k) * 4);
            float s = 0.f;
            for (int q = 0; q < C; ++q) s += ld_dsmem_f32(tc::map_shared(sP + off, q));
            const float v = (s + __ldg(a.bias + static_cast<long long>(slot) * R + k)) * __ldg(a.scale + slot);
            const __nv_bfloat16 hi = __float2bfloat16_rn(v);
            const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
            const uint32_t voff = tc::kmajor_offset(j, k, R);
            const unsigned short hb = *reinterpret_cast<const unsigned short*>(&hi);
            const unsigned short lb = *reinterpret_cast<const unsigned short*>(&lo);
            for (int q = 0; q < C; ++q) {
                st_dsmem_u16(tc::map_shared(sVhi + voff, q), hb);
                st_dsmem_u16(tc::map_shared(sVlo + voff, q), lb);
            }
        }
        tc::cluster_sync();  // V complete in every CTA

        // ---- 4. expand: TMEM[0:512] = V_hi . Bt^T + V_lo . Bt^T
        if (tid == 0) {
            tc::fence_proxy_async();
            tc::fence_after_sync();
            const uint32_t id = tc::idesc_bf16_f32(kTcRows, 256);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t bbase = sBt + half * 32 * (R * 16);  // 256 rows = 32 core-row groups
                uint32_t acc = 0;
#pragma unroll
                for (int k = 0; k < R / 16; ++k) {
                    const uint64_t bd = tc::desc_kmajor(bbase + k * 256, 128, R * 16);
                    tc::mma_bf16(tmem + half * 256, tc::desc_kmajor(sVhi + k * 256, 128, R * 16), bd, id, acc);
                    acc = 1;
                    tc::mma_bf16(tmem + half * 256, tc::desc_kmajor(sVlo + k * 256, 128, R * 16), bd, id, 1u);
                }
            }
            tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1;
        tc::fence_after_sync();

        // ---- 5. epilogue: h_slice += delta (in shared memory), then store rows
        {
            const int q = warp & 3, half = warp >> 2, row = q * 32 + lane;
            const bool live = row < ntok;
#pragma unroll 1
            for (int c0 = 0; c0 < 256; c0 += 16) {
                const int col = half * 256 + c0;
                uint32_t v[16];
                tc::tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + col, v);
                tc::tmem_ld_wait();
                if (live) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        uint4* p = reinterpret_cast<uint4*>(sm + L::H + tc::kmajor_offset(row, col + hh * 8, kTcSlice));
                        uint4 hv = *p;
                        uint32_t* w = reinterpret_cast<uint32_t*>(&hv);
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float lo, hi2;
                            bf16x2_to_acc(w[e], lo, hi2);
                            lo += __uint_as_float(v[hh * 8 + 2 * e]);
                            hi2 += __uint_as_float(v[hh * 8 + 2 * e + 1]);
                            w[e] = f32x2_to_bf16(lo, hi2);
                        }
                        *p = hv;
                    }
                }
            }
        }
        tc::fence_before_sync();
        __syncthreads();
        {
            __nv_bfloat16* hb = a.h + col0;
            for (int i = tid; i < kTcRows * (kTcSlice / 8); i += kTcThreads) {
                const int r8 = i & 7, c8 = (i >> 3) & 63, row = (i >> 9) * 8 + r8;
                const int tok = s_rows[row];
                if (tok >= 0)
                    *reinterpret_cast<uint4*>(hb + static_cast<long long>(tok) * a.ldh + c8 * 8) =
                        *reinterpret_cast<const uint4*>(sm + L::H + tc::kmajor_offset(row, c8 * 8, kTcSlice));
            }
        }
        __syncthreads();
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// returns 0 on launch, PREFT_ERR_* if the shape is not TC-eligible, or -cudaError
int reft_tc_apply(const preft_meta_t* meta, void* h, long long ldh, int d, const void* A, const void* Bt,
                  const void* bias, const void* scale, int r, cudaStream_t stream) {
    if (!Bt || (r != 16 && r != 32) || d % kTcSlice) return PREFT_ERR_SHAPE;
    const int C = d / kTcSlice;
    if (C != 2 && C != 4 && C != 8) return PREFT_ERR_SHAPE;
    if (meta->tile_tokens > kTcRows || (ldh % 8) || (reinterpret_cast<uintptr_t>(h) & 15) ||
        (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(Bt) & 15))
        return PREFT_ERR_SHAPE;
    ReftTcArgs args;
    args.h = static_cast<__nv_bfloat16*>(h);
    args.ldh = ldh;
    args.d = d;
    args.slot_base = meta->slot_split;
    args.A = static_cast<const __nv_bfloat16*>(A);
    args.Bt = static_cast<const __nv_bfloat16*>(Bt);
    args.bias = static_cast<const float*>(bias);
    args.scale = static_cast<const float*>(scale);
    args.tokens = reinterpret_cast<const int2*>(meta->tokens);
    args.tiles = reinterpret_cast<const int4*>(meta->tiles);
    args.counters = meta->counters;
    void (*fn)(ReftTcArgs) = r == 16 ? reft_tc_kernel<16> : reft_tc_kernel<32>;
    const int smem = r == 16 ? TcSmem<16>::TOTAL : TcSmem<32>::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -static_cast<int>(e);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(C * 148);
    int nclusters = 0;
    e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
    if (e != cudaSuccess) return -static_cast<int>(e);
    if (nclusters < 1) return PREFT_ERR_CONFIG;
    cfg.gridDim = dim3(C * nclusters);
    e = cudaLaunchKernelEx(&cfg, fn, args);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
