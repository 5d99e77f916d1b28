// K3-TC — tensor-core ReFT^P for sm_100a (bf16, rank 16 or 32).
//
//     h[t, :] += s_a * ((h[t, :] . A_a^T + b_a) . B_a)      (adapters.py:292-295)
//
// At r >= 16 the residual edit is a real contraction (4*r*d FLOP against
// 4*d bytes per token: 105-315 TFLOP/s at the HBM roofline, beyond SIMT
// FP32), so both products run on tcgen05 with fp32 accumulators in TMEM.
//
// Work unit: one K1 tile = up to 128 slot-sorted tokens of ONE adapter
// (UMMA M = 128).  A thread-block cluster of C = d / SLICE CTAs owns a tile;
// CTA c owns the SLICE columns [SLICE*c, SLICE*(c+1)) of d.  Per tile:
//   1. the tile's h rows (its column slice) land in shared memory in the
//      canonical 128 B-swizzled K-major layout — by TMA (boxes of 128 rows x
//      64 columns) when the tile is 128 consecutive rows (the common case for
//      long prompts), by a cp.async gather otherwise; the adapter's A
//      (r x SLICE) and Bt (SLICE x r) slices are re-staged only when the
//      tile's adapter changes (clusters walk contiguous runs of tiles);
//   2. shrink: TMEM[128 x r] = H_slice . A_slice^T, split over 4 independent
//      accumulators so the UMMA chain is not latency-serialised;
//   3. the C partial rank-r rows are reduced through distributed shared
//      memory: CTA c sums its 128/C rows over the cluster, adds bias, scales,
//      splits v = hi + lo into two bf16 operands (so the expand keeps ~fp32
//      accuracy) and pushes them into every CTA's shared memory;
//   4. expand: TMEM[128 x SLICE] = V_hi . Bt_slice^T + V_lo . Bt_slice^T;
//   5. epilogue: TMEM -> registers, h_slice += delta in shared memory, then
//      the updated rows go back by TMA store (full tiles; it drains while the
//      next tile is staged) or 16 B stores (partial tiles).
// h crosses HBM exactly once in and once out (the algorithmic minimum).
// SLICE is a template parameter (256 fits two CTAs per SM at r = 16 but needs
// 16-CTA clusters for d = 4096, which co-schedule poorly); launches use 512.
// LoRA-class tiles are skipped.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

constexpr int kTcRows = 128;
constexpr int kTcThreads = 256;
constexpr int kTcAcc = 4;  // independent shrink accumulators

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
    long long* prof;  // optional phase timestamps (diagnostics), NULL in production
};

// diagnostics: CTA 0 records clock64() at 8 phase boundaries of its first 16 tiles
static long long* g_tc_prof = nullptr;
#define TC_MARK(p)                                                                              \
    do {                                                                                       \
        if (a.prof && blockIdx.x == 0 && tid == 0 && it < 16) a.prof[it * 8 + (p)] = clock64(); \
    } while (0)

template <int R, int SLICE>
struct TcSmem {
    static constexpr int H = 0;                            // SLICE/64 panels x 128 rows x 128 B (swizzled)
    static constexpr int A = H + kTcRows * SLICE * 2;      // R x SLICE bf16 (core-matrix layout)
    static constexpr int BT = A + R * SLICE * 2;           // SLICE x R bf16
    static constexpr int VHI = BT + SLICE * R * 2;         // 128 x R bf16
    static constexpr int VLO = VHI + kTcRows * R * 2;      // 128 x R bf16
    static constexpr int P = VLO + kTcRows * R * 2;        // 128 x R f32 partials
    static constexpr int TOTAL = P + kTcRows * R * 4;
    static constexpr int TMEM_COLS = SLICE <= 256 ? 256 : 512;
    static constexpr int MIN_BLOCKS = TOTAL <= 110 * 1024 ? 2 : 1;
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

template <int R, int C, int SLICE>
__global__ void __launch_bounds__(kTcThreads, TcSmem<R, SLICE>::MIN_BLOCKS)
    reft_tc_kernel(const __grid_constant__ CUtensorMap tmap, const ReftTcArgs a) {
    using L = TcSmem<R, SLICE>;
    constexpr int PANELS = SLICE / 64;
    constexpr int KSTEPS = SLICE / 16;
    constexpr int rows_per = kTcRows / C;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ int s_rows[kTcRows];
    __shared__ __align__(8) uint64_t mbar;  // MMA completion
    __shared__ __align__(8) uint64_t tbar;  // TMA load completion
    __shared__ uint32_t tslot;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int crank = static_cast<int>(tc::cluster_ctarank());
    const int cluster_id = blockIdx.x / C, nclusters = gridDim.x / C;
    const int col0 = crank * SLICE;
    const uint32_t sbase = tc::smem_u32(sm);
    const uint32_t sH = sbase + L::H, sA = sbase + L::A, sBt = sbase + L::BT;
    const uint32_t sVhi = sbase + L::VHI, sVlo = sbase + L::VLO, sP = sbase + L::P;

    if (warp == 0) tc::tmem_alloc(&tslot, L::TMEM_COLS);
    if (tid == 0) {
        tc::prefetch_tmap(&tmap);
        tc::mbar_init(&mbar, 1);
        tc::mbar_init(&tbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    uint32_t mphase = 0, tphase = 0;
    int cur_slot = -1;
    bool store_pending = false;  // thread 0: a TMA store may still be reading sH
    int it = 0;

    // contiguous run of tiles per cluster: neighbouring tiles share the adapter
    int t0, t1;
    even_share(a.counters[PREFT_CTR_TILES], cluster_id, nclusters, t0, t1);
    for (int t = t0; t < t1; ++t) {
        const int4 tile = a.tiles[t];  // (slot, first sorted position, n tokens, segment)
        if (tile.x < a.slot_base) continue;  // LoRA-class tile: same decision in every CTA of the cluster
        TC_MARK(0);
        const int slot = tile.x - a.slot_base;
        const int ntok = tile.z;
        if (tid < kTcRows) s_rows[tid] = tid < ntok ? a.tokens[tile.y + tid].x : -1;
        if (tid == 0 && store_pending) {
            tc::tma_store_wait_read();  // sH is about to be overwritten
            store_pending = false;
        }
        __syncthreads();
        const int row0 = s_rows[0];
        const bool full = ntok == kTcRows && s_rows[kTcRows - 1] - row0 == kTcRows - 1;

        // ---- 1. stage h rows (and weights when the adapter changes)
        if (full) {
            if (tid == 0) {
                tc::mbar_expect_tx(&tbar, kTcRows * SLICE * 2);
#pragma unroll
                for (int p = 0; p < PANELS; ++p) tc::tma_load_2d(sH + p * kTcRows * 128, &tmap, col0 + p * 64, row0, &tbar);
            }
        } else {
            const __nv_bfloat16* hb = a.h + col0;
            for (int i = tid; i < kTcRows * (SLICE / 8); i += kTcThreads) {
                const int r8 = i & 7, c8 = (i >> 3) % (SLICE / 8), row = (i / SLICE) * 8 + r8;
                const int tok = s_rows[row];
                if (tok >= 0)
                    cp_async16(sH + tc::sw128_offset(row, c8 * 8, kTcRows), hb + static_cast<long long>(tok) * a.ldh + c8 * 8);
            }
        }
        if (slot != cur_slot) {
            const __nv_bfloat16* Ab = a.A + static_cast<long long>(slot) * R * a.d + col0;
            for (int i = tid; i < R * (SLICE / 8); i += kTcThreads) {
                const int r8 = i & 7, c8 = (i >> 3) % (SLICE / 8), k = (i / SLICE) * 8 + r8;
                cp_async16(sA + tc::kmajor_offset(k, c8 * 8, SLICE), Ab + static_cast<long long>(k) * a.d + c8 * 8);
            }
            const __nv_bfloat16* Bb = a.Bt + (static_cast<long long>(slot) * a.d + col0) * R;
            for (int i = tid; i < SLICE * (R / 8); i += kTcThreads) {
                const int n = i / (R / 8), c8 = i % (R / 8);
                cp_async16(sBt + tc::kmajor_offset(n, c8 * 8, R), Bb + static_cast<long long>(n) * R + c8 * 8);
            }
            cur_slot = slot;
        }
        cp_async_wait_all();
        if (full) {
            tc::mbar_wait(&tbar, tphase);
            tphase ^= 1;
        }
        tc::fence_proxy_async();
        __syncthreads();
        TC_MARK(1);

        // ---- 2. shrink: TMEM[acc q: q*R .. q*R+R) = sum_{k % 4 == q} H_k . A_k^T
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t id = tc::idesc_bf16_f32(kTcRows, R);
#pragma unroll
            for (int k = 0; k < KSTEPS; ++k)
                tc::mma_bf16(tmem + (k % kTcAcc) * R, tc::desc_kmajor_sw128(sH + (k >> 2) * kTcRows * 128 + (k & 3) * 32),
                             tc::desc_kmajor(sA + k * 256, 128, SLICE * 16), id, k >= kTcAcc ? 1u : 0u);
            tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, mphase);
        mphase ^= 1;
        tc::fence_after_sync();
        TC_MARK(2);
        if (warp < 4) {
            const int row = warp * 32 + lane;
            float* P = reinterpret_cast<float*>(sm + L::P);
            float s[R];
#pragma unroll
            for (int j = 0; j < R; ++j) s[j] = 0.f;
#pragma unroll
            for (int q = 0; q < kTcAcc; ++q) {
                const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + q * R;
                if constexpr (R == 16) {
                    uint32_t w[16];
                    tc::tmem_ld16(taddr, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) s[j] += __uint_as_float(w[j]);
                } else {
                    uint32_t w[32];
                    tc::tmem_ld32(taddr, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) s[j] += __uint_as_float(w[j]);
                }
            }
#pragma unroll
            for (int j = 0; j < R; j += 4)
                *reinterpret_cast<float4*>(P + row * R + j) = make_float4(s[j], s[j + 1], s[j + 2], s[j + 3]);
        }
        tc::fence_before_sync();
        tc::cluster_sync();  // every CTA's partial rows are visible cluster-wide
        TC_MARK(3);

        // ---- 3. reduce-scatter the partials, push bf16 hi/lo V to every CTA
        for (int idx = tid; idx < rows_per * R; idx += kTcThreads) {
            const int j = crank * rows_per + idx / R, k = idx % R;
            const uint32_t off = static_cast<uint32_t>((j * R + k) * 4);
            float part[C];
#pragma unroll
            for (int q = 0; q < C; ++q) part[q] = ld_dsmem_f32(tc::map_shared(sP + off, q));
            float s = 0.f;
#pragma unroll
            for (int q = 0; q < C; ++q) s += part[q];
            const float v = (s + __ldg(a.bias + static_cast<long long>(slot) * R + k)) * __ldg(a.scale + slot);
            const __nv_bfloat16 hi = __float2bfloat16_rn(v);
            const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
            const uint32_t voff = tc::kmajor_offset(j, k, R);
            const unsigned short hb = *reinterpret_cast<const unsigned short*>(&hi);
            const unsigned short lb = *reinterpret_cast<const unsigned short*>(&lo);
#pragma unroll
            for (int q = 0; q < C; ++q) {
                st_dsmem_u16(tc::map_shared(sVhi + voff, q), hb);
                st_dsmem_u16(tc::map_shared(sVlo + voff, q), lb);
            }
        }
        tc::cluster_sync();  // V complete in every CTA
        TC_MARK(4);

        // ---- 4. expand: TMEM[0:SLICE] = V_hi . Bt^T + V_lo . Bt^T (N = 256 per UMMA)
        if (tid == 0) {
            tc::fence_proxy_async();
            tc::fence_after_sync();
            const uint32_t id = tc::idesc_bf16_f32(kTcRows, 256);
#pragma unroll
            for (int half = 0; half < SLICE / 256; ++half) {
                const uint32_t bbase = sBt + half * 32 * (R * 16);  // 256 rows = 32 core-row groups
#pragma unroll
                for (int k = 0; k < R / 16; ++k) {
                    const uint64_t bd = tc::desc_kmajor(bbase + k * 256, 128, R * 16);
                    tc::mma_bf16(tmem + half * 256, tc::desc_kmajor(sVhi + k * 256, 128, R * 16), bd, id,
                                 k > 0 ? 1u : 0u);
                    tc::mma_bf16(tmem + half * 256, tc::desc_kmajor(sVlo + k * 256, 128, R * 16), bd, id, 1u);
                }
            }
            tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, mphase);
        mphase ^= 1;
        tc::fence_after_sync();
        TC_MARK(5);

        // ---- 5. epilogue: h_slice += delta in shared memory (swizzled rows)
        {
            constexpr int HALF = SLICE / 2;  // columns per warp
            const int q = warp & 3, half = warp >> 2, row = q * 32 + lane;
            const bool live = row < ntok;
            const uint32_t tl = tmem + (static_cast<uint32_t>(q * 32) << 16) + half * HALF;
#pragma unroll 1
            for (int c0 = 0; c0 < HALF; c0 += 64) {
                uint32_t v[64];
                tc::tmem_ld32(tl + c0, *reinterpret_cast<uint32_t(*)[32]>(v));
                tc::tmem_ld32(tl + c0 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                tc::tmem_ld_wait();
                if (live) {
                    const int col = half * HALF + c0;
#pragma unroll
                    for (int hh = 0; hh < 8; ++hh) {
                        uint4* p = reinterpret_cast<uint4*>(sm + L::H + tc::sw128_offset(row, col + hh * 8, kTcRows));
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
        tc::fence_proxy_async();  // epilogue smem writes -> async proxy (TMA store)
        __syncthreads();
        TC_MARK(6);
        if (full) {
            if (tid == 0) {
#pragma unroll
                for (int p = 0; p < PANELS; ++p) tc::tma_store_2d(&tmap, col0 + p * 64, row0, sH + p * kTcRows * 128);
                tc::tma_store_commit();
                store_pending = true;
            }
        } else {
            __nv_bfloat16* hb = a.h + col0;
            for (int i = tid; i < kTcRows * (SLICE / 8); i += kTcThreads) {
                const int r8 = i & 7, c8 = (i >> 3) % (SLICE / 8), row = (i / SLICE) * 8 + r8;
                const int tok = s_rows[row];
                if (tok >= 0)
                    *reinterpret_cast<uint4*>(hb + static_cast<long long>(tok) * a.ldh + c8 * 8) =
                        *reinterpret_cast<const uint4*>(sm + L::H + tc::sw128_offset(row, c8 * 8, kTcRows));
            }
            __syncthreads();
        }
        TC_MARK(7);
        ++it;
    }
    if (tid == 0) tc::tma_store_wait_all();  // bulk stores complete before the CTA (and its smem) retires
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, L::TMEM_COLS);
}

static int g_tc_last_clusters = 0;
void reft_tc_set_profile(long long* buf) { g_tc_prof = buf; }
int reft_tc_last_clusters() { return g_tc_last_clusters; }

template <int R, int C, int SLICE>
static int launch_reft_tc(const ReftTcArgs& args, const CUtensorMap& tmap, cudaStream_t stream) {
    auto fn = reft_tc_kernel<R, C, SLICE>;
    const int smem = TcSmem<R, SLICE>::TOTAL;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -static_cast<int>(e);
    if (C > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return -static_cast<int>(e);
    }
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
    cfg.gridDim = dim3(C * 296);
    int nclusters = 0;
    e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
    if (e != cudaSuccess) return -static_cast<int>(e);
    if (nclusters < 1) return PREFT_ERR_CONFIG;
    g_tc_last_clusters = nclusters;
    cfg.gridDim = dim3(C * nclusters);
    e = cudaLaunchKernelEx(&cfg, fn, tmap, args);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

// returns 0 on launch, PREFT_ERR_SHAPE if the shape is not TC-eligible, or -cudaError
int reft_tc_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A,
                  const void* Bt, const void* bias, const void* scale, int r, cudaStream_t stream) {
    if (!Bt || (r != 16 && r != 32) || d % 512 || rows < 1) return PREFT_ERR_SHAPE;
    if (d != 1024 && d != 2048 && d != 4096) return PREFT_ERR_SHAPE;
    if (meta->tile_tokens > kTcRows || (ldh % 8) || (reinterpret_cast<uintptr_t>(h) & 15) ||
        (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(Bt) & 15))
        return PREFT_ERR_SHAPE;
    CUtensorMap tmap{};
    if (!make_tmap_bf16_sw128(&tmap, h, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(ldh), 64, kTcRows))
        return PREFT_ERR_CONFIG;
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
    args.prof = g_tc_prof;
    // 512-column slices (cluster of d/512).  Measured on B200: 256-column
    // slices fit two CTAs per SM but 16-CTA clusters only reach 7 co-resident
    // clusters (112 CTAs), which loses more than the overlap gains.
    if (r == 16) {
        if (d == 1024) return launch_reft_tc<16, 2, 512>(args, tmap, stream);
        if (d == 2048) return launch_reft_tc<16, 4, 512>(args, tmap, stream);
        return launch_reft_tc<16, 8, 512>(args, tmap, stream);
    }
    if (d == 1024) return launch_reft_tc<32, 2, 512>(args, tmap, stream);
    if (d == 2048) return launch_reft_tc<32, 4, 512>(args, tmap, stream);
    return launch_reft_tc<32, 8, 512>(args, tmap, stream);
}

}  // namespace preft
