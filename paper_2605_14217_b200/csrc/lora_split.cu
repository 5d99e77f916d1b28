// K2 split in two halves around the rank-r intermediate, for tensor-parallel
// LoRA^P (BASELINE config 4: Llama-3.1-70B, 8-way TP, r = 16) and for r >= 16
// on one GPU.
//
//   shrink:  P[t, s*R + k]  = sum_c x[t, c] . A_s[a][k, c]            (f32)
//   (TP)     P <- all-reduce_sum(P) over the tensor-parallel group (NCCL)
//   expand:  y_s[t, :]     += scale_s[a] * sum_k P[t, s*R + k] . Bt_s[a][k, :]
//
// which is the reference's  out[rows] += s * ((X A^T) B^T)  (model.py:449-451,
// adapters.py:284-288) with X A^T computed as a sum of per-rank partials: each
// rank holds A sharded along the input dimension m and B along the output
// dimension n, so the pool shards 8 ways and only T_p x r floats per site
// cross NVLink.  P is indexed by token row (rows of unselected tokens are
// never read).
//
// Two implementations each:
//   tcgen05 (bf16, R in {16, 32}, m % 64 == 0, n % 128 == 0): the M = 64 unit
//     pipeline of the tensor-core ReFT kernel (csrc/reft_tc.cu) cut in half —
//     shrink: TMA x/A panels -> UMMA -> TMEM -> P rows;  expand: P rows ->
//     bf16 hi/lo V -> UMMA against the pre-tiled Bt chunk -> TMEM -> y chunk
//     read-modify-write in shared memory -> TMA store.  One CTA per SM.
//   SIMT (any dtype / rank, one warp per token row) for everything else.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

int grid_for(const void* fn, int threads, int num_sms);

struct SplitSite {
    const void* A;
    const void* Bt;     // row-major [S][R][n] (SIMT)
    const void* Bt_tc;  // core-matrix tiled [S][n/8][R/8][8][8] (tensor cores)
    const void* scale;
    void* y;
    long long ldy;
    int n;
    int pad;
};

struct SplitArgs {
    const void* x;
    long long ldx;
    int m;
    int nsites;
    SplitSite site[3];
    void* P;  // [rows][ldp] acc type
    long long ldp;
    int slot_base;  // LoRA-class slots are < slot_base (meta->slot_split)
    int ks;         // tensor-core shrink: K splits per unit (1 or 2)
    long long* prof;  // diagnostics: clock64 stamps of CTA 0 (NULL in production)
    const int2* tokens;
    const int2* chunks;
    const int4* units;
    const int* counters;
};

// ---------------------------------------------------------------- SIMT halves

template <typename T, bool VEC, int R, int NS, int U>
__global__ void __launch_bounds__(256) shrink_simt_kernel(const SplitArgs a) {
    using V = Vec<T, VEC>;
    using acc_t = typename V::acc_t;
    constexpr int W = V::W;
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    int i0, i1;
    even_share(a.counters[PREFT_CTR_SPLIT], gw, nw, i0, i1);
    const int mv = a.m / W;
    for (int i = i0; i < i1; ++i) {
        const int2 ts = a.tokens[i];
        const T* __restrict__ xr = static_cast<const T*>(a.x) + static_cast<long long>(ts.x) * a.ldx;
        acc_t acc[NS][R];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) acc[s][k] = acc_t(0);
        for (int c0 = lane; c0 < mv; c0 += kWarp * U) {
            typename V::raw_t xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + kWarp * u;
                xv[u] = c < mv ? V::ld_stream(xr + static_cast<long long>(c) * W) : V::zero();
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = c0 + kWarp * u;
                if (c < mv) {
                    acc_t xf[W];
                    V::to_acc(xv[u], xf);
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        const T* As = static_cast<const T*>(a.site[s].A) +
                                      (static_cast<long long>(ts.y) * R) * a.m + static_cast<long long>(c) * W;
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            acc_t af[W];
                            V::to_acc(V::ld_weight(As + static_cast<long long>(k) * a.m), af);
#pragma unroll
                            for (int j = 0; j < W; ++j) acc[s][k] = macc(xf[j], af[j], acc[s][k]);
                        }
                    }
                }
            }
        }
        acc_t* pr = static_cast<acc_t*>(a.P) + static_cast<long long>(ts.x) * a.ldp;
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const acc_t v = warp_sum(acc[s][k]);
                if (lane == ((s * R + k) & 31)) pr[s * R + k] = v;
            }
    }
}

template <typename T, bool VEC, int R, int NS, int U>
__global__ void __launch_bounds__(256) expand_simt_kernel(const SplitArgs a) {
    using V = Vec<T, VEC>;
    using acc_t = typename V::acc_t;
    constexpr int W = V::W;
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    int i0, i1;
    even_share(a.counters[PREFT_CTR_SPLIT], gw, nw, i0, i1);
    for (int i = i0; i < i1; ++i) {
        const int2 ts = a.tokens[i];
        const acc_t* pr = static_cast<const acc_t*>(a.P) + static_cast<long long>(ts.x) * a.ldp;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const acc_t sc = __ldg(static_cast<const acc_t*>(a.site[s].scale) + ts.y);
            acc_t v[R];
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = pr[s * R + k] * sc;
            const int n = a.site[s].n, nv = n / W;
            T* __restrict__ yr = static_cast<T*>(a.site[s].y) + static_cast<long long>(ts.x) * a.site[s].ldy;
            const T* Bs = static_cast<const T*>(a.site[s].Bt) + (static_cast<long long>(ts.y) * R) * n;
            for (int c0 = lane; c0 < nv; c0 += kWarp * U) {
                typename V::raw_t yv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    yv[u] = c < nv ? V::ld_rw(yr + static_cast<long long>(c) * W) : V::zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    if (c < nv) {
                        acc_t yf[W], d[W];
                        V::to_acc(yv[u], yf);
#pragma unroll
                        for (int j = 0; j < W; ++j) d[j] = acc_t(0);
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            acc_t bf[W];
                            V::to_acc(V::ld_weight(Bs + static_cast<long long>(k) * n + static_cast<long long>(c) * W), bf);
#pragma unroll
                            for (int j = 0; j < W; ++j) d[j] = macc(v[k], bf[j], d[j]);
                        }
#pragma unroll
                        for (int j = 0; j < W; ++j) yf[j] += d[j];
                        V::st(yr + static_cast<long long>(c) * W, yf);
                    }
                }
            }
        }
    }
}

// ---------------------------------------------------------------- tcgen05 halves

constexpr int kSpU = 64;                  // unit rows (UMMA M)
constexpr int kSpChunk = PREFT_CHUNK_ROWS;
constexpr int kSpN = 128;                 // expand chunk width (UMMA N) of narrow sites
constexpr int kSpNMax = 256;              // expand chunk width of sites with n % 256 == 0
constexpr int kSpAcc = 4;                 // split shrink accumulators = UMMA-issuing warps
constexpr int kShrinkThreads = 32 * (6 + kSpAcc);

struct SplitMaps {
    CUtensorMap x;       // x [rows][m] (this rank's columns), 16-row x 64-col boxes
    CUtensorMap x64;     // the same with 64-row boxes (a unit of 4 contiguous chunks)
    CUtensorMap A[3];    // A_s [S*R][m], R-row x 64-col boxes
    CUtensorMap y[3];    // y_s [rows][n], 16-row x 64-col boxes
    CUtensorMap y64[3];  // the same with 64-row boxes
};

// A unit whose 4 chunks are consecutive rows of one entry loads as ONE 64-row
// TMA box: a TMA instruction costs ~100 cycles to issue, so per-chunk boxes
// (4 per panel) capped the shrink at ~8 KB per 400 cycles per SM.
__device__ __forceinline__ bool unit_contiguous(const int2* chunks, int4 U) {
    if (U.z != 4) return false;
    const int2 c0 = chunks[U.y], c1 = chunks[U.y + 1], c2 = chunks[U.y + 2], c3 = chunks[U.y + 3];
    return c0.y == kSpChunk && c1.y == kSpChunk && c2.y == kSpChunk && c1.x == c0.x + kSpChunk &&
           c2.x == c0.x + 2 * kSpChunk && c3.x == c0.x + 3 * kSpChunk;
}

constexpr int kPps = 4;  // K panels (64 columns each) per shrink ring stage: amortises the per-stage overheads

template <int R, int NS>
struct ShrinkLayout {
    static constexpr int NSR = NS * R;
    static constexpr int PANEL = kSpU * 128;               // 64 rows x 64 columns
    static constexpr int X_BYTES = kPps * PANEL;
    static constexpr int AP_BYTES = R * 128;
    static constexpr int STAGE = X_BYTES + kPps * NS * AP_BYTES;  // multiple of 1024
    static constexpr int STAGES_FIT = (227 * 1024 - 2048) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 16 ? 16 : STAGES_FIT;
    static constexpr int SMEM = STAGES * STAGE + 1024;
    static constexpr int TMEM_COLS = 2 * kSpAcc * NSR <= 256 ? 256 : 512;
    static_assert(2 * kSpAcc * NSR <= 512, "TMEM budget");
};

// warps: 0 TMA producer (x), 6 TMA producer (A), 1 UMMA issuer, 2..5 TMEM -> P rows (lane quadrant = warp % 4)
template <int R, int NS>
__global__ void __launch_bounds__(kShrinkThreads, 1) shrink_tc_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a) {
    using L = ShrinkLayout<R, NS>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[L::STAGES], empty[L::STAGES];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = (tc::smem_u32(sm_raw) + 1023u) & ~1023u;
    if (warp == 0) tc::tmem_alloc(&tslot, L::TMEM_COLS);
    if (tid == 32) {
        for (int i = 0; i < L::STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], kSpAcc);  // one commit from each UMMA-issuing warp
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], kSpAcc);
            tc::mbar_init(&s_empty[b], 4);
        }
        tc::fence_mbar_init();
        tc::prefetch_tmap(&maps.x);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    // work item = (unit, 1/ks of the K panels): ks = 2 balances launches with
    // ~2 units per SM; the two halves meet in P through f32 atomics, whose
    // order cannot change a two-term sum (0 + a + b == 0 + b + a)
    tc::pdl_launch_dependents();
    tc::pdl_wait();  // everything below reads the previous kernels' output
    const int ks = a.ks;
    int w0, w1;
    even_share(a.counters[PREFT_CTR_UNITS] * ks, blockIdx.x, gridDim.x, w0, w1);
    const int NP = a.m / 64;

    if (warp == 0) {
        // x producer: lane q issues chunk q's box, so a stage's boxes are in
        // flight together (one thread pays ~100+ cycles per TMA issue)
        const uint64_t stream = tc::policy_evict_first();
        int stage = 0, npf = 0;
        uint32_t phase = 0;
        for (int w = w0; w < w1; ++w) {
            const int4 U = a.units[w / ks];
            if (U.x >= a.slot_base) continue;  // ReFT-class unit
            const int p0 = (w % ks) * NP / ks, p1 = (w % ks + 1) * NP / ks;
            const int nch = U.z;
            const int row = lane < nch ? a.chunks[U.y + lane].x : 0;
            const bool contig = unit_contiguous(a.chunks, U);
            const uint32_t bytes = static_cast<uint32_t>(kPps * (nch * kSpChunk * 128 + NS * L::AP_BYTES));
            for (int p = p0; p < p1; p += kPps) {
                if (lane == 0) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    if (a.prof && blockIdx.x == 0 && npf < 128) a.prof[npf * 4 + 0] = clock64();
                    tc::mbar_expect_tx(&full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + stage * L::STAGE;
                const int rq = __shfl_sync(0xffffffffu, row, lane & 3);  // chunk (lane & 3)'s first row, all lanes
                const int r0 = __shfl_sync(0xffffffffu, row, 0);         // the unit's first row
                if (contig) {
                    if (lane < kPps)
                        tc::tma_load_2d_hint(st + lane * L::PANEL, &maps.x64, (p + lane) * 64, r0, &full[stage], stream);
                } else if (lane < 4 * kPps) {
                    const int pp = lane >> 2, q = lane & 3;
                    if (q < nch)
                        tc::tma_load_2d_hint(st + pp * L::PANEL + q * (kSpChunk * 128), &maps.x, (p + pp) * 64, rq,
                                             &full[stage], stream);
                }
                ++npf;
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 6) {
        // second producer: the adapters' A panels (TMA issue costs ~100+ cycles
        // per box from one thread, so x and A boxes are issued from two warps)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int w = w0; w < w1; ++w) {
                const int4 U = a.units[w / ks];
                if (U.x >= a.slot_base) continue;
                const int p0 = (w % ks) * NP / ks, p1 = (w % ks + 1) * NP / ks;
                for (int p = p0; p < p1; p += kPps) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    const uint32_t st = sbase + stage * L::STAGE;
#pragma unroll
                    for (int pp = 0; pp < kPps; ++pp)
#pragma unroll
                        for (int s = 0; s < NS; ++s)
                            tc::tma_load_2d(st + L::X_BYTES + (pp * NS + s) * L::AP_BYTES, &maps.A[s], (p + pp) * 64,
                                            U.x * R, &full[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1 || warp >= 7) {
        // kSpAcc warps issue the UMMAs, K-step k into accumulator k % kSpAcc:
        // one issuing thread is capped at ~140 cycles per UMMA
        const int mw = warp == 1 ? 0 : warp - 6;
        if (lane == 0) {
            // the sites' A panels sit back to back in the stage, so one UMMA with
            // N = NS * R covers all of them (tiny-N UMMAs cost ~60-90 cycles each)
            const uint32_t id = tc::idesc_bf16_f32(kSpU, L::NSR);
            int stage = 0, ub = 0, nmc = 0;
            uint32_t phase = 0;
            for (int w = w0; w < w1; ++w) {
                const int4 U = a.units[w / ks];
                if (U.x >= a.slot_base) continue;
                const int p0 = (w % ks) * NP / ks, p1 = (w % ks + 1) * NP / ks;
                const int sb = ub & 1;
                tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
                tc::fence_after_sync();
                const uint32_t dS = tmem + sb * kSpAcc * L::NSR;
                for (int p = p0; p < p1; p += kPps) {
                    tc::mbar_wait(&full[stage], phase);
                    if (a.prof && blockIdx.x == 0 && mw == 0 && nmc < 128) a.prof[nmc * 4 + 1] = clock64();
                    ++nmc;
                    tc::fence_after_sync();
                    const uint32_t st = sbase + stage * L::STAGE;
#pragma unroll
                    for (int k = mw; k < 4 * kPps; k += kSpAcc) {
                        const int kk = (p - p0) * 4 + k, pp = k >> 2, kq = k & 3;
                        tc::mma_bf16(dS + mw * L::NSR, tc::desc_kmajor_sw128(st + pp * L::PANEL + kq * 32),
                                     tc::desc_kmajor_sw128(st + L::X_BYTES + pp * NS * L::AP_BYTES + kq * 32), id,
                                     kk >= kSpAcc ? 1u : 0u);
                    }
                    tc::mma_commit(&empty[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                tc::mma_commit(&s_full[sb]);
                ++ub;
            }
        }
    } else if (warp < 6) {
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        for (int w = w0; w < w1; ++w) {
            const int4 U = a.units[w / ks];
            if (U.x >= a.slot_base) continue;
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const int sb = ub & 1;
            tc::mbar_wait(&s_full[sb], (ub >> 1) & 1);
            if (a.prof && blockIdx.x == 0 && lane == 0 && q == 0 && ub < 128) a.prof[ub * 4 + 2] = clock64();
            tc::fence_after_sync();
            float s[L::NSR];
#pragma unroll
            for (int c = 0; c < L::NSR; ++c) s[c] = 0.f;
#pragma unroll
            for (int acc = 0; acc < kSpAcc; ++acc)
#pragma unroll
                for (int c0 = 0; c0 < L::NSR; c0 += 16) {
                    uint32_t w[16];
                    tc::tmem_ld16(tmem + lane_base + sb * kSpAcc * L::NSR + acc * L::NSR + c0, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 16; ++c) s[c0 + c] += __uint_as_float(w[c]);
                }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
            if (lane < ch.y) {
                float* pr = static_cast<float*>(a.P) + static_cast<long long>(ch.x + lane) * a.ldp;
                if (ks == 1) {
#pragma unroll
                    for (int c = 0; c < L::NSR; c += 4)
                        *reinterpret_cast<float4*>(pr + c) = make_float4(s[c], s[c + 1], s[c + 2], s[c + 3]);
                } else {
#pragma unroll
                    for (int c = 0; c < L::NSR; ++c) atomicAdd(pr + c, s[c]);
                }
            }
            ++ub;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, L::TMEM_COLS);
    }
}

template <int R, int NS>
struct ExpandLayout {
    static constexpr int Y_BYTES = 4 * kSpU * 128;         // 64 rows x 256 cols (four swizzled panels)
    static constexpr int BT_BYTES = kSpNMax * R * 2;
    static constexpr int STAGE = Y_BYTES + BT_BYTES;       // multiple of 1024
    static constexpr int V_BYTES = kSpU * R * 2;           // one V (hi or lo) of one site
    static constexpr int OFF_V = 0;                        // [2 buffers][NS sites][hi, lo]
    static constexpr int OFF_RING = 4 * NS * V_BYTES;      // multiple of 1024
    static constexpr int STAGES_FIT = (227 * 1024 - 2048 - OFF_RING) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int SMEM = OFF_RING + STAGES * STAGE + 1024;
    static_assert(STAGES >= 3, "expand ring too shallow");
};

// The expand's work item is (unit, block of kExpBlock 128-column chunks) over
// the concatenated chunks of all sites, so a launch balances across CTAs even
// when a batch has few units per SM (Punica-sized steps: ~2 units per CTA,
// but 56 gate/up chunks per unit).  Consecutive items of one unit share its V.
constexpr int kExpBlock = 4;

struct ExpandItems {
    int w0, w1;  // this CTA's contiguous share of items
    int ipu;     // items per unit
    int nc;      // chunks per unit (all sites)
    int off[4];  // first chunk of each site
    int cw[3];   // chunk width of each site: 256 columns (one N = 256 UMMA), else 128
    __device__ void init(const SplitArgs& a, int nsites) {
        nc = 0;
        for (int s = 0; s < nsites; ++s) {
            off[s] = nc;
            cw[s] = a.site[s].n % kSpNMax == 0 ? kSpNMax : kSpN;
            nc += a.site[s].n / cw[s];
        }
        off[nsites] = nc;
        ipu = (nc + kExpBlock - 1) / kExpBlock;
        even_share(a.counters[PREFT_CTR_UNITS] * ipu, blockIdx.x, gridDim.x, w0, w1);
    }
    __device__ void site_of(int c, int nsites, int& s, int& j) const {
        s = 0;
        while (s + 1 < nsites && c >= off[s + 1]) ++s;
        j = c - off[s];
    }
};

// warps: 0 TMA producer, 1 UMMA issuer, 2-3 P rows -> bf16 hi/lo V, 4-11 epilogue
template <int R, int NS>
__global__ void __launch_bounds__(384, 1) expand_tc_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a) {
    using L = ExpandLayout<R, NS>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[L::STAGES], empty[L::STAGES];
    __shared__ __align__(8) uint64_t v_full[2], v_empty[2], d_full[2], d_empty[2];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t raw = tc::smem_u32(sm_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    unsigned char* sgen = sm_raw + (sbase - raw);
    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 32) {
        for (int i = 0; i < L::STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1 + 8);  // MMA commit (Bt read) + 8 epilogue warps (y stored)
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&v_full[b], 2);
            tc::mbar_init(&v_empty[b], 1);
            tc::mbar_init(&d_full[b], 1);
            tc::mbar_init(&d_empty[b], 8);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    tc::pdl_launch_dependents();
    tc::pdl_wait();  // everything below reads the previous kernels' output
    ExpandItems it;
    it.init(a, NS);

    if (warp == 0) {
        // producer: lane 4*pp + q issues y panel pp of chunk q, lane 16 the Bt chunk
        const uint64_t stream = tc::policy_evict_first();
        const int pp = lane >> 2, q = lane & 3;
        int stage = 0, npc = 0;
        uint32_t phase = 0;
        for (int w = it.w0; w < it.w1; ++w) {
            const int4 U = a.units[w / it.ipu];
            if (U.x >= a.slot_base) continue;
            const int nch = U.z;
            const int row = q < nch ? a.chunks[U.y + q].x : 0;
            const int row0 = a.chunks[U.y].x;
            const bool contig = unit_contiguous(a.chunks, U);
            const int c0 = (w % it.ipu) * kExpBlock, c1 = min(it.nc, c0 + kExpBlock);
            for (int c = c0; c < c1; ++c) {
                int s, j;
                it.site_of(c, NS, s, j);
                const int cw = it.cw[s];
                const uint32_t bt_bytes = static_cast<uint32_t>(cw * R * 2);
                if (lane == 0) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    if (a.prof && blockIdx.x == 0 && npc < 128) a.prof[512 + npc * 4 + 0] = clock64();
                    tc::mbar_expect_tx(&full[stage], static_cast<uint32_t>((cw / 64) * nch * kSpChunk * 128) + bt_bytes);
                }
                ++npc;
                __syncwarp();
                const uint32_t st = sbase + L::OFF_RING + stage * L::STAGE;
                if (contig) {
                    if (lane < cw / 64)  // one 64-row box per panel
                        tc::tma_load_2d_hint(st + lane * kSpU * 128, &maps.y64[s], j * cw + lane * 64, row0, &full[stage],
                                             stream);
                } else if (lane < 16 && pp < cw / 64 && q < nch) {
                    tc::tma_load_2d_hint(st + pp * kSpU * 128 + q * (kSpChunk * 128), &maps.y[s], j * cw + pp * 64, row,
                                         &full[stage], stream);
                }
                if (lane == 16)
                    tc::bulk_load_1d(st + L::Y_BYTES,
                                     static_cast<const unsigned char*>(a.site[s].Bt_tc) +
                                         static_cast<long long>(U.x) * a.site[s].n * R * 2 +
                                         static_cast<long long>(j) * bt_bytes,
                                     bt_bytes, &full[stage]);
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t id128 = tc::idesc_bf16_f32(kSpU, kSpN), id256 = tc::idesc_bf16_f32(kSpU, kSpNMax);
            int stage = 0, visit = 0, dc = 0, prev = -1;
            uint32_t phase = 0;
            for (int w = it.w0; w < it.w1; ++w) {
                const int u = w / it.ipu;
                const int4 U = a.units[u];
                if (U.x >= a.slot_base) continue;
                const int vb = visit & 1;
                if (u != prev) {
                    tc::mbar_wait(&v_full[vb], (visit >> 1) & 1);
                    tc::fence_after_sync();
                    prev = u;
                }
                const int c0 = (w % it.ipu) * kExpBlock, c1 = min(it.nc, c0 + kExpBlock);
                for (int c = c0; c < c1; ++c) {
                    int s, j;
                    it.site_of(c, NS, s, j);
                    const uint32_t vhi = sbase + L::OFF_V + ((vb * NS + s) * 2) * L::V_BYTES, vlo = vhi + L::V_BYTES;
                    tc::mbar_wait(&full[stage], phase);
                    const int db = dc & 1;
                    tc::mbar_wait(&d_empty[db], ((dc >> 1) & 1) ^ 1u);
                    tc::fence_after_sync();
                    if (a.prof && blockIdx.x == 0 && dc < 128) a.prof[512 + dc * 4 + 1] = clock64();
                    const uint32_t bt = sbase + L::OFF_RING + stage * L::STAGE + L::Y_BYTES;
                    const uint32_t dD = tmem + db * kSpNMax;
                    const uint32_t id = it.cw[s] == kSpNMax ? id256 : id128;
#pragma unroll
                    for (int k = 0; k < R / 16; ++k) {
                        const uint64_t bd = tc::desc_kmajor(bt + k * 256, 128, R * 16);
                        tc::mma_bf16(dD, tc::desc_kmajor(vhi + k * 256, 128, R * 16), bd, id, k > 0 ? 1u : 0u);
                        tc::mma_bf16(dD, tc::desc_kmajor(vlo + k * 256, 128, R * 16), bd, id, 1u);
                    }
                    tc::mma_commit(&d_full[db]);
                    tc::mma_commit(&empty[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                    ++dc;
                }
                // the unit's V buffer is free once its last item has been issued
                const bool last = w + 1 >= it.w1 || (w + 1) / it.ipu != u;
                if (last) {
                    tc::mma_commit(&v_empty[vb]);
                    ++visit;
                    prev = -1;
                }
            }
        }
    } else if (warp < 4) {
        // P rows -> V = scale * P (bf16 hi + lo), 32 rows per warp, once per unit visit
        int visit = 0, prev = -1;
        for (int w = it.w0; w < it.w1; ++w) {
            const int u = w / it.ipu;
            const int4 U = a.units[u];
            if (U.x >= a.slot_base) continue;
            if (u == prev) continue;
            prev = u;
            const int vb = visit & 1;
            const int m = (warp - 2) * 32 + lane, q = m >> 4, rr = m & 15;
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const bool valid = rr < ch.y;
            const float* pr = static_cast<const float*>(a.P) + static_cast<long long>(ch.x + rr) * a.ldp;
            tc::mbar_wait(&v_empty[vb], ((visit >> 1) & 1) ^ 1u);
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const float sc = __ldg(static_cast<const float*>(a.site[s].scale) + U.x);
                unsigned char* vhi = sgen + L::OFF_V + ((vb * NS + s) * 2) * L::V_BYTES;
#pragma unroll
                for (int k0 = 0; k0 < R; k0 += 8) {
                    float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
                    if (valid) {
                        p0 = *reinterpret_cast<const float4*>(pr + s * R + k0);
                        p1 = *reinterpret_cast<const float4*>(pr + s * R + k0 + 4);
                    }
                    const float v[8] = {p0.x * sc, p0.y * sc, p0.z * sc, p0.w * sc,
                                        p1.x * sc, p1.y * sc, p1.z * sc, p1.w * sc};
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        hi[e] = f32x2_to_bf16(v[2 * e], v[2 * e + 1]);
                        float h0, h1;
                        bf16x2_to_acc(hi[e], h0, h1);
                        lo[e] = f32x2_to_bf16(v[2 * e] - h0, v[2 * e + 1] - h1);
                    }
                    const uint32_t off = tc::kmajor_offset(m, k0, R);
                    *reinterpret_cast<uint4*>(vhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(vhi + L::V_BYTES + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&v_full[vb]);
            ++visit;
        }
    } else {
        // epilogue: D -> registers, y chunk += D in shared memory, TMA store
        const int q = warp & 3, hf = (warp - 4) >> 2;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        const uint64_t stream = tc::policy_evict_first();
        const int r1 = lane >> 2, cp = 2 * (lane & 3);
        int stage = 0, dc = 0, pend = -1;
        uint32_t phase = 0;
        for (int w = it.w0; w < it.w1; ++w) {
            const int4 U = a.units[w / it.ipu];
            if (U.x >= a.slot_base) continue;
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const int c0 = (w % it.ipu) * kExpBlock, c1 = min(it.nc, c0 + kExpBlock);
            for (int c = c0; c < c1; ++c) {
                int s, j;
                it.site_of(c, NS, s, j);
                const int cw = it.cw[s], npw = cw / 128;  // 64-column panels per warp: 1 or 2
                const int db = dc & 1;
                tc::mbar_wait(&d_full[db], (dc >> 1) & 1);
                tc::mbar_wait(&full[stage], phase);
                tc::fence_after_sync();
                if (a.prof && blockIdx.x == 0 && warp == 4 && lane == 0 && dc < 128) a.prof[512 + dc * 4 + 2] = clock64();
                uint32_t v[2][32];
                // both loads unconditionally, then the wait: a tcgen05.ld whose
                // issue sits under a branch lets the compiler merge its output
                // registers at the join BEFORE tcgen05.wait::ld, i.e. copy
                // registers the load has not written yet (found as stale D
                // columns 120-127 of 256-wide chunks).  For 128-wide chunks the
                // second load reads the other half's columns and is ignored.
                tc::tmem_ld_16x256b_x8(tmem + lane_base + db * kSpNMax + hf * (cw / 2), v[0]);
                tc::tmem_ld_16x256b_x8(tmem + lane_base + db * kSpNMax + hf * (cw / 2) + 64, v[1]);
                tc::tmem_ld_wait();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&d_empty[db]);
                if (ch.y > 0) {
#pragma unroll
                    for (int pw = 0; pw < 2; ++pw) {
                        if (pw >= npw) break;
                        const int pan = hf * npw + pw;  // 64-column panel of the chunk
                        const uint32_t panel = L::OFF_RING + stage * L::STAGE + pan * kSpU * 128;
                        uint32_t hv[16];
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half)
                                hv[2 * i + half] = *reinterpret_cast<const uint32_t*>(
                                    sgen + panel + tc::sw128_offset(q * kSpChunk + r1 + 8 * half, 8 * i + cp, 64));
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
                                float lo, hi;
                                bf16x2_to_acc(hv[2 * i + half], lo, hi);
                                lo += __uint_as_float(v[pw][4 * i + 2 * half]);
                                hi += __uint_as_float(v[pw][4 * i + 2 * half + 1]);
                                hv[2 * i + half] = f32x2_to_bf16(lo, hi);
                            }
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half)
                                *reinterpret_cast<uint32_t*>(
                                    sgen + panel + tc::sw128_offset(q * kSpChunk + r1 + 8 * half, 8 * i + cp, 64)) =
                                    hv[2 * i + half];
                    }
                    tc::fence_proxy_async();
                    __syncwarp();
                    for (int pw = 0; pw < npw; ++pw) {
                        const int pan = hf * npw + pw;
                        const uint32_t panel = L::OFF_RING + stage * L::STAGE + pan * kSpU * 128;
                        if (ch.y == kSpChunk) {
                            if (lane == 0)
                                tc::tma_store_2d_hint(&maps.y[s], j * cw + pan * 64, ch.x,
                                                      sbase + panel + q * (kSpChunk * 128), stream);
                        } else {
                            __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(a.site[s].y);
                            for (int idx = lane; idx < ch.y * 8; idx += 32) {
                                const int rr = idx >> 3, c16 = idx & 7;
                                const uint4 val = *reinterpret_cast<const uint4*>(
                                    sgen + panel + tc::sw128_offset(q * kSpChunk + rr, c16 * 8, 64));
                                *reinterpret_cast<uint4*>(yb + static_cast<long long>(ch.x + rr) * a.site[s].ldy +
                                                          j * cw + pan * 64 + c16 * 8) = val;
                            }
                        }
                    }
                }
                if (lane == 0) {
                    // release the PREVIOUS stage once its store has read shared
                    // memory: the store of this chunk drains while the next is processed
                    tc::tma_store_commit();
                    tc::tma_store_wait_read_1();
                    if (pend >= 0) tc::mbar_arrive(&empty[pend]);
                    pend = stage;
                    if (a.prof && blockIdx.x == 0 && warp == 4 && dc < 128) a.prof[512 + dc * 4 + 3] = clock64();
                }
                __syncwarp();
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
                ++dc;
            }
        }
        if (lane == 0) {
            tc::tma_store_wait_all();
            if (pend >= 0) tc::mbar_arrive(&empty[pend]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------- dispatch

using SplitFn = void (*)(SplitArgs);

template <typename T, bool VEC, int NS, bool SHRINK>
SplitFn pick_split_rank(int r) {
    constexpr int U = VEC ? 4 : 2;
#define PREFT_SPLIT_CASE(RR)                                                                       \
    case RR:                                                                                       \
        if constexpr (NS * RR <= 64)                                                               \
            return SHRINK ? shrink_simt_kernel<T, VEC, RR, NS, U> : expand_simt_kernel<T, VEC, RR, NS, U>; \
        else                                                                                       \
            return nullptr;
    switch (r) {
        PREFT_SPLIT_CASE(1)
        PREFT_SPLIT_CASE(2)
        PREFT_SPLIT_CASE(4)
        PREFT_SPLIT_CASE(8)
        PREFT_SPLIT_CASE(16)
        PREFT_SPLIT_CASE(32)
        PREFT_SPLIT_CASE(64)
        default: return nullptr;
    }
#undef PREFT_SPLIT_CASE
}

template <typename T, bool SHRINK>
SplitFn pick_split(bool vec, int nsites, int r) {
    if (nsites == 1) return vec ? pick_split_rank<T, true, 1, SHRINK>(r) : pick_split_rank<T, false, 1, SHRINK>(r);
    if (nsites == 2) return vec ? pick_split_rank<T, true, 2, SHRINK>(r) : pick_split_rank<T, false, 2, SHRINK>(r);
    return vec ? pick_split_rank<T, true, 3, SHRINK>(r) : pick_split_rank<T, false, 3, SHRINK>(r);
}

bool pdl_enabled();

template <typename K>
static int launch_tc(K kernel, int smem, int threads, const SplitMaps& maps, const SplitArgs& args, int num_sms,
                     cudaStream_t stream) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -static_cast<int>(e);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(num_sms);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kernel, maps, args);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

static int fill_common(SplitArgs& args, const preft_meta_t* meta, const preft_lora_site_t* sites, int nsites,
                       void* P, long long ldp) {
    args.nsites = nsites;
    for (int s = 0; s < nsites; ++s) {
        args.site[s].A = sites[s].A;
        args.site[s].Bt = sites[s].Bt;
        args.site[s].Bt_tc = sites[s].Bt_tc;
        args.site[s].scale = sites[s].scale;
        args.site[s].y = sites[s].y;
        args.site[s].ldy = sites[s].ldy;
        args.site[s].n = sites[s].n;
    }
    args.P = P;
    args.ldp = ldp;
    args.slot_base = meta->slot_split;
    args.tokens = reinterpret_cast<const int2*>(meta->tokens);
    args.chunks = reinterpret_cast<const int2*>(meta->chunks);
    args.units = reinterpret_cast<const int4*>(meta->units);
    args.counters = meta->counters;
    return PREFT_OK;
}

static long long* g_split_prof = nullptr;
void split_set_profile(long long* buf) { g_split_prof = buf; }

static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// -1 automatic, 0 SIMT only, 1 tensor cores only (env PREFT_SPLIT_VARIANT=simt|tc)
static int g_split_variant = -2;
int split_variant() {
    if (g_split_variant == -2) {
        const char* env = getenv("PREFT_SPLIT_VARIANT");
        g_split_variant = (env && env[0] == 's') ? 0 : (env && env[0] == 't') ? 1 : -1;
    }
    return g_split_variant;
}
void set_split_variant(int v) { g_split_variant = v; }

// Can the tcgen05 pair (shrink + expand) run this group?  Shared by the split
// entry points and by lora_apply's r >= 16 route.
static bool shrink_tc_ok(const preft_meta_t* meta, const void* x, long long ldx, int m,
                         const preft_lora_site_t* sites, int nsites, int r, int dtype, const void* P, long long ldp) {
    bool ok = dtype == PREFT_DTYPE_BF16 && (r == 16 || r == 32) && m % (64 * kPps) == 0 && ldx % 8 == 0 &&
              ldp % 4 == 0 && al16(x) && al16(P) && meta->chunks && meta->units && nsites * r <= 64;
    for (int s = 0; s < nsites; ++s) ok = ok && sites[s].A && al16(sites[s].A);
    return ok;
}

static bool expand_tc_ok(const preft_meta_t* meta, const void* P, long long ldp, const preft_lora_site_t* sites,
                         int nsites, int r, int dtype) {
    bool ok = dtype == PREFT_DTYPE_BF16 && (r == 16 || r == 32) && ldp % 4 == 0 && al16(P) && meta->chunks &&
              meta->units && nsites * r <= 64;
    for (int s = 0; s < nsites; ++s)
        ok = ok && sites[s].Bt_tc && sites[s].n % kSpN == 0 && sites[s].ldy % 8 == 0 && al16(sites[s].y) &&
             al16(sites[s].Bt_tc);
    return ok;
}

bool lora_tc_route_ok(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
                      int nsites, int r, int dtype) {
    if (!meta->lora_part || split_variant() == 0) return false;
    const long long ldp = static_cast<long long>(nsites) * r;
    if (meta->lora_part_floats < static_cast<long long>(meta->T_cap) * ldp) return false;
    return shrink_tc_ok(meta, x, ldx, m, sites, nsites, r, dtype, meta->lora_part, ldp) &&
           expand_tc_ok(meta, meta->lora_part, ldp, sites, nsites, r, dtype);
}

int lora_shrink(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
                const preft_lora_site_t* sites, int nsites, int r, int dtype, void* P, long long ldp,
                cudaStream_t stream, int num_sms) {
    if (!meta || !x || !sites || !P || nsites < 1 || nsites > 3 || m < 1 || ldx < m || rows < 1) return PREFT_ERR_SHAPE;
    if (r < 1 || r > 64 || (r & (r - 1)) || nsites * r > 64) return PREFT_ERR_RANK;
    if (ldp < static_cast<long long>(nsites) * r) return PREFT_ERR_SHAPE;
    if (dtype != PREFT_DTYPE_F32 && dtype != PREFT_DTYPE_BF16 && dtype != PREFT_DTYPE_F64) return PREFT_ERR_DOMAIN;
    for (int s = 0; s < nsites; ++s)
        if (!sites[s].A) return PREFT_ERR_SHAPE;
    SplitArgs args{};
    args.x = x;
    args.ldx = ldx;
    args.m = m;
    fill_common(args, meta, sites, nsites, P, ldp);
    const int variant = split_variant();
    const bool tc_ok = shrink_tc_ok(meta, x, ldx, m, sites, nsites, r, dtype, P, ldp);
    if (variant == 1 && !tc_ok) return PREFT_ERR_SHAPE;
    if (variant != 0 && tc_ok) {
        SplitMaps maps{};
        if (!make_tmap_bf16_sw128(&maps.x, x, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(m),
                                  static_cast<unsigned long long>(ldx), 64, kSpChunk) ||
            !make_tmap_bf16_sw128(&maps.x64, x, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(m),
                                  static_cast<unsigned long long>(ldx), 64, kSpU))
            return PREFT_ERR_CONFIG;
        for (int s = 0; s < nsites; ++s)
            if (!make_tmap_bf16_sw128(&maps.A[s], sites[s].A, 1ull << 20, static_cast<unsigned long long>(m),
                                      static_cast<unsigned long long>(m), 64, static_cast<unsigned>(r)))
                return PREFT_ERR_CONFIG;
        // two K halves per unit when the unit's K range is long enough to split
        // (P must start at zero: the halves accumulate into it)
        args.ks = getenv("PREFT_SPLIT_KS") ? atoi(getenv("PREFT_SPLIT_KS")) : 1;
        args.prof = g_split_prof;
        if (args.ks > 1) {
            const cudaError_t e = cudaMemsetAsync(P, 0, static_cast<size_t>(rows) * ldp * sizeof(float), stream);
            if (e != cudaSuccess) return -static_cast<int>(e);
        }
        if (r == 16) {
            if (nsites == 1) return launch_tc(shrink_tc_kernel<16, 1>, ShrinkLayout<16, 1>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
            if (nsites == 2) return launch_tc(shrink_tc_kernel<16, 2>, ShrinkLayout<16, 2>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
            return launch_tc(shrink_tc_kernel<16, 3>, ShrinkLayout<16, 3>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
        }
        if (nsites == 1) return launch_tc(shrink_tc_kernel<32, 1>, ShrinkLayout<32, 1>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
        if (nsites == 2) return launch_tc(shrink_tc_kernel<32, 2>, ShrinkLayout<32, 2>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
        return PREFT_ERR_RANK;  // 3 x 32 > 64 columns of P per row (checked above)
    }
    const int W = dtype == PREFT_DTYPE_BF16 ? 8 : dtype == PREFT_DTYPE_F32 ? 4 : 2;
    bool vec = m % W == 0 && ldx % W == 0 && al16(x);
    for (int s = 0; s < nsites; ++s) vec = vec && al16(sites[s].A);
    SplitFn fn = dtype == PREFT_DTYPE_BF16  ? pick_split<__nv_bfloat16, true>(vec, nsites, r)
                 : dtype == PREFT_DTYPE_F32 ? pick_split<float, true>(vec, nsites, r)
                                            : pick_split<double, true>(vec, nsites, r);
    if (!fn) return PREFT_ERR_RANK;
    fn<<<grid_for(reinterpret_cast<const void*>(fn), 256, num_sms), 256, 0, stream>>>(args);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

int lora_expand(const preft_meta_t* meta, const void* P, long long ldp, long long rows, const preft_lora_site_t* sites,
                int nsites, int r, int dtype, cudaStream_t stream, int num_sms) {
    if (!meta || !P || !sites || nsites < 1 || nsites > 3 || rows < 1) return PREFT_ERR_SHAPE;
    if (r < 1 || r > 64 || (r & (r - 1)) || nsites * r > 64) return PREFT_ERR_RANK;
    if (ldp < static_cast<long long>(nsites) * r) return PREFT_ERR_SHAPE;
    if (dtype != PREFT_DTYPE_F32 && dtype != PREFT_DTYPE_BF16 && dtype != PREFT_DTYPE_F64) return PREFT_ERR_DOMAIN;
    for (int s = 0; s < nsites; ++s)
        if (!sites[s].scale || !sites[s].y || sites[s].n < 1 || sites[s].ldy < sites[s].n) return PREFT_ERR_SHAPE;
    SplitArgs args{};
    fill_common(args, meta, sites, nsites, const_cast<void*>(P), ldp);
    args.prof = g_split_prof;
    const int variant = split_variant();
    const bool tc_ok = expand_tc_ok(meta, P, ldp, sites, nsites, r, dtype);
    if (variant == 1 && !tc_ok) return PREFT_ERR_SHAPE;
    if (variant != 0 && tc_ok) {
        SplitMaps maps{};
        for (int s = 0; s < nsites; ++s)
            if (!make_tmap_bf16_sw128(&maps.y[s], sites[s].y, static_cast<unsigned long long>(rows),
                                      static_cast<unsigned long long>(sites[s].n),
                                      static_cast<unsigned long long>(sites[s].ldy), 64, kSpChunk) ||
                !make_tmap_bf16_sw128(&maps.y64[s], sites[s].y, static_cast<unsigned long long>(rows),
                                      static_cast<unsigned long long>(sites[s].n),
                                      static_cast<unsigned long long>(sites[s].ldy), 64, kSpU))
                return PREFT_ERR_CONFIG;
        if (r == 16) {
            if (nsites == 1) return launch_tc(expand_tc_kernel<16, 1>, ExpandLayout<16, 1>::SMEM, 384, maps, args, num_sms, stream);
            if (nsites == 2) return launch_tc(expand_tc_kernel<16, 2>, ExpandLayout<16, 2>::SMEM, 384, maps, args, num_sms, stream);
            return launch_tc(expand_tc_kernel<16, 3>, ExpandLayout<16, 3>::SMEM, 384, maps, args, num_sms, stream);
        }
        if (nsites == 1) return launch_tc(expand_tc_kernel<32, 1>, ExpandLayout<32, 1>::SMEM, 384, maps, args, num_sms, stream);
        if (nsites == 2) return launch_tc(expand_tc_kernel<32, 2>, ExpandLayout<32, 2>::SMEM, 384, maps, args, num_sms, stream);
        return PREFT_ERR_RANK;
    }
    const int W = dtype == PREFT_DTYPE_BF16 ? 8 : dtype == PREFT_DTYPE_F32 ? 4 : 2;
    bool vec = true;
    for (int s = 0; s < nsites; ++s) {
        if (!sites[s].Bt) return PREFT_ERR_SHAPE;  // the SIMT expand reads the row-major Bt
        vec = vec && sites[s].n % W == 0 && sites[s].ldy % W == 0 && al16(sites[s].y) && al16(sites[s].Bt);
    }
    SplitFn fn = dtype == PREFT_DTYPE_BF16  ? pick_split<__nv_bfloat16, false>(vec, nsites, r)
                 : dtype == PREFT_DTYPE_F32 ? pick_split<float, false>(vec, nsites, r)
                                            : pick_split<double, false>(vec, nsites, r);
    if (!fn) return PREFT_ERR_RANK;
    fn<<<grid_for(reinterpret_cast<const void*>(fn), 256, num_sms), 256, 0, stream>>>(args);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
