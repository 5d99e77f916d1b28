// K3-TC-R — tensor-core ReFT^P that reads h from HBM exactly once (sm_100a,
// bf16, rank 16 or 32).
//
//     h[t, :] += s_a * ((h[t, :] . A_a^T + b_a) . B_a)      (adapters.py:292-295)
//
// Same work units as K3-TC (reft_tc.cu: <= 4 chunks of <= 16 rows of one
// adapter, one M = 64 UMMA tile, chunk q in TMEM lane quadrant q).  A cluster
// of C = d / COLS CTAs owns a unit, COLS = 1024 (or 512) columns each, and
// the unit's slice of h is PARKED IN TENSOR MEMORY between the shrink and the
// epilogue: an M = 64 tile only uses TMEM lanes 0-15 of each 32-lane quadrant,
// so lanes 16-31 x 512 columns (128 KB) are free and hold 16 panels of
// 64 rows x 64 columns bf16.  The streaming K3-TC re-reads each panel from L2
// after the shrink; under 148 SMs' worth of traffic ~40% of those re-reads
// miss and cost HBM bandwidth.  Here h crosses HBM once in and once out.
//
// Panel g (the g-th 64-column panel this CTA loads) flows
//   HBM -(TMA)-> smem ring slot g % RING -(shrink MMA, and the stash warps'
//   LDS + tcgen05.st)-> TMEM block g % 16 -(epilogue tcgen05.ld, + D)->
//   smem staging -(TMA store)-> HBM
// so the smem ring only covers HBM latency and the shrink of unit u+1 can
// finish while the epilogue of unit u is a quarter done.
//
//   warp 0      producer: h panel (4 x 16-row boxes, evict_first) + A panel
//   warp 1      shrink MMA: TMEM S[64 x R] += H_panel . A_panel^T
//   warp 2      Bt producer (pre-tiled chunk, one bulk copy)
//   warp 3      expand MMA: TMEM D[64 x 128] = V_hi . Bt^T + V_lo . Bt^T
//   warps 4-11  epilogue, two groups on alternate chunks: D + parked h ->
//               bf16 -> staging -> TMA store
//   warps 12-15 V: exchange the partial S with the cluster peers (st.async
//               with complete_tx on the peer's barrier), V = s*(S + b) -> bf16
//               hi + lo
//   warps 16-19 stash: smem panel -> registers -> TMEM lanes 16-31 of their
//               quadrant, in the register layout the epilogue loads back
#include <cuda_bf16.h>

#include <mutex>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

void reft_tc_note_grid(int grid);  // reft_tc.cu: diagnostics (preft_diag_reft_tc)

namespace {

constexpr int kRows = 64;                  // UMMA M
constexpr int kChunkR = PREFT_CHUNK_ROWS;  // 16 rows: one TMA box, one TMEM lane quadrant
constexpr int kN = 128;                    // expand / epilogue chunk width
constexpr int kThreads = 640;              // 20 warps
constexpr int kAcc = 2;                    // split shrink accumulators
constexpr int kTBlocks = 16;               // TMEM parking blocks: 32 columns x lanes 16-31 each
constexpr int kStashBatch = 4;             // panels per TMEM store wait

template <int R, int C, int COLS, bool XG>
struct ResLayout {
    static constexpr int NP = COLS / 64;  // panels per unit slice
    static constexpr int NJ = COLS / kN;  // chunks (even: the epilogue groups alternate)
    static_assert(NP <= kTBlocks, "a unit slice must fit in the TMEM parking lanes");
    static constexpr int H_BYTES = kRows * 128;
    static constexpr int AP_BYTES = R * 128;
    static constexpr int SLOT = H_BYTES + AP_BYTES;  // h panel, then its A panel
    static constexpr int BT_BYTES = kN * R * 2;
    static constexpr int BT_STAGES = R == 16 ? 3 : 2;
    static constexpr int V_BYTES = kRows * R * 2;    // one of V_hi / V_lo
    static constexpr int IN_BYTES = kRows * R * 4;   // one peer's partial S (f32)
    static constexpr int OUT_BYTES = kRows * 128;         // one panel of a chunk (64 rows, 128 B-swizzled)
    static constexpr int OUT_TOTAL = 2 * 2 * OUT_BYTES;   // [2 epilogue groups][2 panels]
    static constexpr int NIN = XG ? 0 : C - 1;      // DSMEM inbox slots (cluster exchange only)
    static constexpr int OTHER = BT_STAGES * BT_BYTES + 4 * V_BYTES + NIN * IN_BYTES + OUT_TOTAL;
    static constexpr int RING_FIT = (227 * 1024 - 2048 - OTHER) / SLOT;  // - alignment, static smem
    static constexpr int RING = RING_FIT > 16 ? 16 : RING_FIT;
    static_assert(RING >= 6, "smem ring too shallow");
    static constexpr int OFF_RING = 0;
    static constexpr int OFF_OUT = RING * SLOT;
    static constexpr int OFF_BT = OFF_OUT + OUT_TOTAL;
    static constexpr int OFF_V = OFF_BT + BT_STAGES * BT_BYTES;  // [2 buffers][hi, lo]
    static constexpr int OFF_IN = OFF_V + 4 * V_BYTES;           // [C-1 peers], single-buffered
    static constexpr int SMEM = OFF_IN + NIN * IN_BYTES + 1024;
    static constexpr int S_COLS = kAcc * R;
    static constexpr int D_COL0 = 256;
    static_assert(2 * S_COLS <= D_COL0, "TMEM budget");
    static_assert(SMEM + 1024 <= 227 * 1024, "shared memory budget");
};

struct ResArgs {
    __nv_bfloat16* h;
    long long ldh;
    int d;
    int slot_base;
    const unsigned char* Bt;  // [S][d/8][R/8][8][8] bf16
    const float* bias;        // [S][R]
    const float* scale;       // [S]
    const int2* chunks;
    const int4* units;
    const int* counters;
    // exchange through L2 (XG): [header: epoch u64, done u32][flags u64 per CTA
    // and quadrant][partials f32: group, unit parity, rank, 64 x R]
    unsigned char* xs;
    long long* prof;  // diagnostics: clock64 stamps of CTA prof_cta (NULL in production)
    int prof_cta;
    int part_lo, part_hi;  // this launch takes units [N*lo/4096, N*hi/4096) (co-launch split)
};

constexpr int kXsHeader = 256;
__host__ __device__ constexpr long long xs_flags_bytes(int grid) { return static_cast<long long>(grid) * 4 * 8; }

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// diagnostics: unit stamps at prof[ub * 8 + k] (first 16 units), chunk stamps
// at prof[128 + dc * 8 + k] (first 64 chunks)
#define RPROF_U(k) \
    if (a.prof && blockIdx.x == a.prof_cta && lane == 0 && ub < 16) a.prof[ub * 8 + (k)] = clock64()
#define RPROF_C(k, dcx) \
    if (a.prof && blockIdx.x == a.prof_cta && lane == 0 && (dcx) < 64) a.prof[128 + (dcx) * 8 + (k)] = clock64()

// the unit's chunks are 64 consecutive rows (the last chunk may be short when
// `full` is false: a load box may read past it, a store box may not)
__device__ __forceinline__ bool unit_rows_consecutive(const int2* chunks, int4 U, bool full) {
    if (U.z != 4) return false;
    const int2 c0 = chunks[U.y], c1 = chunks[U.y + 1], c2 = chunks[U.y + 2], c3 = chunks[U.y + 3];
    return c0.y == kChunkR && c1.y == kChunkR && c2.y == kChunkR && (!full || c3.y == kChunkR) &&
           c1.x == c0.x + kChunkR && c2.x == c0.x + 2 * kChunkR && c3.x == c0.x + 3 * kChunkR;
}

__device__ __forceinline__ void group_bar(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

template <int R, int C, int COLS, bool XG>
__global__ void __launch_bounds__(kThreads, 1)
    reft_res_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmH64,
                    const __grid_constant__ CUtensorMap tmA, const ResArgs a) {
    using L = ResLayout<R, C, COLS, XG>;
    static_assert(L::NJ % 2 == 0, "two epilogue groups alternate chunks");
    constexpr int NP = L::NP, NJ = L::NJ, RING = L::RING;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t h_full[RING], h_empty[RING], t_full[kTBlocks], t_empty[kTBlocks];
    __shared__ __align__(8) uint64_t bt_full[L::BT_STAGES], bt_empty[L::BT_STAGES];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2], v_full[2], v_empty[2], d_full[2], d_empty[2];
    __shared__ __align__(8) uint64_t p_full, p_empty;  // cluster exchange of partial S (C > 1)
    __shared__ uint32_t tslot;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t raw = tc::smem_u32(sm_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;  // 128 B-swizzled operands need 1024 B alignment
    unsigned char* sgen = sm_raw + (sbase - raw);

    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 32) {
        for (int i = 0; i < RING; ++i) {
            tc::mbar_init(&h_full[i], 1);
            tc::mbar_init(&h_empty[i], 1 + 4);  // shrink-MMA commit + the 4 stash warps
        }
        for (int i = 0; i < kTBlocks; ++i) {
            tc::mbar_init(&t_full[i], 4);   // the 4 stash warps
            tc::mbar_init(&t_empty[i], 4);  // the 4 warps of the epilogue group that reads the block
        }
        for (int i = 0; i < L::BT_STAGES; ++i) {
            tc::mbar_init(&bt_full[i], 1);
            tc::mbar_init(&bt_empty[i], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], 1);
            tc::mbar_init(&s_empty[b], 4);  // the 4 V warps
            tc::mbar_init(&v_full[b], 4);
            tc::mbar_init(&v_empty[b], 1);
            tc::mbar_init(&d_full[b], 1);
            tc::mbar_init(&d_empty[b], 4);  // D buffer b belongs to epilogue group b
        }
        tc::mbar_init(&p_full, 4);             // the 4 local V warps (expect_tx of the peers' bytes)
        tc::mbar_init(&p_empty, 4 * (C - 1));  // the 4 V warps of each peer
        tc::fence_mbar_init();
        tc::prefetch_tmap(&tmH);
        tc::prefetch_tmap(&tmH64);
        tc::prefetch_tmap(&tmA);
    }
    tc::fence_before_sync();
    if constexpr (C > 1 && !XG) tc::cluster_sync();  // peers' barriers initialised before any remote arrive
    else __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;

    const int crank = C == 1 ? 0 : XG ? static_cast<int>(blockIdx.x % C) : static_cast<int>(tc::cluster_ctarank());
    // L2 exchange: this launch's epoch (bumped by the last CTA of the previous launch)
    unsigned long long epoch = 0;
    if constexpr (XG && C > 1) epoch = *reinterpret_cast<volatile unsigned long long*>(a.xs) << 32;
    int u0, u1;
    {
        const long long nu = a.counters[PREFT_CTR_UNITS];
        const int ulo = static_cast<int>(nu * a.part_lo >> 12), uhi = static_cast<int>(nu * a.part_hi >> 12);
        even_share(uhi - ulo, blockIdx.x / C, gridDim.x / C, u0, u1);  // contiguous runs share adapters
        u0 += ulo;
        u1 += ulo;
    }
    const int pc0 = crank * NP, jc0 = crank * NJ;  // first global panel / chunk of this CTA
    const int r1 = lane >> 2, cp = 2 * (lane & 3);   // 16x256b layout: rows r1, r1 + 8; columns 8i + cp + {0, 1}

    if (warp >= 16) {
        // ------------------------------------------------ stash: smem panel -> TMEM lanes 16-31
        // the smem slot is released as soon as the panel is in registers (the
        // TMEM store consumed them); the TMEM blocks are published in batches
        // of kStashBatch panels, one store wait per batch, and at unit ends
        const int q = warp & 3;
        const uint32_t park = tmem + (static_cast<uint32_t>(q * 32 + 16) << 16);
        int g = 0, pend0 = 0, npend = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const bool live = q < U.z;
            for (int p = 0; p < NP; ++p, ++g) {
                const int rs = g % RING, tb = g % kTBlocks;
                tc::mbar_wait(&h_full[rs], (g / RING) & 1);
                if (warp == 16 && a.prof && blockIdx.x == a.prof_cta && lane == 0 && g / NP < 16 && (p == 0 || p == NP - 1))
                    a.prof[640 + (g / NP) * 4 + (p ? 2 : 0)] = clock64();
                tc::mbar_wait(&t_empty[tb], ((g / kTBlocks) & 1) ^ 1u);
                if (warp == 16 && a.prof && blockIdx.x == a.prof_cta && lane == 0 && g / NP < 16 && (p == 0 || p == NP - 1))
                    a.prof[640 + (g / NP) * 4 + (p ? 3 : 1)] = clock64();
                if (warp == 16) RPROF_C(6, g);
                tc::fence_after_sync();
                if (live) {
                    const unsigned char* panel = sgen + L::OFF_RING + rs * L::SLOT;
                    uint32_t hv[16];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int half = 0; half < 2; ++half)
                            hv[2 * i + half] = *reinterpret_cast<const uint32_t*>(
                                panel + tc::sw128_offset(q * kChunkR + r1 + 8 * half, 8 * i + cp, 64));
                    tc::tmem_st_16x256b_x4(park + tb * 32, hv);  // issues once the loads have returned
                }
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&h_empty[rs]);
                if (warp == 16) RPROF_C(7, g);
                if (npend++ == 0) pend0 = g;
                if (npend == kStashBatch || p == NP - 1) {
                    tc::tmem_st_wait();
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0)
                        for (int x = 0; x < npend; ++x) tc::mbar_arrive(&t_full[(pend0 + x) % kTBlocks]);
                    npend = 0;
                }
            }
        }
    } else if (warp >= 12) {
        // ------------------------------------------------ V warps: V = s * (S + b) -> bf16 hi + lo
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int slot = U.x - a.slot_base;
            const int sb = ub & 1;
            tc::mbar_wait(&s_full[sb], (ub >> 1) & 1);
            if (warp == 12) RPROF_U(0);
            tc::fence_after_sync();
            float s[R];
#pragma unroll
            for (int k = 0; k < R; ++k) s[k] = 0.f;
#pragma unroll
            for (int acc = 0; acc < kAcc; ++acc) {
                const uint32_t taddr = tmem + lane_base + sb * L::S_COLS + acc * R;
                if constexpr (R == 16) {
                    uint32_t w[16];
                    tc::tmem_ld16(taddr, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 16; ++k) s[k] += __uint_as_float(w[k]);
                } else {
                    uint32_t w[32];
                    tc::tmem_ld32(taddr, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int k = 0; k < 32; ++k) s[k] += __uint_as_float(w[k]);
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
            if constexpr (C > 1 && XG) {
                // S is a partial sum over this CTA's columns: publish this warp's 16
                // rows in L2, raise its flag, wait for the peers' flags of the same
                // quadrant and add their rows (double-buffered by unit parity: a
                // peer re-writes a buffer only after it saw our flag for the unit
                // in between, which we raise after reading the buffer)
                const int m = q * kChunkR + (lane & 15);
                const int gb = blockIdx.x - crank;  // first CTA of the group
                float* part = reinterpret_cast<float*>(a.xs + kXsHeader + xs_flags_bytes(gridDim.x)) +
                              (static_cast<long long>(gb / C) * 2 + (ub & 1)) * C * kRows * R;
                unsigned long long* flags = reinterpret_cast<unsigned long long*>(a.xs + kXsHeader);
                if (lane < kChunkR) {
                    float* dst = part + (crank * kRows + m) * R;
#pragma unroll
                    for (int k = 0; k < R; k += 4)
                        __stcg(reinterpret_cast<float4*>(dst + k), make_float4(s[k], s[k + 1], s[k + 2], s[k + 3]));
                }
                __syncwarp();
                const unsigned long long want = epoch | static_cast<unsigned long long>(ub + 1);
                if (lane == 0) {
                    __threadfence();  // cumulative over the warp's stores (ordered by __syncwarp)
                    st_relaxed_u64(flags + (blockIdx.x * 4 + q), want);
                }
                if (lane < C - 1) {
                    const unsigned long long* f = flags + ((gb + (crank + 1 + lane) % C) * 4 + q);
                    while (ld_acquire_u64(f) < want) __nanosleep(32);
                }
                __syncwarp();
                if (warp == 12) RPROF_U(1);
                if (lane < kChunkR) {
#pragma unroll
                    for (int x = 1; x < C; ++x) {
                        const float* src = part + (((crank + x) % C) * kRows + m) * R;
#pragma unroll
                        for (int k = 0; k < R; k += 4) {
                            const float4 t = __ldcg(reinterpret_cast<const float4*>(src + k));
                            s[k] += t.x;
                            s[k + 1] += t.y;
                            s[k + 2] += t.z;
                            s[k + 3] += t.w;
                        }
                    }
                }
            } else if constexpr (C > 1) {
                // S is a partial sum over this CTA's columns: push it into every
                // peer's inbox (the bytes complete on the peer's p_full), then
                // add the peers' partials from our own inbox
                const int m = q * kChunkR + (lane & 15);
                if (lane == 0) tc::mbar_expect_tx(&p_full, (C - 1) * kChunkR * R * 4);
                tc::mbar_wait(&p_empty, (ub & 1) ^ 1u);  // peers done with our previous push
#pragma unroll
                for (int x = 1; x < C; ++x) {
                    const int peer = (crank + x) % C;  // our slot in the peer's inbox: C - 1 - x
                    const uint32_t dst =
                        tc::map_shared(sbase + L::OFF_IN + (C - 1 - x) * L::IN_BYTES + m * R * 4, peer);
                    const uint32_t bar = tc::map_shared(tc::smem_u32(&p_full), peer);
                    if (lane < kChunkR) {
#pragma unroll
                        for (int k = 0; k < R; k += 4)
                            tc::st_async_f4(dst + k * 4, make_float4(s[k], s[k + 1], s[k + 2], s[k + 3]), bar);
                    }
                }
                tc::mbar_wait(&p_full, ub & 1);
                if (warp == 12) RPROF_U(1);
                if (lane < kChunkR) {
#pragma unroll
                    for (int x = 0; x < C - 1; ++x) {
                        const float* in = reinterpret_cast<const float*>(sgen + L::OFF_IN + x * L::IN_BYTES + m * R * 4);
#pragma unroll
                        for (int k = 0; k < R; k += 4) {
                            const float4 t = *reinterpret_cast<const float4*>(in + k);
                            s[k] += t.x;
                            s[k + 1] += t.y;
                            s[k + 2] += t.z;
                            s[k + 3] += t.w;
                        }
                    }
                }
            }
            tc::mbar_wait(&v_empty[sb], ((ub >> 1) & 1) ^ 1u);
            if (lane < kChunkR) {
                const int m = q * kChunkR + lane;
                const float sc = __ldg(a.scale + slot);
                const float* bb = a.bias + static_cast<long long>(slot) * R;
                unsigned char* vhi = sgen + L::OFF_V + sb * 2 * L::V_BYTES;
#pragma unroll
                for (int k0 = 0; k0 < R; k0 += 8) {
                    uint32_t hi[4], lo[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float v0 = (s[k0 + 2 * e] + __ldg(bb + k0 + 2 * e)) * sc;
                        const float v1 = (s[k0 + 2 * e + 1] + __ldg(bb + k0 + 2 * e + 1)) * sc;
                        hi[e] = f32x2_to_bf16(v0, v1);
                        float h0, h1;
                        bf16x2_to_acc(hi[e], h0, h1);
                        lo[e] = f32x2_to_bf16(v0 - h0, v1 - h1);
                    }
                    const uint32_t off = tc::kmajor_offset(m, k0, R);
                    *reinterpret_cast<uint4*>(vhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(vhi + L::V_BYTES + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            tc::fence_proxy_async();  // V (generic writes) -> tensor-core operand reads
            __syncwarp();
            if (warp == 12) RPROF_U(2);
            if (lane == 0) {
                tc::mbar_arrive(&v_full[sb]);
                // the inbox was consumed into V (written above, in issue order after
                // the inbox loads returned): the peers may push their next partial
                if constexpr (C > 1 && !XG) {
#pragma unroll
                    for (int x = 1; x < C; ++x)
                        tc::mbar_arrive_remote_relaxed(tc::map_shared(tc::smem_u32(&p_empty), (crank + x) % C));
                }
            }
            ++ub;
        }
    } else if (warp == 0) {
        // ------------------------------------------------ producer: h panels + A panels
        // lane 0 owns the barriers; lane q issues chunk q's 16-row box, lane 4
        // the A panel, so a panel's boxes are in flight together
        const uint64_t once = tc::policy_evict_first();  // read exactly once
        int g = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int slot = U.x - a.slot_base, nch = U.z;
            const int row = lane < nch ? a.chunks[U.y + lane].x : 0;
            // 64 consecutive rows: one 64-row box instead of four (TMA issue slots are the scarce resource)
            const bool box64 = unit_rows_consecutive(a.chunks, U, false);
            const uint32_t bytes = static_cast<uint32_t>(nch * kChunkR * 128 + L::AP_BYTES);
            const int ub = g / NP;
            for (int p = 0; p < NP; ++p, ++g) {
                const int rs = g % RING;
                if (lane == 0) {
                    tc::mbar_wait(&h_empty[rs], ((g / RING) & 1) ^ 1u);
                    tc::mbar_expect_tx(&h_full[rs], bytes);
                    if (p == 0) RPROF_U(5);
                    if (p == NP - 1) RPROF_U(6);
                }
                __syncwarp();
                const uint32_t st = sbase + L::OFF_RING + rs * L::SLOT;
                if (box64) {
                    if (lane == 0) tc::tma_load_2d_hint(st, &tmH64, (pc0 + p) * 64, row, &h_full[rs], once);
                } else if (lane < nch) {
                    tc::tma_load_2d_hint(st + lane * (kChunkR * 128), &tmH, (pc0 + p) * 64, row, &h_full[rs], once);
                }
                if (lane == 4)
                    tc::tma_load_2d(st + L::H_BYTES, &tmA, (pc0 + p) * 64, slot * R, &h_full[rs]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ shrink MMA
        if (lane == 0) {
            const uint32_t id = tc::idesc_bf16_f32(kRows, R);
            int g = 0, ub = 0;
            for (int u = u0; u < u1; ++u) {
                const int4 U = a.units[u];
                if (U.x < a.slot_base) continue;
                const int sb = ub & 1;
                tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
                tc::fence_after_sync();
                const uint32_t dS = tmem + sb * L::S_COLS;
                for (int p = 0; p < NP; ++p, ++g) {
                    const int rs = g % RING;
                    tc::mbar_wait(&h_full[rs], (g / RING) & 1);
                    if (p == 0) RPROF_U(3);
                    if (p == NP - 1) RPROF_U(4);
                    tc::fence_after_sync();
                    const uint32_t hp = sbase + L::OFF_RING + rs * L::SLOT, ap = hp + L::H_BYTES;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int kk = p * 4 + k;
                        tc::mma_bf16(dS + (kk % kAcc) * R, tc::desc_kmajor_sw128(hp + k * 32),
                                     tc::desc_kmajor_sw128(ap + k * 32), id, kk >= kAcc ? 1u : 0u);
                    }
                    tc::mma_commit(&h_empty[rs]);
                }
                tc::mma_commit(&s_full[sb]);
                ++ub;
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ Bt producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = u0; u < u1; ++u) {
                const int4 U = a.units[u];
                if (U.x < a.slot_base) continue;
                const unsigned char* bt = a.Bt + static_cast<long long>(U.x - a.slot_base) * a.d * R * 2;
                for (int j = 0; j < NJ; ++j) {
                    tc::mbar_wait(&bt_empty[stage], phase ^ 1u);
                    tc::mbar_expect_tx(&bt_full[stage], L::BT_BYTES);
                    tc::bulk_load_1d(sbase + L::OFF_BT + stage * L::BT_BYTES,
                                     bt + static_cast<long long>(jc0 + j) * L::BT_BYTES, L::BT_BYTES, &bt_full[stage]);
                    if (++stage == L::BT_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------ expand MMA
        if (lane == 0) {
            const uint32_t id = tc::idesc_bf16_f32(kRows, kN);
            int stage = 0, ub = 0, dc = 0;
            uint32_t phase = 0;
            for (int u = u0; u < u1; ++u) {
                const int4 U = a.units[u];
                if (U.x < a.slot_base) continue;
                const int vb = ub & 1;
                tc::mbar_wait(&v_full[vb], (ub >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t vhi = sbase + L::OFF_V + vb * 2 * L::V_BYTES, vlo = vhi + L::V_BYTES;
                for (int j = 0; j < NJ; ++j, ++dc) {
                    tc::mbar_wait(&bt_full[stage], phase);
                    RPROF_C(3, dc);
                    const int db = dc & 1;
                    tc::mbar_wait(&d_empty[db], ((dc >> 1) & 1) ^ 1u);
                    RPROF_C(4, dc);
                    tc::fence_after_sync();
                    const uint32_t bt = sbase + L::OFF_BT + stage * L::BT_BYTES;
                    const uint32_t dD = tmem + L::D_COL0 + db * kN;
#pragma unroll
                    for (int k = 0; k < R / 16; ++k) {
                        const uint64_t bd = tc::desc_kmajor(bt + k * 256, 128, R * 16);
                        tc::mma_bf16(dD, tc::desc_kmajor(vhi + k * 256, 128, R * 16), bd, id, k > 0 ? 1u : 0u);
                        tc::mma_bf16(dD, tc::desc_kmajor(vlo + k * 256, 128, R * 16), bd, id, 1u);
                    }
                    tc::mma_commit(&d_full[db]);
                    tc::mma_commit(&bt_empty[stage]);
                    RPROF_C(5, dc);
                    if (++stage == L::BT_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                tc::mma_commit(&v_empty[vb]);
                ++ub;
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 4..11)
        // group g takes the chunks j with j % 2 == g (NJ is even, so also D
        // buffer g); a warp covers its TMEM lane quadrant's 16 rows across the
        // chunk's two panels: D (lanes 0-15) + parked h (lanes 16-31) -> bf16 ->
        // the group's staging -> TMA store (two 64-row boxes when the unit's
        // rows are consecutive, else one 16-row box per warp and panel)
        const int q = warp & 3;
        const int grp = (warp - 4) >> 2;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        const uint32_t park = tmem + (static_cast<uint32_t>(q * 32 + 16) << 16);
        const uint64_t out = tc::policy_evict_first();
        const uint32_t stg = L::OFF_OUT + grp * 2 * L::OUT_BYTES;  // the group's [2 panels] of staging
        int g0 = 0, dc = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const bool box64 = unit_rows_consecutive(a.chunks, U, true);
            for (int j = grp; j < NJ; j += 2) {
                const int dcj = dc + j;
                tc::mbar_wait(&d_full[grp], (dcj >> 1) & 1);
                if (q == 0) RPROF_C(0, dcj);
                if (lane == 0) tc::tma_store_wait_read();  // this thread's previous stores have read the staging
                group_bar(1 + grp);
#pragma unroll 1
                for (int hf = 0; hf < 2; ++hf) {
                    const int g = g0 + 2 * j + hf, tb = g % kTBlocks;
                    tc::mbar_wait(&t_full[tb], (g / kTBlocks) & 1);
                    tc::fence_after_sync();
                    if (ch.y > 0) {
                        uint32_t v[32], hv[16];
                        tc::tmem_ld_16x256b_x8(tmem + lane_base + L::D_COL0 + grp * kN + hf * 64, v);
                        tc::tmem_ld_16x256b_x4(park + tb * 32, hv);
                        tc::tmem_ld_wait();
                        tc::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) {
                            tc::mbar_arrive(&t_empty[tb]);
                            if (hf == 1) tc::mbar_arrive(&d_empty[grp]);
                        }
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
                                float lo, hi;
                                bf16x2_to_acc(hv[2 * i + half], lo, hi);
                                lo += __uint_as_float(v[4 * i + 2 * half]);
                                hi += __uint_as_float(v[4 * i + 2 * half + 1]);
                                *reinterpret_cast<uint32_t*>(
                                    sgen + stg + hf * L::OUT_BYTES +
                                    tc::sw128_offset(q * kChunkR + r1 + 8 * half, 8 * i + cp, kRows)) =
                                    f32x2_to_bf16(lo, hi);
                            }
                    } else {
                        __syncwarp();
                        if (lane == 0) {
                            tc::mbar_arrive(&t_empty[tb]);
                            if (hf == 1) tc::mbar_arrive(&d_empty[grp]);
                        }
                    }
                }
                if (q == 0) RPROF_C(1, dcj);
                tc::fence_proxy_async();  // staging writes -> TMA store reads
                if (box64) {
                    group_bar(1 + grp);
                    if (q == 0 && lane == 0) {
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
                            tc::tma_store_2d_hint(&tmH64, (jc0 + j) * kN + hf * 64, ch.x, sbase + stg + hf * L::OUT_BYTES,
                                                  out);
                        tc::tma_store_commit();
                    }
                } else if (ch.y == kChunkR) {
                    __syncwarp();
                    if (lane == 0) {
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
                            tc::tma_store_2d_hint(&tmH, (jc0 + j) * kN + hf * 64, ch.x,
                                                  sbase + stg + hf * L::OUT_BYTES + q * (kChunkR * 128), out);
                        tc::tma_store_commit();
                    }
                } else if (ch.y > 0) {
                    // partial chunk (end of a prompt): only its valid rows go back
                    __syncwarp();
                    for (int idx = lane; idx < ch.y * 16; idx += 32) {
                        const int rr = idx >> 4, hf = (idx >> 3) & 1, c16 = idx & 7;
                        const uint4 val = *reinterpret_cast<const uint4*>(
                            sgen + stg + hf * L::OUT_BYTES + tc::sw128_offset(q * kChunkR + rr, c16 * 8, kRows));
                        *reinterpret_cast<uint4*>(a.h + static_cast<long long>(ch.x + rr) * a.ldh + (jc0 + j) * kN +
                                                  hf * 64 + c16 * 8) = val;
                    }
                }
                __syncwarp();
                if (q == 0) RPROF_C(2, dcj);
            }
            g0 += NP;
            dc += NJ;
        }
        if (lane == 0) tc::tma_store_wait_all();  // bulk stores complete before the CTA retires
    }
    tc::fence_before_sync();
    if constexpr (C > 1 && !XG) tc::cluster_sync();  // no peer still writes our inbox / barriers
    else __syncthreads();
    if constexpr (XG && C > 1) {
        if (tid == 0) {
            // the last CTA out bumps the epoch: the next launch's flags compare above every flag of this one
            __threadfence();
            unsigned int* done = reinterpret_cast<unsigned int*>(a.xs + 8);
            if (atomicAdd(done, 1u) == gridDim.x - 1) {
                *done = 0;
                *reinterpret_cast<volatile unsigned long long*>(a.xs) = (epoch >> 32) + 1;
                __threadfence();
            }
        }
    }
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, 512);
    }
}

template <int R, int C, int COLS, bool XG>
int launch_res(const ResArgs& args, const CUtensorMap& tmH, const CUtensorMap& tmH64, const CUtensorMap& tmA, int num_sms,
               cudaStream_t stream, bool dry = false) {
    auto fn = reft_res_kernel<R, C, COLS, XG>;
    const int smem = ResLayout<R, C, COLS, XG>::SMEM;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -static_cast<int>(e);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    if (XG) {
        // the groups spin on each other's flags: every CTA must be resident
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    } else {
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
    }
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = C > 1 ? 1 : 0;
    int grid = (num_sms / C) * C;
    if (C > 1 && !XG) {
        static int nc = 0;  // co-resident clusters for this instantiation, measured once
        if (nc == 0) {
            cfg.gridDim = dim3(grid);
            e = cudaOccupancyMaxActiveClusters(&nc, fn, &cfg);
            if (e != cudaSuccess) return -static_cast<int>(e);
            if (nc < 1) return PREFT_ERR_CONFIG;
        }
        grid = min(grid, nc * C);
    }
    if (dry) return grid;
    cfg.gridDim = dim3(grid);
    reft_tc_note_grid(grid);
    e = cudaLaunchKernelEx(&cfg, fn, tmH, tmH64, tmA, args);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace

// columns per CTA: 1024 (the TMEM parking lanes hold one 128 KB slice; a
// group of d / 1024 CTAs per unit)
constexpr int kCols = 1024;

long long* reft_tc_profile_buffer();

bool reft_res_eligible(int d, int r) {
    if ((r != 16 && r != 32) || d % kCols) return false;
    const int c = d / kCols;
    return c == 1 || c == 2 || c == 4 || (c == 8 && r == 16);
}

// partial-S exchange between the CTAs of a unit: through DSMEM in a
// thread-block cluster (default), or through L2 with flags in a cooperative
// grid (every SM works whatever the GPC floor-sweeping leaves for 4-CTA
// clusters, 148 vs 132 CTAs, but the fence + flag round trip costs more than
// the extra SMs bring: 58% vs 63% of HBM at d = 4096, 52% vs 68% at 2048).
// Env PREFT_REFT_RES_XCHG=l2|dsmem (A/B measurement).
static bool res_xchg_l2() {
    static int v = -1;
    if (v < 0) {
        const char* env = getenv("PREFT_REFT_RES_XCHG");
        v = (env && env[0] == 'l') ? 1 : 0;
    }
    return v == 1;
}

// automatic choice between this kernel and the streaming K3-TC (measured,
// profiles/reft_bench_r01g.json)
bool reft_res_preferred(int d, int r) {
    if (!reft_res_eligible(d, r)) return false;
    // clusters of 4 get 132 of the 148 SMs (GPC packing): at d = 4096 the
    // L2-streaming kernel on all SMs is as fast (62-69% vs 62-65% across boxes)
    return d / kCols <= 2;
}

// L2 exchange scratch, one per (device, stream): launches on one stream are
// ordered, so they may share flags and partial buffers; zeroed once
struct XsEntry {
    int device;
    cudaStream_t stream;
    unsigned char* ptr;
    long long bytes;
};
static std::mutex g_xs_mu;
static XsEntry g_xs[32];
static int g_nxs = 0;

static int xs_for(cudaStream_t stream, int num_sms, unsigned char** out) {
    int dev = 0;
    cudaGetDevice(&dev);
    const long long need = kXsHeader + xs_flags_bytes(num_sms) + static_cast<long long>(num_sms) * 2 * kRows * 32 * 4;
    std::lock_guard<std::mutex> lk(g_xs_mu);
    for (int i = 0; i < g_nxs; ++i)
        if (g_xs[i].device == dev && g_xs[i].stream == stream && g_xs[i].bytes >= need) {
            *out = g_xs[i].ptr;
            return PREFT_OK;
        }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return PREFT_ERR_SHAPE;  // no allocation inside a capture: the caller falls back
    if (g_nxs == 32) return PREFT_ERR_SHAPE;
    void* p = nullptr;
    if (cudaMalloc(&p, need) != cudaSuccess) return PREFT_ERR_SHAPE;
    if (cudaMemset(p, 0, need) != cudaSuccess) return PREFT_ERR_SHAPE;
    g_xs[g_nxs++] = {dev, stream, static_cast<unsigned char*>(p), need};
    *out = static_cast<unsigned char*>(p);
    return PREFT_OK;
}

int reft_res_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A,
                   const void* Bt, const void* bias, const void* scale, int r, cudaStream_t stream, int num_sms,
                   int part_lo, int part_hi, bool dry) {
    if (!Bt || !reft_res_eligible(d, r) || rows < 1) return PREFT_ERR_SHAPE;
    if (!meta->chunks || !meta->units || (ldh % 8) || (reinterpret_cast<uintptr_t>(h) & 15) ||
        (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(Bt) & 15))
        return PREFT_ERR_SHAPE;
    CUtensorMap tmH{}, tmH64{}, tmA{};
    if (!make_tmap_bf16_sw128(&tmH, h, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(ldh), 64, kChunkR) ||
        !make_tmap_bf16_sw128(&tmH64, h, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(ldh), 64, kRows))
        return PREFT_ERR_CONFIG;
    if (!make_tmap_bf16_sw128(&tmA, A, 1ull << 20, static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(d), 64, static_cast<unsigned>(r)))
        return PREFT_ERR_CONFIG;
    ResArgs args;
    args.h = static_cast<__nv_bfloat16*>(h);
    args.ldh = ldh;
    args.d = d;
    args.slot_base = meta->slot_split;
    args.Bt = static_cast<const unsigned char*>(Bt);
    args.bias = static_cast<const float*>(bias);
    args.scale = static_cast<const float*>(scale);
    args.chunks = reinterpret_cast<const int2*>(meta->chunks);
    args.units = reinterpret_cast<const int4*>(meta->units);
    args.counters = meta->counters;
    args.part_lo = part_lo;
    args.part_hi = part_hi;
    args.prof = reft_tc_profile_buffer();
    {
        const char* pc = args.prof ? getenv("PREFT_REFT_PROF_CTA") : nullptr;
        args.prof_cta = pc ? atoi(pc) : 0;
    }
    const int c = d / kCols;
    const bool xg = c > 1 && res_xchg_l2();
    args.xs = nullptr;
    if (xg && !dry) {
        const int rc = xs_for(stream, num_sms, &args.xs);
        if (rc != PREFT_OK) return rc;
    }
#define PREFT_RES(RR, CC, XG_) \
    if (r == RR && c == CC && xg == XG_) return launch_res<RR, CC, kCols, XG_>(args, tmH, tmH64, tmA, num_sms, stream, dry);
    PREFT_RES(16, 1, false)
    PREFT_RES(16, 2, false)
    PREFT_RES(16, 4, false)
    PREFT_RES(16, 8, false)
    PREFT_RES(16, 2, true)
    PREFT_RES(16, 4, true)
    PREFT_RES(16, 8, true)
    PREFT_RES(32, 1, false)
    PREFT_RES(32, 2, false)
    PREFT_RES(32, 4, false)
    PREFT_RES(32, 2, true)
    PREFT_RES(32, 4, true)
#undef PREFT_RES
    return PREFT_ERR_SHAPE;
}

}  // namespace preft
