// K3-TC — tensor-core ReFT^P for sm_100a (bf16, rank 16 or 32).
//
//     h[t, :] += s_a * ((h[t, :] . A_a^T + b_a) . B_a)      (adapters.py:292-295)
//
// At r >= 16 the residual edit is a real contraction (4*r*d FLOP against
// 4*d bytes per token: 105-315 TFLOP/s at the HBM roofline, beyond SIMT
// FP32), so both products run on tcgen05 with fp32 accumulators in TMEM.
//
// Work unit (built by K1): up to 4 chunks of <= 16 consecutive h rows of ONE
// adapter, i.e. one M = 64 UMMA tile whose chunk q lands in TMEM lane
// quadrant q (lanes 32q .. 32q+15; the M = 64 data-path layout).  Each chunk
// is one 16-row TMA box, so ragged prompts cost at most 15 extra rows read
// per entry and never a gather.
//
// A cluster of C CTAs (C = 2 at d = 4096, 4 at d = 8192) owns a unit; CTA c
// owns the columns [c*d/C, (c+1)*d/C).  One CTA per SM, warp-specialised,
// every hand-off an mbarrier ring:
//   warp 0   shrink producer: TMA h panels (64 rows x 64 cols, evict_last)
//            and the adapter's A panel (R x 64) into a 5-10 stage ring; it
//            stays at most one unit ahead of the epilogue
//   warp 1   shrink MMA: TMEM S[64 x R] += H_panel . A_panel^T over this
//            CTA's columns, 2 split accumulators, S double-buffered
//   warp 2   epilogue producer: TMA the unit's h rows AGAIN, 128 columns at a
//            time (an L2 hit: the rows were read moments ago with evict_last),
//            plus the adapter's Bt chunk (pre-tiled in the pool, one bulk copy)
//   warp 3   expand MMA: TMEM D[64 x 128] = V_hi . Bt_chunk^T + V_lo . Bt_chunk^T,
//            D double-buffered
//   warps 4-11 epilogue: (warps 4-7) exchange the partial S with the cluster
//            peers through distributed shared memory (remote mbarrier arrives,
//            no cluster-wide barrier), V = s*(S + b) split into bf16 hi + lo
//            (so the expand keeps ~fp32 accuracy); (all 8) D -> registers,
//            h_chunk += D in shared memory, TMA store (evict_first)
// h crosses HBM once in and once out (the algorithmic minimum).  The second
// read is served by L2 because each CTA has at most ~2 x 256 KB of h between
// first read and re-read (~50 MB across the GPU against a 126 MB L2; a single
// CTA per unit at d = 4096 would need ~150 MB and miss).  The tensor pipe,
// TMA and the epilogue math overlap, so the kernel streams at HBM speed
// instead of alternating load and compute phases.  LoRA-class units are
// skipped.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

constexpr int kUnitRows = 64;             // UMMA M
constexpr int kChunk = PREFT_CHUNK_ROWS;  // 16 rows: one TMA box, one TMEM lane quadrant
constexpr int kEpiN = 128;                // expand / epilogue chunk width (UMMA N)
constexpr int kTcThreads = 512;           // 16 warps
constexpr int kNacc = 2;                  // split shrink accumulators
constexpr int kEpiWarps = 8;
// K panels per shrink ring stage: issuing several panels of the same rows
// together amortises the per-stage costs and gives DRAM longer runs per row
constexpr int spps_for(int R, int C) { return R == 16 && C == 2 ? 4 : 2; }

template <int R, int C>
struct TcLayout {
    static constexpr int H_BYTES = kUnitRows * 128;      // 64 rows x 64 bf16 (one 128 B-swizzled panel)
    static constexpr int AP_BYTES = R * 128;             // A panel: R rows x 64 bf16
    static constexpr int SPPS = spps_for(R, C);
    static constexpr int SH_STAGE = SPPS * (H_BYTES + AP_BYTES);  // SPPS panels of h, then their A panels
    static constexpr int EH_BYTES = 2 * H_BYTES;         // 128 columns = two panels
    static constexpr int BT_BYTES = kEpiN * R * 2;       // Bt chunk: 128 rows x R (core-matrix layout)
    static constexpr int EPI_STAGE = EH_BYTES + BT_BYTES;
    static constexpr int V_BYTES = kUnitRows * R * 2;    // one of V_hi / V_lo
    // the epilogue re-read is an L2 hit (~1.5k cycles) and needs a short
    // ring; the shrink streams from HBM (~4-5k cycles under load) and gets
    // every byte left
    static constexpr int EPI_STAGES = 4;
    static constexpr int FIXED = EPI_STAGES * EPI_STAGE + 4 * V_BYTES + 2 * (C - 1) * kUnitRows * R * 4 + 1024;
    static constexpr int SH_FIT = (227 * 1024 - 1024 - FIXED) / SH_STAGE;  // - static smem (barriers)
    static constexpr int SH_STAGES = SH_FIT > 14 ? 14 : SH_FIT;
    static_assert(SH_STAGES >= 2, "shrink ring too shallow");
    static constexpr int OFF_SH = 0;
    static constexpr int OFF_EPI = SH_STAGES * SH_STAGE;
    static constexpr int OFF_V = OFF_EPI + EPI_STAGES * EPI_STAGE;  // [2 buffers][hi, lo]
    static constexpr int IN_BYTES = kUnitRows * R * 4;                // one peer's partial S (f32)
    static constexpr int OFF_IN = OFF_V + 4 * V_BYTES;                // [2 buffers][C-1 peers]
    static constexpr int TOTAL = OFF_IN + 2 * (C - 1) * IN_BYTES;
    static constexpr int SMEM = TOTAL + 1024;            // + alignment slack
    static constexpr int S_COLS = kNacc * R;             // TMEM columns per S buffer
    static constexpr int D_COL0 = 256;                   // D buffers: columns 256 .. 511
    static_assert(2 * S_COLS <= D_COL0, "TMEM budget");
    static_assert(SMEM + 1024 <= 227 * 1024, "shared memory budget (dynamic + static)");
};

struct ReftTcArgs {
    __nv_bfloat16* h;
    long long ldh;
    int d;
    int slot_base;
    const unsigned char* Bt;  // [S][d/8][R/8][8][8] bf16 (UMMA core-matrix order)
    const float* bias;        // [S][R]
    const float* scale;       // [S]
    const int2* chunks;
    const int4* units;
    const int* counters;
    int flags;  // diagnostics knobs: bit 0 immediate stage release, bit 1 pace the shrink behind the
                // epilogue, bit 2 no one-unit throttle of the shrink, bit 3 let the
                // epilogue producer read ahead of the shrink, bit 4 no L2 hints, bit 5
                // reduce epilogue (bf16 delta added into h by TMA in L2, no re-read)
    int look;   // with bit 1: panels the shrink may run ahead of the epilogue's re-read
    long long* prof;  // diagnostics: clock64 stamps of CTA prof_cta (NULL in production)
    int prof_cta;
    int part_lo, part_hi;  // this launch takes units [N*lo/4096, N*hi/4096) (co-launch split)
};

// diagnostics: warp 4 lane 0 of CTA 0 stamps chunk phases (first 64 chunks) and unit phases
#define PROF(k) \
    if (a.prof && blockIdx.x == a.prof_cta && (warp == 4 || warp == 8) && lane == 0 && dc < 64) a.prof[dc * 8 + (k)] = clock64()
#define XPROF(k, v) \
    if (a.prof && blockIdx.x == a.prof_cta && warp == 12 && lane == 0 && ub < 16) a.prof[608 + ub * 8 + (k)] = (v)
#define UPROF(k) \
    if (a.prof && blockIdx.x == a.prof_cta && warp == 12 && lane == 0 && ub < 16) a.prof[512 + ub * 4 + (k)] = clock64()

template <int R, int C>
__global__ void __launch_bounds__(kTcThreads, 1)
    reft_tc_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmA,
                   const ReftTcArgs a) {
    using L = TcLayout<R, C>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t sh_full[L::SH_STAGES], sh_empty[L::SH_STAGES];
    __shared__ __align__(8) uint64_t epi_full[L::EPI_STAGES], epi_empty[L::EPI_STAGES];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2], v_full[2], v_empty[2], d_full[2], d_empty[2];
    __shared__ __align__(8) uint64_t p_full[2], p_empty[2];  // cluster exchange of partial S (C > 1)
    __shared__ uint32_t tslot;
    __shared__ int s_epi_done;  // epilogue chunks finished (warp 4), read by the shrink producer when pacing
    __shared__ int s_shrunk;    // h panels landed and consumed by the shrink MMA (monotonic across units)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t raw = tc::smem_u32(sm_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;  // 128 B-swizzled operands need 1024 B alignment
    unsigned char* sgen = sm_raw + (sbase - raw);

    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 32) {
        s_epi_done = 0;
        s_shrunk = 0;
        for (int i = 0; i < L::SH_STAGES; ++i) {
            tc::mbar_init(&sh_full[i], 1);
            tc::mbar_init(&sh_empty[i], 1);
        }
        for (int i = 0; i < L::EPI_STAGES; ++i) {
            tc::mbar_init(&epi_full[i], 1);
            tc::mbar_init(&epi_empty[i], 1 + kEpiWarps / 2);  // expand-MMA commit + the owning group's warps
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], 1);
            tc::mbar_init(&s_empty[b], 4);  // the 4 V warps
            tc::mbar_init(&v_full[b], 4);
            tc::mbar_init(&v_empty[b], 1);
            tc::mbar_init(&d_full[b], 1);
            tc::mbar_init(&d_empty[b], kEpiWarps / 2);  // D buffer b belongs to epilogue group b
            tc::mbar_init(&p_full[b], 4);             // the 4 local V warps (expect_tx of the peers' st.async bytes)
            tc::mbar_init(&p_empty[b], 4 * (C - 1));  // the 4 V warps of each peer
        }
        tc::fence_mbar_init();
        tc::prefetch_tmap(&tmH);
        tc::prefetch_tmap(&tmA);
    }
    tc::fence_before_sync();
    if constexpr (C > 1) tc::cluster_sync();  // peers' barriers initialised before any remote arrive
    else __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;

    // a cluster of C CTAs owns each unit; CTA `crank` owns columns [crank*d/C, (crank+1)*d/C)
    const int crank = C > 1 ? static_cast<int>(tc::cluster_ctarank()) : 0;
    int u0, u1;
    {
        const long long nu = a.counters[PREFT_CTR_UNITS];
        const int ulo = static_cast<int>(nu * a.part_lo >> 12), uhi = static_cast<int>(nu * a.part_hi >> 12);
        even_share(uhi - ulo, blockIdx.x / C, gridDim.x / C, u0, u1);  // contiguous runs share adapters
        u0 += ulo;
        u1 += ulo;
    }
    const int NP = a.d / (64 * C), NJ = a.d / (kEpiN * C);
    const int pc0 = crank * NP, jc0 = crank * NJ;  // first global panel / chunk of this CTA

    if (warp >= 12) {
        // ------------------------------------------------ V warps (12..15): V = s * (S + b) -> bf16 hi + lo
        const int q = warp & 3;  // the TMEM lane quadrant this warp may access
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int slot = U.x - a.slot_base;
            const int sb = ub & 1;
            // V = s * (S + b) for this quadrant's 16 rows -> bf16 hi + lo
            tc::mbar_wait(&s_full[sb], (ub >> 1) & 1);
            UPROF(0);
            tc::fence_after_sync();
            float s[R];
#pragma unroll
            for (int k = 0; k < R; ++k) s[k] = 0.f;
#pragma unroll
            for (int acc = 0; acc < kNacc; ++acc) {
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
            UPROF(1);
            if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
            if constexpr (C > 1) {
                // S is a partial sum over this CTA's columns: push it to every
                // peer's inbox, then add the peers' partials from our own
                const int m = q * kChunk + (lane & 15);
                // every peer's st.async completes its bytes on our p_full: expect them
                if (lane == 0) tc::mbar_expect_tx(&p_full[sb], (C - 1) * kChunk * R * 4);
                tc::mbar_wait(&p_empty[sb], ((ub >> 1) & 1) ^ 1u);  // peers done with unit u-2 (flow control only)
                XPROF(0, clock64());
                XPROF(4, static_cast<long long>(tc::globaltimer()));
#pragma unroll
                for (int x = 1; x < C; ++x) {
                    const int peer = (crank + x) % C;  // our slot in peer's inbox: C - 1 - x
                    const uint32_t dst = tc::map_shared(
                        sbase + L::OFF_IN + (sb * (C - 1) + (C - 1 - x)) * L::IN_BYTES + m * R * 4, peer);
                    const uint32_t bar = tc::map_shared(tc::smem_u32(&p_full[sb]), peer);
                    if (lane < kChunk) {
#pragma unroll
                        for (int k = 0; k < R; k += 4)
                            tc::st_async_f4(dst + k * 4, make_float4(s[k], s[k + 1], s[k + 2], s[k + 3]), bar);
                    }
                }
                XPROF(1, clock64());
                tc::mbar_wait(&p_full[sb], (ub >> 1) & 1);
                XPROF(2, clock64());
                XPROF(5, static_cast<long long>(tc::globaltimer()));
                if (lane < kChunk) {
#pragma unroll
                    for (int x = 0; x < C - 1; ++x) {
                        const float* in = reinterpret_cast<const float*>(
                            sgen + L::OFF_IN + (sb * (C - 1) + x) * L::IN_BYTES + m * R * 4);
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
            UPROF(2);
            if (lane < kChunk) {
                const int m = q * kChunk + lane;
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
            if (lane == 0) {
                tc::mbar_arrive(&v_full[sb]);
                // the inbox was consumed into V (written above, in issue order after the
                // inbox loads returned): the peers may overwrite it with unit u+2
                if constexpr (C > 1) {
#pragma unroll
                    for (int x = 1; x < C; ++x)
                        tc::mbar_arrive_remote_relaxed(tc::map_shared(tc::smem_u32(&p_empty[sb]), (crank + x) % C));
                }
            }
            UPROF(3);
        
            ++ub;
        }
    } else if (warp == 0) {
        // ------------------------------------------------ shrink producer
        // lane 0 owns the barriers; lane q issues chunk q's box and lane 4 the
        // A panel, so a stage's boxes are in flight together (a single thread
        // pays ~100+ cycles per TMA issue)
        const uint64_t keep = tc::policy_evict_last();
        int stage = 0, ub = 0;
        uint32_t phase = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int slot = U.x - a.slot_base, nch = U.z;
            // stay at most one unit ahead of the epilogue: the unit being
            // re-read plus the one being streamed must fit in L2
            if (lane == 0 && ub > 0 && !(a.flags & 4)) tc::mbar_wait(&v_full[(ub - 1) & 1], ((ub - 1) >> 1) & 1);
            ++ub;
            const int row = lane < nch ? a.chunks[U.y + lane].x : 0;
            const uint32_t bytes = static_cast<uint32_t>(L::SPPS * (nch * kChunk * 128 + L::AP_BYTES));
            const int rq = __shfl_sync(0xffffffffu, row, lane & 3);
            for (int p = 0; p < NP; p += L::SPPS) {
                if (lane == 0) {
                    tc::mbar_wait(&sh_empty[stage], phase ^ 1u);
                    if ((a.flags & 2) && ub > 1) {
                        // panel p of this unit may load once the epilogue re-read columns p*64 - look*64 of the previous one
                        const int need = (ub - 2) * NJ + min(NJ, max(0, (p - a.look) * 64 / kEpiN + 1));
                        while (atomicOr(&s_epi_done, 0) < need) __nanosleep(64);
                    }
                    tc::mbar_expect_tx(&sh_full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + L::OFF_SH + stage * L::SH_STAGE;
                const int pp = lane >> 2, q = lane & 3;  // lane 4*pp + q: panel pp of chunk q; lanes 16+: A panels
                if (lane < 4 * L::SPPS) {
                    if (q < nch)
                        tc::tma_load_2d_hint(st + pp * L::H_BYTES + q * (kChunk * 128), &tmH, (pc0 + p + pp) * 64, rq,
                                             &sh_full[stage], keep);
                } else if (lane >= 16 && lane < 16 + L::SPPS) {
                    tc::tma_load_2d(st + L::SPPS * L::H_BYTES + (lane - 16) * L::AP_BYTES, &tmA, (pc0 + p + lane - 16) * 64,
                                    slot * R, &sh_full[stage]);
                }
                if (++stage == L::SH_STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ shrink MMA
        if (lane == 0) {
            const uint32_t id = tc::idesc_bf16_f32(kUnitRows, R);
            int stage = 0, ub = 0;
            uint32_t phase = 0;
            for (int u = u0; u < u1; ++u) {
                const int4 U = a.units[u];
                if (U.x < a.slot_base) continue;
                const int sb = ub & 1;
                tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
                tc::fence_after_sync();
                const uint32_t dS = tmem + sb * L::S_COLS;
                for (int p = 0; p < NP; p += L::SPPS) {
                    tc::mbar_wait(&sh_full[stage], phase);
                    // these rows are in L2 now: the epilogue producer may re-read them
                    atomicMax(&s_shrunk, (ub * NP) + p + L::SPPS);  // shared-memory atomics: an explicit, race-free flag
                    if (a.prof && blockIdx.x == a.prof_cta && ub < 16 && (p == 0 || p + L::SPPS >= NP))
                        a.prof[576 + ub * 2 + (p ? 1 : 0)] = clock64();
                    tc::fence_after_sync();
                    const uint32_t st = sbase + L::OFF_SH + stage * L::SH_STAGE;
#pragma unroll
                    for (int k = 0; k < 4 * L::SPPS; ++k) {
                        const int kk = p * 4 + k, pp = k >> 2, kq = k & 3;
                        tc::mma_bf16(dS + (kk % kNacc) * R, tc::desc_kmajor_sw128(st + pp * L::H_BYTES + kq * 32),
                                     tc::desc_kmajor_sw128(st + L::SPPS * L::H_BYTES + pp * L::AP_BYTES + kq * 32), id,
                                     kk >= kNacc ? 1u : 0u);
                    }
                    tc::mma_commit(&sh_empty[stage]);
                    if (++stage == L::SH_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                tc::mma_commit(&s_full[sb]);
                ++ub;
            }
        }
    } else if (warp == 2) {
        // ------------------------------------------------ epilogue producer
        // lane 4*pp + q issues panel pp of chunk q, lane 8 the Bt chunk
        const uint64_t stream = tc::policy_evict_first();
        const int pp = lane >> 2, q = lane & 3;
        int stage = 0, ub = 0;
        uint32_t phase = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int slot = U.x - a.slot_base, nch = U.z;
            const int unit_base = ub * NP;
            ++ub;
            const int row = q < nch ? a.chunks[U.y + q].x : 0;
            const unsigned char* bt = a.Bt + static_cast<long long>(slot) * a.d * R * 2;
            const bool reduce = a.flags & 32;  // epilogue adds delta in L2: no re-read of h
            const uint32_t bytes = static_cast<uint32_t>((reduce ? 0 : 2 * nch * kChunk * 128) + L::BT_BYTES);
            for (int j = 0; j < NJ; ++j) {
                if (lane == 0) {
                    tc::mbar_wait(&epi_empty[stage], phase ^ 1u);
                    if (!(a.flags & 8) && !reduce) {
                        // never re-read columns before the shrink has read them: an
                        // early (evict_first) epilogue read would miss, and could
                        // evict the lines before the shrink gets to them
                        const int need = unit_base + min(NP, (j + 1) * (kEpiN / 64));
                        while (atomicOr(&s_shrunk, 0) < need) __nanosleep(32);
                    }
                    tc::mbar_expect_tx(&epi_full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + L::OFF_EPI + stage * L::EPI_STAGE;
                if (lane < 8 && q < nch && !reduce)
                    tc::tma_load_2d_hint(st + pp * L::H_BYTES + q * (kChunk * 128), &tmH, (jc0 + j) * kEpiN + pp * 64,
                                         row, &epi_full[stage], stream);
                else if (lane == 8)
                    tc::bulk_load_1d(st + L::EH_BYTES, bt + static_cast<long long>(jc0 + j) * L::BT_BYTES, L::BT_BYTES,
                                     &epi_full[stage]);
                if (++stage == L::EPI_STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 3) {
        // ------------------------------------------------ expand MMA
        if (lane == 0) {
            const uint32_t id = tc::idesc_bf16_f32(kUnitRows, kEpiN);
            int stage = 0, ub = 0, dc = 0;
            uint32_t phase = 0;
            for (int u = u0; u < u1; ++u) {
                const int4 U = a.units[u];
                if (U.x < a.slot_base) continue;
                const int vb = ub & 1;
                tc::mbar_wait(&v_full[vb], (ub >> 1) & 1);
                tc::fence_after_sync();
                const uint32_t vhi = sbase + L::OFF_V + vb * 2 * L::V_BYTES, vlo = vhi + L::V_BYTES;
                for (int j = 0; j < NJ; ++j) {
                    tc::mbar_wait(&epi_full[stage], phase);
                    if (a.prof && blockIdx.x == a.prof_cta && dc < 64) a.prof[dc * 8 + 0] = clock64();
                    const int db = dc & 1;
                    tc::mbar_wait(&d_empty[db], ((dc >> 1) & 1) ^ 1u);
                    if (a.prof && blockIdx.x == a.prof_cta && dc < 64) a.prof[dc * 8 + 1] = clock64();
                    tc::fence_after_sync();
                    const uint32_t bt = sbase + L::OFF_EPI + stage * L::EPI_STAGE + L::EH_BYTES;
                    const uint32_t dD = tmem + L::D_COL0 + db * kEpiN;
#pragma unroll
                    for (int k = 0; k < R / 16; ++k) {
                        const uint64_t bd = tc::desc_kmajor(bt + k * 256, 128, R * 16);
                        tc::mma_bf16(dD, tc::desc_kmajor(vhi + k * 256, 128, R * 16), bd, id, k > 0 ? 1u : 0u);
                        tc::mma_bf16(dD, tc::desc_kmajor(vlo + k * 256, 128, R * 16), bd, id, 1u);
                    }
                    tc::mma_commit(&d_full[db]);
                    tc::mma_commit(&epi_empty[stage]);  // Bt chunk no longer read
                    if (a.prof && blockIdx.x == a.prof_cta && dc < 64) a.prof[dc * 8 + 2] = clock64();
                    if (++stage == L::EPI_STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                    ++dc;
                }
                tc::mma_commit(&v_empty[vb]);
                ++ub;
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 4..11)
        // two groups of four warps take alternate chunks (group g: the chunks with
        // dc % 2 == g, hence D buffer g and the stages of parity g); a warp covers
        // its TMEM lane quadrant's 16 rows across the whole 128-column chunk, so two
        // chunks' latency chains (TMEM load, smem RMW, TMA store) overlap
        const int q = warp & 3;             // the TMEM lane quadrant this warp may access
        const int grp = (warp - 4) >> 2;    // chunk parity this group owns
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        const uint64_t stream = (a.flags & 16) ? tc::policy_evict_normal() : tc::policy_evict_first();
        int stage = 0, ub = 0, dc = 0, pend = -1;
        uint32_t phase = 0;
        for (int u = u0; u < u1; ++u) {
            const int4 U = a.units[u];
            if (U.x < a.slot_base) continue;
            const int nch = U.z;
            const int2 ch = q < nch ? a.chunks[U.y + q] : make_int2(0, 0);
            const int r1 = lane >> 2, cp = 2 * (lane & 3);
            for (int j = 0; j < NJ; ++j, ++dc) {
                const int st0 = stage;
                const uint32_t ph0 = phase;
                if (++stage == L::EPI_STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
                if ((dc & 1) != grp) continue;
                const int db = grp;
                tc::mbar_wait(&d_full[db], (dc >> 1) & 1);
                PROF(3);
                tc::mbar_wait(&epi_full[st0], ph0);
                PROF(4);
                tc::fence_after_sync();
#pragma unroll 1
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t v[32];
                    tc::tmem_ld_16x256b_x8(tmem + lane_base + L::D_COL0 + db * kEpiN + hf * 64, v);
                    tc::tmem_ld_wait();
                    if (hf == 1) {
                        tc::fence_before_sync();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&d_empty[db]);
                        PROF(5);
                    }
                    const uint32_t panel = L::OFF_EPI + st0 * L::EPI_STAGE + hf * L::H_BYTES;
                    if (ch.y > 0 && (a.flags & 32)) {
                        // reduce epilogue: stage the bf16 delta (-0.0 in rows past the
                        // chunk: the additive identity that keeps every bit, -0.0
                        // included) and let TMA add it into h in L2
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
                                const int rr = r1 + 8 * half;
                                const uint32_t d = rr < ch.y ? f32x2_to_bf16(__uint_as_float(v[4 * i + 2 * half]),
                                                                              __uint_as_float(v[4 * i + 2 * half + 1]))
                                                             : 0x80008000u;
                                *reinterpret_cast<uint32_t*>(sgen + panel +
                                                             tc::sw128_offset(q * kChunk + rr, 8 * i + cp, 64)) = d;
                            }
                    } else if (ch.y > 0) {
                        // all 16 loads first, then the math, then the stores (the
                        // addresses are disjoint but not provably so to the compiler)
                        uint32_t hv[16];
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half)
                                hv[2 * i + half] = *reinterpret_cast<const uint32_t*>(
                                    sgen + panel + tc::sw128_offset(q * kChunk + r1 + 8 * half, 8 * i + cp, 64));
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
                                float lo, hi;
                                bf16x2_to_acc(hv[2 * i + half], lo, hi);
                                lo += __uint_as_float(v[4 * i + 2 * half]);
                                hi += __uint_as_float(v[4 * i + 2 * half + 1]);
                                hv[2 * i + half] = f32x2_to_bf16(lo, hi);
                            }
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half)
                                *reinterpret_cast<uint32_t*>(sgen + panel + tc::sw128_offset(q * kChunk + r1 + 8 * half,
                                                                                             8 * i + cp, 64)) =
                                    hv[2 * i + half];
                    }
                }
                if (ch.y > 0) {
                    tc::fence_proxy_async();  // epilogue smem writes -> TMA reads
                    __syncwarp();
                    PROF(6);
                    const uint32_t panel0 = L::OFF_EPI + st0 * L::EPI_STAGE;
                    if (a.flags & 32) {
                        if (lane == 0)
                            for (int hf = 0; hf < 2; ++hf)
                                tc::tma_reduce_add_2d(&tmH, (jc0 + j) * kEpiN + hf * 64, ch.x,
                                                      sbase + panel0 + hf * L::H_BYTES + q * (kChunk * 128));
                    } else if (ch.y == kChunk) {
                        if (lane == 0)
                            for (int hf = 0; hf < 2; ++hf)
                                tc::tma_store_2d_hint(&tmH, (jc0 + j) * kEpiN + hf * 64, ch.x,
                                                      sbase + panel0 + hf * L::H_BYTES + q * (kChunk * 128), stream);
                    } else {
                        // partial chunk (end of a prompt): only its valid rows go back
                        for (int idx = lane; idx < ch.y * 16; idx += 32) {
                            const int rr = idx >> 4, hf = (idx >> 3) & 1, c16 = idx & 7;
                            const uint4 val = *reinterpret_cast<const uint4*>(
                                sgen + panel0 + hf * L::H_BYTES + tc::sw128_offset(q * kChunk + rr, c16 * 8, 64));
                            *reinterpret_cast<uint4*>(a.h + static_cast<long long>(ch.x + rr) * a.ldh +
                                                      (jc0 + j) * kEpiN + hf * 64 + c16 * 8) = val;
                        }
                    }
                }
                if (lane == 0) {
                    tc::tma_store_commit();
                    if (a.flags & 1) {
                        // release this stage once its stores have read shared memory
                        tc::tma_store_wait_read();
                        tc::mbar_arrive(&epi_empty[st0]);
                    } else {
                        // release the group's PREVIOUS stage once its stores have read
                        tc::tma_store_wait_read_1();
                        if (pend >= 0) tc::mbar_arrive(&epi_empty[pend]);
                        pend = st0;
                    }
                    if (q == 0) atomicAdd(&s_epi_done, 1);
                }
                __syncwarp();
                PROF(7);
            }
            ++ub;
        }
        if (lane == 0) {
            tc::tma_store_wait_all();  // bulk stores complete before the CTA retires
            if (pend >= 0) tc::mbar_arrive(&epi_empty[pend]);
        }
    }
    tc::fence_before_sync();
    if constexpr (C > 1) tc::cluster_sync();  // no peer still writes our inbox / barriers
    else __syncthreads();
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, 512);
    }
}

static int g_tc_last_grid = 0;
static int g_tc_flags = -1, g_tc_look = -1;  // -1: from the environment (PREFT_REFT_TC_FLAGS / _LOOK)
void reft_tc_set_flags(int flags, int look) {
    g_tc_flags = flags;
    g_tc_look = look;
}
static long long* g_tc_prof = nullptr;
int reft_tc_last_grid() { return g_tc_last_grid; }
void reft_tc_note_grid(int grid) { g_tc_last_grid = grid; }
void reft_tc_set_profile(long long* buf) { g_tc_prof = buf; }
long long* reft_tc_profile_buffer() { return g_tc_prof; }

template <int R, int C>
static int launch_reft_tc(const ReftTcArgs& args, const CUtensorMap& tmH, const CUtensorMap& tmA, int num_sms,
                          cudaStream_t stream) {
    auto fn = reft_tc_kernel<R, C>;
    const int smem = TcLayout<R, C>::SMEM;
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
    int grid = (num_sms / C) * C;
    if (C > 1) {
        static int cached[3] = {0, 0, 0};  // co-resident clusters per (C), measured once
        int& nc = cached[C == 2 ? 1 : 2];
        if (nc == 0) {
            cfg.gridDim = dim3(grid);
            e = cudaOccupancyMaxActiveClusters(&nc, fn, &cfg);
            if (e != cudaSuccess) return -static_cast<int>(e);
            if (nc < 1) return PREFT_ERR_CONFIG;
        }
        grid = min(grid, nc * C);
    }
    cfg.gridDim = dim3(grid);
    g_tc_last_grid = grid;
    e = cudaLaunchKernelEx(&cfg, fn, tmH, tmA, args);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

// Cluster size: split d over C CTAs so one unit is <= 2048 columns (256 KB of
// h per CTA): the rows read by the shrink are still in L2 when the epilogue
// re-reads them.  Env PREFT_REFT_TC_CLUSTER=1|2|4 overrides (A/B measurement).
static int tc_cluster_for(int d) {
    static int forced = -1;
    if (forced < 0) {
        const char* env = getenv("PREFT_REFT_TC_CLUSTER");
        forced = env ? atoi(env) : 0;
    }
    int c = d >= 8192 && d % 512 == 0 ? 4 : d >= 2048 && d % 256 == 0 ? 2 : 1;
    if (forced == 1 || forced == 2 || forced == 4) c = forced;
    while (c > 1 && d % (kEpiN * c)) c >>= 1;
    return c;
}

// returns 0 on launch, PREFT_ERR_SHAPE if the shape is not TC-eligible, or -cudaError
int reft_tc_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A,
                  const void* Bt, const void* bias, const void* scale, int r, cudaStream_t stream, int num_sms,
                  int part_lo, int part_hi) {
    if (!Bt || (r != 16 && r != 32) || d < 128 || d % 128 || rows < 1) return PREFT_ERR_SHAPE;
    if ((d / tc_cluster_for(d)) % (64 * spps_for(r, tc_cluster_for(d)))) return PREFT_ERR_SHAPE;
    if (!meta->chunks || !meta->units || (ldh % 8) || (reinterpret_cast<uintptr_t>(h) & 15) ||
        (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(Bt) & 15))
        return PREFT_ERR_SHAPE;
    CUtensorMap tmH{}, tmA{};
    if (!make_tmap_bf16_sw128(&tmH, h, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(ldh), 64, kChunk))
        return PREFT_ERR_CONFIG;
    // A slab of this layer viewed as [slots * r][d]; the box row is always a
    // registered slot, so the row extent only needs to cover the pool
    if (!make_tmap_bf16_sw128(&tmA, A, 1ull << 20, static_cast<unsigned long long>(d),
                              static_cast<unsigned long long>(d), 64, static_cast<unsigned>(r)))
        return PREFT_ERR_CONFIG;
    ReftTcArgs args;
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
    {
        int& flags = g_tc_flags;
        int& look = g_tc_look;
        if (flags < 0) {
            const char* f = getenv("PREFT_REFT_TC_FLAGS");
            const char* l = getenv("PREFT_REFT_TC_LOOK");
            flags = f ? atoi(f) : 7;  // immediate stage release, shrink paced by the epilogue, no unit throttle
            look = l ? atoi(l) : -1;
        }
        args.flags = flags;
        // the shrink may run 3/4 of a unit ahead of the epilogue's re-read
        args.look = look >= 0 ? look : (d / 64) / tc_cluster_for(d) * 3 / 4;
        args.prof = g_tc_prof;
        const char* pc = g_tc_prof ? getenv("PREFT_REFT_PROF_CTA") : nullptr;
        args.prof_cta = pc ? atoi(pc) : 0;
    }
    const int c = tc_cluster_for(d);
    if (r == 16)
        return c == 4 ? launch_reft_tc<16, 4>(args, tmH, tmA, num_sms, stream)
               : c == 2 ? launch_reft_tc<16, 2>(args, tmH, tmA, num_sms, stream)
                        : launch_reft_tc<16, 1>(args, tmH, tmA, num_sms, stream);
    return c == 4 ? launch_reft_tc<32, 4>(args, tmH, tmA, num_sms, stream)
           : c == 2 ? launch_reft_tc<32, 2>(args, tmH, tmA, num_sms, stream)
                    : launch_reft_tc<32, 1>(args, tmH, tmA, num_sms, stream);
}

}  // namespace preft
