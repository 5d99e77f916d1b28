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
//   tcgen05 (bf16, R in {16, 32}, m % 256 == 0, n % 128 == 0): persistent
//     warp-specialised kernels over K1's M = 64 units — shrink: TMA x/A
//     panels -> UMMA -> TMEM -> P rows;  expand: P rows -> bf16 hi/lo V ->
//     UMMA against the pre-tiled Bt block -> TMEM -> y tile read-modify-write
//     in shared memory -> TMA store.  Each CTA takes a contiguous,
//     cost-balanced range of (unit, column block) items (see item_range):
//     with short prompts there are only ~1.6 units per SM, and whole-unit
//     shares left the slowest CTA with 2-4x the mean work.
//   SIMT (any dtype / rank, one warp per token row) for everything else.
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"
#include "tmap.cuh"
#include "split.cuh"
#include "expand.cuh"

namespace preft {

int grid_for(const void* fn, int threads, int num_sms);

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



// Items are (unit, block of kPps K panels); a CTA accumulates its run of a
// unit's blocks (a "visit") in TMEM.  When several CTAs share a unit (at most
// max_planes), each writes its partial to plane (cta - first owner) and the
// last to arrive sums the planes in plane order into P — a fixed summation
// order, so results do not depend on which CTA finishes last.
//
// warps: 0 TMA producer (x), 6 TMA producer (A), 1 + 7..9 UMMA issuers,
//        2..5 TMEM -> P rows (lane quadrant = warp % 4)
template <int R, int NS>
__global__ void __launch_bounds__(kShrinkThreads, 1) shrink_tc_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a) {
    using L = ShrinkLayout<R, NS>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[L::STAGES], empty[L::STAGES];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
    __shared__ uint32_t tslot;
    __shared__ int s_u[2];
    __shared__ int s_last;
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
    tc::pdl_launch_dependents();

    // K blocks of kPps panels; with one plane a unit is never split
    Blocks bl;
    CostModel cm;
    shrink_model(bl, cm, a.units, a.counters, a.m, NS * R, a.max_planes, gridDim.x, a.beta_s);
    int k0, k1;
    // the schedule reads only K1's units and counters, written by a meta
    // build that completed before the first kernel of this PDL chain could
    // start (K1 never triggers its dependents early), so it is found while the
    // previous kernel drains; x, A and P are touched only after the wait
    item_range(cm, bl, s_u, k0, k1);
    const int nc = bl.nc;
    tc::pdl_wait();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1536 + 2 * blockIdx.x] = tc::globaltimer();

    if (warp == 0) {
        // x producer: lane q issues chunk q's boxes, so a stage's boxes are in
        // flight together
        const uint64_t stream = tc::policy_evict_first();
        int stage = 0, npf = 0, pu = -1, row = 0, r0 = 0, nch = 0;
        bool contig = false;
        uint32_t phase = 0;
        for (int k = k0; k < k1; ++k) {
            const int u = k / nc, g = k - u * nc;
            if (u != pu) {
                const int4 U = a.units[u];
                nch = U.z;
                row = lane < nch ? a.chunks[U.y + lane].x : 0;
                r0 = __shfl_sync(0xffffffffu, row, 0);
                contig = unit_contiguous(a.chunks, U);
                pu = u;
            }
            const int p = g * (bl.cw[0] / 64);
            const int np = bl.cw[0] / 64;
            const uint32_t bytes = static_cast<uint32_t>(kPps * (nch * kSpChunk * 128 + NS * L::AP_BYTES));
            for (int pi = 0; pi < np; pi += kPps) {
                if (lane == 0) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    if (a.prof && blockIdx.x == 0 && npf < 128) a.prof[npf * 4 + 0] = clock64();
                    tc::mbar_expect_tx(&full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + stage * L::STAGE;
                const int rq = __shfl_sync(0xffffffffu, row, lane & 3);  // chunk (lane & 3)'s first row
                if (contig) {
                    if (lane < kPps)
                        tc::tma_load_2d_hint(st + lane * L::PANEL, &maps.x64, (p + pi + lane) * 64, r0, &full[stage],
                                             stream);
                } else if (lane < 4 * kPps) {
                    const int pp = lane >> 2, q = lane & 3;
                    if (q < nch)
                        tc::tma_load_2d_hint(st + pp * L::PANEL + q * (kSpChunk * 128), &maps.x, (p + pi + pp) * 64,
                                             rq, &full[stage], stream);
                }
                ++npf;
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 6) {
        // second producer: the adapters' A panels, lane (panel, site) issues one
        // box, so a stage's kPps x NS boxes go out together (one thread issuing
        // them back to back took ~100-200 cycles per box)
        {
            int stage = 0, pu = -1, slot = 0;
            uint32_t phase = 0;
            const int pp = lane / NS, s = lane - pp * NS;
            for (int k = k0; k < k1; ++k) {
                const int u = k / nc, g = k - u * nc;
                if (u != pu) {
                    slot = a.units[u].x;
                    pu = u;
                }
                const int np = bl.cw[0] / 64, p = g * np;
                for (int pi = 0; pi < np; pi += kPps) {
                    if (lane == 0) tc::mbar_wait(&empty[stage], phase ^ 1u);
                    __syncwarp();
                    const uint32_t st = sbase + stage * L::STAGE;
                    if (lane < kPps * NS)
                        tc::tma_load_2d(st + L::X_BYTES + (pp * NS + s) * L::AP_BYTES, &maps.A[s], (p + pi + pp) * 64,
                                        slot * R, &full[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1 || warp >= 7) {
        // kSpAcc warps issue the UMMAs, K-step k into accumulator k % kSpAcc
        const int mw = warp == 1 ? 0 : warp - 6;
        if (lane == 0) {
            // the sites' A panels sit back to back in the stage, so one UMMA with
            // N = NS * R covers all of them
            const uint32_t id = tc::idesc_bf16_f32(kSpU, L::NSR);
            int stage = 0, ub = 0, nmc = 0, kk = 0;
            uint32_t phase = 0;
            for (int k = k0; k < k1; ++k) {
                const int u = k / nc;
                const bool first = k == k0 || (k - 1) / nc != u;
                const bool last = k + 1 == k1 || (k + 1) / nc != u;
                const int sb = ub & 1;
                const uint32_t dS = tmem + sb * kSpAcc * L::NSR;
                if (first) {
                    tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
                    tc::fence_after_sync();
                    kk = 0;
                }
                const int np = bl.cw[0] / 64;
                for (int pi = 0; pi < np; pi += kPps) {
                    tc::mbar_wait(&full[stage], phase);
                    if (a.prof && blockIdx.x == 0 && mw == 0 && nmc < 128) a.prof[nmc * 4 + 1] = clock64();
                    ++nmc;
                    tc::fence_after_sync();
                    const uint32_t st = sbase + stage * L::STAGE;
#pragma unroll
                    for (int j = mw; j < 4 * kPps; j += kSpAcc) {
                        const int pp = j >> 2, kq = j & 3;
                        tc::mma_bf16(dS + mw * L::NSR, tc::desc_kmajor_sw128(st + pp * L::PANEL + kq * 32),
                                     tc::desc_kmajor_sw128(st + L::X_BYTES + pp * NS * L::AP_BYTES + kq * 32), id,
                                     kk + j >= kSpAcc ? 1u : 0u);
                    }
                    kk += 4 * kPps;
                    tc::mma_commit(&empty[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                if (last) {
                    tc::mma_commit(&s_full[sb]);
                    ++ub;
                }
            }
        }
    } else if (warp < 6) {
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        for (int k = k0; k < k1; ++k) {
            const int u = k / nc;
            if (!(k + 1 == k1 || (k + 1) / nc != u)) continue;  // act once per visit, at its last item
            const int4 U = a.units[u];
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            // which plane: this CTA's index among the CTAs sharing the unit
            int plane = 0, np = 1;
            if (nc > 1) {
                plane = static_cast<int>(blockIdx.x) - unit_first_cta(cm, bl, u);
                np = unit_pieces(cm, bl, u, U.z);
            }
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
            float* P0 = static_cast<float*>(a.P);
            float* dst = plane == 0 ? P0 : a.planes + plane * a.plane_stride;
            if (lane < ch.y) {
                float* pr = dst + static_cast<long long>(ch.x + lane) * a.ldp;
#pragma unroll
                for (int c = 0; c < L::NSR; c += 4)
                    *reinterpret_cast<float4*>(pr + c) = make_float4(s[c], s[c + 1], s[c + 2], s[c + 3]);
            }
            if (np > 1) {
                // arrive (the CUDA threadFenceReduction pattern: the barrier
                // orders the four warps' plane rows before one thread's fence
                // + atomic); the last of the unit's np CTAs sums the planes
                readout_bar();
                if (warp == 2 && lane == 0) {
                    __threadfence();
                    s_last = atomicAdd(a.sync + u, 1) == np - 1;
                    if (s_last) __threadfence();
                }
                readout_bar();
                if (s_last) {
                    if (lane < ch.y) {
                        const long long row = static_cast<long long>(ch.x + lane) * a.ldp;
#pragma unroll
                        for (int c = 0; c < L::NSR; c += 4) {
                            float4 v = __ldcg(reinterpret_cast<const float4*>(P0 + row + c));
                            for (int p = 1; p < np; ++p) {
                                const float4 w = __ldcg(reinterpret_cast<const float4*>(a.planes + p * a.plane_stride + row + c));
                                v.x += w.x;
                                v.y += w.y;
                                v.z += w.z;
                                v.w += w.w;
                            }
                            *reinterpret_cast<float4*>(P0 + row + c) = v;
                        }
                    }
                    if (warp == 2 && lane == 0) a.sync[u] = 0;  // every contributor has arrived
                }
                readout_bar();  // s_last is rewritten by the next visit
            }
            ++ub;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1537 + 2 * blockIdx.x] = tc::globaltimer();
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, L::TMEM_COLS);
    }
}


// LPT shrink (opt-in, PREFT_SPLIT_LPT=1; needs K1's size order): whole units
// handed out largest first — the CTA's own index first, then from a global
// counter one grab ahead — through a 4-slot shared-memory queue that every
// role walks.  At ~1.6 units per CTA the cost-balanced contiguous ranges
// left the slowest CTA at ~1.7x the mean (whole units cannot be split
// without summing partials, which costs more than it saves); greedy
// largest-first brings it to ~1.2x.  Grab counters: LaunchSeq (split.cuh).
//
// warps: 0 grabs + TMA producer (x), 6 TMA producer (A), 1 + 7..9 UMMA
// issuers, 2..5 TMEM -> P rows (lane quadrant = warp % 4)
template <int R, int NS>
__global__ void __launch_bounds__(kShrinkThreads, 1) shrink_lpt_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a) {
    using L = ShrinkLayout<R, NS>;
    constexpr int Q = 4, CONSUMERS = 1 + kSpAcc + 4;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[L::STAGES], empty[L::STAGES];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2];
    __shared__ __align__(8) uint64_t q_full[Q], q_empty[Q];
    __shared__ int q_u[Q];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = (tc::smem_u32(sm_raw) + 1023u) & ~1023u;
    if (warp == 0) tc::tmem_alloc(&tslot, L::TMEM_COLS);
    if (tid == 32) {
        for (int i = 0; i < L::STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], kSpAcc);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], kSpAcc);
            tc::mbar_init(&s_empty[b], 4);
        }
        for (int i = 0; i < Q; ++i) {
            tc::mbar_init(&q_full[i], 1);
            tc::mbar_init(&q_empty[i], CONSUMERS);
        }
        tc::fence_mbar_init();
        tc::prefetch_tmap(&maps.x);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    tc::pdl_launch_dependents();
    const int nlu = a.counters[PREFT_CTR_LORA_UNITS];
    const int* order = a.unit_order;
    // K1's output: the first grab is known before the wait
    int first_u = -1;
    if (warp == 0 && lane == 0 && static_cast<int>(blockIdx.x) < nlu) first_u = order[blockIdx.x];
    tc::pdl_wait();  // x, A, P and the launch-sequence counters from here on
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1536 + 2 * blockIdx.x] = tc::globaltimer();
    const int np = a.m / 64;
    int* seqb = a.sched + kSeqInts;
    const LaunchSeq seq = launch_seq_begin(seqb);
    int* ctr = seq.grab;

    // consumers: every posted unit in order
    auto walk = [&](auto&& body) {
        int qi = 0;
        uint32_t qph = 0;
        while (true) {
            if (lane == 0) tc::mbar_wait(&q_full[qi], qph);
            __syncwarp();
            const int u = *reinterpret_cast<volatile int*>(&q_u[qi]);
            __syncwarp();
            if (u < 0) break;
            if (lane == 0) tc::mbar_arrive(&q_empty[qi]);
            body(u);
            if (++qi == Q) {
                qi = 0;
                qph ^= 1u;
            }
        }
    };

    if (warp == 0) {
        const uint64_t stream = tc::policy_evict_first();
        int stage = 0, qi = 0;
        uint32_t phase = 0, qph = 0;
        int cur_u = first_u;      // lane 0
        int next_g = -1;          // lane 0: the next grab index, in flight
        if (lane == 0 && cur_u >= 0) next_g = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
        while (true) {
            if (lane == 0) {
                tc::mbar_wait(&q_empty[qi], qph ^ 1u);
                q_u[qi] = cur_u;
                tc::mbar_arrive(&q_full[qi]);
            }
            const int u = __shfl_sync(0xffffffffu, cur_u, 0);
            if (++qi == Q) {
                qi = 0;
                qph ^= 1u;
            }
            if (u < 0) break;
            // the next unit: its order[] load and the grab after it go out now,
            // their round trips overlap this unit's loads
            int nu_ = -1;
            if (lane == 0) {
                if (next_g < nlu) {
                    nu_ = order[next_g];
                    next_g = atomicAdd(ctr, 1) + static_cast<int>(gridDim.x);
                }
            }
            const int4 U = a.units[u];
            const int n = U.z;
            const int row = lane < n ? a.chunks[U.y + lane].x : 0;
            const int r0 = __shfl_sync(0xffffffffu, row, 0);
            const bool contig = unit_contiguous(a.chunks, U);
            const uint32_t bytes = static_cast<uint32_t>(kPps * (n * kSpChunk * 128 + NS * L::AP_BYTES));
            const int rq = __shfl_sync(0xffffffffu, row, lane & 3);
            for (int p = 0; p < np; p += kPps) {
                if (lane == 0) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    tc::mbar_expect_tx(&full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + stage * L::STAGE;
                if (contig) {
                    if (lane < kPps)
                        tc::tma_load_2d_hint(st + lane * L::PANEL, &maps.x64, (p + lane) * 64, r0, &full[stage], stream);
                } else if (lane < 4 * kPps) {
                    const int pp = lane >> 2, q = lane & 3;
                    if (q < n)
                        tc::tma_load_2d_hint(st + pp * L::PANEL + q * (kSpChunk * 128), &maps.x, (p + pp) * 64, rq,
                                             &full[stage], stream);
                }
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            cur_u = nu_;
        }
    } else if (warp == 6) {
        int stage = 0;
        uint32_t phase = 0;
        const int pp = lane / NS, s = lane - pp * NS;  // lane-parallel box issue (see shrink_tc_kernel)
        walk([&](int u) {
            const int slot = a.units[u].x;
            for (int p = 0; p < np; p += kPps) {
                if (lane == 0) tc::mbar_wait(&empty[stage], phase ^ 1u);
                __syncwarp();
                const uint32_t st = sbase + stage * L::STAGE;
                if (lane < kPps * NS)
                    tc::tma_load_2d(st + L::X_BYTES + (pp * NS + s) * L::AP_BYTES, &maps.A[s], (p + pp) * 64,
                                    slot * R, &full[stage]);
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        });
    } else if (warp == 1 || warp >= 7) {
        const int mw = warp == 1 ? 0 : warp - 6;
        const uint32_t id = tc::idesc_bf16_f32(kSpU, L::NSR);
        int stage = 0, ub = 0;
        uint32_t phase = 0;
        walk([&](int) {
            if (lane != 0) return;
            const int sb = ub & 1;
            const uint32_t dS = tmem + sb * kSpAcc * L::NSR;
            tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
            tc::fence_after_sync();
            for (int p = 0; p < np; p += kPps) {
                tc::mbar_wait(&full[stage], phase);
                tc::fence_after_sync();
                const uint32_t st = sbase + stage * L::STAGE;
#pragma unroll
                for (int j = mw; j < 4 * kPps; j += kSpAcc) {
                    const int pp = j >> 2, kq = j & 3;
                    tc::mma_bf16(dS + mw * L::NSR, tc::desc_kmajor_sw128(st + pp * L::PANEL + kq * 32),
                                 tc::desc_kmajor_sw128(st + L::X_BYTES + pp * NS * L::AP_BYTES + kq * 32), id,
                                 p * 4 + j >= kSpAcc ? 1u : 0u);
                }
                tc::mma_commit(&empty[stage]);
                if (++stage == L::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            tc::mma_commit(&s_full[sb]);
            ++ub;
        });
    } else if (warp < 6) {
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        walk([&](int u) {
            const int4 U = a.units[u];
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const int sb = ub & 1;
            tc::mbar_wait(&s_full[sb], (ub >> 1) & 1);
            tc::fence_after_sync();
            float s[L::NSR];
#pragma unroll
            for (int c = 0; c < L::NSR; ++c) s[c] = 0.f;
#pragma unroll
            for (int acc = 0; acc < kSpAcc; ++acc)
#pragma unroll
                for (int cc = 0; cc < L::NSR; cc += 16) {
                    uint32_t w[16];
                    tc::tmem_ld16(tmem + lane_base + sb * kSpAcc * L::NSR + acc * L::NSR + cc, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 16; ++c) s[cc + c] += __uint_as_float(w[c]);
                }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
            if (lane < ch.y) {
                float* pr = static_cast<float*>(a.P) + static_cast<long long>(ch.x + lane) * a.ldp;
#pragma unroll
                for (int c = 0; c < L::NSR; c += 4)
                    *reinterpret_cast<float4*>(pr + c) = make_float4(s[c], s[c + 1], s[c + 2], s[c + 3]);
            }
            ++ub;
        });
    }
    tc::fence_before_sync();
    __syncthreads();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1537 + 2 * blockIdx.x] = tc::globaltimer();
    if (tid == 0) launch_seq_end(seqb, seq.n);
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, L::TMEM_COLS);
    }
}

// The expand (the pipeline in expand.cuh): static cost-balanced item ranges,
// or dynamic grabs (a.sched) for wide groups — the static ranges finished at
// max/mean 1.29 across CTAs at config-4 gate/up although every item ran at
// the SM's share of HBM.  Grab counters come from the launch sequence
// (split.cuh), so no CTA waits on an end-of-kernel handshake.
template <int R, int NS>
__global__ void __launch_bounds__(384, 1) expand_tc_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a) {
    using L = ExpandLayout<R, NS>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[L::STAGES], empty[L::STAGES];
    __shared__ __align__(8) uint64_t v_full[2], v_empty[2], d_full[2], d_empty[2];
    __shared__ __align__(8) uint64_t q_full[kExpQ], q_empty[kExpQ];
    __shared__ int q_lo[kExpQ], q_hi[kExpQ];
    __shared__ uint32_t tslot;
    __shared__ int s_u[2];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t raw = tc::smem_u32(sm_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    unsigned char* sgen = sm_raw + (sbase - raw);
    const ExpandBars B{full, empty, v_full, v_empty, d_full, d_empty, q_full, q_empty, q_lo, q_hi};
    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 32) {
        expand_bars_init(B, L::STAGES);
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    tc::pdl_launch_dependents();
    Blocks bl;
    expand_blocks(bl, a, NS);
    ExpandWork W{0, 0, a.sched, a.grab, 0};
    if (!a.sched) {
        CostModel cm;
        cm.units = a.units;
        cm.load(a.counters);
        cm.alpha = kSpChunk * 4;          // y read + write per column per chunk
        cm.beta = 2 * R + 16 + a.beta_e;  // Bt bytes per column + per-item overhead
        cm.G = gridDim.x;
        item_range(cm, bl, s_u, W.k0, W.k1);  // K1's output only: before the wait (see the shrink)
    }
    W.total = a.counters[PREFT_CTR_LORA_UNITS] * bl.nc;
    tc::pdl_wait();  // P, y and the launch-sequence counters from here on
    LaunchSeq seq{0, nullptr};
    if (a.sched) {
        seq = launch_seq_begin(a.sched);
        W.sched = seq.grab;
    }
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1792 + 2 * blockIdx.x] = tc::globaltimer();
    SplitVSrc vs{static_cast<const float*>(a.P), a.ldp};
    expand_pipeline<R, NS>(maps, a, bl, sbase, sgen, tmem, B, W, vs);
    tc::fence_before_sync();
    __syncthreads();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1793 + 2 * blockIdx.x] = tc::globaltimer();
    if (tid == 0 && a.sched) launch_seq_end(a.sched, seq.n);
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

static int launch_expand(const SplitMaps& maps, const SplitArgs& args, int nsites, int r, int num_sms, cudaStream_t stream) {
    if (r == 16) {
        if (nsites == 1) return launch_tc(expand_tc_kernel<16, 1>, ExpandLayout<16, 1>::SMEM, 384, maps, args, num_sms, stream);
        if (nsites == 2) return launch_tc(expand_tc_kernel<16, 2>, ExpandLayout<16, 2>::SMEM, 384, maps, args, num_sms, stream);
        return launch_tc(expand_tc_kernel<16, 3>, ExpandLayout<16, 3>::SMEM, 384, maps, args, num_sms, stream);
    }
    if (nsites == 1) return launch_tc(expand_tc_kernel<32, 1>, ExpandLayout<32, 1>::SMEM, 384, maps, args, num_sms, stream);
    if (nsites == 2) return launch_tc(expand_tc_kernel<32, 2>, ExpandLayout<32, 2>::SMEM, 384, maps, args, num_sms, stream);
    return PREFT_ERR_RANK;
}

static long long* g_split_prof = nullptr;
void split_set_profile(long long* buf) { g_split_prof = buf; }
long long* split_profile_buffer() { return g_split_prof; }

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

// Floats of meta->lora_part the tensor-core split uses: kPlanes planes of
// [T_cap][64] f32 (plane 0 is P itself on the preft_lora_apply route) and
// one int per unit (the shrink's per-unit arrival counters, kept zero
// between launches).
long long xchg_region_bytes(int tp, int planes, int T_cap, int U_cap);

// floats of the split pair's part of meta->lora_part (P / planes / counters)
long long lora_split_floats(const preft_meta_t* meta) {
    return (static_cast<long long>(kPlanes) * meta->T_cap * 64 + meta->chunk_cap + kSchedInts + 3) / 4 * 4;
}

// the dynamic expand's grab counter + finished-CTA counter (zero between
// launches), after the per-unit arrival counters in meta->lora_part
static int* split_sched(const preft_meta_t* meta) {
    if (!meta->lora_part || meta->lora_part_floats < lora_split_floats(meta)) return nullptr;
    return reinterpret_cast<int*>(meta->lora_part + static_cast<long long>(kPlanes) * meta->T_cap * 64 + meta->chunk_cap);
}

// ... followed by the single-rank exchange region of the fused kernel
// (lora_fused.cu), which the r >= 16 route of preft_lora_apply uses
long long lora_part_floats_needed(const preft_meta_t* meta) {
    return lora_split_floats(meta) + (xchg_region_bytes(1, kPlanes, meta->T_cap, meta->chunk_cap) + 3) / 4;
}

// cost-model overheads (bytes-equivalent per column per item) beyond the
// defaults: env PREFT_SPLIT_BETA_S / PREFT_SPLIT_BETA_E
static void split_tuning(SplitArgs& args) {
    static int bs = -1, be = -1;
    if (bs < 0) {
        const char* e = getenv("PREFT_SPLIT_BETA_S");
        bs = e ? atoi(e) : kBetaS;
        e = getenv("PREFT_SPLIT_BETA_E");
        be = e ? atoi(e) : kBetaE;
    }
    args.beta_s = bs;
    args.beta_e = be;
}

// the shrink's partial planes (p >= 1) and arrival counters, from the meta's
// workspace; one plane (whole units per CTA) without it
static void split_planes(SplitArgs& args, const preft_meta_t* meta) {
    args.max_planes = 1;
    args.planes = nullptr;
    args.plane_stride = 0;
    args.sync = nullptr;
    // default one plane (whole units per CTA): at config-4 shapes the K-split
    // schedule balances the CTAs (busy max/mean 1.3 -> 1.1) but its
    // per-visit fixup (fence + atomic + plane sum) costs more than it saves
    // (cfg4 12.0 ms/step with whole units vs 14.2 with 4 planes, r02i)
    const char* env = getenv("PREFT_SPLIT_PLANES");
    const int want = env ? atoi(env) : 1;
    if (meta->lora_part && meta->lora_part_floats >= lora_part_floats_needed(meta) && want > 1) {
        args.max_planes = want < kPlanes ? want : kPlanes;
        args.planes = meta->lora_part;
        args.plane_stride = static_cast<long long>(meta->T_cap) * 64;
        args.sync = reinterpret_cast<int*>(meta->lora_part + static_cast<long long>(kPlanes) * meta->T_cap * 64);
    }
}

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
        split_planes(args, meta);
        args.prof = g_split_prof;
        split_tuning(args);
        // largest-first whole units from K1's size order: opt-in (PREFT_SPLIT_LPT=1).
        // Measured (profiles/split_tuning_r02c.txt): 8B r16 shrink 4.88 -> 4.61 ms/step,
        // but config 4 4.18 -> 4.46 — the size order separates units of one adapter,
        // whose A panels then come from DRAM twice instead of once plus L2
        static int lpt = -1;
        if (lpt < 0) {
            const char* e = getenv("PREFT_SPLIT_LPT");
            lpt = (e && e[0] == '1') ? 1 : 0;
        }
        args.sched = split_sched(meta);
        args.unit_order = meta->units + 4 * static_cast<long long>(meta->chunk_cap);
        if (lpt && args.max_planes <= 1 && args.sched && (meta->meta_flags & PREFT_META_UNIT_ORDER)) {
            if (r == 16) {
                if (nsites == 1) return launch_tc(shrink_lpt_kernel<16, 1>, ShrinkLayout<16, 1>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
                if (nsites == 2) return launch_tc(shrink_lpt_kernel<16, 2>, ShrinkLayout<16, 2>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
                return launch_tc(shrink_lpt_kernel<16, 3>, ShrinkLayout<16, 3>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
            }
            if (nsites == 1) return launch_tc(shrink_lpt_kernel<32, 1>, ShrinkLayout<32, 1>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
            if (nsites == 2) return launch_tc(shrink_lpt_kernel<32, 2>, ShrinkLayout<32, 2>::SMEM, kShrinkThreads, maps, args, num_sms, stream);
            return PREFT_ERR_RANK;
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
    split_tuning(args);
    {
        // dynamic item grabs for wide groups: measured (profiles/split_tuning_r02c.txt) they
        // win where a unit has >= 28 output blocks (gate/up: 8B 119 -> 103 us per launch,
        // config 4 31.5 -> 30.5) and lose on narrower groups, whose few items per CTA the
        // static cost-balanced ranges split better.  PREFT_SPLIT_DYN=0/1 forces off/on.
        static int dyn = -2;
        if (dyn == -2) {
            const char* e = getenv("PREFT_SPLIT_DYN");
            dyn = e ? (e[0] == '0' ? 0 : 1) : -1;
        }
        int blocks = 0;
        for (int s = 0; s < nsites; ++s) blocks += sites[s].n / (sites[s].n % kSpNMax == 0 ? kSpNMax : kSpN);
        const bool want = dyn == 1 || (dyn == -1 && blocks >= 28);
        args.sched = want ? split_sched(meta) : nullptr;
        // items per grab: 8 for the widest groups; 6 below 64 blocks (config-4 gate/up,
        // 28 blocks: 11.06 -> 10.95 ms/step against 4, 11.01 at 8; r02h sweep)
        args.grab = blocks >= 64 ? 8 : 6;
        if (const char* e = getenv("PREFT_SPLIT_GRAB")) args.grab = atoi(e) > 0 ? atoi(e) : args.grab;
    }
    {
        const char* h = getenv("PREFT_SPLIT_HINTS");  // default on (+0.3%, profiles/split_tuning_r02c.txt)
        args.flags = (h && h[0] == '0') ? 0 : kSplitHints;
    }
    const int variant = split_variant();
    const bool tc_ok = expand_tc_ok(meta, P, ldp, sites, nsites, r, dtype);
    if (variant == 1 && !tc_ok) return PREFT_ERR_SHAPE;
    if (variant != 0 && tc_ok) {
        SplitMaps maps{};
        for (int s = 0; s < nsites; ++s) {
            const unsigned npan = (sites[s].n % kSpNMax == 0 ? kSpNMax : kSpN) / 64;
            if (!make_tmap_bf16_panels(&maps.y[s], sites[s].y, static_cast<unsigned long long>(rows),
                                       static_cast<unsigned long long>(sites[s].n),
                                       static_cast<unsigned long long>(sites[s].ldy), kSpChunk, npan))
                return PREFT_ERR_CONFIG;
        }
        return launch_expand(maps, args, nsites, r, num_sms, stream);
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
