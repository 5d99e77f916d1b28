// K2f — LoRA^P shrink -> cross-rank exchange -> expand in ONE persistent
// tcgen05 kernel (BASELINE config 4's tensor-parallel path and the r >= 16
// single-GPU route).  The reference delta is out[rows] += s * ((X A^T) B^T)
// (model.py:449-451, adapters.py:284-288); under tensor parallelism X A^T is
// the sum of every rank's partial over its m-slice.
//
// The split pair (lora_split.cu) runs this as shrink, NCCL all-reduce of P,
// expand: three launches per site group, each with its own ramp-up, tail and
// (for the collective) ~10-20 us of latency.  Here one grid does all of it:
//
//   phase 1 (shrink): every CTA takes a cost-balanced range of
//     (unit, K block) items — a unit may be split by K across up to
//     `planes` CTAs — accumulates its piece in TMEM and stores the partial
//     rows into EVERY rank's exchange region (P2P stores over NVLink when
//     tp > 1), then publishes the piece's flag = this launch's tag.
//   phase 2 (expand): the same CTA takes a cost-balanced range of
//     (unit, output block) items; before a unit's first block it waits for
//     the tp x pieces flags of that unit in its own region, sums the partials
//     in (src rank, piece) order — the same order on every rank, so every
//     rank's V is bit-identical, like an all-reduce — and runs the expand of
//     lora_split.cu (bf16 hi/lo V, UMMA against the pre-tiled Bt, TMA
//     reduce-add of the bf16 delta into y).
//
// Both phases are balanced independently, so the CTAs reach phase 2 at about
// the same time and the waits are short; the K-split pieces that the
// stand-alone shrink could not afford (a fixup pass per shared unit) cost
// nothing extra here, because the expand already sums partials.
//
// Exchange protocol (see preft_xchg_t in include/preft.h): flags carry the
// launch's tag (device-side launch count + 1), so they never need resetting;
// consecutive launches alternate between two parities of the region, so a
// rank that runs ahead into the next launch never overwrites partials a slow
// rank is still reading (it cannot get two launches ahead: the next launch
// waits for this rank's own partials).
#include <cuda_bf16.h>

#include "common.cuh"
#include "split.cuh"
#include "expand.cuh"
#include "tc.cuh"
#include "tmap.cuh"

namespace preft {

struct XchgArgs {
    float* part[PREFT_XCHG_MAX_TP];
    int* flag[PREFT_XCHG_MAX_TP];
    int* state;
    int tp, rank, planes, sys;
    int T_cap, U_cap;
    long long spin_ns;
    int beta_s, beta_e;  // cost-model tuning (env PREFT_FUSED_BETA_S / _E)
    int knobs;           // experiments: bit 0 no producer fence
    int dyn, grab;       // phase 2: dynamic item grabs (LaunchSeq at state + 16), items per grab
};


__host__ __device__ __forceinline__ long long xchg_part_off(int par, int src, int plane, int tp, int planes, int T_cap) {
    return ((static_cast<long long>(par) * tp + src) * planes + plane) * T_cap * 64;
}
__host__ __device__ __forceinline__ long long xchg_flag_off(int par, int src, int plane, int u, int tp, int planes,
                                                            int U_cap) {
    return ((static_cast<long long>(par) * tp + src) * planes + plane) * U_cap + u;
}

__device__ __forceinline__ void st_flag(int* p, int v, bool sys) {
    if (sys)
        asm volatile("st.relaxed.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
    else
        asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_flag(const int* p, bool sys) {
    int v;
    if (sys)
        asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// release fence of the publishing lane: it follows the readout warps' partial
// stores through the named barrier, so a cumulative acq_rel fence orders all
// of them before the flag store
__device__ __forceinline__ void fence_release(bool sys) {
    if (sys)
        asm volatile("fence.acq_rel.sys;" ::: "memory");
    else
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// phase 2's rank-r rows: wait for every (source rank, piece) flag of the
// unit, then sum the partials in (source, piece) order — the same order on
// every rank, so every rank's V is bit-identical, like an all-reduce's
struct XchgVSrc {
    const float* part;  // this rank's region
    const int* flag;
    int* state;
    const CostModel* cs;
    const Blocks* bs;
    int tp, planes, T_cap, U_cap, par, tag;
    bool sys;
    long long spin_ns;
    int npc;
    __device__ __forceinline__ void prepare(int u, const int4& U) {
        const int lane = threadIdx.x & 31;
        npc = unit_pieces(*cs, *bs, u, U.z);
        const int nflags = tp * npc;
        bool ok = lane >= nflags;
        const int* fp = ok ? nullptr : flag + xchg_flag_off(par, lane / npc, lane % npc, u, tp, planes, U_cap);
        uint64_t t0 = 0;
        while (true) {
            if (!ok) ok = ld_flag(fp, sys) == tag;
            if (__all_sync(0xffffffffu, ok)) break;
            const uint64_t now = tc::globaltimer();
            if (t0 == 0) t0 = now;
            if (static_cast<long long>(now - t0) > spin_ns) {
                if (lane == 0) atomicOr(state + 2, 1);
                break;
            }
            __nanosleep(64);
        }
        // every flag was read with ld.acquire by some lane; the warp barrier
        // orders the other lanes' partial loads after those acquires
        __syncwarp();
    }
    __device__ __forceinline__ void load(long long row, int col, float4& p0, float4& p1) const {
        p0 = make_float4(0.f, 0.f, 0.f, 0.f);
        p1 = p0;
        for (int src = 0; src < tp; ++src)
            for (int pl = 0; pl < npc; ++pl) {
                const float* pr = part + xchg_part_off(par, src, pl, tp, planes, T_cap) + row * 64 + col;
                const float4 w0 = __ldcg(reinterpret_cast<const float4*>(pr));
                const float4 w1 = __ldcg(reinterpret_cast<const float4*>(pr + 4));
                p0.x += w0.x;
                p0.y += w0.y;
                p0.z += w0.z;
                p0.w += w0.w;
                p1.x += w1.x;
                p1.y += w1.y;
                p1.z += w1.z;
                p1.w += w1.w;
            }
    }
};

template <int R, int NS>
struct FusedLayout {
    using LS = ShrinkLayout<R, NS>;
    using LE = ExpandLayout<R, NS>;
    static constexpr int SMEM = LS::SMEM > LE::SMEM ? LS::SMEM : LE::SMEM;
};

// warps: phase 1 — 0 TMA x, 6 TMA A, 1 + 7..9 UMMA, 2..5 TMEM -> partial rows -> every rank;
//        phase 2 — 0 TMA Bt, 1 UMMA, 2..3 flags -> sum of partials -> bf16 hi/lo V,
//                  4..7 / 8..11 epilogue groups (even / odd items)
template <int R, int NS>
__global__ void __launch_bounds__(384, 1)
    lora_fused_kernel(const __grid_constant__ SplitMaps maps, const SplitArgs a, const XchgArgs xa) {
    using LS = ShrinkLayout<R, NS>;
    using LE = ExpandLayout<R, NS>;
    extern __shared__ unsigned char sm_raw[];
    __shared__ __align__(8) uint64_t full[LS::STAGES], empty[LS::STAGES], s_full[2], s_empty[2];
    __shared__ __align__(8) uint64_t efull[LE::STAGES], eempty[LE::STAGES];
    __shared__ __align__(8) uint64_t v_full[2], v_empty[2], d_full[2], d_empty[2];
    __shared__ __align__(8) uint64_t q_full[kExpQ], q_empty[kExpQ];
    __shared__ int q_lo[kExpQ], q_hi[kExpQ];
    __shared__ uint32_t tslot;
    __shared__ int s_u[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t raw = tc::smem_u32(sm_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    unsigned char* sgen = sm_raw + (sbase - raw);
    const ExpandBars EB{efull, eempty, v_full, v_empty, d_full, d_empty, q_full, q_empty, q_lo, q_hi};
    if (warp == 0) tc::tmem_alloc(&tslot, 512);
    if (tid == 32) {
        for (int i = 0; i < LS::STAGES; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], kSpAcc);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&s_full[b], kSpAcc);
            tc::mbar_init(&s_empty[b], 4);
        }
        expand_bars_init(EB, LE::STAGES);
        tc::fence_mbar_init();
        tc::prefetch_tmap(&maps.x);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tslot;
    tc::pdl_launch_dependents();
    const bool sys = xa.sys != 0;

    // ---- schedules (K1's units and counters only: found before the PDL wait)
    Blocks bs;
    CostModel cs;
    shrink_model(bs, cs, a.units, a.counters, a.m, NS * R, xa.planes, gridDim.x, xa.beta_s);
    int s0, s1;
    item_range(cs, bs, s_u, s0, s1);
    __syncthreads();
    Blocks be;
    expand_blocks(be, a, NS);
    CostModel ce;
    ce.units = a.units;
    ce.load(a.counters);
    ce.alpha = kSpChunk * 4;
    ce.beta = 2 * R + 16 + xa.beta_e;
    ce.G = gridDim.x;
    int e0, e1;
    item_range(ce, be, s_u, e0, e1);
    const int ncs = bs.nc, nce = be.nc;

    tc::pdl_wait();
    // the launch's tag: every CTA's own launch count + 1 (LaunchSeq, split.cuh) —
    // the same on every CTA and, with the same launch sequence, on every rank
    int* seqb = xa.state + 16;
    const LaunchSeq seq = launch_seq_begin(seqb);
    const int tag = seq.n + 1, par = tag & 1;
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1536 + 2 * blockIdx.x] = tc::globaltimer();

    // ================================================================ phase 1: shrink
    if (warp == 0) {
        const uint64_t stream = tc::policy_evict_first();
        int stage = 0, pu = -1, row = 0, r0 = 0, nch = 0;
        bool contig = false;
        uint32_t phase = 0;
        for (int k = s0; k < s1; ++k) {
            const int u = k / ncs, g = k - u * ncs;
            if (u != pu) {
                const int4 U = a.units[u];
                nch = U.z;
                row = lane < nch ? a.chunks[U.y + lane].x : 0;
                r0 = __shfl_sync(0xffffffffu, row, 0);
                contig = unit_contiguous(a.chunks, U);
                pu = u;
            }
            const int np = bs.cw[0] / 64, p = g * np;
            const uint32_t bytes = static_cast<uint32_t>(kPps * (nch * kSpChunk * 128 + NS * LS::AP_BYTES));
            for (int pi = 0; pi < np; pi += kPps) {
                if (lane == 0) {
                    tc::mbar_wait(&empty[stage], phase ^ 1u);
                    tc::mbar_expect_tx(&full[stage], bytes);
                }
                __syncwarp();
                const uint32_t st = sbase + stage * LS::STAGE;
                const int rq = __shfl_sync(0xffffffffu, row, lane & 3);
                if (contig) {
                    if (lane < kPps)
                        tc::tma_load_2d_hint(st + lane * LS::PANEL, &maps.x64, (p + pi + lane) * 64, r0, &full[stage],
                                             stream);
                } else if (lane < 4 * kPps) {
                    const int pp = lane >> 2, q = lane & 3;
                    if (q < nch)
                        tc::tma_load_2d_hint(st + pp * LS::PANEL + q * (kSpChunk * 128), &maps.x, (p + pi + pp) * 64,
                                             rq, &full[stage], stream);
                }
                if (++stage == LS::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 6) {
        int stage = 0, pu = -1, slot = 0;
        uint32_t phase = 0;
        const int pp = lane / NS, s = lane - pp * NS;  // lane-parallel box issue
        for (int k = s0; k < s1; ++k) {
            const int u = k / ncs, g = k - u * ncs;
            if (u != pu) {
                slot = a.units[u].x;
                pu = u;
            }
            const int np = bs.cw[0] / 64, p = g * np;
            for (int pi = 0; pi < np; pi += kPps) {
                if (lane == 0) tc::mbar_wait(&empty[stage], phase ^ 1u);
                __syncwarp();
                const uint32_t st = sbase + stage * LS::STAGE;
                if (lane < kPps * NS)
                    tc::tma_load_2d(st + LS::X_BYTES + (pp * NS + s) * LS::AP_BYTES, &maps.A[s], (p + pi + pp) * 64,
                                    slot * R, &full[stage]);
                if (++stage == LS::STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1 || (warp >= 7 && warp <= 9)) {
        const int mw = warp == 1 ? 0 : warp - 6;
        if (lane == 0) {
            const uint32_t id = tc::idesc_bf16_f32(kSpU, LS::NSR);
            int stage = 0, ub = 0, kk = 0;
            uint32_t phase = 0;
            for (int k = s0; k < s1; ++k) {
                const int u = k / ncs;
                const bool first = k == s0 || (k - 1) / ncs != u;
                const bool last = k + 1 == s1 || (k + 1) / ncs != u;
                const int sb = ub & 1;
                const uint32_t dS = tmem + sb * kSpAcc * LS::NSR;
                if (first) {
                    tc::mbar_wait(&s_empty[sb], ((ub >> 1) & 1) ^ 1u);
                    tc::fence_after_sync();
                    kk = 0;
                }
                const int np = bs.cw[0] / 64;
                for (int pi = 0; pi < np; pi += kPps) {
                    tc::mbar_wait(&full[stage], phase);
                    tc::fence_after_sync();
                    const uint32_t st = sbase + stage * LS::STAGE;
#pragma unroll
                    for (int j = mw; j < 4 * kPps; j += kSpAcc) {
                        const int pp = j >> 2, kq = j & 3;
                        tc::mma_bf16(dS + mw * LS::NSR, tc::desc_kmajor_sw128(st + pp * LS::PANEL + kq * 32),
                                     tc::desc_kmajor_sw128(st + LS::X_BYTES + pp * NS * LS::AP_BYTES + kq * 32), id,
                                     kk + j >= kSpAcc ? 1u : 0u);
                    }
                    kk += 4 * kPps;
                    tc::mma_commit(&empty[stage]);
                    if (++stage == LS::STAGES) {
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
    } else if (warp >= 2 && warp <= 5) {
        // TMEM -> this CTA's partial rows of the unit -> every rank's region
        const int q = warp & 3;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        int ub = 0;
        for (int k = s0; k < s1; ++k) {
            const int u = k / ncs;
            if (!(k + 1 == s1 || (k + 1) / ncs != u)) continue;  // once per visit, at its last item
            const int4 U = a.units[u];
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            int plane = 0;
            if (ncs > 1) plane = static_cast<int>(blockIdx.x) - unit_first_cta(cs, bs, u);
            const int sb = ub & 1;
            tc::mbar_wait(&s_full[sb], (ub >> 1) & 1);
            tc::fence_after_sync();
            float s[LS::NSR];
#pragma unroll
            for (int c = 0; c < LS::NSR; ++c) s[c] = 0.f;
#pragma unroll
            for (int acc = 0; acc < kSpAcc; ++acc)
#pragma unroll
                for (int c0 = 0; c0 < LS::NSR; c0 += 16) {
                    uint32_t w[16];
                    tc::tmem_ld16(tmem + lane_base + sb * kSpAcc * LS::NSR + acc * LS::NSR + c0, w);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int c = 0; c < 16; ++c) s[c0 + c] += __uint_as_float(w[c]);
                }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&s_empty[sb]);
            if (lane < ch.y) {
                const long long off = xchg_part_off(par, xa.rank, plane, xa.tp, xa.planes, xa.T_cap) +
                                      static_cast<long long>(ch.x + lane) * 64;
                for (int d = 0; d < xa.tp; ++d) {
                    float* pr = xa.part[d] + off;
#pragma unroll
                    for (int c = 0; c < LS::NSR; c += 4)
                        *reinterpret_cast<float4*>(pr + c) = make_float4(s[c], s[c + 1], s[c + 2], s[c + 3]);
                }
            }
            // publish the piece once all four quadrants' rows are stored
            readout_bar();
            if (warp == 2 && lane < xa.tp) {
                if (!(xa.knobs & 1)) fence_release(sys);
                st_flag(xa.flag[lane] + xchg_flag_off(par, xa.rank, plane, u, xa.tp, xa.planes, xa.U_cap), tag, sys);
            }
            ++ub;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1537 + 2 * blockIdx.x] = tc::globaltimer();

    // ================================================================ phase 2: expand
    {
        ExpandWork W{e0, e1, xa.dyn ? seq.grab : nullptr, xa.grab, a.counters[PREFT_CTR_LORA_UNITS] * nce};
        XchgVSrc vs{xa.part[xa.rank], xa.flag[xa.rank], xa.state, &cs, &bs, xa.tp, xa.planes, xa.T_cap, xa.U_cap,
                    par, tag, sys, xa.spin_ns, 1};
        expand_pipeline<R, NS>(maps, a, be, sbase, sgen, tmem, EB, W, vs);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (a.prof && tid == 0 && blockIdx.x < 128) a.prof[1280 + blockIdx.x] = tc::globaltimer();
    if (tid == 0) launch_seq_end(seqb, seq.n);
    if (warp == 0) {
        __syncwarp();
        tc::tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------- host

bool pdl_enabled();
long long* split_profile_buffer();

long long xchg_region_bytes(int tp, int planes, int T_cap, int U_cap) {
    return 2ll * tp * planes * T_cap * 64 * 4 + 2ll * tp * planes * U_cap * 4 + (16 + kSeqInts) * 4;
}

int xchg_init(preft_xchg_t* xg, void* const* bases, int tp, int rank, int planes, int T_cap, int U_cap, int peer_sys) {
    if (!xg || !bases || tp < 1 || tp > PREFT_XCHG_MAX_TP || rank < 0 || rank >= tp || planes < 1 || planes > kPlanes ||
        T_cap < 1 || U_cap < 1)
        return PREFT_ERR_SHAPE;
    *xg = preft_xchg_t{};
    xg->tp_size = tp;
    xg->tp_rank = rank;
    xg->planes = planes;
    xg->T_cap = T_cap;
    xg->U_cap = U_cap;
    xg->peer_sys = peer_sys ? 1 : 0;
    const long long part_bytes = 2ll * tp * planes * T_cap * 64 * 4;
    const long long flag_bytes = 2ll * tp * planes * U_cap * 4;
    for (int d = 0; d < tp; ++d) {
        if (!bases[d] || (reinterpret_cast<uintptr_t>(bases[d]) & 15u)) return PREFT_ERR_SHAPE;
        unsigned char* b = static_cast<unsigned char*>(bases[d]);
        xg->part[d] = reinterpret_cast<float*>(b);
        xg->flag[d] = reinterpret_cast<int32_t*>(b + part_bytes);
    }
    xg->state = reinterpret_cast<int32_t*>(static_cast<unsigned char*>(bases[rank]) + part_bytes + flag_bytes);
    xg->spin_ns = 2000000000ll;
    return PREFT_OK;
}

static bool al16f(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool lora_fused_ok(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
                   int nsites, int r, int dtype) {
    bool ok = dtype == PREFT_DTYPE_BF16 && (r == 16 || r == 32) && nsites >= 1 && nsites <= 3 && nsites * r <= 64 &&
              m % (64 * kPps) == 0 && ldx % 8 == 0 && al16f(x) && meta && meta->chunks && meta->units;
    for (int s = 0; ok && s < nsites; ++s)
        ok = sites[s].A && al16f(sites[s].A) && sites[s].Bt_tc && al16f(sites[s].Bt_tc) && sites[s].scale &&
             sites[s].y && sites[s].n % kSpN == 0 && sites[s].ldy % 8 == 0 && al16f(sites[s].y);
    return ok;
}

template <int R, int NS>
static int launch_fused(const SplitMaps& maps, const SplitArgs& args, const XchgArgs& xa, int num_sms,
                        cudaStream_t stream) {
    auto kernel = lora_fused_kernel<R, NS>;
    const int smem = FusedLayout<R, NS>::SMEM;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return -static_cast<int>(e);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(num_sms);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kernel, maps, args, xa);
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

int lora_fused(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
               const preft_lora_site_t* sites, int nsites, int r, int dtype, const preft_xchg_t* xg,
               cudaStream_t stream, int num_sms) {
    if (!meta || !x || !sites || !xg || nsites < 1 || nsites > 3 || m < 1 || ldx < m || rows < 1)
        return PREFT_ERR_SHAPE;
    if (r < 1 || r > 64 || (r & (r - 1)) || nsites * r > 64) return PREFT_ERR_RANK;
    if (dtype != PREFT_DTYPE_BF16) return PREFT_ERR_DOMAIN;
    if (!lora_fused_ok(meta, x, ldx, m, sites, nsites, r, dtype)) return PREFT_ERR_SHAPE;
    if (xg->T_cap < meta->T_cap || xg->U_cap < meta->chunk_cap || !xg->state || xg->tp_size < 1 ||
        xg->tp_size > PREFT_XCHG_MAX_TP || xg->planes < 1 || xg->planes > kPlanes)
        return PREFT_ERR_CONFIG;
    SplitArgs args{};
    args.x = x;
    args.ldx = ldx;
    args.m = m;
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
    args.slot_base = meta->slot_split;
    args.tokens = reinterpret_cast<const int2*>(meta->tokens);
    args.chunks = reinterpret_cast<const int2*>(meta->chunks);
    args.units = reinterpret_cast<const int4*>(meta->units);
    args.counters = meta->counters;
    args.prof = split_profile_buffer();
    XchgArgs xa{};
    for (int d = 0; d < xg->tp_size; ++d) {
        xa.part[d] = xg->part[d];
        xa.flag[d] = xg->flag[d];
        if (!xa.part[d] || !xa.flag[d]) return PREFT_ERR_CONFIG;
    }
    xa.state = xg->state;
    xa.tp = xg->tp_size;
    xa.rank = xg->tp_rank;
    xa.planes = xg->planes;
    xa.sys = xg->peer_sys;
    xa.T_cap = xg->T_cap;
    xa.U_cap = xg->U_cap;
    xa.spin_ns = xg->spin_ns > 0 ? xg->spin_ns : 2000000000ll;
    {
        // phase 2's dynamic grabs for the widest groups (>= 64 output blocks per
        // unit: 8B gate/up, step 14.75 -> 13.98 ms, now level with the split
        // pair); at 28 blocks (config-4 gate/up) the grabs meet units whose
        // shrink is still running and lose (12.14 -> 12.75 ms).
        // PREFT_SPLIT_DYN=0/1 forces off/on.
        int blocks = 0;
        for (int s = 0; s < nsites; ++s) blocks += sites[s].n / (sites[s].n % kSpNMax == 0 ? kSpNMax : kSpN);
        const char* e = getenv("PREFT_SPLIT_DYN");
        xa.dyn = e ? (e[0] != '0') : blocks >= 64;
        xa.grab = blocks >= 64 ? 8 : 4;
    }
    xa.beta_s = kBetaS;
    xa.beta_e = kBetaE;
    if (const char* e = getenv("PREFT_FUSED_BETA_S")) xa.beta_s = atoi(e);
    if (const char* e = getenv("PREFT_FUSED_BETA_E")) xa.beta_e = atoi(e);
    if (const char* e = getenv("PREFT_FUSED_KNOBS")) xa.knobs = atoi(e);
    // the planes K-split needs whole 4-panel blocks
    if (xa.planes > 1 && (m / 64) % kPps) xa.planes = 1;
    SplitMaps maps{};
    if (!make_tmap_bf16_sw128(&maps.x, x, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(m),
                              static_cast<unsigned long long>(ldx), 64, kSpChunk) ||
        !make_tmap_bf16_sw128(&maps.x64, x, static_cast<unsigned long long>(rows), static_cast<unsigned long long>(m),
                              static_cast<unsigned long long>(ldx), 64, kSpU))
        return PREFT_ERR_CONFIG;
    for (int s = 0; s < nsites; ++s) {
        if (!make_tmap_bf16_sw128(&maps.A[s], sites[s].A, 1ull << 20, static_cast<unsigned long long>(m),
                                  static_cast<unsigned long long>(m), 64, static_cast<unsigned>(r)))
            return PREFT_ERR_CONFIG;
        const unsigned npan = (sites[s].n % kSpNMax == 0 ? kSpNMax : kSpN) / 64;
        if (!make_tmap_bf16_panels(&maps.y[s], sites[s].y, static_cast<unsigned long long>(rows),
                                   static_cast<unsigned long long>(sites[s].n),
                                   static_cast<unsigned long long>(sites[s].ldy), kSpChunk, npan))
            return PREFT_ERR_CONFIG;
    }
    if (xg->grid > 0) num_sms = xg->grid;
    if (r == 16) {
        if (nsites == 1) return launch_fused<16, 1>(maps, args, xa, num_sms, stream);
        if (nsites == 2) return launch_fused<16, 2>(maps, args, xa, num_sms, stream);
        return launch_fused<16, 3>(maps, args, xa, num_sms, stream);
    }
    if (nsites == 1) return launch_fused<32, 1>(maps, args, xa, num_sms, stream);
    if (nsites == 2) return launch_fused<32, 2>(maps, args, xa, num_sms, stream);
    return PREFT_ERR_RANK;
}

int xchg_errors(const preft_xchg_t* xg, cudaStream_t stream, int* out) {
    if (!xg || !xg->state || !out) return PREFT_ERR_SHAPE;
    int v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, xg->state + 2, sizeof(int), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return -static_cast<int>(e);
    *out = v;
    return PREFT_OK;
}

}  // namespace preft
