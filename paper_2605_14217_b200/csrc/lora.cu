// K2 — fused segmented-gather LoRA^P for sm_100a (SIMT path, rank <= 64).
//
// For every selected token t (adapter slot a) and every site s of a group of
// sites that share the input x (q/k/v or gate/up or a single projection):
//
//     y_s[t, :] += scale_s[a] * (x[t, :] . A_s[a]^T) . Bt_s[a]
//
// which is the reference's  out[rows] += s * ((X A^T) B^T)   (model.py:449-451,
// adapters.py:284-288) with the scalar folded onto the rank-r intermediate.
// An optional per-slot bias b (added before the scale) makes the same kernel
// compute the ReFT delta s * ((H A^T + b) B) into a separate output
// (adapters.py:292-295), which the out-of-place drop-in delta_for_rows uses.
//
// Mapping (HBM-bound for every rank this path is used at):
//   - one warp owns one token row at a time: the shrink streams x[t,:] with
//     128-bit loads (U loads in flight per lane), the rank-r partial sums stay
//     in registers and are reduced with warp shuffles, the expand streams
//     y_s[t,:] read-modify-write with 128-bit accesses — no shared memory, no
//     block barrier, no atomics, deterministic;
//   - warps take contiguous, balanced runs of the slot-sorted token list built
//     by K1, so neighbouring warps (same CTA, same SM) work on the same
//     adapter and its A/Bt rows are served from L1 after the first touch;
//   - the grid is persistent (a multiple of the SM count) and reads the token
//     count from device memory, so the launch is CUDA-graph safe.
// Unselected tokens are never touched, so their rows stay bit-identical.
#include "common.cuh"

namespace preft {

struct LoraSiteDev {
    const void* A;
    const void* Bt;
    const void* scale;
    const void* bias;
    void* y;
    long long ldy;
    int n;
    int pad;
};

struct LoraArgs {
    const void* x;
    long long ldx;
    int m;
    int nsites;
    LoraSiteDev site[3];
    const int2* tokens;
    const int* counters;
};

template <typename T, bool VEC, int R, int NS, int U>
__global__ void __launch_bounds__(256) lora_kernel(const LoraArgs a) {
    using V = Vec<T, VEC>;
    using acc_t = typename V::acc_t;
    constexpr int W = V::W;
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    pdl_begin();  // programmatic dependent launch: wait for the previous kernel's writes
    const int n_tok = a.counters[PREFT_CTR_SPLIT];  // LoRA-class tokens: sorted [0, split)
    int i0, i1;
    even_share(n_tok, gw, nw, i0, i1);

    const T* __restrict__ x = static_cast<const T*>(a.x);
    const int mv = a.m / W;

    for (int i = i0; i < i1; ++i) {
        const int2 ts = a.tokens[i];  // (token row, adapter slot)
        const T* __restrict__ xr = x + static_cast<long long>(ts.x) * a.ldx;

        acc_t acc[NS][R];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) acc[s][k] = acc_t(0);

        // ---- shrink: acc[s][k] = x[t,:] . A_s[a][k,:]
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
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const acc_t sc = __ldg(static_cast<const acc_t*>(a.site[s].scale) + ts.y);
            const acc_t* bias = static_cast<const acc_t*>(a.site[s].bias);
#pragma unroll
            for (int k = 0; k < R; ++k) {
                acc_t v = warp_sum(acc[s][k]);
                if (bias) v += __ldg(bias + static_cast<long long>(ts.y) * R + k);
                acc[s][k] = v * sc;
            }
        }

        // ---- expand: y_s[t,:] += sum_k acc[s][k] * Bt_s[a][k,:]
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int n = a.site[s].n;
            const int nv = n / W;
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
                            V::to_acc(V::ld_weight(Bs + static_cast<long long>(k) * n + static_cast<long long>(c) * W),
                                      bf);
#pragma unroll
                            for (int j = 0; j < W; ++j) d[j] = macc(acc[s][k], bf[j], d[j]);
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

#include "lora_team.cuh"

// ------------------------------------------------------------------ dispatch

using LoraFn = void (*)(LoraArgs);

template <typename T, bool VEC, int NS>
LoraFn pick_rank(int r) {
    constexpr int U = VEC ? 8 : 4;
    switch (r) {
        case 1: return lora_kernel<T, VEC, 1, NS, U>;
        case 2: return lora_kernel<T, VEC, 2, NS, U>;
        case 4: return lora_kernel<T, VEC, 4, NS, U>;
        case 8: return lora_kernel<T, VEC, 8, NS, U>;
        case 16: return lora_kernel<T, VEC, 16, NS, U>;
        case 32: if constexpr (NS <= 2) return lora_kernel<T, VEC, 32, NS, U>; else return nullptr;
        case 64: if constexpr (NS == 1) return lora_kernel<T, VEC, 64, NS, 4>; else return nullptr;
        default: return nullptr;
    }
}

template <typename T>
LoraFn pick_lora(bool vec, int nsites, int r) {
    if (vec) {
        if (nsites == 1) return pick_rank<T, true, 1>(r);
        if constexpr (!std::is_same<T, double>::value) {
            if (nsites == 2) return pick_rank<T, true, 2>(r);
            if (nsites == 3) return pick_rank<T, true, 3>(r);
        }
        return nullptr;
    }
    return nsites == 1 ? pick_rank<T, false, 1>(r) : nullptr;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// -1 = automatic, 0 = warp-per-row only, 1 = CTA-per-row where eligible
static int g_lora_variant = -2;
int lora_variant() {
    if (g_lora_variant == -2) {
        const char* env = getenv("PREFT_LORA_VARIANT");
        g_lora_variant = -1;
        if (env && env[0] == 'w') g_lora_variant = 0;
        if (env && (env[0] == '1' || env[0] == '2' || env[0] == '4' || env[0] == '8')) g_lora_variant = env[0] - '0';
    }
    return g_lora_variant;
}
void set_lora_variant(int v) { g_lora_variant = v; }

int grid_for(const void* fn, int threads, int num_sms);
bool pdl_enabled();
bool lora_tc_route_ok(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
                      int nsites, int r, int dtype);
int lora_shrink(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
                const preft_lora_site_t* sites, int nsites, int r, int dtype, void* P, long long ldp,
                cudaStream_t stream, int num_sms);
int lora_expand(const preft_meta_t* meta, const void* P, long long ldp, long long rows, const preft_lora_site_t* sites,
                int nsites, int r, int dtype, cudaStream_t stream, int num_sms);
long long lora_split_floats(const preft_meta_t* meta);
long long lora_part_floats_needed(const preft_meta_t* meta);
int xchg_init(preft_xchg_t* xg, void* const* bases, int tp, int rank, int planes, int T_cap, int U_cap, int peer_sys);
bool lora_fused_ok(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
                   int nsites, int r, int dtype);
int lora_fused(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
               const preft_lora_site_t* sites, int nsites, int r, int dtype, const preft_xchg_t* xg,
               cudaStream_t stream, int num_sms);

// fused shrink -> expand (one launch, lora_fused.cu) for the r >= 16 route
// where it measured faster: inputs of >= 4096 columns (the 8B r16 step 14.58
// -> 13.81 ms, bench lora16 line).  On narrow inputs (config-4 shards: m =
// 1024) the split pair is faster.  PREFT_LORA_FUSED=0/1 forces off/on.
// The fused kernel (one launch: shrink -> one-rank exchange -> expand) for
// inputs of >= 8192 columns, the split pair below that.  Measured at the 8B
// r16 step (tools/split_breakdown.py --shape 8b --tp 1 --fused 1, r02h):
// split / fused q/k/v (m 4096) 2.36 / 2.44 ms, o 1.61 / 1.60, gate/up 6.59 /
// 6.61, down (m 14336) 3.22 / 3.07.  PREFT_LORA_FUSED=0/1 forces either
// route, PREFT_LORA_FUSED_MIN_M moves the threshold.
static bool lora_fused_wanted(int m) {
    static int on = -2, min_m = 8192;
    if (on == -2) {
        const char* e = getenv("PREFT_LORA_FUSED");
        on = e ? (e[0] == '1' ? 1 : 0) : -1;
        if (const char* t = getenv("PREFT_LORA_FUSED_MIN_M")) min_m = atoi(t);
    }
    return on == 1 || (on == -1 && m >= min_m);
}

int lora_apply(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
               int nsites, int r, int dtype, cudaStream_t stream, int num_sms) {
    if (!meta || !x || !sites || nsites < 1 || nsites > 3 || m < 1 || ldx < m) return PREFT_ERR_SHAPE;
    if (r < 1 || r > 64 || (r & (r - 1)) || nsites * r > 64) return PREFT_ERR_RANK;
    if (dtype != PREFT_DTYPE_F32 && dtype != PREFT_DTYPE_BF16 && dtype != PREFT_DTYPE_F64) return PREFT_ERR_DOMAIN;
    const int W = dtype == PREFT_DTYPE_BF16 ? 8 : dtype == PREFT_DTYPE_F32 ? 4 : 2;
    bool vec = (m % W == 0) && (ldx % W == 0) && aligned16(x);
    for (int s = 0; s < nsites; ++s) {
        const preft_lora_site_t& st = sites[s];
        if (!st.A || !st.Bt || !st.scale || !st.y || st.n < 1 || st.ldy < st.n) return PREFT_ERR_SHAPE;
        vec = vec && (st.n % W == 0) && (st.ldy % W == 0) && aligned16(st.y) && aligned16(st.A) && aligned16(st.Bt);
    }
    // r >= 16 (bf16): ~10 FLOP/B at r = 16, beyond SIMT FP32 at the HBM
    // roofline, so the delta goes through the tcgen05 split pair with the
    // rank-r intermediate in the meta's workspace (T x nsites x r f32, stays
    // in L2 between the two launches).  Both kernels only touch rows of the
    // K1 units, so the TMA bound T_cap never exposes rows beyond the batch.
    if (lora_variant() != 0 && lora_fused_wanted(m) && meta->lora_part &&
        meta->lora_part_floats >= lora_part_floats_needed(meta) && lora_fused_ok(meta, x, ldx, m, sites, nsites, r, dtype)) {
        // one rank: the exchange region is the tail of the meta's workspace
        preft_xchg_t xg;
        void* base = meta->lora_part + lora_split_floats(meta);
        const int rc = xchg_init(&xg, &base, 1, 0, 1, meta->T_cap, meta->chunk_cap, 0);
        if (rc) return rc;
        return lora_fused(meta, x, meta->T_cap, ldx, m, sites, nsites, r, dtype, &xg, stream, num_sms);
    }
    if (lora_variant() != 0 && lora_tc_route_ok(meta, x, ldx, m, sites, nsites, r, dtype)) {
        const long long ldp = static_cast<long long>(nsites) * r;
        int rc = lora_shrink(meta, x, meta->T_cap, ldx, m, sites, nsites, r, dtype, meta->lora_part, ldp, stream,
                             num_sms);
        if (rc) return rc;
        return lora_expand(meta, meta->lora_part, ldp, meta->T_cap, sites, nsites, r, dtype, stream, num_sms);
    }
    if ((!vec || dtype == PREFT_DTYPE_F64) && nsites > 1) {  // one launch per site
        for (int s = 0; s < nsites; ++s) {
            const int rc = lora_apply(meta, x, ldx, m, sites + s, 1, r, dtype, stream, num_sms);
            if (rc) return rc;
        }
        return PREFT_OK;
    }
    LoraArgs args{};
    args.x = x;
    args.ldx = ldx;
    args.m = m;
    args.nsites = nsites;
    for (int s = 0; s < nsites; ++s) {
        args.site[s].A = sites[s].A;
        args.site[s].Bt = sites[s].Bt;
        args.site[s].scale = sites[s].scale;
        args.site[s].bias = sites[s].bias;
        args.site[s].y = sites[s].y;
        args.site[s].ldy = sites[s].ldy;
        args.site[s].n = sites[s].n;
    }
    args.tokens = reinterpret_cast<const int2*>(meta->tokens);
    args.counters = meta->counters;
    // variant: team kernel (lora_team.cuh) for aligned rank<=4 bf16/f32 rows,
    // team size from the row widths unless forced (preft_set_lora_variant:
    // 0 = warp kernel above, 1/2/4/8 = team warps; PREFT_LORA_VARIANT env)
    const int variant = lora_variant();
    LoraFn fn = nullptr;
    if (variant != 0 && vec && r <= 4 && dtype != PREFT_DTYPE_F64) {
        int nvt = 0;
        for (int s = 0; s < nsites; ++s) nvt += sites[s].n / W;
        (void)nvt;
        const int team = variant > 0 ? variant : auto_team_warps(meta->rows_hint, num_sms);
        fn = reinterpret_cast<LoraFn>(dtype == PREFT_DTYPE_BF16 ? pick_lora_team<__nv_bfloat16>(nsites, r, team)
                                                                : pick_lora_team<float>(nsites, r, team));
    }
    if (!fn)
        fn = dtype == PREFT_DTYPE_BF16  ? pick_lora<__nv_bfloat16>(vec, nsites, r)
             : dtype == PREFT_DTYPE_F32 ? pick_lora<float>(vec, nsites, r)
                                        : pick_lora<double>(vec, nsites, r);
    if (!fn) return PREFT_ERR_RANK;
    const int grid = grid_for(reinterpret_cast<const void*>(fn), 256, num_sms);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, fn, args);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
