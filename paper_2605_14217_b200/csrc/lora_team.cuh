// K2 "team" variant: a team of TEAM warps (1, 2, 4 or 8) owns one token row
// at a time; a 256-thread CTA runs 8/TEAM teams side by side.
//
// Why teams: the row widths of one transformer layer differ by 14x (k/v
// 1024, q/o 4096, gate/up 14336), and a memory-bound row kernel wants every
// thread to have a full batch of 128-bit loads in flight for ONE row, with
// enough rows per SM to cover the memory latency.  A team sized to the row
// (host heuristic: ~16 vectors per thread for the wider phase) gives each
// thread one batch of loads for the whole row — gate/up: 8 warps x 14 loads;
// q/k/v: 2 warps, 4 rows per CTA — instead of a warp walking a wide row in
// dependent batches (the warp kernel) or 8 warps sharing a narrow row.
//
// Per row: shrink (x chunks x A chunks, fp32 FMA), warp-shuffle reduction,
// cross-warp reduction through shared memory behind a named barrier per team
// (bar.sync 1+team, TEAM*32), then expand (y chunks += v . Bt chunks).  Loads
// are issued unconditionally from clamped in-bounds addresses; only the
// stores are predicated, so the compiler keeps a whole batch in flight.
// Teams take balanced contiguous runs of the slot-sorted tokens (neighbouring
// teams = same CTA = same SM share an adapter's A/Bt chunks through L1).
// Included from lora.cu inside namespace preft (uses LoraArgs).

constexpr int kTeamCtaThreads = 256;
constexpr int kTeamCtaWarps = kTeamCtaThreads / 32;

template <int TEAM>
__device__ __forceinline__ void team_barrier(int team) {
    if constexpr (TEAM == 1) {
        __syncwarp();
    } else if constexpr (TEAM == kTeamCtaWarps) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TEAM * 32) : "memory");
    }
}

template <typename T, int R, int NS, int U, int TEAM, int MINB = 2>
__global__ void __launch_bounds__(kTeamCtaThreads, MINB) lora_team_kernel(const LoraArgs a) {
    using V = Vec<T, true>;
    using acc_t = typename V::acc_t;
    constexpr int W = V::W;
    constexpr int NR = NS * R;
    constexpr int TT = TEAM * 32;  // threads per team
    constexpr int TEAMS = kTeamCtaWarps / TEAM;
    __shared__ acc_t red[kTeamCtaWarps][NR];
    __shared__ acc_t vsh[TEAMS][NR];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int team = warp / TEAM, tt = threadIdx.x % TT;
    pdl_begin();  // programmatic dependent launch: wait for the previous kernel's writes
    const int n_tok = a.counters[PREFT_CTR_SPLIT];
    int i0, i1;
    even_share(n_tok, blockIdx.x * TEAMS + team, gridDim.x * TEAMS, i0, i1);
    const T* __restrict__ x = static_cast<const T*>(a.x);
    const int mv = a.m / W;

    for (int i = i0; i < i1; ++i) {
        const int2 ts = a.tokens[i];
        const T* __restrict__ xr = x + static_cast<long long>(ts.x) * a.ldx;
        // multi-warp teams (small batches, one row per team: latency-bound) load
        // the row's scale and bias with the x batch, not after the reduction —
        // one dependent round trip fewer (Punica step 567k -> 587k tokens/s).
        // Single-warp teams keep the late load: the two registers per site held
        // across the shrink cost the big-batch groups ~0.2%.
        acc_t sc[NS], bi[NS][R];
        if constexpr (TEAM >= 2) {
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                sc[s] = __ldg(static_cast<const acc_t*>(a.site[s].scale) + ts.y);
                const acc_t* bias = static_cast<const acc_t*>(a.site[s].bias);
#pragma unroll
                for (int k = 0; k < R; ++k)
                    bi[s][k] = bias ? __ldg(bias + static_cast<long long>(ts.y) * R + k) : acc_t(0);
            }
        }
        acc_t acc[NS][R];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int k = 0; k < R; ++k) acc[s][k] = acc_t(0);

        // ---- shrink
        for (int c0 = tt; c0 < mv; c0 += TT * U) {
            typename V::raw_t xv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = min(c0 + TT * u, mv - 1);
                xv[u] = V::ld_stream(xr + static_cast<long long>(c) * W);
            }
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const T* As = static_cast<const T*>(a.site[s].A) + (static_cast<long long>(ts.y) * R) * a.m;
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    typename V::raw_t av[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int c = min(c0 + TT * u, mv - 1);
                        av[u] = V::ld_weight(As + static_cast<long long>(k) * a.m + static_cast<long long>(c) * W);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        // branch-free: a clamped (duplicate) vector past the row end
                        // contributes x = 0.  A branch here let the compiler sink each
                        // u's x load into its branch, serialising the batch's round trips
                        const bool ok = c0 + TT * u < mv;
                        acc_t xf[W], af[W];
                        V::to_acc(xv[u], xf);
                        V::to_acc(av[u], af);
#pragma unroll
                        for (int j = 0; j < W; ++j) acc[s][k] = macc(ok ? xf[j] : acc_t(0), af[j], acc[s][k]);
                    }
                }
            }
        }

        // ---- reduce over the team: shuffle, then shared memory
        acc_t v[NR];
        if constexpr (TEAM == 1) {
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    acc_t t = warp_sum(acc[s][k]);
                    const acc_t* bias = static_cast<const acc_t*>(a.site[s].bias);
                    if (bias) t += __ldg(bias + static_cast<long long>(ts.y) * R + k);
                    v[s * R + k] = t * __ldg(static_cast<const acc_t*>(a.site[s].scale) + ts.y);
                }
        } else {
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int k = 0; k < R; ++k) {
                    const acc_t t = warp_sum(acc[s][k]);
                    if (lane == 0) red[warp][s * R + k] = t;
                }
            team_barrier<TEAM>(team);
            if (tt < NR) {
                acc_t t = acc_t(0);
#pragma unroll
                for (int w = 0; w < TEAM; ++w) t += red[team * TEAM + w][tt];
                acc_t b_ = acc_t(0), s_ = acc_t(0);
#pragma unroll
                for (int q = 0; q < NS; ++q)
#pragma unroll
                    for (int kk = 0; kk < R; ++kk)
                        if (q * R + kk == tt) b_ = bi[q][kk], s_ = sc[q];
                vsh[team][tt] = (t + b_) * s_;
            }
            team_barrier<TEAM>(team);
#pragma unroll
            for (int q = 0; q < NR; ++q) v[q] = vsh[team][q];
        }

        // ---- expand
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            const int n = a.site[s].n;
            const int nv = n / W;
            T* __restrict__ yr = static_cast<T*>(a.site[s].y) + static_cast<long long>(ts.x) * a.site[s].ldy;
            const T* Bs = static_cast<const T*>(a.site[s].Bt) + (static_cast<long long>(ts.y) * R) * n;
            for (int c0 = tt; c0 < nv; c0 += TT * U) {
                typename V::raw_t yv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = min(c0 + TT * u, nv - 1);
                    yv[u] = V::ld_rw(yr + static_cast<long long>(c) * W);
                }
                if constexpr (R == 1) {
                    typename V::raw_t bv[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int c = min(c0 + TT * u, nv - 1);
                        bv[u] = V::ld_weight(Bs + static_cast<long long>(c) * W);
                    }
                    // every u's update before any (predicated) store, so no load is
                    // sunk behind a store branch
                    acc_t yf[U][W];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc_t bf[W];
                        V::to_acc(yv[u], yf[u]);
                        V::to_acc(bv[u], bf);
#pragma unroll
                        for (int j = 0; j < W; ++j) yf[u][j] = macc(v[s], bf[j], yf[u][j]);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int c = c0 + TT * u;
                        if (c < nv) V::st(yr + static_cast<long long>(c) * W, yf[u]);
                    }
                } else {
                    acc_t d[U][W];
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int j = 0; j < W; ++j) d[u][j] = acc_t(0);
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        typename V::raw_t bv[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            const int c = min(c0 + TT * u, nv - 1);
                            bv[u] = V::ld_weight(Bs + static_cast<long long>(k) * n + static_cast<long long>(c) * W);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            acc_t bf[W];
                            V::to_acc(bv[u], bf);
#pragma unroll
                            for (int j = 0; j < W; ++j) d[u][j] = macc(v[s * R + k], bf[j], d[u][j]);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        acc_t yf[W];
                        V::to_acc(yv[u], yf);  // outside the store branch: keeps the y load in the batch
#pragma unroll
                        for (int j = 0; j < W; ++j) d[u][j] += yf[j];
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int c = c0 + TT * u;
                        if (c < nv) V::st(yr + static_cast<long long>(c) * W, d[u]);
                    }
                }
            }
        }
        // no trailing barrier: the next row writes red[] only for its own warp
        // and vsh[] only after its first barrier, which every reader of this
        // row's vsh[] must pass first
    }
}

// single-warp teams: (unroll, min CTAs/SM) configurations, PREFT_LORA_T1CFG
// selects one for A/B measurement (0 = default)
// Measured (tools/kbench.py, cfg2 batch, L2 flushed): fused 2-3 site groups
// prefer U=4 at 3 CTAs/SM, single sites U=8 at 3 CTAs/SM.
template <typename T, int R, int NS>
void* pick_team1(int cfg) {
    constexpr int U = R == 1 ? 8 : 4;
    if (cfg == 0) cfg = NS > 1 ? 1 : 3;
    switch (cfg) {
        case 1: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, 4, 1, 3>);
        case 2: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, 4, 1, 4>);
        case 3: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, U, 1, 3>);
        default: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, U, 1, 2>);
    }
}

inline int team1_cfg() {
    const char* e = getenv("PREFT_LORA_T1CFG");
    return e ? (e[0] - '0') : 0;
}

template <typename T, int R, int NS>
void* pick_team_size(int team) {
    constexpr int U = R == 1 ? 8 : 4;
    switch (team) {
        case 1: return pick_team1<T, R, NS>(team1_cfg());
        case 2: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, U, 2>);
        case 4: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, U, 4>);
        case 8: return reinterpret_cast<void*>(lora_team_kernel<T, R, NS, U, 8>);
        default: return nullptr;
    }
}

template <typename T>
void* pick_lora_team(int nsites, int r, int team) {
    switch (nsites * 8 + r) {
        case 8 + 1: return pick_team_size<T, 1, 1>(team);
        case 8 + 2: return pick_team_size<T, 2, 1>(team);
        case 8 + 4: return pick_team_size<T, 4, 1>(team);
        case 16 + 1: return pick_team_size<T, 1, 2>(team);
        case 16 + 2: return pick_team_size<T, 2, 2>(team);
        case 16 + 4: return pick_team_size<T, 4, 2>(team);
        case 24 + 1: return pick_team_size<T, 1, 3>(team);
        case 24 + 2: return pick_team_size<T, 2, 3>(team);
        case 24 + 4: return pick_team_size<T, 4, 3>(team);
        default: return nullptr;
    }
}

// Warps per team from the expected row count (meta->rows_hint, host-known).
// Measured on B200 (tools/kbench.py, profiles/): with thousands of rows one
// warp per row wins for every Llama-3.1-8B site group (wider teams only add
// barrier latency); with few rows (a Punica-sized step, ~850 tokens) there
// are too few warps to cover memory latency and 2-warp teams win.  Aim for
// about half the resident warps (SMs x 16) busy.
inline int auto_team_warps(int rows_hint, int num_sms) {
    if (rows_hint <= 0) return 1;
    const int target = num_sms * 8;
    int team = 1;
    while (team < 8 && rows_hint * team < target) team *= 2;
    return team;
}
