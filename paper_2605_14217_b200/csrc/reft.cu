// K3 — fused ReFT^P residual edit for sm_100a (SIMT path, rank <= 64).
//
// For every selected token t (adapter slot a):
//
//     h[t, :] += scale[a] * ((h[t, :] . A[a]^T + b[a]) . B[a])
//
//   DiReFT: A, B, b exactly as the reference stores them       (adapters.py:292-293)
//   LoReFT: A := W - R (folded in f64 at registration), B := R  (adapters.py:294-295)
//
// One warp per token row.  When the row fits in registers (KEEP vectors per
// lane, e.g. d = 4096 in bf16 -> 16 x 128-bit per lane) it is loaded once,
// used for the shrink and updated in registers for the expand, so h moves
// HBM->SM->HBM exactly once — the algorithmic minimum 2*d*e bytes per token.
// Wider rows re-read h for the expand (an L1/L2 hit in practice).
#include <mutex>

#include "common.cuh"

namespace preft {

struct ReftArgs {
    void* h;
    long long ldh;
    int d;
    int slot_base;
    const void* A;
    const void* B;
    const void* bias;
    const void* scale;
    const int2* tokens;
    const int* counters;
};

template <typename T, bool VEC, int R, int U, int KEEP>
__global__ void __launch_bounds__(256) reft_kernel(const ReftArgs a) {
    using V = Vec<T, VEC>;
    using acc_t = typename V::acc_t;
    constexpr int W = V::W;
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    // ReFT-class tokens: sorted positions [split, n_selected), slots >= slot_base
    const int lo = a.counters[PREFT_CTR_SPLIT];
    int i0, i1;
    even_share(a.counters[PREFT_CTR_SEL_TOKENS] - lo, gw, nw, i0, i1);
    const int dv = a.d / W;
    const long long d = a.d;

    for (int i = lo + i0; i < lo + i1; ++i) {
        int2 ts = a.tokens[i];
        ts.y -= a.slot_base;
        T* __restrict__ hr = static_cast<T*>(a.h) + static_cast<long long>(ts.x) * a.ldh;
        const T* As = static_cast<const T*>(a.A) + (static_cast<long long>(ts.y) * R) * d;
        const T* Bs = static_cast<const T*>(a.B) + (static_cast<long long>(ts.y) * R) * d;
        const acc_t sc = __ldg(static_cast<const acc_t*>(a.scale) + ts.y);
        const acc_t* bb = static_cast<const acc_t*>(a.bias) + static_cast<long long>(ts.y) * R;

        acc_t acc[R];
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = acc_t(0);

        if constexpr (KEEP > 0) {
            // whole row resident in registers: dv <= 32 * KEEP (checked by the host)
            typename V::raw_t hv[KEEP];
#pragma unroll
            for (int u = 0; u < KEEP; ++u) {
                const int c = lane + kWarp * u;
                hv[u] = c < dv ? V::ld_rw(hr + static_cast<long long>(c) * W) : V::zero();
            }
#pragma unroll
            for (int u = 0; u < KEEP; ++u) {
                const int c = lane + kWarp * u;
                if (c < dv) {
                    acc_t hf[W];
                    V::to_acc(hv[u], hf);
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        acc_t af[W];
                        V::to_acc(V::ld_weight(As + k * d + static_cast<long long>(c) * W), af);
#pragma unroll
                        for (int j = 0; j < W; ++j) acc[k] = macc(hf[j], af[j], acc[k]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k] = (warp_sum(acc[k]) + __ldg(bb + k)) * sc;
#pragma unroll
            for (int u = 0; u < KEEP; ++u) {
                const int c = lane + kWarp * u;
                if (c < dv) {
                    acc_t hf[W], dl[W];
                    V::to_acc(hv[u], hf);
#pragma unroll
                    for (int j = 0; j < W; ++j) dl[j] = acc_t(0);
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        acc_t bf[W];
                        V::to_acc(V::ld_weight(Bs + k * d + static_cast<long long>(c) * W), bf);
#pragma unroll
                        for (int j = 0; j < W; ++j) dl[j] = macc(acc[k], bf[j], dl[j]);
                    }
#pragma unroll
                    for (int j = 0; j < W; ++j) hf[j] += dl[j];
                    V::st(hr + static_cast<long long>(c) * W, hf);
                }
            }
        } else {
            for (int c0 = lane; c0 < dv; c0 += kWarp * U) {
                typename V::raw_t hv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    hv[u] = c < dv ? V::ld_rw(hr + static_cast<long long>(c) * W) : V::zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    if (c < dv) {
                        acc_t hf[W];
                        V::to_acc(hv[u], hf);
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            acc_t af[W];
                            V::to_acc(V::ld_weight(As + k * d + static_cast<long long>(c) * W), af);
#pragma unroll
                            for (int j = 0; j < W; ++j) acc[k] = macc(hf[j], af[j], acc[k]);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) acc[k] = (warp_sum(acc[k]) + __ldg(bb + k)) * sc;
            for (int c0 = lane; c0 < dv; c0 += kWarp * U) {
                typename V::raw_t hv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    hv[u] = c < dv ? V::ld_rw(hr + static_cast<long long>(c) * W) : V::zero();
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int c = c0 + kWarp * u;
                    if (c < dv) {
                        acc_t hf[W], dl[W];
                        V::to_acc(hv[u], hf);
#pragma unroll
                        for (int j = 0; j < W; ++j) dl[j] = acc_t(0);
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            acc_t bf[W];
                            V::to_acc(V::ld_weight(Bs + k * d + static_cast<long long>(c) * W), bf);
#pragma unroll
                            for (int j = 0; j < W; ++j) dl[j] = macc(acc[k], bf[j], dl[j]);
                        }
#pragma unroll
                        for (int j = 0; j < W; ++j) hf[j] += dl[j];
                        V::st(hr + static_cast<long long>(c) * W, hf);
                    }
                }
            }
        }
    }
}

using ReftFn = void (*)(ReftArgs);

template <typename T, bool VEC, int KEEP>
ReftFn pick_reft_rank(int r) {
    constexpr int U = VEC ? 8 : 4;
    switch (r) {
        case 1: return reft_kernel<T, VEC, 1, U, KEEP>;
        case 2: return reft_kernel<T, VEC, 2, U, KEEP>;
        case 4: return reft_kernel<T, VEC, 4, U, KEEP>;
        case 8: return reft_kernel<T, VEC, 8, U, KEEP>;
        case 16: return reft_kernel<T, VEC, 16, U, KEEP>;
        case 32: return reft_kernel<T, VEC, 32, U, KEEP>;
        case 64: if constexpr (KEEP == 0) return reft_kernel<T, VEC, 64, 4, 0>; else return nullptr;
        default: return nullptr;
    }
}

static bool aligned16r(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(const void* fn, int threads, int num_sms);

int reft_tc_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A, const void* Bt,
                  const void* bias, const void* scale, int r, cudaStream_t stream, int num_sms, int part_lo,
                  int part_hi);
int reft_res_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A,
                   const void* Bt, const void* bias, const void* scale, int r, cudaStream_t stream, int num_sms,
                   int part_lo, int part_hi, bool dry);
bool reft_res_preferred(int d, int r);
bool reft_res_eligible(int d, int r);

// Co-launch (d = 4096): clusters of d/1024 CTAs for the TMEM-parked kernel
// pack only ~132 of the 148 SMs, so the streaming kernel runs on the SMs left
// over, on a forked stream, over the last part of the unit list (the units
// split in proportion to the two kernels' per-SM rates).  Env
// PREFT_REFT_COLAUNCH=0 disables, PREFT_REFT_COSPLIT=<fraction*4096 for the
// parked kernel> overrides the split.
struct CoStreams {
    int device = -1;
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
static CoStreams g_co[16];
// held from the fork record to the join wait: two host threads co-launching
// (on any streams) cannot interleave record(fork) / wait(aux, fork), so each
// aux half always waits for its own caller stream's prior work.  One pair per
// device (created at the first eager co-launch) keeps a later capture on any
// stream able to fork.
static std::mutex g_co_mu;

static CoStreams* co_streams_locked(cudaStream_t stream) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
    CoStreams& c = g_co[dev];
    if (c.device < 0) {
        // creating streams/events is not allowed while a capture is open: the
        // first co-launch must run eagerly (a warm-up); until then, one kernel
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
        if (cudaStreamCreateWithFlags(&c.aux, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        if (cudaEventCreateWithFlags(&c.join, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        c.device = dev;
    }
    return &c;
}

static int colaunch_split() {
    static int v = -2;
    if (v == -2) {
        const char* off = getenv("PREFT_REFT_COLAUNCH");
        const char* sp = getenv("PREFT_REFT_COSPLIT");
        v = (off && off[0] == '0') ? -1 : sp ? atoi(sp) : 0;
    }
    return v;  // -1 off, 0 automatic, else the parked kernel's share in 1/4096
}

static int reft_colaunch(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A,
                         const void* Bt, const void* bias, const void* scale, int r, cudaStream_t stream,
                         int num_sms) {
    const int sp = colaunch_split();
    // measured win at clusters of 4 (d = 4096, r = 16: 68% vs 65%); clusters of 8 run the
    // parked kernel at 54% and would drag the pair down
    if (sp < 0 || !reft_res_eligible(d, r) || d / 1024 != 4) return PREFT_ERR_SHAPE;
    const int g = reft_res_apply(meta, h, rows, ldh, d, A, Bt, bias, scale, r, stream, num_sms, 0, 4096, true);
    const int left = num_sms - g;  // (a dry run returns the grid; error codes are < 32)
    if (g < 32 || left < 2) return PREFT_ERR_SHAPE;
    std::lock_guard<std::mutex> lk(g_co_mu);
    CoStreams* c = co_streams_locked(stream);
    if (!c) return PREFT_ERR_SHAPE;
    // units split in proportion to the kernels' per-SM rates: swept at
    // config 3 (profiles/reft_cosplit_r02c.txt) the best share of the parked
    // kernel is 88.5-89% (rate ~0.97x the streaming kernel's per SM; 71.1%
    // of HBM peak vs 68.8% at the old 1.2x guess); the optimum is sharp
    // (+-1.5% of the units costs 2-6 points)
    const int f = sp > 0 ? min(4095, sp) : static_cast<int>(4096.0 * 0.97 * g / (0.97 * g + left));
    if (cudaEventRecord(c->fork, stream) != cudaSuccess) return PREFT_ERR_CONFIG;
    if (cudaStreamWaitEvent(c->aux, c->fork, 0) != cudaSuccess) return PREFT_ERR_CONFIG;
    int rc = reft_res_apply(meta, h, rows, ldh, d, A, Bt, bias, scale, r, stream, num_sms, 0, f, false);
    const int rc2 = reft_tc_apply(meta, h, rows, ldh, d, A, Bt, bias, scale, r, c->aux, left, f, 4096);
    // always join, so a failed half never leaves the aux stream forked off a capture
    cudaEventRecord(c->join, c->aux);
    cudaStreamWaitEvent(stream, c->join, 0);
    if (rc == PREFT_OK) rc = rc2;
    // once a half may have launched, a failure must not read as "ineligible"
    // (PREFT_ERR_SHAPE): the caller would re-run the whole unit list and
    // apply the delta twice to the units that did run
    if (rc == PREFT_ERR_SHAPE) rc = PREFT_ERR_CONFIG;
    return rc;
}

// -1 automatic (tensor cores when eligible), 0 SIMT only, 1 tensor cores only
// (resident kernel when eligible, else streaming), 2 streaming tensor-core
// kernel only, 3 resident tensor-core kernel only
static int g_reft_variant = -2;
int reft_variant() {
    if (g_reft_variant == -2) {
        const char* env = getenv("PREFT_REFT_VARIANT");
        g_reft_variant = !env ? -1 : env[0] == 's' ? 0 : env[0] == 't' ? 1 : env[0] == 'p' ? 2 : env[0] == 'r' ? 3 : -1;
    }
    return g_reft_variant;
}
void set_reft_variant(int v) { g_reft_variant = v; }

int reft_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A, const void* B,
               const void* Bt, const void* bias, const void* scale, int r, int dtype, cudaStream_t stream,
               int num_sms) {
    if (!meta || !h || !A || !B || !bias || !scale || d < 1 || ldh < d) return PREFT_ERR_SHAPE;
    if (r < 1 || r > 64 || (r & (r - 1))) return PREFT_ERR_RANK;
    if (dtype != PREFT_DTYPE_F32 && dtype != PREFT_DTYPE_BF16 && dtype != PREFT_DTYPE_F64) return PREFT_ERR_DOMAIN;
    const int variant = reft_variant();
    if (variant != 0 && Bt && dtype == PREFT_DTYPE_BF16) {
        int rc = PREFT_ERR_SHAPE;
        if (variant == 3 || (variant != 2 && reft_res_preferred(d, r)))
            rc = reft_res_apply(meta, h, rows, ldh, d, A, Bt, bias, scale, r, stream, num_sms, 0, 4096, false);
        if (rc != PREFT_ERR_SHAPE || variant == 3) return rc;  // launched, failed, or resident forced
        if (variant != 2 && r == 16) {
            rc = reft_colaunch(meta, h, rows, ldh, d, A, Bt, bias, scale, r, stream, num_sms);
            if (rc != PREFT_ERR_SHAPE) return rc;
        }
        rc = reft_tc_apply(meta, h, rows, ldh, d, A, Bt, bias, scale, r, stream, num_sms, 0, 4096);
        if (rc != PREFT_ERR_SHAPE || variant >= 1) return rc;  // launched, failed, or TC forced
    } else if (variant >= 1) {
        return PREFT_ERR_SHAPE;
    }
    const int W = dtype == PREFT_DTYPE_BF16 ? 8 : dtype == PREFT_DTYPE_F32 ? 4 : 2;
    const bool vec = (d % W == 0) && (ldh % W == 0) && aligned16r(h) && aligned16r(A) && aligned16r(B);
    const int dv = vec ? d / W : d;
    ReftArgs args{};
    args.h = h;
    args.ldh = ldh;
    args.d = d;
    args.slot_base = meta->slot_split;
    args.A = A;
    args.B = B;
    args.bias = bias;
    args.scale = scale;
    args.tokens = reinterpret_cast<const int2*>(meta->tokens);
    args.counters = meta->counters;
    ReftFn fn = nullptr;
    if (dtype == PREFT_DTYPE_BF16) {
        if (vec && dv <= 32 * 16 && r <= 32) fn = pick_reft_rank<__nv_bfloat16, true, 16>(r);
        else if (vec) fn = pick_reft_rank<__nv_bfloat16, true, 0>(r);
        else fn = pick_reft_rank<__nv_bfloat16, false, 0>(r);
    } else if (dtype == PREFT_DTYPE_F32) {
        if (vec && dv <= 32 * 8 && r <= 32) fn = pick_reft_rank<float, true, 8>(r);
        else if (vec) fn = pick_reft_rank<float, true, 0>(r);
        else fn = pick_reft_rank<float, false, 0>(r);
    } else {
        fn = vec ? pick_reft_rank<double, true, 0>(r) : pick_reft_rank<double, false, 0>(r);
    }
    if (!fn) return PREFT_ERR_RANK;
    const int grid = grid_for(reinterpret_cast<const void*>(fn), 256, num_sms);
    fn<<<grid, 256, 0, stream>>>(args);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : -static_cast<int>(e);
}

}  // namespace preft
