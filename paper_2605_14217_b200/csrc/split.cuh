// Shared pieces of the tensor-core LoRA split kernels (lora_split.cu) and
// the fused shrink -> exchange -> expand kernel (lora_fused.cu): argument
// structs, K1-unit work items and their cost-balanced ranges, and the
// shared-memory layouts of the two halves.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "tc.cuh"

namespace preft {

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
    int slot_base;  // LoRA-class slots are < slot_split (meta->slot_split)
    int max_planes; // tensor-core shrink: CTAs that may share one unit (1 = whole units)
    float* planes;  // partial planes p >= 1 at planes + p * plane_stride (row stride ldp)
    long long plane_stride;
    int* sync;      // per-unit arrival counters (zero between launches)
    int flags;      // kSplitHints
    int* sched;     // dynamic schedules: launch-sequence counters (LaunchSeq) of the expand at sched,
                    //   of the LPT shrink at sched + kSeqInts; NULL = static ranges
    const int* unit_order;  // K1's size order of the LoRA units (PREFT_META_UNIT_ORDER)
    int grab;       // items per grab
    int beta_s;     // added to the shrink / expand cost models' per-column item overhead
    int beta_e;     //   (tuning; env PREFT_SPLIT_BETA_S / _E)
    long long* prof;  // diagnostics: clock64 stamps of CTA 0 (NULL in production)
    const int2* tokens;
    const int2* chunks;
    const int4* units;
    const int* counters;
};

// ---------------------------------------------------------------- tcgen05 halves

constexpr int kSpU = 64;                  // unit rows (UMMA M)
constexpr int kSpChunk = PREFT_CHUNK_ROWS;
constexpr int kSpN = 128;                 // expand block width (UMMA N) of narrow sites
constexpr int kSpNMax = 256;              // expand block width of sites with n % 256 == 0
constexpr int kSpAcc = 4;                 // split shrink accumulators = UMMA-issuing warps
constexpr int kShrinkThreads = 32 * (6 + kSpAcc);
constexpr int kPps = 4;                   // K panels (64 columns) per shrink item / ring stage
constexpr int kPlanes = 4;                // max CTAs sharing one unit's shrink (P partial planes)
// extra per-item overheads of the cost models (bytes-equivalent per column):
// an item's fixed cost (barriers, UMMA issue, TMEM round trip, TMA issue)
// is worth ~128 B per column more than its bytes; measured on config 4
// (12.1 -> 11.4-11.7 ms/step) and the 8B r16 step
constexpr int kBetaS = 128;
constexpr int kBetaE = 128;
constexpr int kSplitHints = 2;  // expand: Bt loads evict_last, y reduce-adds evict_first
constexpr int kMaxGrid = 1024;  // CTAs per launch the launch-sequence counters cover
constexpr int kSeqInts = 8 + kMaxGrid;
constexpr int kSchedInts = 2 * kSeqInts;  // the dynamic schedules' counters in meta->lora_part (expand, LPT shrink)

// Launch-local counters without an end-of-kernel handshake.  Every CTA keeps
// its own launch count at base[8 + blockIdx.x] — on one stream all CTAs of a
// kernel's launches see the same count, so it numbers the launch — and grab
// counters form a ring of three: launch n grabs from base[n % 3] and zeroes
// base[(n + 2) % 3], which launch n - 1 used (it has completed: launches on a
// stream run one after another past the PDL wait) and launch n + 2 will use.
// The count is read after the PDL wait and written back by the CTA at its end;
// the next launch reads it after its own wait.  The grid must not change
// between launches that share a base.
struct LaunchSeq {
    int n;      // this launch's number
    int* grab;  // this launch's grab counter
};
__device__ __forceinline__ LaunchSeq launch_seq_begin(int* base) {
    const int n = *reinterpret_cast<volatile int*>(base + 8 + blockIdx.x);
    if (blockIdx.x == 0 && threadIdx.x == 0) base[(n + 2) % 3] = 0;
    return {n, base + n % 3};
}
__device__ __forceinline__ void launch_seq_end(int* base, int n) {  // one thread per CTA
    base[8 + blockIdx.x] = n + 1;
}

struct SplitMaps {
    CUtensorMap x;       // x [rows][m] (this rank's columns), 16-row x 64-col boxes
    CUtensorMap x64;     // the same with 64-row boxes (a unit of 4 contiguous chunks)
    CUtensorMap A[3];    // A_s [S*R][m], R-row x 64-col boxes
    CUtensorMap y[3];    // y_s as [panels][rows][64] (make_tmap_bf16_panels), box {64, 16, block/64}
};

// A unit whose 4 chunks are consecutive rows of one entry loads as ONE 64-row
// TMA box per panel (a TMA instruction costs ~30-100 cycles to issue).
__device__ __forceinline__ bool unit_contiguous(const int2* chunks, int4 U) {
    if (U.z != 4) return false;
    const int2 c0 = chunks[U.y], c1 = chunks[U.y + 1], c2 = chunks[U.y + 2], c3 = chunks[U.y + 3];
    return c0.y == kSpChunk && c1.y == kSpChunk && c2.y == kSpChunk && c1.x == c0.x + kSpChunk &&
           c2.x == c0.x + 2 * kSpChunk && c3.x == c0.x + 3 * kSpChunk;
}

// ---- cost-balanced work ranges
//
// Work items are (unit u, column block c) over the LoRA-class units (K1 lists
// them first; counters[PREFT_CTR_LORA_UNITS]), c over `nc` blocks of a unit's
// columns (the expand: every site's output columns; the shrink: the input
// columns, kPps panels per block).  Item (u, c) costs
//     width(c) * (alpha * nch_u + beta)        (bytes-equivalent)
// alpha per column per 16-row chunk (activation traffic), beta per column
// (the adapter's weights plus a fixed per-item overhead).  The cost ahead of
// unit u is  W * (alpha * ch0(u) + beta * u)  with ch0(u) = units[u].y, K1's
// exclusive prefix of chunk counts.  Each CTA takes the items whose start
// cost falls in its 1/G of the total, found by a two-level parallel search
// over the units — no host round trip, so the launch stays graph-safe.
struct Blocks {
    int nc;        // blocks per unit
    int nsites;
    int first[4];  // first block of each site (first[nsites] = nc)
    int cw[3];     // block width of each site
    int coff[3];   // first column of each site among the unit's columns
    long long W;   // columns per unit
    __device__ __forceinline__ int site(int c) const {
        int s = 0;
        while (s + 1 < nsites && c >= first[s + 1]) ++s;
        return s;
    }
    __device__ __forceinline__ long long off(int c) const {
        const int s = site(c);
        return coff[s] + static_cast<long long>(c - first[s]) * cw[s];
    }
    // first block whose column offset is >= X (nc if none)
    __device__ __forceinline__ int first_at_least(long long X) const {
        if (X <= 0) return 0;
        for (int s = 0; s < nsites; ++s) {
            const long long last = coff[s] + static_cast<long long>(first[s + 1] - first[s] - 1) * cw[s];
            if (X <= last) {
                const long long j = (X - coff[s] + cw[s] - 1) / cw[s];
                return first[s] + (j > 0 ? static_cast<int>(j) : 0);
            }
        }
        return nc;
    }
};

struct CostModel {
    const int4* units;
    int nu;
    int nch_tot;  // chunks of the LoRA-class units (counters[PREFT_CTR_LORA_CHUNKS])
    long long alpha, beta;
    int G;  // CTAs sharing the items (CTAs >= G get none)
    long long tot;
    __device__ __forceinline__ long long prefix(int u, const Blocks& b) const {
        const int ch0 = u < nu ? units[u].y : nch_tot;
        return b.W * (alpha * ch0 + beta * u);
    }
    __device__ __forceinline__ void load(const int* counters) {
        nu = counters[PREFT_CTR_LORA_UNITS];
        nch_tot = counters[PREFT_CTR_LORA_CHUNKS];
    }
    __device__ __forceinline__ long long target(int cta) const { return tot * cta / G; }
    // the CTA whose share holds cost position S
    __device__ __forceinline__ int owner(long long S) const {
        int b = static_cast<int>(S * G / tot);
        b = b < G - 1 ? b : G - 1;
        while (b + 1 < G && target(b + 1) <= S) ++b;
        while (b > 0 && target(b) > S) --b;
        return b;
    }
    // first item of unit u (or u + 1) whose start cost is >= t
    __device__ __forceinline__ int first_item(int u, long long t, const Blocks& b) const {
        const long long base = prefix(u, b), per = alpha * units[u].z + beta;
        const long long X = t > base ? (t - base + per - 1) / per : 0;
        return u * b.nc + b.first_at_least(X);
    }
};

// The shrink's schedule: items (unit, K block of kPps panels) over an input of
// width m; with max_planes > 1 a unit may be split by K between up to
// max_planes CTAs (G is capped so that a CTA's share covers at least one
// item of any unit).  Shared by the shrink and by the fused kernel, whose
// expand phase sums the pieces.
__device__ __forceinline__ void shrink_model(Blocks& bl, CostModel& cm, const int4* units, const int* counters, int m,
                                             int nsr, int max_planes, int grid, int beta_extra) {
    const int NP = m / 64;
    bl.nsites = 1;
    bl.nc = max_planes > 1 ? NP / kPps : 1;
    bl.cw[0] = bl.nc == 1 ? m : 64 * kPps;
    bl.coff[0] = 0;
    bl.first[0] = 0;
    bl.first[1] = bl.nc;
    bl.W = m;
    cm.units = units;
    cm.load(counters);
    cm.alpha = kSpChunk * 2;            // x bytes per column per chunk
    cm.beta = nsr * 2 + 16 + beta_extra;  // A bytes per column + per-item overhead
    cm.G = grid;
    cm.tot = cm.nu > 0 ? cm.prefix(cm.nu, bl) : 0;
    if (max_planes > 1 && cm.nu > 0) {
        // a unit may span at most max_planes CTAs: cap the CTAs sharing the
        // work so that one CTA's share is >= max_unit / f, f = max(1,
        // max_planes - 2) (a unit then meets at most f + 1 CTAs, with one
        // to spare for the rounding of the share boundaries)
        const long long umax = bl.W * (cm.alpha * PREFT_UNIT_CHUNKS + cm.beta);
        const long long f = max_planes > 3 ? max_planes - 2 : 1;
        const long long g = f * cm.tot / umax;
        cm.G = static_cast<int>(g < 1 ? 1 : g < cm.G ? g : cm.G);
    }
}

// first CTA of unit u's shrink and the number of CTAs (pieces) that share it
__device__ __forceinline__ int unit_first_cta(const CostModel& cm, const Blocks& bl, int u) {
    return cm.owner(cm.prefix(u, bl));
}
__device__ __forceinline__ int unit_pieces(const CostModel& cm, const Blocks& bl, int u, int nch) {
    if (bl.nc <= 1) return 1;
    const long long base = cm.prefix(u, bl), per = cm.alpha * nch + cm.beta;
    return cm.owner(base + bl.off(bl.nc - 1) * per) - cm.owner(base) + 1;
}

// [k0, k1) of this CTA; every thread of the block must call it
static __device__ void item_range(CostModel& cm, const Blocks& b, int* s_u, int& k0, int& k1) {
    k0 = k1 = 0;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int nu = cm.nu;
    if (nu <= 0) return;
    cm.tot = cm.prefix(nu, b);
    if (static_cast<int>(blockIdx.x) >= cm.G || cm.tot <= 0) return;
    const long long t0 = cm.target(blockIdx.x), t1 = cm.target(blockIdx.x + 1);
    const int step = (nu + nt - 1) / nt;
    if (tid < 2) s_u[tid] = 0;
    __syncthreads();
    int u = tid * step;
    if (u < nu) {
        const long long p = cm.prefix(u, b);
        if (p <= t0) atomicMax(&s_u[0], u);
        if (p <= t1) atomicMax(&s_u[1], u);
    }
    __syncthreads();
    const int l0 = s_u[0], l1 = s_u[1];
    __syncthreads();
    if (tid < step) {
        u = l0 + tid;
        if (u < nu && cm.prefix(u, b) <= t0) atomicMax(&s_u[0], u);
        u = l1 + tid;
        if (u < nu && cm.prefix(u, b) <= t1) atomicMax(&s_u[1], u);
    }
    __syncthreads();
    k0 = cm.first_item(s_u[0], t0, b);
    k1 = static_cast<int>(blockIdx.x) + 1 == cm.G ? nu * b.nc : cm.first_item(s_u[1], t1, b);
}

// ---- shrink

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

__device__ __forceinline__ void readout_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// ---- expand

// The expand's shared-memory layout: Bt blocks in a ring (TMA bulk copies),
// the unit's V (hi / lo, double-buffered) and the epilogue's bf16 staging
// tiles, from which a TMA reduce-add adds the delta into y in L2 (rows of a
// partial chunk beyond the entry's own are padded with -0.0, which leaves any
// value and the sign of zero unchanged), so y never passes through the SM.
template <int R, int NS>
struct ExpandLayout {
    static constexpr int QS = 4 * kSpChunk * 128;         // one chunk's rows of a block: <= 4 panels x 16 rows x 128 B
    static constexpr int BT_BYTES = kSpNMax * R * 2;
    static constexpr int STAGE = BT_BYTES;                // multiple of 1024
    static constexpr int V_BYTES = kSpU * R * 2;          // one V (hi or lo) of one site
    static constexpr int OFF_V = 0;                       // [2 buffers][NS sites][hi, lo]
    static constexpr int OFF_STG = 4 * NS * V_BYTES;      // reduce staging [2 groups][2 buffers][4 chunks] x QS
    static constexpr int STG_BYTES = 2 * 2 * 4 * QS;
    static constexpr int OFF_RING = OFF_STG + STG_BYTES;  // multiple of 1024
    static constexpr int STAGES_FIT = (227 * 1024 - 2048 - OFF_RING) / STAGE;
    static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
    static constexpr int SMEM = OFF_RING + STAGES * STAGE + 1024;
    static_assert(STAGES >= 3, "expand ring too shallow");
};

__device__ __forceinline__ void expand_blocks(Blocks& b, const SplitArgs& a, int nsites) {
    b.nsites = nsites;
    b.nc = 0;
    long long W = 0;
    for (int s = 0; s < nsites; ++s) {
        b.first[s] = b.nc;
        b.cw[s] = a.site[s].n % kSpNMax == 0 ? kSpNMax : kSpN;
        b.coff[s] = static_cast<int>(W);
        b.nc += a.site[s].n / b.cw[s];
        W += a.site[s].n;
    }
    b.first[nsites] = b.nc;
    b.W = W;
}

}  // namespace preft
