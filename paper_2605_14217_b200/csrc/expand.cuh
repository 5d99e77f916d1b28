// The tcgen05 expand pipeline shared by the split pair's expand kernel
// (lora_split.cu) and phase 2 of the fused tensor-parallel kernel
// (lora_fused.cu):
//
//   y_s[rows of unit u, block c] += V_u . Bt_s,a[block c]      (bf16 delta, TMA reduce-add in L2)
//
// Work items are (unit u, output block c) in unit-major order.  They reach
// the CTA's roles as [lo, hi) ranges through a kExpQ-slot shared-memory queue
// that the producer warp fills:
//   * static mode: one range, the CTA's cost-balanced share (item_range);
//   * dynamic mode: grabs of G consecutive items, the CTA's own index first
//     and then from a global counter (one grab ahead, so the atomic's round
//     trip hides behind the current grab's loads).  A CTA that meets slower
//     memory simply takes fewer grabs; the caller resets the counter.
// Every role walks the same ranges in the same order, so the CTA's item
// sequence (and its parity, which splits the epilogue between two warp
// groups) is the same for all of them; a "visit" — one V build — is a run of
// items of one unit in that sequence.
//
// warps: 0 producer (grabs + Bt bulk copies), 1 UMMA issuer, 2-3 V builders
// (VSrc supplies the rank-r rows: P of the split pair, or the exchange's
// partials for the fused kernel), 4-7 / 8-11 epilogue groups.
#pragma once

#include "split.cuh"

namespace preft {

constexpr int kExpQ = 4;
constexpr int kExpConsumers = 1 + 2 + 8;  // warps that read each queue slot (lane 0 arrives)

struct ExpandBars {
    uint64_t* full;
    uint64_t* empty;  // [STAGES]
    uint64_t* v_full;
    uint64_t* v_empty;
    uint64_t* d_full;
    uint64_t* d_empty;  // [2]
    uint64_t* q_full;
    uint64_t* q_empty;  // [kExpQ]
    int* q_lo;
    int* q_hi;  // [kExpQ]
};

// one thread
__device__ __forceinline__ void expand_bars_init(const ExpandBars& b, int stages) {
    for (int i = 0; i < stages; ++i) {
        tc::mbar_init(&b.full[i], 1);
        tc::mbar_init(&b.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
        tc::mbar_init(&b.v_full[i], 2);
        tc::mbar_init(&b.v_empty[i], 1);
        tc::mbar_init(&b.d_full[i], 1);
        tc::mbar_init(&b.d_empty[i], 4);
    }
    for (int i = 0; i < kExpQ; ++i) {
        tc::mbar_init(&b.q_full[i], 1);
        tc::mbar_init(&b.q_empty[i], kExpConsumers);
    }
}

struct ExpandWork {
    int k0, k1;  // static mode: this CTA's items
    int* sched;  // dynamic mode: grab counter (NULL = static)
    int G;       // items per grab
    int total;   // items of the launch
};

// split pair: the rank-r rows are P (one row per token, ldp floats)
struct SplitVSrc {
    const float* P;
    long long ldp;
    __device__ __forceinline__ void prepare(int, const int4&) {}
    __device__ __forceinline__ void load(long long row, int col, float4& p0, float4& p1) const {
        const float* pr = P + row * ldp + col;
        p0 = *reinterpret_cast<const float4*>(pr);
        p1 = *reinterpret_cast<const float4*>(pr + 4);
    }
};

template <int R, int NS, class VSrc>
__device__ __forceinline__ void expand_pipeline(const SplitMaps& maps, const SplitArgs& a, const Blocks& bl,
                                                uint32_t sbase, unsigned char* sgen, uint32_t tmem,
                                                const ExpandBars& B, const ExpandWork& W, VSrc& vs) {
    using L = ExpandLayout<R, NS>;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nc = bl.nc;

    // every consumer warp walks the queue: body(k, jt) for each item k, jt = its index in the CTA's sequence
    auto walk = [&](auto&& body) {
        int qi = 0, jt = 0;
        uint32_t qph = 0;
        while (true) {
            if (lane == 0) tc::mbar_wait(&B.q_full[qi], qph);
            __syncwarp();
            const int lo = *reinterpret_cast<volatile int*>(&B.q_lo[qi]);
            const int hi = *reinterpret_cast<volatile int*>(&B.q_hi[qi]);
            __syncwarp();
            if (lo < 0) break;
            if (lane == 0) tc::mbar_arrive(&B.q_empty[qi]);
            for (int k = lo; k < hi; ++k) body(k, jt++);
            if (++qi == kExpQ) {
                qi = 0;
                qph ^= 1u;
            }
        }
    };

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t keep = tc::policy_evict_last();  // Bt: reused by the adapter's next unit
            int stage = 0, qi = 0;
            uint32_t phase = 0, qph = 0;
            const int ngrabs = W.sched ? (W.total + W.G - 1) / W.G : 0;
            int next = W.sched ? static_cast<int>(blockIdx.x) : 0;
            bool posted_static = false;
            while (true) {
                int lo, hi;
                if (W.sched) {
                    const int cur = next;
                    if (cur < ngrabs) {
                        next = atomicAdd(W.sched, 1) + static_cast<int>(gridDim.x);  // consumed next iteration
                        lo = cur * W.G;
                        hi = min(W.total, lo + W.G);
                    } else {
                        lo = hi = -1;
                    }
                } else if (!posted_static && W.k0 < W.k1) {
                    lo = W.k0;
                    hi = W.k1;
                    posted_static = true;
                } else {
                    lo = hi = -1;
                }
                tc::mbar_wait(&B.q_empty[qi], qph ^ 1u);
                B.q_lo[qi] = lo;
                B.q_hi[qi] = hi;
                tc::mbar_arrive(&B.q_full[qi]);
                if (++qi == kExpQ) {
                    qi = 0;
                    qph ^= 1u;
                }
                if (lo < 0) break;
                for (int k = lo; k < hi; ++k) {
                    const int u = k / nc, c = k - u * nc;
                    const int s = bl.site(c), j = c - bl.first[s], cw = bl.cw[s];
                    const uint32_t bt_bytes = static_cast<uint32_t>(cw * R * 2);
                    tc::mbar_wait(&B.empty[stage], phase ^ 1u);
                    tc::mbar_expect_tx(&B.full[stage], bt_bytes);
                    const unsigned char* src = static_cast<const unsigned char*>(a.site[s].Bt_tc) +
                                               static_cast<long long>(a.units[u].x) * a.site[s].n * R * 2 +
                                               static_cast<long long>(j) * bt_bytes;
                    if (a.flags & kSplitHints)
                        tc::bulk_load_1d_hint(sbase + L::OFF_RING + stage * L::STAGE, src, bt_bytes, &B.full[stage], keep);
                    else
                        tc::bulk_load_1d(sbase + L::OFF_RING + stage * L::STAGE, src, bt_bytes, &B.full[stage]);
                    if (++stage == L::STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        const uint32_t id128 = tc::idesc_bf16_f32(kSpU, kSpN), id256 = tc::idesc_bf16_f32(kSpU, kSpNMax);
        int stage = 0, visit = -1, pu = -1;
        uint32_t phase = 0;
        walk([&](int k, int jt) {
            if (lane != 0) return;
            const int u = k / nc, c = k - u * nc;
            if (u != pu) {
                // a commit covers every UMMA issued before it: the previous visit's V is free
                if (visit >= 0) tc::mma_commit(&B.v_empty[visit & 1]);
                ++visit;
                pu = u;
                tc::mbar_wait(&B.v_full[visit & 1], (visit >> 1) & 1);
                tc::fence_after_sync();
            }
            const int vb = visit & 1, s = bl.site(c);
            const uint32_t vhi = sbase + L::OFF_V + ((vb * NS + s) * 2) * L::V_BYTES, vlo = vhi + L::V_BYTES;
            tc::mbar_wait(&B.full[stage], phase);
            const int db = jt & 1;
            tc::mbar_wait(&B.d_empty[db], ((jt >> 1) & 1) ^ 1u);
            tc::fence_after_sync();
            const uint32_t bt = sbase + L::OFF_RING + stage * L::STAGE;
            const uint32_t dD = tmem + db * kSpNMax;
            const uint32_t id = bl.cw[s] == kSpNMax ? id256 : id128;
#pragma unroll
            for (int kk = 0; kk < R / 16; ++kk) {
                const uint64_t bd = tc::desc_kmajor(bt + kk * 256, 128, R * 16);
                tc::mma_bf16(dD, tc::desc_kmajor(vhi + kk * 256, 128, R * 16), bd, id, kk > 0 ? 1u : 0u);
                tc::mma_bf16(dD, tc::desc_kmajor(vlo + kk * 256, 128, R * 16), bd, id, 1u);
            }
            tc::mma_commit(&B.d_full[db]);
            tc::mma_commit(&B.empty[stage]);
            if (++stage == L::STAGES) {
                stage = 0;
                phase ^= 1u;
            }
        });
    } else if (warp < 4) {
        // V = scale * (rank-r row) as bf16 hi + lo, 32 rows per warp, once per visit
        int visit = -1, pu = -1;
        walk([&](int k, int) {
            const int u = k / nc;
            if (u == pu) return;
            pu = u;
            ++visit;
            const int4 U = a.units[u];
            vs.prepare(u, U);
            const int vb = visit & 1;
            const int m = (warp - 2) * 32 + lane, q = m >> 4, rr = m & 15;
            const int2 ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
            const bool valid = rr < ch.y;
            tc::mbar_wait(&B.v_empty[vb], ((visit >> 1) & 1) ^ 1u);
#pragma unroll
            for (int s = 0; s < NS; ++s) {
                const float sc = __ldg(static_cast<const float*>(a.site[s].scale) + U.x);
                unsigned char* vhi = sgen + L::OFF_V + ((vb * NS + s) * 2) * L::V_BYTES;
#pragma unroll
                for (int k0v = 0; k0v < R; k0v += 8) {
                    float4 p0 = make_float4(0.f, 0.f, 0.f, 0.f), p1 = p0;
                    if (valid) vs.load(static_cast<long long>(ch.x + rr), s * R + k0v, p0, p1);
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
                    const uint32_t off = tc::kmajor_offset(m, k0v, R);
                    *reinterpret_cast<uint4*>(vhi + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(vhi + L::V_BYTES + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                }
            }
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&B.v_full[vb]);
        });
    } else {
        // epilogue group g: D -> bf16 staging tile -> TMA reduce-add into y
        const int q = warp & 3, g = (warp - 4) >> 2;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
        const uint64_t stream = tc::policy_evict_first();
        const int r1 = lane >> 2, cp = 2 * (lane & 3);
        int pu = -1;
        int2 ch = make_int2(0, 0);
        walk([&](int k, int jt) {
            if ((jt & 1) != g) return;
            const int u = k / nc, c = k - u * nc;
            if (u != pu) {
                const int4 U = a.units[u];
                ch = q < U.z ? a.chunks[U.y + q] : make_int2(0, 0);
                pu = u;
            }
            const int s = bl.site(c), j = c - bl.first[s], cw = bl.cw[s], npan = cw / 64;
            tc::mbar_wait(&B.d_full[g], (jt >> 1) & 1);
            tc::fence_after_sync();
            const int sb = (jt >> 1) & 1;
            const uint32_t tile = L::OFF_STG + ((g * 2 + sb) * 4 + q) * L::QS;
            if (lane == 0) tc::tma_store_wait_read_1();  // this buffer's reduce of 2 items ago has read it
            __syncwarp();
            if (ch.y > 0) {
                for (int pass = 0; pass < npan / 2; ++pass) {
                    // loads, wait and every use of v stay in one block: a
                    // tcgen05.ld whose registers are live across a branch join
                    // can have them copied before tcgen05.wait::ld (stale D)
                    uint32_t v[2][32];
                    tc::tmem_ld_16x256b_x8(tmem + lane_base + g * kSpNMax + pass * 128, v[0]);
                    tc::tmem_ld_16x256b_x8(tmem + lane_base + g * kSpNMax + pass * 128 + 64, v[1]);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int pw = 0; pw < 2; ++pw) {
                        const uint32_t panel = tile + (2 * pass + pw) * (kSpChunk * 128);
#pragma unroll
                        for (int i = 0; i < 8; ++i)
#pragma unroll
                            for (int half = 0; half < 2; ++half) {
                                const int r = r1 + 8 * half;
                                const uint32_t w = r < ch.y ? f32x2_to_bf16(__uint_as_float(v[pw][4 * i + 2 * half]),
                                                                             __uint_as_float(v[pw][4 * i + 2 * half + 1]))
                                                            : 0x80008000u;  // -0.0: y + (-0) == y bit for bit
                                *reinterpret_cast<uint32_t*>(sgen + panel + tc::sw128_offset(r, 8 * i + cp, kSpChunk)) = w;
                            }
                    }
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&B.d_empty[g]);
            if (ch.y > 0) {
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    if (a.flags & kSplitHints)
                        tc::tma_reduce_add_3d_hint(&maps.y[s], 0, ch.x, j * npan, sbase + tile, stream);
                    else
                        tc::tma_reduce_add_3d(&maps.y[s], 0, ch.x, j * npan, sbase + tile);
                }
            }
            if (lane == 0) tc::tma_store_commit();
            __syncwarp();
        });
        if (lane == 0) tc::tma_store_wait_all();
    }
}

}  // namespace preft
