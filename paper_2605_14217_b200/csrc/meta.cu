// K1 — device batch-metadata builder.
//
// Restates compute_position_mask (reference pkg/src/prefillsim/model.py:305-319)
// on the device and adds what the fused kernels need: the selected tokens
// grouped by adapter slot into segments, and a work list of token tiles.
//
//   selected(entry) = adapter_id is not None
//                     and (phase is PREFILL or schedule is ALL_POSITIONS)   model.py:314-318
//   mask[t]         = selected(entry owning t), constant over the entry's span
//
// Two launches, both graph-capturable (E and T are read from device memory):
//   meta_sort_kernel    1 CTA x 1024 threads: validate query_start_loc, stable
//                       sort of selected entries by (slot, entry index) with an
//                       in-smem bitonic sort of 64-bit keys, block scans for the
//                       sorted token offsets, segment heads and tile counts.
//   meta_scatter_kernel grid over entries: writes mask[] and the sorted
//                       (token, slot) list; ~5 B per token of traffic.
#include "common.cuh"

namespace preft {

constexpr int kSortThreads = 1024;

// exclusive block-wide prefix sum of one int per thread; *total gets the sum
__device__ int block_exclusive_sum(int v, int* s_warp, int* s_total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const int nwarps = blockDim.x >> 5;
        int w = lane < nwarps ? s_warp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < nwarps) s_warp[lane] = wi - w;  // exclusive warp offsets
        if (lane == 31) *s_total = wi;
    }
    __syncthreads();
    const int out = s_warp[wid] + inc - v;
    __syncthreads();  // s_warp reusable by the caller afterwards
    return out;
}

// in-place exclusive scan of arr[0..n) held in shared memory; returns the total
__device__ int block_scan_array(int* arr, int n, int* s_warp, int* s_total) {
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int beg = min(n, static_cast<int>(threadIdx.x) * per);
    const int end = min(n, beg + per);
    int local = 0;
    for (int i = beg; i < end; ++i) local += arr[i];
    int run = block_exclusive_sum(local, s_warp, s_total);
    for (int i = beg; i < end; ++i) {
        const int v = arr[i];
        arr[i] = run;
        run += v;
    }
    __syncthreads();
    return *s_total;
}

__device__ __forceinline__ bool entry_selected(int slot, int flags) {
    // model.py:314-316: no adapter -> unselected; prefill tokens are prompt
    // positions (covered by both schedules); decode tokens only by ALL_POSITIONS
    if (slot < 0) return false;
    return !(flags & PREFT_ENTRY_DECODE) || (flags & PREFT_ENTRY_ALL_POSITIONS);
}

__global__ void __launch_bounds__(kSortThreads, 1) meta_sort_kernel(const preft_meta_t m) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_warp[32];
    __shared__ int s_total;
    __shared__ int s_split;
    __shared__ int s_lora_units, s_lora_chunks;
    __shared__ int s_err;

    const int tid = threadIdx.x;
    const int* ent = m.entries;
    const int E = ent[0];
    const int T = ent[1];

    if (tid == 0) {
        int err = 0;
        if (E < 1 || E > m.E_cap) err |= PREFT_META_ERR_E_RANGE;
        if (T < 1 || T > m.T_cap) err |= PREFT_META_ERR_T_RANGE;
        s_err = err;
    }
    __syncthreads();
    if (s_err & PREFT_META_ERR_E_RANGE) {
        if (tid < PREFT_NUM_COUNTERS) m.counters[tid] = tid == PREFT_CTR_ERR ? s_err : 0;
        return;
    }
    const int* qsl = ent + 2;
    const int* slots = qsl + E + 1;
    const int* flags = slots + E;

    // query_start_loc must be a strictly increasing prefix sum 0 .. T (model.py:250-258)
    for (int i = tid; i < E; i += blockDim.x) {
        if (qsl[i + 1] <= qsl[i]) atomicOr(&s_err, PREFT_META_ERR_QSL);
        m.entry_offset[i] = -1;
    }
    if (tid == 0 && (qsl[0] != 0 || qsl[E] != T)) atomicOr(&s_err, PREFT_META_ERR_QSL);

    int P = 1;
    while (P < E) P <<= 1;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem_raw);
    int* A = reinterpret_cast<int*>(keys + P);  // per sorted entry: length -> token offset
    int* B = A + P;                             // per sorted entry: head flag -> segment id
    int* C = B + P;                             // per segment: tile count -> tile offset (P + 1)
    int* D = C + P + 1;                         // per sorted entry: chunk count -> chunk offset

    for (int i = tid; i < P; i += blockDim.x) {
        unsigned long long k = ~0ull;
        if (i < E && entry_selected(slots[i], flags[i]))
            k = (static_cast<unsigned long long>(static_cast<unsigned>(slots[i])) << 32) |
                static_cast<unsigned>(i);
        keys[i] = k;
    }
    __syncthreads();
    if (s_err) {  // malformed batch: publish the error, select nothing
        if (tid < PREFT_NUM_COUNTERS)
            m.counters[tid] = tid == PREFT_CTR_ERR ? s_err
                              : tid == PREFT_CTR_E ? E
                              : tid == PREFT_CTR_T ? T
                                                   : 0;
        return;
    }

    // bitonic sort, ascending; keys are unique (entry index in the low word)
    // so the order is the stable order by slot
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = keys[i], b = keys[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        keys[i] = b;
                        keys[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    }

    // number of selected entries
    int local = 0;
    for (int i = tid; i < E; i += blockDim.x) local += keys[i] != ~0ull;
    block_exclusive_sum(local, s_warp, &s_total);
    const int nsel = s_total;
    __syncthreads();

    for (int i = tid; i < nsel; i += blockDim.x) {
        const unsigned long long k = keys[i];
        const int e = static_cast<int>(k & 0xffffffffu);
        A[i] = qsl[e + 1] - qsl[e];
        B[i] = (i == 0 || (k >> 32) != (keys[i - 1] >> 32)) ? 1 : 0;
        D[i] = (A[i] + PREFT_CHUNK_ROWS - 1) / PREFT_CHUNK_ROWS;
    }
    __syncthreads();
    const int n_tok = block_scan_array(A, nsel, s_warp, &s_total);
    const int nseg = block_scan_array(B, nsel, s_warp, &s_total);
    const int nchunks = block_scan_array(D, nsel, s_warp, &s_total);

    // tokens below the LoRA/ReFT slot split (own shared slot: s_total may
    // still be being read by threads returning from the last scan)
    if (tid == 0) s_split = n_tok;
    __syncthreads();
    for (int i = tid; i < nsel; i += blockDim.x) {
        const int sl = static_cast<int>(keys[i] >> 32);
        if (sl >= m.slot_split && (i == 0 || static_cast<int>(keys[i - 1] >> 32) < m.slot_split)) s_split = A[i];
    }
    __syncthreads();
    const int n_split = s_split;
    for (int i = tid; i < nsel; i += blockDim.x) {
        const unsigned long long k = keys[i];
        const int e = static_cast<int>(k & 0xffffffffu);
        m.entry_offset[e] = A[i];
        const bool head = (i == 0 || (k >> 32) != (keys[i - 1] >> 32));
        if (head) {
            const int s = B[i];  // exclusive count of earlier heads = segment id
            m.segments[3 * s + 0] = static_cast<int>(k >> 32);
            m.segments[3 * s + 1] = A[i];
            C[s] = A[i];  // segment begin, turned into a tile count below
        }
    }
    __syncthreads();
    const int tt = m.tile_tokens;
    for (int s = tid; s < nseg; s += blockDim.x) {
        const int begin = C[s];
        const int end = (s + 1 < nseg) ? C[s + 1] : n_tok;
        m.segments[3 * s + 2] = end - begin;
        A[s] = begin;  // A no longer needed per entry; keep segment begins here
    }
    __syncthreads();
    for (int s = tid; s < nseg; s += blockDim.x) {
        const int begin = A[s];
        const int end = (s + 1 < nseg) ? A[s + 1] : n_tok;
        C[s] = (end - begin + tt - 1) / tt;
    }
    __syncthreads();
    int ntiles = block_scan_array(C, nseg, s_warp, &s_total);
    if (tid == 0) C[nseg] = ntiles;
    int err = 0;
    if (ntiles > m.tile_cap) {
        err |= PREFT_META_ERR_TILES;
        ntiles = 0;
    }
    __syncthreads();
    for (int j = tid; j < ntiles; j += blockDim.x) {
        int lo = 0, hi = nseg - 1;  // last segment with C[s] <= j
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (C[mid] <= j) lo = mid;
            else hi = mid - 1;
        }
        const int s = lo;
        const int begin = A[s];
        const int end = (s + 1 < nseg) ? A[s + 1] : n_tok;
        const int t0 = begin + (j - C[s]) * tt;
        int4 tile;
        tile.x = m.segments[3 * s + 0];
        tile.y = t0;
        tile.z = min(tt, end - t0);
        tile.w = s;
        reinterpret_cast<int4*>(m.tiles)[j] = tile;
    }

    // ---- chunks and tensor-core units.  Every selected entry is cut into
    // chunks of <= PREFT_CHUNK_ROWS consecutive rows (so each chunk is one TMA
    // box); a unit is up to PREFT_UNIT_CHUNKS consecutive chunks of one
    // segment (one slot).  C (tile offsets) and A (segment token begins) are
    // dead now and are reused per segment: A = first chunk, C = unit offset.
    int nunits = 0;
    const bool chunks_fit = nchunks <= m.chunk_cap;
    __syncthreads();
    if (chunks_fit) {
        for (int i = tid; i < nsel; i += blockDim.x) {
            const unsigned long long k = keys[i];
            const int e = static_cast<int>(k & 0xffffffffu);
            const int row0 = qsl[e], len = qsl[e + 1] - qsl[e];
            const int c0 = D[i];
            for (int c = 0; c * PREFT_CHUNK_ROWS < len; ++c)
                reinterpret_cast<int2*>(m.chunks)[c0 + c] =
                    make_int2(row0 + c * PREFT_CHUNK_ROWS, min(PREFT_CHUNK_ROWS, len - c * PREFT_CHUNK_ROWS));
            if (i == 0 || (k >> 32) != (keys[i - 1] >> 32)) A[B[i]] = c0;  // segment's first chunk
        }
        __syncthreads();
        for (int s = tid; s < nseg; s += blockDim.x) {
            const int end = (s + 1 < nseg) ? A[s + 1] : nchunks;
            C[s] = (end - A[s] + PREFT_UNIT_CHUNKS - 1) / PREFT_UNIT_CHUNKS;
        }
        __syncthreads();
        nunits = block_scan_array(C, nseg, s_warp, &s_total);
        // LoRA-class units (slot < slot_split) come first: their count is the
        // unit offset of the first ReFT-class segment
        if (tid == 0) {
            s_lora_units = nunits;
            s_lora_chunks = nchunks;
        }
        __syncthreads();
        for (int s = tid; s < nseg; s += blockDim.x) {
            const int sl = m.segments[3 * s + 0];
            if (sl >= m.slot_split && (s == 0 || m.segments[3 * (s - 1) + 0] < m.slot_split)) {
                s_lora_units = C[s];
                s_lora_chunks = A[s];
            }
        }
        __syncthreads();
        for (int j = tid; j < nunits; j += blockDim.x) {
            int lo = 0, hi = nseg - 1;  // last segment with C[s] <= j
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (C[mid] <= j) lo = mid;
                else hi = mid - 1;
            }
            const int s = lo;
            const int end = (s + 1 < nseg) ? A[s + 1] : nchunks;
            const int first = A[s] + (j - C[s]) * PREFT_UNIT_CHUNKS;
            reinterpret_cast<int4*>(m.units)[j] =
                make_int4(m.segments[3 * s + 0], first, min(PREFT_UNIT_CHUNKS, end - first), 0);
        }
        // the LoRA-class units in size order (4 chunks first, ..., 1 last; K1 order
        // within a size) for the largest-first (LPT) tensor-core shrink: at ~1.6
        // units per CTA it brings the slowest CTA's share from ~1.7x to ~1.2x the
        // mean in a cost simulation (profiles/split_tuning_r02c.txt has the
        // measurement, where adapter locality costs most of that back)
        if (m.meta_flags & PREFT_META_UNIT_ORDER) {
            __syncthreads();
            int* order = m.units + 4 * m.chunk_cap;
            const int nlu = s_lora_units;
            const int per = (nlu + blockDim.x - 1) / blockDim.x;
            const int beg = min(nlu, tid * per), end = min(nlu, beg + per);
            int base = 0;
            for (int z = PREFT_UNIT_CHUNKS; z >= 1; --z) {
                int local = 0;
                for (int j = beg; j < end; ++j) local += reinterpret_cast<const int4*>(m.units)[j].z == z;
                int run = base + block_exclusive_sum(local, s_warp, &s_total);
                for (int j = beg; j < end; ++j)
                    if (reinterpret_cast<const int4*>(m.units)[j].z == z) order[run++] = j;
                base += s_total;
                __syncthreads();  // s_total is rewritten by the next scan
            }
        }
    } else {
        err |= PREFT_META_ERR_UNITS;
    }
    if (tid == 0) {
        m.counters[PREFT_CTR_CHUNKS] = chunks_fit ? nchunks : 0;
        m.counters[PREFT_CTR_UNITS] = nunits;
        m.counters[PREFT_CTR_LORA_UNITS] = chunks_fit ? s_lora_units : 0;
        m.counters[PREFT_CTR_LORA_CHUNKS] = chunks_fit ? s_lora_chunks : 0;
        m.counters[PREFT_CTR_SEL_TOKENS] = n_tok;
        m.counters[PREFT_CTR_SEGMENTS] = nseg;
        m.counters[PREFT_CTR_TILES] = ntiles;
        m.counters[PREFT_CTR_ERR] = err;
        m.counters[PREFT_CTR_SEL_ENTRIES] = nsel;
        m.counters[PREFT_CTR_T] = T;
        m.counters[PREFT_CTR_E] = E;
        m.counters[PREFT_CTR_SPLIT] = n_split;
    }
}

__global__ void __launch_bounds__(256) meta_scatter_kernel(const preft_meta_t m) {
    const int* ent = m.entries;
    const int E = ent[0];
    if (m.counters[PREFT_CTR_ERR] & (PREFT_META_ERR_E_RANGE | PREFT_META_ERR_T_RANGE | PREFT_META_ERR_QSL))
        return;
    const int* qsl = ent + 2;
    const int* slots = qsl + E + 1;
    for (int e = blockIdx.x; e < E; e += gridDim.x) {
        const int b = qsl[e], en = qsl[e + 1];
        const int off = m.entry_offset[e];
        const unsigned char sel = off >= 0 ? 1 : 0;
        const int slot = slots[e];
        for (int t = b + threadIdx.x; t < en; t += blockDim.x) {
            m.mask[t] = sel;
            if (sel) reinterpret_cast<int2*>(m.tokens)[off + (t - b)] = make_int2(t, slot);
        }
    }
}

size_t meta_sort_smem_bytes(int E_cap) {
    int P = 1;
    while (P < E_cap) P <<= 1;
    return static_cast<size_t>(P) * 8 + static_cast<size_t>(P) * 4 * 3 + (static_cast<size_t>(P) + 1) * 4;
}

int meta_build(const preft_meta_t* m, cudaStream_t stream, int num_sms) {
    const size_t smem = meta_sort_smem_bytes(m->E_cap);
    cudaError_t e = cudaFuncSetAttribute(meta_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return -static_cast<int>(e);
    meta_sort_kernel<<<1, kSortThreads, smem, stream>>>(*m);
    e = cudaGetLastError();
    if (e != cudaSuccess) return -static_cast<int>(e);
    meta_scatter_kernel<<<2 * num_sms, 256, 0, stream>>>(*m);
    e = cudaGetLastError();
    if (e != cudaSuccess) return -static_cast<int>(e);
    return 0;
}

}  // namespace preft
