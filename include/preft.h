/*
 * preft.h — C ABI of libpreft, the B200 (sm_100a) PreFT hot path.
 *
 * The reference (arxiv 2605.14217, package `prefillsim`) is pure Python; its
 * "FFI" for this path is the Python operator API.  Each entry point below
 * replaces one piece of that API (file:line relative to /root/reference):
 *
 *   preft_meta_build      <- compute_position_mask   pkg/src/prefillsim/model.py:305-319
 *                            (+ the per-entry row selection inside
 *                             forward_chunk, model.py:474-475,509,538; the
 *                             grouping of selected tokens by adapter has no
 *                             reference counterpart)
 *   preft_lora_apply      <- _project's low-rank delta  model.py:442-452
 *                            via delta_for_rows        adapters.py:278-288
 *                            (in place on the base output y; one call covers
 *                             every entry of the batch and 1-3 sites that
 *                             share the same input x: q/k/v, gate/up)
 *   preft_reft_apply      <- the residual-stream hook   model.py:543-546
 *                            via delta_for_rows        adapters.py:289-295
 *                            (DiReFT and LoReFT; LoReFT arrives with
 *                             A := W - R folded at registration)
 *   preft_convert_2d      <- AdapterParams construction adapters.py:129-185
 *                            (f64 bundle -> bf16/f32 pool slab slot; the
 *                             upload half of weight sync, engine.py:676-697)
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless stated otherwise;
 *   - every call is stream-ordered on `stream` (a cudaStream_t passed as
 *     void*), never synchronises the host, and is CUDA-graph capturable:
 *     sizes that change per step (E, T) are read from device memory;
 *   - return value 0 = success, otherwise a PREFT_ERR_* code.  Codes 1-8 map
 *     one-to-one onto prefillsim.errors (errors.py:8-37); the Python shim
 *     raises the matching exception class.
 */
#ifndef PREFT_H
#define PREFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PREFT_ABI_VERSION 2

/* status codes (errors.py:8-37) */
#define PREFT_OK 0
#define PREFT_ERR_SHAPE 1      /* ShapeError  */
#define PREFT_ERR_RANK 2       /* RankError   */
#define PREFT_ERR_DOMAIN 3     /* DomainError */
#define PREFT_ERR_CONFIG 4     /* ConfigError */
#define PREFT_ERR_BATCH 5      /* BatchError  */
#define PREFT_ERR_STATE 6      /* StateError  */
#define PREFT_ERR_SYNC 7       /* SyncError   */
#define PREFT_ERR_INFEASIBLE 8 /* InfeasibleBatchError */
#define PREFT_ERR_CUDA 16      /* a CUDA runtime/launch error (RuntimeError) */

/* element types of activations and pool slabs */
#define PREFT_DTYPE_F32 0  /* fp32 I/O, fp32 accumulate: the "fp32 mode" (<= 1e-5 rel)   */
#define PREFT_DTYPE_BF16 1 /* bf16 I/O, fp32 accumulate: the serving mode (<= 2e-2 rel)  */
#define PREFT_DTYPE_F64 2  /* f64 I/O, f64 accumulate: the reference's own precision     */

/* per-entry flag bits (SeqEntry.phase / .schedule, model.py:223-242) */
#define PREFT_ENTRY_DECODE 1        /* Phase.DECODE (else PREFILL) */
#define PREFT_ENTRY_ALL_POSITIONS 2 /* PositionSchedule.ALL_POSITIONS */

/* device-side error bits written to counters[PREFT_CTR_ERR] by preft_meta_build */
#define PREFT_META_ERR_E_RANGE 1   /* E < 1 or E > E_cap            */
#define PREFT_META_ERR_T_RANGE 2   /* T < 1 or T > T_cap            */
#define PREFT_META_ERR_QSL 4       /* query_start_loc not a strictly increasing prefix sum from 0 to T */
#define PREFT_META_ERR_TILES 8     /* work list would exceed tile_cap */
#define PREFT_META_ERR_UNITS 16    /* chunk list would exceed chunk_cap */

/* counters[] slots */
#define PREFT_CTR_SEL_TOKENS 0  /* selected (adapter-carrying) tokens      */
#define PREFT_CTR_SEGMENTS 1    /* segments = runs of one adapter slot      */
#define PREFT_CTR_TILES 2       /* work tiles of <= tile_tokens tokens      */
#define PREFT_CTR_ERR 3         /* PREFT_META_ERR_* bits                    */
#define PREFT_CTR_SEL_ENTRIES 4 /* entries whose tokens are selected        */
#define PREFT_CTR_T 5           /* T as read from the entry buffer          */
#define PREFT_CTR_E 6           /* E as read from the entry buffer          */
#define PREFT_CTR_SPLIT 7       /* selected tokens whose slot < slot_split  */
#define PREFT_CTR_CHUNKS 8      /* row chunks (<= PREFT_CHUNK_ROWS rows of one entry) */
#define PREFT_CTR_UNITS 9       /* tensor-core work units (<= 4 chunks of one slot)  */
#define PREFT_CTR_LORA_UNITS 10 /* units whose slot < slot_split (they come first)   */
#define PREFT_CTR_LORA_CHUNKS 11 /* chunks of those units (they come first as well)   */
#define PREFT_NUM_COUNTERS 12

/* rows per chunk: one TMA box / one TMEM lane quadrant of an M = 64 UMMA */
#define PREFT_CHUNK_ROWS 16
#define PREFT_UNIT_CHUNKS 4
#define PREFT_META_UNIT_ORDER 1

/*
 * Batch-metadata workspace.  All arrays are device memory at fixed addresses
 * (allocated once by the host, reused every step, so a captured CUDA graph
 * stays valid).  The host writes `entries` (one H2D copy per step):
 *
 *   entries[0]                 = E  (number of SeqEntry)
 *   entries[1]                 = T  (total query tokens)
 *   entries[2 .. 2+E]          = query_start_loc[0..E]      (model.py:248)
 *   entries[3+E .. 3+2E)       = adapter slot per entry, -1 = no adapter
 *   entries[3+2E .. 3+3E)      = PREFT_ENTRY_* flags per entry
 *
 * preft_meta_build fills:
 *   mask[T]            1 where the reference's PositionMask is True (bit-exact)
 *   tokens[2*n_sel]    (token index, slot) pairs of the selected tokens, stably
 *                      sorted by slot (ties keep batch order)
 *   segments[3*nseg]   (slot, first sorted position, length)
 *   tiles[4*ntiles]    (slot, first sorted position, n tokens, segment id)
 *   entry_offset[E]    sorted position of the entry's first token, -1 if unselected
 *   chunks[2*nchunks]  (first h row, n rows): every selected entry cut into runs
 *                      of <= PREFT_CHUNK_ROWS consecutive rows, in sorted order
 *   units[4*nunits]    (slot, first chunk, n chunks, 0): up to PREFT_UNIT_CHUNKS
 *                      consecutive chunks of one slot — the tensor-core ReFT
 *                      kernel's work item (one M = 64 UMMA tile, one chunk per
 *                      TMEM lane quadrant, each chunk one TMA box)
 *   counters[12]       PREFT_CTR_*
 *
 * Slot classes: one pool serves LoRA and ReFT adapters side by side (a batch
 * may mix them, BASELINE config 1).  LoRA adapters own slots [0, slot_split),
 * ReFT adapters slots [slot_split, ...).  Because tokens are sorted by slot,
 * the LoRA tokens are sorted positions [0, counters[SPLIT]) and the ReFT
 * tokens [counters[SPLIT], counters[SEL_TOKENS]): preft_lora_apply walks the
 * first range, preft_reft_apply the second (indexing its slabs with
 * slot - slot_split).
 */
typedef struct preft_meta {
    int32_t* entries;
    uint8_t* mask;
    int32_t* tokens;
    int32_t* segments;
    int32_t* tiles;
    int32_t* entry_offset;
    int32_t* counters;
    int32_t E_cap;       /* <= PREFT_MAX_ENTRIES */
    int32_t T_cap;
    int32_t tile_cap;    /* >= E_cap + T_cap / tile_tokens + 1 */
    int32_t tile_tokens; /* tokens per work tile (>= 1) */
    int32_t slot_split;  /* first ReFT slot; slots below it are LoRA slots */
    int32_t rows_hint;   /* host's expected token count (0 = unknown): picks the
                            K2 team size at launch; never affects results */
    int32_t* chunks;
    int32_t* units;
    int32_t chunk_cap;   /* >= E_cap + T_cap / PREFT_CHUNK_ROWS + 1 (bounds chunks and units) */
    int32_t meta_flags;  /* PREFT_META_UNIT_ORDER: units[] holds 5 * chunk_cap ints and K1 appends,
                            at units + 4 * chunk_cap, the LoRA-class units in size order (4 chunks
                            first, then 3, 2, 1; K1 order within a size) — the tensor-core shrink
                            hands them out largest first */
    float* lora_part;    /* NULL, or a [T_cap][nsites * r_max] f32 workspace for the rank-r
                            intermediate of tensor-core LoRA launches (bf16, r_max 16/32) */
    int64_t lora_part_floats; /* capacity of lora_part in floats */
} preft_meta_t;

#define PREFT_MAX_ENTRIES 4096

/* number of int32 words `entries` must hold for E_cap entries */
size_t preft_meta_entries_words(int32_t E_cap);

/* K1: device metadata builder (replaces compute_position_mask, model.py:305). */
int preft_meta_build(const preft_meta_t* meta, void* stream);

/*
 * One LoRA site of a fused group (all sites of a group read the same x).
 * Pool layout for this (layer, site): A  [S][r_max][m], Bt [S][r_max][n]
 * (the reference's B is (n, r), adapters.py:159; it is stored transposed so
 * the expand streams contiguous rows), scale [S] = scaling_prefactor
 * (adapters.py:109-117) in the accumulator type (f32 for F32/BF16, f64 for
 * F64).  Rows k >= rank of a slot are zero.
 */
typedef struct preft_lora_site {
    const void* A;
    const void* Bt;
    const void* scale;
    const void* bias; /* NULL, or [S][r_max] added to the rank-r intermediate before
                         the scale (lets this kernel compute the ReFT delta
                         s*((h A^T + b) B) out of place, adapters.py:292-295) */
    void* y;        /* base output [T][ldy], updated in place on selected rows */
    int64_t ldy;
    int32_t n;
    int32_t reserved;
    const void* Bt_tc; /* NULL, or Bt pre-tiled in UMMA core-matrix order
                          [S][n/8][r_max/8][8][8] (bf16, r_max 16/32): lets
                          preft_lora_expand run on tensor cores */
} preft_lora_site_t;

/*
 * K2: y_s[t,:] += s_a * (x[t,:] . A_s,a^T) . Bt_s,a   for every selected token t
 * (adapter a = its slot) and every site s of the group (adapters.py:288).
 * Unselected rows of y are never read or written.
 *   x: [T][ldx] (dtype), m = input width; nsites in 1..3; r_max in
 *   {1,2,4,8,16,32,64} with nsites * r_max <= 64.
 * bf16 with r_max 16/32 (where the delta is a real contraction, ~10 FLOP/B
 * at r = 16), m % 256 == 0, every n % 128 == 0, every site's Bt_tc given and
 * meta->lora_part large enough runs on tcgen05: for inputs of >= 8192
 * columns the fused kernel (preft_lora_fused with a one-rank exchange in
 * meta->lora_part: one launch), otherwise the split shrink into
 * meta->lora_part (L2-resident, T x nsites x r f32) then the split expand
 * (the kernels of preft_lora_shrink / preft_lora_expand, no collective).
 * PREFT_LORA_FUSED=0/1 forces either; PREFT_LORA_FUSED_MIN_M moves the
 * threshold.
 * Everything else runs the SIMT kernels (team / warp per row).
 */
int preft_lora_apply(const preft_meta_t* meta, const void* x, int64_t ldx, int32_t m,
                     const preft_lora_site_t* sites, int32_t nsites, int32_t r_max,
                     int32_t dtype, void* stream);

/*
 * K2 split at the rank-r intermediate (tensor-parallel LoRA^P, BASELINE
 * config 4; also the r >= 16 path on one GPU).  With A sharded along the
 * input dimension and B along the output dimension across a TP group:
 *
 *   preft_lora_shrink:  P[t][s*r_max + k] = x[t, :] . A_s[a][k, :]
 *                       (this rank's partial; P in the accumulator type: f32
 *                       for BF16/F32, f64 for F64; P is indexed by token row,
 *                       ldp >= nsites * r_max; rows of unselected tokens are
 *                       left untouched)
 *   (caller)            P <- all-reduce-sum of P over the TP group (NCCL)
 *   preft_lora_expand:  y_s[t, :] += scale_s[a] * P[t][s*r_max ..] . Bt_s[a]
 *
 * which together equal preft_lora_apply when the group has one rank
 * (adapters.py:284-288, model.py:449-451).  x / y_s are this rank's column
 * slices (pass the pointer of the first owned column with the full leading
 * dimension).  bf16 with r_max in {16, 32}, m % 64 == 0 (shrink) and
 * n % 128 == 0 with sites[s].Bt_tc given (expand) run on tcgen05 (M = 64
 * units from meta->units); everything else on the SIMT path.  `rows` is the
 * number of allocated rows of x / y (TMA bounds).
 */
int preft_lora_shrink(const preft_meta_t* meta, const void* x, int64_t rows, int64_t ldx, int32_t m,
                      const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype,
                      void* P, int64_t ldp, void* stream);
int preft_lora_expand(const preft_meta_t* meta, const void* P, int64_t ldp, int64_t rows,
                      const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype,
                      void* stream);
/* Floats the tensor-core split wants in meta->lora_part (zero-initialised):
 * P and its partial planes (K-split shrinks, opt-in), one arrival counter per
 * unit, the dynamic schedules' launch-sequence counters (split.cuh LaunchSeq:
 * without them every expand uses static ranges) and a one-rank exchange
 * region for the opt-in fused route of preft_lora_apply (PREFT_LORA_FUSED=1). */
int64_t preft_lora_part_floats(const preft_meta_t* meta);
/*
 * Fused tensor-parallel LoRA^P: shrink -> cross-rank exchange of the rank-r
 * partials -> expand in ONE persistent tcgen05 kernel (replaces the
 * preft_lora_shrink + NCCL all-reduce + preft_lora_expand sequence above for
 * the same model.py:449-451 / adapters.py:284-288 delta).
 *
 * Every rank owns one exchange region (preft_xchg_region_bytes, zeroed once)
 * that its peers can address (cudaIpc / the same device when tp_size == 1):
 *   part [2 parities][tp src][planes][T_cap][64] f32 — src's partial P rows
 *   flag [2 parities][tp src][planes][U_cap] int32 — tag of the launch that
 *                                                      wrote them
 *   state int32 — [2] error bits; from [16] the launch-sequence counters
 *        (each CTA's launch count, which numbers the launch and is its tag;
 *        the grid must therefore stay the same on an exchange)
 * A CTA that finishes a unit's shrink piece stores its partial rows into
 * every rank's region (P2P stores over NVLink) and then the piece's flag
 * (system-scope release); the expand of that unit waits for all tp x pieces
 * flags of the launch and sums the partials in (src, piece) order, so every
 * rank computes the same V bit for bit.  Consecutive launches alternate
 * parities (the device-side launch count), which is what lets a fast rank
 * start the next launch while a slow one still reads this one.  All ranks
 * must issue the same sequence of fused launches on their exchanges.
 * A wait that exceeds spin_ns (default 2 s) sets state[2] bit 0 and gives up
 * (the output is then wrong; preft_xchg_errors reads the bits).
 */
#define PREFT_XCHG_MAX_TP 8
typedef struct preft_xchg {
    int32_t tp_size;
    int32_t tp_rank;
    int32_t planes;    /* K-split pieces per unit and rank, 1..4 */
    int32_t T_cap;     /* rows of every partial plane (>= meta->T_cap) */
    int32_t U_cap;     /* units (>= meta->chunk_cap) */
    int32_t peer_sys;  /* 1: the peers are other devices (system-scope ordering) */
    int32_t grid;      /* CTAs per launch, 0 = the SM count; must match on every rank */
    int32_t reserved;
    float* part[PREFT_XCHG_MAX_TP];    /* part[d]: rank d's partial planes, as mapped here */
    int32_t* flag[PREFT_XCHG_MAX_TP];  /* flag[d]: rank d's flags */
    int32_t* state;                    /* this rank's state words */
    int64_t spin_ns;
} preft_xchg_t;
int64_t preft_xchg_region_bytes(int32_t tp_size, int32_t planes, int32_t T_cap, int32_t U_cap);
/* fill part/flag/state from the base address of every rank's region */
int preft_xchg_init(preft_xchg_t* xg, void* const* region_bases, int32_t tp_size, int32_t tp_rank,
                    int32_t planes, int32_t T_cap, int32_t U_cap, int32_t peer_sys);
int preft_lora_fused(const preft_meta_t* meta, const void* x, int64_t rows, int64_t ldx, int32_t m,
                     const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype,
                     const preft_xchg_t* xchg, void* stream);
/* state[2] of this rank's region (stream-ordered read; synchronises the stream) */
int preft_xchg_errors(const preft_xchg_t* xchg, void* stream, int32_t* out);
/* cudaIpc plumbing for the exchange regions of a multi-GPU TP group:
 * a zeroed device allocation, its 64-byte IPC handle, and the peer mapping */
int preft_dev_alloc(int64_t bytes, void** out);
int preft_dev_free(void* p);
int preft_ipc_handle(void* dev_ptr, void* handle_out /* 64 bytes */);
int preft_ipc_open(const void* handle /* 64 bytes */, void** dev_ptr_out);
int preft_ipc_close(void* dev_ptr);
/* split-kernel variant: -1 automatic, 0 SIMT only, 1 tensor cores only
 * (PREFT_ERR_SHAPE when ineligible).  Env: PREFT_SPLIT_VARIANT=simt|tc. */
int preft_set_split_variant(int32_t variant);
/* Diagnostic: clock64() stamps of CTA 0 of the tensor-core shrink (4 per
 * stage / unit at [0, 512)) and expand (4 + 4 per item at [512, 1024) and
 * [1024, 1536)), then per-CTA globaltimer windows of CTAs 0-127 (shrink at
 * [1536, 1792), expand at [1792, 2048)); 2048
 * int64, NULL = off. */
int preft_diag_split(long long* device_buffer);

/*
 * K3 (h has `rows` allocated rows; TMA bounds): h[t,:] += s_a * ((h[t,:] . A_a^T + b_a) . B_a)   for every selected token
 * (adapters.py:292-295).  DiReFT: A, B as stored by the reference.  LoReFT:
 * A = W - R, B = R.  Pool layout for this layer: A [S][r_max][d],
 * B [S][r_max][d], bias [S][r_max], scale [S] (bias/scale in the accumulator
 * type: f32 for F32/BF16, f64 for F64).  r_max in {1,2,4,8,16,32,64}.
 * Bt (may be NULL) is B transposed and pre-tiled for the tensor-core expand:
 * per slot a [d/8][r_max/8][8][8] bf16 block, i.e. element (n, k) of B^T at
 * ((n/8)*(r_max/8) + k/8)*64 + (n%8)*8 + k%8 — the UMMA K-major core-matrix
 * order, so any 128-row chunk is one contiguous bulk copy.  When given, bf16
 * with r_max in {16, 32} and d % 128 == 0 runs the tcgen05 kernel (one
 * persistent CTA per SM, M = 64 units from meta->units, TMA rings, TMEM
 * accumulators); everything else runs the SIMT kernel.
 */
int preft_reft_apply(const preft_meta_t* meta, void* h, int64_t rows, int64_t ldh, int32_t d,
                     const void* A, const void* B, const void* Bt, const void* bias,
                     const void* scale, int32_t r_max, int32_t dtype, void* stream);

/* K3 kernel variant: -1 automatic (default), 0 SIMT only, 1 tensor cores
 * only (resident kernel when eligible, else streaming; PREFT_ERR_SHAPE when
 * neither applies), 2 streaming tensor-core kernel only, 3 resident
 * tensor-core kernel only.  Env: PREFT_REFT_VARIANT=simt|tc|pass|res. */
int preft_set_reft_variant(int32_t variant);

/* Tensor-core ReFT pipeline knobs (diagnostics / A-B measurement; results
 * never change): bit 0 immediate ring-stage release, bit 1 pace the shrink
 * behind the epilogue (`look` panels ahead, -1 = 3/4 of a unit), bit 2 no
 * one-unit throttle, bit 3 let the epilogue re-read run ahead of the shrink,
 * bit 4 no L2 cache hints, bit 5 reduce epilogue (TMA adds the bf16 delta
 * into h in L2 instead of re-reading h).  flags = -1 restores the default
 * (environment PREFT_REFT_TC_FLAGS / PREFT_REFT_TC_LOOK, else 7). */
int preft_set_reft_tc_flags(int32_t flags, int32_t look);

/*
 * K4: dst[i*dst_ld + j] = convert(src[i*src_stride_row + j*src_stride_col])
 * for i < rows_valid, j < cols; rows in [rows_valid, rows) are zero-filled.
 * src is a DEVICE float64 buffer; round-to-nearest-even into dst_dtype.
 */
int preft_convert_2d(void* dst, int32_t dst_dtype, int64_t dst_ld, const double* src,
                     int64_t src_stride_row, int64_t src_stride_col, int64_t rows_valid,
                     int64_t rows, int64_t cols, void* stream);

/*
 * Step plan: the native executor that replaces forward_chunk's Python
 * `layer x entry` loop (model.py:504-546).  A plan holds a copy of the meta
 * descriptor and an ordered list of LoRA-group / ReFT launches with fixed
 * pointers; preft_plan_run issues K1 (optional) and every launch on `stream`
 * with one call, and is CUDA-graph capturable while timing is off.  Launches
 * whose `tag` equals the timing tag are bracketed by CUDA events (bench.py's
 * per-kernel roofline figure).
 */
typedef struct preft_plan preft_plan_t;
preft_plan_t* preft_plan_create(const preft_meta_t* meta);
void preft_plan_destroy(preft_plan_t* plan);
int preft_plan_set_slot_split(preft_plan_t* plan, int32_t slot_split);
/* expected selected rows per step: the K2 launch shape (team size) of every
 * later run; a plan created before its meta's first build would otherwise
 * keep the hint 0 (one-warp teams).  Never affects results. */
int preft_plan_set_rows_hint(preft_plan_t* plan, int32_t rows_hint);
/* re-copy the meta descriptor (e.g. after its lora_part workspace was
 * attached); the plan keeps its own slot_split and rows_hint */
int preft_plan_refresh_meta(preft_plan_t* plan, const preft_meta_t* meta);
int preft_plan_add_lora(preft_plan_t* plan, const void* x, int64_t ldx, int32_t m,
                        const preft_lora_site_t* sites, int32_t nsites, int32_t r_max,
                        int32_t dtype, int32_t tag);
int preft_plan_add_reft(preft_plan_t* plan, void* h, int64_t rows, int64_t ldh, int32_t d, const void* A,
                        const void* B, const void* Bt, const void* bias, const void* scale,
                        int32_t r_max, int32_t dtype, int32_t tag);
int preft_plan_num_ops(const preft_plan_t* plan);
int preft_plan_set_timing(preft_plan_t* plan, int32_t tag, int32_t reserve_pairs);
int preft_plan_run(preft_plan_t* plan, int32_t run_meta, void* stream);
int preft_plan_collect_timing(preft_plan_t* plan, double* total_ms, int32_t* count);

/* K2 kernel variant: -1 automatic (default: team kernel with the team size
 * chosen from the row widths), 0 warp-per-row kernel only, 1/2/4/8 team
 * kernel with that many warps per row where eligible (aligned rows,
 * r_max <= 4, bf16/f32).  For A/B measurement and for testing every code
 * path; results agree to the stated tolerance.  Env: PREFT_LORA_VARIANT. */
int preft_set_lora_variant(int32_t variant);

/* Diagnostic: D[128 x N] (f32) = A[128 x K] . B[N x K]^T (bf16, row-major,
 * device) through the tcgen05/TMEM path the tensor-core kernels use
 * (K % 16 == 0, N % 16 == 0, 16 <= N <= 256).  mode 0: A staged by threads,
 * no swizzle; 1: threads, 128 B swizzle; 2: TMA, 128 B swizzle (K % 64 == 0).
 * Pins the UMMA descriptors, the swizzle and the TMA tensor maps. */
int preft_tc_selftest(const void* A, const void* B, float* D, int32_t K, int32_t N, int32_t mode,
                      void* stream);

/* Diagnostic: route clock64() stamps of the tensor-core ReFT kernel's CTA 0
 * (8 per chunk for 64 chunks, 4 per unit and 2 shrink stamps per unit for 16
 * units; device buffer of >= 736 int64, NULL = off) and return the grid size of the last launch. */
int preft_diag_reft_tc(long long* device_buffer);

/* library / device introspection */
int preft_abi_version(void);
const char* preft_status_string(int status);
const char* preft_last_cuda_error(void);
int preft_num_sms(void);

#ifdef __cplusplus
}
#endif

#endif /* PREFT_H */
