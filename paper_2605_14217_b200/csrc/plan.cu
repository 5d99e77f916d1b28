// Native step executor: a pre-validated list of hot-path launches for one
// step (K1, then every LoRA group / ReFT site of every layer) issued by ONE
// C call.  Replaces the reference's Python `layer x entry` loop
// (model.py:504-546) with a launch list built once; all pointers are fixed,
// so the same plan serves every step (and can be captured in a CUDA graph
// when timing is off).  Optional CUDA-event timing of one tagged launch
// class (e.g. the gate/up group) feeds bench.py's roofline numbers.
#include <vector>

#include "common.cuh"

namespace preft {
int meta_build(const preft_meta_t* m, cudaStream_t stream, int num_sms);
int lora_apply(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
               int nsites, int r, int dtype, cudaStream_t stream, int num_sms);
int reft_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A, const void* B,
               const void* Bt, const void* bias, const void* scale, int r, int dtype, cudaStream_t stream,
               int num_sms);
int plan_num_sms();
int plan_record_cuda(cudaError_t e);
}  // namespace preft

struct PlanOp {
    int kind;  // 0 = lora group, 1 = reft
    int tag;
    const void* x;
    void* h;
    long long rows;
    long long ld;
    int width;
    int nsites;
    int r;
    int dtype;
    preft_lora_site_t sites[3];
    const void *A, *B, *Bt, *bias, *scale;
};

struct preft_plan {
    preft_meta_t meta;
    std::vector<PlanOp> ops;
    int timing_tag = -1;
    std::vector<cudaEvent_t> pool;  // start/end pairs
    size_t used = 0;
};

using namespace preft;

static int plan_launch(preft_plan* p, const PlanOp& op, cudaStream_t s, int sms) {
    if (op.kind == 0) return lora_apply(&p->meta, op.x, op.ld, op.width, op.sites, op.nsites, op.r, op.dtype, s, sms);
    return reft_apply(&p->meta, op.h, op.rows, op.ld, op.width, op.A, op.B, op.Bt, op.bias, op.scale, op.r, op.dtype, s, sms);
}

extern "C" {

preft_plan* preft_plan_create(const preft_meta_t* meta) {
    if (!meta) return nullptr;
    preft_plan* p = new preft_plan();
    p->meta = *meta;
    return p;
}

void preft_plan_destroy(preft_plan* p) {
    if (!p) return;
    for (cudaEvent_t e : p->pool) cudaEventDestroy(e);
    delete p;
}

int preft_plan_set_slot_split(preft_plan* p, int32_t split) {
    if (!p) return PREFT_ERR_STATE;
    p->meta.slot_split = split;
    return PREFT_OK;
}

int preft_plan_set_rows_hint(preft_plan* p, int32_t rows) {
    if (!p || rows < 0) return PREFT_ERR_STATE;
    p->meta.rows_hint = rows;
    return PREFT_OK;
}

int preft_plan_refresh_meta(preft_plan* p, const preft_meta_t* meta) {
    if (!p || !meta) return PREFT_ERR_STATE;
    const int32_t split = p->meta.slot_split, hint = p->meta.rows_hint;
    p->meta = *meta;
    p->meta.slot_split = split;
    p->meta.rows_hint = hint;
    return PREFT_OK;
}

int preft_plan_add_lora(preft_plan* p, const void* x, int64_t ldx, int32_t m, const preft_lora_site_t* sites,
                        int32_t nsites, int32_t r_max, int32_t dtype, int32_t tag) {
    if (!p || !sites || nsites < 1 || nsites > 3) return PREFT_ERR_SHAPE;
    PlanOp op{};
    op.kind = 0;
    op.tag = tag;
    op.x = x;
    op.ld = ldx;
    op.width = m;
    op.nsites = nsites;
    op.r = r_max;
    op.dtype = dtype;
    for (int i = 0; i < nsites; ++i) op.sites[i] = sites[i];
    p->ops.push_back(op);
    return PREFT_OK;
}

int preft_plan_add_reft(preft_plan* p, void* h, int64_t rows, int64_t ldh, int32_t d, const void* A, const void* B,
                        const void* Bt, const void* bias, const void* scale, int32_t r_max, int32_t dtype,
                        int32_t tag) {
    if (!p) return PREFT_ERR_SHAPE;
    PlanOp op{};
    op.kind = 1;
    op.tag = tag;
    op.h = h;
    op.rows = rows;
    op.ld = ldh;
    op.width = d;
    op.A = A;
    op.B = B;
    op.Bt = Bt;
    op.bias = bias;
    op.scale = scale;
    op.r = r_max;
    op.dtype = dtype;
    p->ops.push_back(op);
    return PREFT_OK;
}

int preft_plan_num_ops(const preft_plan* p) { return p ? static_cast<int>(p->ops.size()) : 0; }

// time launches whose tag == `tag` with CUDA events (-1 = off); reserve
// `reserve_pairs` event pairs up front so no event is created while timing
int preft_plan_set_timing(preft_plan* p, int32_t tag, int32_t reserve_pairs) {
    if (!p) return PREFT_ERR_STATE;
    p->timing_tag = tag;
    while (static_cast<int>(p->pool.size()) < 2 * reserve_pairs) {
        cudaEvent_t e;
        const cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) return plan_record_cuda(err);
        p->pool.push_back(e);
    }
    p->used = 0;
    return PREFT_OK;
}

// launch the whole step on `stream`: K1 (if run_meta) then every op in order
int preft_plan_run(preft_plan* p, int32_t run_meta, void* stream) {
    if (!p) return PREFT_ERR_STATE;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int sms = plan_num_sms();
    if (run_meta) {
        const int rc = meta_build(&p->meta, s, sms);
        if (rc) return rc < 0 ? plan_record_cuda(static_cast<cudaError_t>(-rc)) : rc;
    }
    // under stream capture the timing events become external event-record
    // nodes, re-recorded at every replay of the graph (so a graph of K steps
    // yields its K steps' launch times)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (p->timing_tag >= 0) cudaStreamIsCapturing(s, &cap);
    const unsigned rec_flags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : 0u;
    for (const PlanOp& op : p->ops) {
        const bool timed = p->timing_tag >= 0 && op.tag == p->timing_tag;
        if (timed) {
            if (p->used + 2 > p->pool.size()) return PREFT_ERR_STATE;  // reserve more pairs
            cudaEventRecordWithFlags(p->pool[p->used], s, rec_flags);
        }
        const int rc = plan_launch(p, op, s, sms);
        if (rc) return rc < 0 ? plan_record_cuda(static_cast<cudaError_t>(-rc)) : rc;
        if (timed) {
            cudaEventRecordWithFlags(p->pool[p->used + 1], s, rec_flags);
            p->used += 2;
        }
    }
    return PREFT_OK;
}

// wait for the recorded pairs, return their summed duration and count, reset
int preft_plan_collect_timing(preft_plan* p, double* total_ms, int32_t* count) {
    if (!p || !total_ms || !count) return PREFT_ERR_SHAPE;
    double sum = 0.0;
    for (size_t i = 0; i + 1 < p->used; i += 2) {
        cudaError_t e = cudaEventSynchronize(p->pool[i + 1]);
        if (e != cudaSuccess) return plan_record_cuda(e);
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, p->pool[i], p->pool[i + 1]);
        if (e != cudaSuccess) return plan_record_cuda(e);
        sum += ms;
    }
    *total_ms = sum;
    *count = static_cast<int32_t>(p->used / 2);
    p->used = 0;
    return PREFT_OK;
}

}  // extern "C"
