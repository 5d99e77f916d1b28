// extern "C" surface of libpreft (declared in include/preft.h) and K4, the
// f64 -> pool-slab conversion used by adapter registration / weight sync.
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"

namespace preft {

int meta_build(const preft_meta_t* m, cudaStream_t stream, int num_sms);
int lora_apply(const preft_meta_t* meta, const void* x, long long ldx, int m, const preft_lora_site_t* sites,
               int nsites, int r, int dtype, cudaStream_t stream, int num_sms);
int reft_apply(const preft_meta_t* meta, void* h, long long rows, long long ldh, int d, const void* A, const void* B,
               const void* Bt, const void* bias, const void* scale, int r, int dtype, cudaStream_t stream,
               int num_sms);
void set_reft_variant(int v);
void set_split_variant(int v);
void split_set_profile(long long* buf);
long long lora_part_floats_needed(const preft_meta_t* meta);
int lora_shrink(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
                const preft_lora_site_t* sites, int nsites, int r, int dtype, void* P, long long ldp,
                cudaStream_t stream, int num_sms);
int lora_expand(const preft_meta_t* meta, const void* P, long long ldp, long long rows, const preft_lora_site_t* sites,
                int nsites, int r, int dtype, cudaStream_t stream, int num_sms);
int reft_tc_last_grid();
long long xchg_region_bytes(int tp, int planes, int T_cap, int U_cap);
int xchg_init(preft_xchg_t* xg, void* const* bases, int tp, int rank, int planes, int T_cap, int U_cap, int peer_sys);
int lora_fused(const preft_meta_t* meta, const void* x, long long rows, long long ldx, int m,
               const preft_lora_site_t* sites, int nsites, int r, int dtype, const preft_xchg_t* xg,
               cudaStream_t stream, int num_sms);
int xchg_errors(const preft_xchg_t* xg, cudaStream_t stream, int* out);
void reft_tc_set_profile(long long* buf);
void reft_tc_set_flags(int flags, int look);

// programmatic dependent launch of the tensor-core kernels (PREFT_PDL=0 disables)
bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("PREFT_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

static thread_local char g_last_cuda_error[256] = "";

static int record_cuda(cudaError_t e) {
    snprintf(g_last_cuda_error, sizeof(g_last_cuda_error), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
    return PREFT_ERR_CUDA;
}

// kernel launch helpers return 0, a PREFT_ERR_* code (> 0) or -cudaError_t
static int finish(int rc) {
    if (rc < 0) return record_cuda(static_cast<cudaError_t>(-rc));
    return rc;
}

static int current_num_sms() {
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) sms = 148;
    cache[dev] = sms;
    return sms;
}

// persistent grid: SM count x resident CTAs per SM for this kernel
int grid_for(const void* fn, int threads, int num_sms) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(fn);
        if (it != cache.end()) per_sm = it->second;
    }
    if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        std::lock_guard<std::mutex> lock(mu);
        cache[fn] = per_sm;
    }
    return num_sms * per_sm;
}

void set_lora_variant(int v);
int tc_selftest(const void* A, const void* B, float* D, int K, int N, int mode, cudaStream_t s);
int plan_num_sms() { return current_num_sms(); }
int plan_record_cuda(cudaError_t e) { return record_cuda(e); }

template <typename T>
__device__ __forceinline__ T cvt_from_f64(double v);
template <>
__device__ __forceinline__ float cvt_from_f64<float>(double v) {
    return __double2float_rn(v);
}
template <>
__device__ __forceinline__ double cvt_from_f64<double>(double v) {
    return v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_from_f64<__nv_bfloat16>(double v) {
    // single rounding f64 -> bf16 (round to nearest even), no double rounding via f32
    return __double2bfloat16(v);
}

template <typename T>
__global__ void convert_2d_kernel(T* dst, long long dst_ld, const double* src, long long srow, long long scol,
                                  long long rows_valid, long long rows, long long cols) {
    const long long total = rows * cols;
    for (long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = idx / cols, j = idx % cols;
        const double v = i < rows_valid ? src[i * srow + j * scol] : 0.0;
        dst[i * dst_ld + j] = cvt_from_f64<T>(v);
    }
}

}  // namespace preft

using namespace preft;

extern "C" {

int preft_abi_version(void) { return PREFT_ABI_VERSION; }

const char* preft_status_string(int status) {
    switch (status) {
        case PREFT_OK: return "ok";
        case PREFT_ERR_SHAPE: return "ShapeError";
        case PREFT_ERR_RANK: return "RankError";
        case PREFT_ERR_DOMAIN: return "DomainError";
        case PREFT_ERR_CONFIG: return "ConfigError";
        case PREFT_ERR_BATCH: return "BatchError";
        case PREFT_ERR_STATE: return "StateError";
        case PREFT_ERR_SYNC: return "SyncError";
        case PREFT_ERR_INFEASIBLE: return "InfeasibleBatchError";
        case PREFT_ERR_CUDA: return "CudaError";
        default: return "unknown";
    }
}

const char* preft_last_cuda_error(void) { return g_last_cuda_error; }

int preft_num_sms(void) { return current_num_sms(); }

int preft_tc_selftest(const void* A, const void* B, float* D, int32_t K, int32_t N, int32_t mode, void* stream) {
    return finish(tc_selftest(A, B, D, K, N, mode, static_cast<cudaStream_t>(stream)));
}

int preft_set_lora_variant(int32_t variant) {
    if (variant != -1 && variant != 0 && variant != 1 && variant != 2 && variant != 4 && variant != 8)
        return PREFT_ERR_DOMAIN;
    set_lora_variant(variant);
    return PREFT_OK;
}

size_t preft_meta_entries_words(int32_t E_cap) { return 2 + static_cast<size_t>(E_cap) * 3 + 1; }

int preft_meta_build(const preft_meta_t* meta, void* stream) {
    if (!meta || !meta->entries || !meta->mask || !meta->tokens || !meta->segments || !meta->tiles ||
        !meta->entry_offset || !meta->counters || !meta->chunks || !meta->units)
        return PREFT_ERR_SHAPE;
    if (meta->E_cap < 1 || meta->E_cap > PREFT_MAX_ENTRIES || meta->T_cap < 1 || meta->tile_tokens < 1)
        return PREFT_ERR_CONFIG;
    if (static_cast<long long>(meta->tile_cap) <
        static_cast<long long>(meta->E_cap) + meta->T_cap / meta->tile_tokens + 1)
        return PREFT_ERR_CONFIG;
    if (static_cast<long long>(meta->chunk_cap) <
        static_cast<long long>(meta->E_cap) + meta->T_cap / PREFT_CHUNK_ROWS + 1)
        return PREFT_ERR_CONFIG;
    return finish(meta_build(meta, static_cast<cudaStream_t>(stream), current_num_sms()));
}

int preft_lora_apply(const preft_meta_t* meta, const void* x, int64_t ldx, int32_t m, const preft_lora_site_t* sites,
                     int32_t nsites, int32_t r_max, int32_t dtype, void* stream) {
    return finish(lora_apply(meta, x, ldx, m, sites, nsites, r_max, dtype, static_cast<cudaStream_t>(stream),
                             current_num_sms()));
}

int preft_reft_apply(const preft_meta_t* meta, void* h, int64_t rows, int64_t ldh, int32_t d, const void* A, const void* B,
                     const void* Bt, const void* bias, const void* scale, int32_t r_max, int32_t dtype, void* stream) {
    return finish(reft_apply(meta, h, rows, ldh, d, A, B, Bt, bias, scale, r_max, dtype, static_cast<cudaStream_t>(stream),
                             current_num_sms()));
}

int preft_lora_shrink(const preft_meta_t* meta, const void* x, int64_t rows, int64_t ldx, int32_t m,
                      const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype, void* P,
                      int64_t ldp, void* stream) {
    return finish(lora_shrink(meta, x, rows, ldx, m, sites, nsites, r_max, dtype, P, ldp,
                              static_cast<cudaStream_t>(stream), current_num_sms()));
}

int preft_lora_expand(const preft_meta_t* meta, const void* P, int64_t ldp, int64_t rows,
                      const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype, void* stream) {
    return finish(lora_expand(meta, P, ldp, rows, sites, nsites, r_max, dtype, static_cast<cudaStream_t>(stream),
                              current_num_sms()));
}

int64_t preft_xchg_region_bytes(int32_t tp_size, int32_t planes, int32_t T_cap, int32_t U_cap) {
    if (tp_size < 1 || tp_size > PREFT_XCHG_MAX_TP || planes < 1 || T_cap < 1 || U_cap < 1) return 0;
    return xchg_region_bytes(tp_size, planes, T_cap, U_cap);
}

int preft_xchg_init(preft_xchg_t* xg, void* const* region_bases, int32_t tp_size, int32_t tp_rank, int32_t planes,
                    int32_t T_cap, int32_t U_cap, int32_t peer_sys) {
    return xchg_init(xg, region_bases, tp_size, tp_rank, planes, T_cap, U_cap, peer_sys);
}

int preft_lora_fused(const preft_meta_t* meta, const void* x, int64_t rows, int64_t ldx, int32_t m,
                     const preft_lora_site_t* sites, int32_t nsites, int32_t r_max, int32_t dtype,
                     const preft_xchg_t* xchg, void* stream) {
    return finish(lora_fused(meta, x, rows, ldx, m, sites, nsites, r_max, dtype, xchg,
                             static_cast<cudaStream_t>(stream), current_num_sms()));
}

int preft_xchg_errors(const preft_xchg_t* xchg, void* stream, int32_t* out) {
    return finish(xchg_errors(xchg, static_cast<cudaStream_t>(stream), out));
}

int preft_dev_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 1) return PREFT_ERR_SHAPE;
    *out = nullptr;
    cudaError_t e = cudaMalloc(out, static_cast<size_t>(bytes));
    if (e == cudaSuccess) e = cudaMemset(*out, 0, static_cast<size_t>(bytes));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    return e == cudaSuccess ? PREFT_OK : record_cuda(e);
}

int preft_dev_free(void* p) {
    const cudaError_t e = cudaFree(p);
    return e == cudaSuccess ? PREFT_OK : record_cuda(e);
}

int preft_ipc_handle(void* dev_ptr, void* handle_out) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (!dev_ptr || !handle_out) return PREFT_ERR_SHAPE;
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
    if (e != cudaSuccess) return record_cuda(e);
    memcpy(handle_out, &h, sizeof(h));
    return PREFT_OK;
}

int preft_ipc_open(const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return PREFT_ERR_SHAPE;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    const cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? PREFT_OK : record_cuda(e);
}

int preft_ipc_close(void* dev_ptr) {
    const cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? PREFT_OK : record_cuda(e);
}

int64_t preft_lora_part_floats(const preft_meta_t* meta) {
    return meta ? lora_part_floats_needed(meta) : 0;
}

int preft_diag_split(long long* device_buffer) {
    split_set_profile(device_buffer);
    return PREFT_OK;
}

int preft_set_split_variant(int32_t variant) {
    if (variant < -1 || variant > 1) return PREFT_ERR_DOMAIN;
    set_split_variant(variant);
    return PREFT_OK;
}

int preft_diag_reft_tc(long long* device_buffer) {
    reft_tc_set_profile(device_buffer);
    return reft_tc_last_grid();
}

int preft_set_reft_tc_flags(int32_t flags, int32_t look) {
    if (flags < -1 || flags > 127) return PREFT_ERR_DOMAIN;
    reft_tc_set_flags(flags, look);
    return PREFT_OK;
}

int preft_set_reft_variant(int32_t variant) {
    if (variant < -1 || variant > 3) return PREFT_ERR_DOMAIN;
    set_reft_variant(variant);
    return PREFT_OK;
}

int preft_convert_2d(void* dst, int32_t dst_dtype, int64_t dst_ld, const double* src, int64_t src_stride_row,
                     int64_t src_stride_col, int64_t rows_valid, int64_t rows, int64_t cols, void* stream) {
    if (!dst || (!src && rows_valid > 0) || rows < 0 || cols < 0 || rows_valid < 0 || rows_valid > rows ||
        dst_ld < cols)
        return PREFT_ERR_SHAPE;
    if (rows == 0 || cols == 0) return PREFT_OK;
    const long long total = rows * cols;
    const int threads = 256;
    const int grid = static_cast<int>(min(static_cast<long long>(current_num_sms()) * 8, (total + threads - 1) / threads));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dst_dtype == PREFT_DTYPE_BF16)
        convert_2d_kernel<__nv_bfloat16><<<grid, threads, 0, s>>>(static_cast<__nv_bfloat16*>(dst), dst_ld, src,
                                                                  src_stride_row, src_stride_col, rows_valid, rows, cols);
    else if (dst_dtype == PREFT_DTYPE_F32)
        convert_2d_kernel<float><<<grid, threads, 0, s>>>(static_cast<float*>(dst), dst_ld, src, src_stride_row,
                                                          src_stride_col, rows_valid, rows, cols);
    else if (dst_dtype == PREFT_DTYPE_F64)
        convert_2d_kernel<double><<<grid, threads, 0, s>>>(static_cast<double*>(dst), dst_ld, src, src_stride_row,
                                                           src_stride_col, rows_valid, rows, cols);
    else
        return PREFT_ERR_DOMAIN;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PREFT_OK : record_cuda(e);
}

}  // extern "C"
