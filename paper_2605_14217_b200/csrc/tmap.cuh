// Host-side TMA tensor-map encoding (driver entry point fetched through the
// runtime, so libpreft does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

namespace preft {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// bf16 [rows x cols] row-major matrix with leading dimension ld (elements),
// boxes of box_rows x box_cols, 128-byte swizzle (box_cols * 2 == 128)
inline bool make_tmap_bf16_sw128(CUtensorMap* m, const void* base, unsigned long long rows, unsigned long long cols,
                                 unsigned long long ld, unsigned box_cols, unsigned box_rows) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The same matrix seen as [panels][rows][64 columns]: dim 0 = the 64 columns
// of a 128-byte panel, dim 1 = rows (stride ld), dim 2 = panels (stride 128 B).
// One box of {64, box_rows, box_panels} lands in shared memory as box_panels
// consecutive swizzled [box_rows][128 B] panels — the layout the 2D boxes
// build one panel at a time — so a 16-row x 256-column tile is ONE TMA
// instruction instead of four (per-instruction TMA issue cost bounds the
// short-unit tensor-core kernels).  cols % 64 == 0.
inline bool make_tmap_bf16_panels(CUtensorMap* m, const void* base, unsigned long long rows, unsigned long long cols,
                                  unsigned long long ld, unsigned box_rows, unsigned box_panels) {
    auto enc = tmap_encoder();
    if (!enc || cols % 64) return false;
    cuuint64_t dims[3] = {64, rows, cols / 64};
    cuuint64_t strides[2] = {ld * 2, 128};
    cuuint32_t box[3] = {64, box_rows, box_panels};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace preft
