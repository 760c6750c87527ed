// Host-side TMA tensor-map construction (driver entry point resolved through
// the runtime, so libtcb.so does not link libcuda directly).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tcb {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Row-major bf16 matrix [rows][cols] (cols contiguous, cols % 8 == 0) read in
// boxes of box_rows x 64 columns with the 128-byte swizzle the UMMA K-major
// SW128 descriptor expects. Out-of-bounds rows/cols read as zero.
inline bool make_tmap_bf16_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols = 64,
                              CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_128B) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// `planes` contiguous row-major bf16 matrices [rows][cols] as one 3-D map
// (the plane index is the third coordinate), boxes of box_rows x box_cols x 1.
inline bool make_tmap_bf16_3d(CUtensorMap* map, const void* base, uint64_t planes, uint64_t rows, uint64_t cols,
                              uint32_t box_rows, uint32_t box_cols = 64) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {cols, rows, planes};
    const cuuint64_t strides[2] = {cols * 2, rows * cols * 2};
    const cuuint32_t box[3] = {box_cols, box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// KRSC bf16 filter bank viewed as [K][R*S][C] (C contiguous), read in boxes of
// 64 filters x 1 tap x 64 channels: an MN-major (channel-contiguous) 128B-
// swizzled operand tile for the dgrad GEMM, taken straight from the weights.
inline bool make_tmap_filters_bf16(CUtensorMap* map, const void* base, uint64_t k, uint64_t taps,
                                   uint64_t c) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {c, taps, k};
    const cuuint64_t strides[2] = {c * 2, taps * c * 2};
    const cuuint32_t box[3] = {64, 1, 64};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box,
              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC bf16 tensor [n][h][w][c] read in tiled boxes of 64 channels x bw pixels x
// bh rows x 1 image (128-byte swizzle): a conv "window" of whole padded input
// rows; out-of-image rows/columns (the padding) read as zero.
inline bool make_tmap_window_bf16(CUtensorMap* map, const void* base, int n, int h, int w, int c,
                                  uint32_t bw, uint32_t bh) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[4] = {cuuint64_t(c), cuuint64_t(w), cuuint64_t(h), cuuint64_t(n)};
    const cuuint64_t strides[3] = {cuuint64_t(c) * 2, cuuint64_t(w) * c * 2, cuuint64_t(h) * w * c * 2};
    const cuuint32_t box[4] = {64, bw, bh, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeIm2colFn encode_im2col_fn() {
    static EncodeIm2colFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeIm2colFn>(p);
    }
    return fn;
}

// im2col view of an NHWC bf16 tensor [n][h][w][c]: each load brings
// `pixels` consecutive filter-base positions (w fastest, then h, then n,
// inside the bounding box [lower, dim - 1 + upper] stepped by the traversal
// strides) x 64 channels, with the 128-byte swizzle; out-of-image taps read 0.
inline bool make_tmap_im2col_bf16(CUtensorMap* map, const void* base, int n, int h, int w, int c,
                                  int lower_w, int lower_h, int upper_w, int upper_h,
                                  int stride_w, int stride_h, uint32_t pixels,
                                  uint32_t channels = 64) {
    EncodeIm2colFn fn = encode_im2col_fn();
    if (!fn) return false;
    const cuuint64_t dims[4] = {cuuint64_t(c), cuuint64_t(w), cuuint64_t(h), cuuint64_t(n)};
    const cuuint64_t strides[3] = {cuuint64_t(c) * 2, cuuint64_t(w) * c * 2,
                                   cuuint64_t(h) * w * c * 2};
    const int lower[2] = {lower_w, lower_h};
    const int upper[2] = {upper_w, upper_h};
    const cuuint32_t estr[4] = {1, cuuint32_t(stride_w), cuuint32_t(stride_h), 1};
    // 64 channels = 128-byte rows (SWIZZLE_128B); 8 channels = 16-byte rows written
    // densely (no swizzle), i.e. UMMA "interleaved" 8x16B core matrices.
    const CUtensorMapSwizzle swz =
        channels * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lower,
           upper, channels, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    // Driver <= 13.1 mis-handles im2col maps of tensors under 128 KB unless bit 21
    // of descriptor word 1 is cleared (same workaround CUTLASS applies).
    int drv = 0;
    cudaDriverGetVersion(&drv);
    if (drv <= 13010 && size_t(n) * h * w * c * 2 < 131072)
        reinterpret_cast<uint64_t*>(map)[1] &= ~(uint64_t(1) << 21);
    return true;
}

// fp32 variants (the TF32 tensor-core mode: fp32 storage, tf32 math). 32
// fp32 = one 128-byte row. K-major operands use SWIZZLE_128B; MN-major ones
// SWIZZLE_128B_ATOM_32B (= the UMMA SWIZZLE_128B_BASE32B layout tf32 needs).
inline bool make_tmap_f32_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                             uint32_t box_rows, CUtensorMapSwizzle swizzle) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 4};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// KRSC fp32 filters as [K][R*S][C]: boxes of 32 channels x 1 tap x 32 filters,
// MN-major (channels along the 128-byte row) for the tf32 dgrad B operand
inline bool make_tmap_filters_f32(CUtensorMap* map, const void* base, uint64_t k, uint64_t taps, uint64_t c) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {c, taps, k};
    const cuuint64_t strides[2] = {c * 4, taps * c * 4};
    const cuuint32_t box[3] = {32, 1, 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// im2col view of an NHWC fp32 tensor: `pixels` filter-base positions x 32 channels
inline bool make_tmap_im2col_f32(CUtensorMap* map, const void* base, int n, int h, int w, int c, int lower_w,
                                 int lower_h, int upper_w, int upper_h, int stride_w, int stride_h,
                                 uint32_t pixels, CUtensorMapSwizzle swizzle, uint32_t channels = 32) {
    EncodeIm2colFn fn = encode_im2col_fn();
    if (!fn) return false;
    const cuuint64_t dims[4] = {cuuint64_t(c), cuuint64_t(w), cuuint64_t(h), cuuint64_t(n)};
    const cuuint64_t strides[3] = {cuuint64_t(c) * 4, cuuint64_t(w) * c * 4, cuuint64_t(h) * w * c * 4};
    const int lower[2] = {lower_w, lower_h};
    const int upper[2] = {upper_w, upper_h};
    const cuuint32_t estr[4] = {1, cuuint32_t(stride_w), cuuint32_t(stride_h), 1};
    if (fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, lower, upper,
           channels, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    int drv = 0;
    cudaDriverGetVersion(&drv);
    if (drv <= 13010 && size_t(n) * h * w * c * 4 < 131072)
        reinterpret_cast<uint64_t*>(map)[1] &= ~(uint64_t(1) << 21);
    return true;
}

}  // namespace tcb
