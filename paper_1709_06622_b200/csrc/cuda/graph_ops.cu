// Graph operators for branched (Inception-style) networks, NHWC, bf16 / fp32:
//   slice_copy   strided channel-slice copy: concat forward (branch -> its
//                channel range of the concatenated tensor) and concat
//                backward (the range -> the branch's gradient)
//   avgpool2d    windowed average pool (count_include_pad: / f*f), forward and
//                an owner-computes backward (each input pixel sums the output
//                windows covering it — no atomics), optional fused ReLU mask
// All HBM-bound; 16-byte vectors over the channel axis where the layout allows.
#include <algorithm>

#include "common.cuh"

namespace tcb {
namespace {

constexpr int kBlock = 256;

inline int grid_for(size_t n, int per_thread = 1) {
    size_t blocks = (n + size_t(kBlock) * per_thread - 1) / (size_t(kBlock) * per_thread);
    return static_cast<int>(std::max<size_t>(1, std::min(blocks, size_t(num_sms()) * 16)));
}

template <typename T>
struct Vec {
    static constexpr int N = 16 / sizeof(T);
};

template <typename T>
__device__ __forceinline__ void load_vec(const T* p, float (&f)[Vec<T>::N]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int i = 0; i < Vec<T>::N; ++i) f[i] = to_f32<T>(e[i]);
}

template <typename T>
__device__ __forceinline__ void store_vec(T* p, const float (&f)[Vec<T>::N]) {
    uint4 u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int i = 0; i < Vec<T>::N; ++i) e[i] = from_f32<T>(f[i]);
    *reinterpret_cast<uint4*>(p) = u;
}

// rows x width elements, 16-byte chunks (all pitches / offsets in chunks)
__global__ void slice_copy_vec_kernel(const uint4* __restrict__ src, size_t src_pitch, uint4* __restrict__ dst,
                                      size_t dst_pitch, int width, size_t rows) {
    pdl_wait();
    pdl_trigger();
    const size_t total = rows * width;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / width;
        const int c = static_cast<int>(i - r * width);
        dst[r * dst_pitch + c] = src[r * src_pitch + c];
    }
}

// slice copy fused with a ReLU mask (bf16: the concat input's gradient is its
// channel slice of the concat gradient times [activation > 0]; one pass instead
// of a copy and an in-place mask). mask rows use the destination pitch.
__global__ void slice_copy_mask_bf16_kernel(const uint4* __restrict__ src, size_t src_pitch, uint4* __restrict__ dst,
                                            size_t dst_pitch, int width, size_t rows,
                                            const uint4* __restrict__ mask) {
    pdl_wait();
    pdl_trigger();
    const size_t total = rows * width;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / width;
        const int c = static_cast<int>(i - r * width);
        uint4 v = src[r * src_pitch + c];
        const uint4 m = __ldg(mask + r * dst_pitch + c);
        uint32_t* vw = reinterpret_cast<uint32_t*>(&v);
        const uint32_t* mw = reinterpret_cast<const uint32_t*>(&m);
        const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            vw[j] &= __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&mw[j]), zero2);
        dst[r * dst_pitch + c] = v;
    }
}

template <typename T>
__global__ void slice_copy_kernel(const T* __restrict__ src, size_t src_pitch, T* __restrict__ dst,
                                  size_t dst_pitch, int width, size_t rows) {
    const size_t total = rows * width;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / width;
        const int c = static_cast<int>(i - r * width);
        dst[r * dst_pitch + c] = src[r * src_pitch + c];
    }
}

struct PoolShape {
    int n, h, w, c, ho, wo, f, s, p;
};

// one thread per (output pixel, V channels). K3: 3x3 / stride 1 / pad 1 (the Inception branch
// pools) with the 9 window loads issued together (raw 16-byte vectors, converted while
// summing in the generic loop's order) instead of one dependent loop iteration each.
template <typename T, bool K3 = false>
__global__ void avgpool2d_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, PoolShape ps) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int cv = ps.c / V;
    const uint32_t total = static_cast<uint32_t>(size_t(ps.n) * ps.ho * ps.wo * cv);  // < 2^32 (host)
    const float inv = 1.f / static_cast<float>(ps.f * ps.f);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int cg = static_cast<int>(i % static_cast<uint32_t>(cv));
        uint32_t pix = i / static_cast<uint32_t>(cv);
        const int j = static_cast<int>(pix % static_cast<uint32_t>(ps.wo));
        pix /= static_cast<uint32_t>(ps.wo);
        const int oi = static_cast<int>(pix % static_cast<uint32_t>(ps.ho));
        const int b = static_cast<int>(pix / static_cast<uint32_t>(ps.ho));
        float acc[V] = {};
        if constexpr (K3) {
            uint4 raw[9];
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const int hh = oi - 1 + t / 3, ww = j - 1 + t % 3;
                raw[t] = (hh >= 0 && hh < ps.h && ww >= 0 && ww < ps.w)
                             ? __ldg(reinterpret_cast<const uint4*>(x + ((size_t(b) * ps.h + hh) * ps.w + ww) * ps.c +
                                                                    cg * V))
                             : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                const T* e8 = reinterpret_cast<const T*>(&raw[t]);
#pragma unroll
                for (int e = 0; e < V; ++e) acc[e] += to_f32<T>(e8[e]);
            }
        } else {
            for (int r = 0; r < ps.f; ++r) {
                const int hh = oi * ps.s - ps.p + r;
                if (hh < 0 || hh >= ps.h) continue;
                for (int q = 0; q < ps.f; ++q) {
                    const int ww = j * ps.s - ps.p + q;
                    if (ww < 0 || ww >= ps.w) continue;
                    float v[V];
                    load_vec(x + ((size_t(b) * ps.h + hh) * ps.w + ww) * ps.c + cg * V, v);
#pragma unroll
                    for (int e = 0; e < V; ++e) acc[e] += v[e];
                }
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] *= inv;
        store_vec(y + size_t(i) * V, acc);
    }
}

// one thread per (input pixel, V channels): sum of the covering windows' dy / f^2
template <typename T>
__global__ void avgpool2d_bwd_kernel(const T* __restrict__ dy, T* dx, PoolShape ps, const T* __restrict__ mask,
                                     const T* residual) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int cv = ps.c / V;
    const size_t total = size_t(ps.n) * ps.h * ps.w * cv;
    const float inv = 1.f / static_cast<float>(ps.f * ps.f);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int cg = static_cast<int>(i % cv);
        size_t pix = i / cv;
        const int ww = static_cast<int>(pix % ps.w);
        pix /= ps.w;
        const int hh = static_cast<int>(pix % ps.h);
        const int b = static_cast<int>(pix / ps.h);
        // windows oi with oi*s - p <= hh <= oi*s - p + f - 1
        const int i0 = max(0, (hh + ps.p - ps.f + ps.s) / ps.s), i1 = min(ps.ho - 1, (hh + ps.p) / ps.s);
        const int j0 = max(0, (ww + ps.p - ps.f + ps.s) / ps.s), j1 = min(ps.wo - 1, (ww + ps.p) / ps.s);
        float acc[V] = {};
        for (int oi = i0; oi <= i1; ++oi)
            for (int oj = j0; oj <= j1; ++oj) {
                float v[V];
                load_vec(dy + ((size_t(b) * ps.ho + oi) * ps.wo + oj) * ps.c + cg * V, v);
#pragma unroll
                for (int e = 0; e < V; ++e) acc[e] += v[e];
            }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] *= inv;
        if (residual) {  // may alias dx: read before the write below, same thread
            float r[V];
            load_vec(residual + i * V, r);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] += r[e];
        }
        if (mask) {
            float m[V];
            load_vec(mask + i * V, m);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] = m[e] > 0.f ? acc[e] : 0.f;
        }
        store_vec(dx + i * V, acc);
    }
}

// 3x3 / stride 1 / pad 1 average pool (Inception branch pools), one block per output row:
// the block's threads sweep (column, channel vector) of that row, so the 3 input rows its 9
// taps read stay in L1 (the flat grid-stride kernel spread a pixel's 9 readers over SMs and
// re-read every input vector 9 times from L2). Loads issued together; the generic kernel's
// summation order (rows, then columns).
template <typename T>
__global__ void __launch_bounds__(256) avgpool3_fwd_rows_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                                PoolShape ps) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int cv = ps.c / V;
    const int b = blockIdx.x / ps.ho, oi = blockIdx.x - b * ps.ho;
    const float inv = 1.f / 9.f;
    const T* xb = x + size_t(b) * ps.h * ps.w * ps.c;
    T* yr = y + size_t(blockIdx.x) * ps.wo * ps.c;
    for (int i = threadIdx.x; i < ps.wo * cv; i += blockDim.x) {
        const int j = i / cv, cg = i - j * cv;
        uint4 raw[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int hh = oi - 1 + t / 3, ww = j - 1 + t % 3;
            raw[t] = (hh >= 0 && hh < ps.h && ww >= 0 && ww < ps.w)
                         ? __ldg(reinterpret_cast<const uint4*>(xb + (size_t(hh) * ps.w + ww) * ps.c + cg * V))
                         : make_uint4(0, 0, 0, 0);
        }
        float acc[V] = {};
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const T* e8 = reinterpret_cast<const T*>(&raw[t]);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] += to_f32<T>(e8[e]);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] *= inv;
        store_vec(yr + size_t(i) * V, acc);
    }
}

// its backward, one block per input row: dx = [mask > 0] * (residual + sum of the 9
// covering windows' dy / 9), windows (oi, oj) in [h - 1, h + 1] x [w - 1, w + 1]
template <typename T>
__global__ void __launch_bounds__(256) avgpool3_bwd_rows_kernel(const T* __restrict__ dy, T* dx, PoolShape ps,
                                                                const T* __restrict__ mask, const T* residual) {
    pdl_wait();
    pdl_trigger();
    constexpr int V = Vec<T>::N;
    const int cv = ps.c / V;
    const int b = blockIdx.x / ps.h, hh = blockIdx.x - b * ps.h;
    const float inv = 1.f / 9.f;
    const T* db = dy + size_t(b) * ps.ho * ps.wo * ps.c;
    const size_t rbase = size_t(blockIdx.x) * ps.w * cv;  // this row's first vector
    for (int i = threadIdx.x; i < ps.w * cv; i += blockDim.x) {
        const int ww = i / cv, cg = i - ww * cv;
        uint4 raw[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int oi = hh - 1 + t / 3, oj = ww - 1 + t % 3;
            raw[t] = (oi >= 0 && oi < ps.ho && oj >= 0 && oj < ps.wo)
                         ? __ldg(reinterpret_cast<const uint4*>(db + (size_t(oi) * ps.wo + oj) * ps.c + cg * V))
                         : make_uint4(0, 0, 0, 0);
        }
        float acc[V] = {};
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const T* e8 = reinterpret_cast<const T*>(&raw[t]);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] += to_f32<T>(e8[e]);
        }
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] *= inv;
        const size_t o = (rbase + i) * V;
        if (residual) {  // may alias dx: read before the write below, same thread
            float r[V];
            load_vec(residual + o, r);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] += r[e];
        }
        if (mask) {
            float m[V];
            load_vec(mask + o, m);
#pragma unroll
            for (int e = 0; e < V; ++e) acc[e] = m[e] > 0.f ? acc[e] : 0.f;
        }
        store_vec(dx + o, acc);
    }
}

inline bool a16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }

}  // namespace

cudaError_t slice_copy(DType dt, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                       size_t rows, cudaStream_t st) {
    if (rows == 0 || width == 0) return cudaSuccess;
    const size_t es = dtype_size(dt), v = 16 / es;
    if (a16(src) && a16(dst) && src_pitch % v == 0 && dst_pitch % v == 0 && width % v == 0) {
        const int wv = static_cast<int>(width / v);
        return launch_pdl(slice_copy_vec_kernel, dim3(grid_for(rows * wv, 2)), dim3(kBlock), 0, st,
                          static_cast<const uint4*>(src), src_pitch / v, static_cast<uint4*>(dst), dst_pitch / v,
                          wv, rows);
    }
    if (dt == DType::F32)
        slice_copy_kernel<float><<<grid_for(rows * width, 2), kBlock, 0, st>>>(
            static_cast<const float*>(src), src_pitch, static_cast<float*>(dst), dst_pitch, width, rows);
    else
        slice_copy_kernel<__nv_bfloat16><<<grid_for(rows * width, 2), kBlock, 0, st>>>(
            static_cast<const __nv_bfloat16*>(src), src_pitch, static_cast<__nv_bfloat16*>(dst), dst_pitch,
            width, rows);
    return cudaGetLastError();
}

bool slice_copy_mask_supported(DType dt, const void* src, size_t src_pitch, const void* dst, size_t dst_pitch,
                               int width, const void* mask) {
    return dt == DType::BF16 && a16(src) && a16(dst) && a16(mask) && src_pitch % 8 == 0 && dst_pitch % 8 == 0 &&
           width % 8 == 0;
}

cudaError_t slice_copy_mask(DType dt, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                            size_t rows, const void* mask, cudaStream_t st) {
    if (!slice_copy_mask_supported(dt, src, src_pitch, dst, dst_pitch, width, mask)) return cudaErrorInvalidValue;
    if (rows == 0 || width == 0) return cudaSuccess;
    const int wv = width / 8;
    return launch_pdl(slice_copy_mask_bf16_kernel, dim3(grid_for(rows * wv, 2)), dim3(kBlock), 0, st,
                      static_cast<const uint4*>(src), src_pitch / 8, static_cast<uint4*>(dst), dst_pitch / 8, wv,
                      rows, static_cast<const uint4*>(mask));
}

bool avgpool2d_supported(DType dt, int c) { return c % static_cast<int>(16 / dtype_size(dt)) == 0; }

cudaError_t avgpool2d_fwd(DType dt, const void* x, void* y, int n, int h, int w, int c, int f, int s, int p,
                          cudaStream_t st) {
    if (!avgpool2d_supported(dt, c) || !a16(x) || !a16(y)) return cudaErrorInvalidValue;
    PoolShape ps{n, h, w, c, (h + 2 * p - f) / s + 1, (w + 2 * p - f) / s + 1, f, s, p};
    const size_t total = size_t(n) * ps.ho * ps.wo * c / (16 / dtype_size(dt));
    static const int env_k3 = [] { const char* e = getenv("TCB_AVGPOOL_K3"); return e ? atoi(e) : 2; }();
    const bool k3 = env_k3 != 0 && f == 3 && s == 1 && p == 1;
    if (k3 && env_k3 == 2) {  // one block per output row
        if (dt == DType::F32)
            return launch_pdl(avgpool3_fwd_rows_kernel<float>, dim3(n * ps.ho), dim3(256), 0, st,
                              static_cast<const float*>(x), static_cast<float*>(y), ps);
        return launch_pdl(avgpool3_fwd_rows_kernel<__nv_bfloat16>, dim3(n * ps.ho), dim3(256), 0, st,
                          static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), ps);
    }
    if (dt == DType::F32)
        return launch_pdl(k3 ? avgpool2d_fwd_kernel<float, true> : avgpool2d_fwd_kernel<float>,
                          dim3(grid_for(total, 2)), dim3(kBlock), 0, st, static_cast<const float*>(x),
                          static_cast<float*>(y), ps);
    return launch_pdl(k3 ? avgpool2d_fwd_kernel<__nv_bfloat16, true> : avgpool2d_fwd_kernel<__nv_bfloat16>,
                      dim3(grid_for(total, 2)), dim3(kBlock), 0, st, static_cast<const __nv_bfloat16*>(x),
                      static_cast<__nv_bfloat16*>(y), ps);
}

cudaError_t avgpool2d_bwd(DType dt, const void* dy, void* dx, int n, int h, int w, int c, int f, int s, int p,
                          cudaStream_t st, const void* mask, const void* residual) {
    if (!avgpool2d_supported(dt, c) || !a16(dy) || !a16(dx) || (mask && !a16(mask)) || (residual && !a16(residual)))
        return cudaErrorInvalidValue;
    PoolShape ps{n, h, w, c, (h + 2 * p - f) / s + 1, (w + 2 * p - f) / s + 1, f, s, p};
    const size_t total = size_t(n) * h * w * c / (16 / dtype_size(dt));
    static const int env_k3b = [] { const char* e = getenv("TCB_AVGPOOL_K3"); return e ? atoi(e) : 2; }();
    if (env_k3b == 2 && f == 3 && s == 1 && p == 1) {  // one block per input row
        if (dt == DType::F32)
            return launch_pdl(avgpool3_bwd_rows_kernel<float>, dim3(n * h), dim3(256), 0, st,
                              static_cast<const float*>(dy), static_cast<float*>(dx), ps,
                              static_cast<const float*>(mask), static_cast<const float*>(residual));
        return launch_pdl(avgpool3_bwd_rows_kernel<__nv_bfloat16>, dim3(n * h), dim3(256), 0, st,
                          static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx), ps,
                          static_cast<const __nv_bfloat16*>(mask), static_cast<const __nv_bfloat16*>(residual));
    }
    if (dt == DType::F32)
        return launch_pdl(avgpool2d_bwd_kernel<float>, dim3(grid_for(total, 2)), dim3(kBlock), 0, st,
                          static_cast<const float*>(dy), static_cast<float*>(dx), ps,
                          static_cast<const float*>(mask), static_cast<const float*>(residual));
    return launch_pdl(avgpool2d_bwd_kernel<__nv_bfloat16>, dim3(grid_for(total, 2)), dim3(kBlock), 0, st,
                      static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx), ps,
                      static_cast<const __nv_bfloat16*>(mask), static_cast<const __nv_bfloat16*>(residual));
}

}  // namespace tcb
