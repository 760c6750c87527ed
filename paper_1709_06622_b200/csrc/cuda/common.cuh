// Shared device helpers: fast integer division, the implicit-GEMM view of a
// convolution, dtype load/store, launch checks.
#pragma once
#include <utility>

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tcb/kernels.h"

namespace tcb {

// Unsigned division by a runtime constant via multiply-high (Granlund-Montgomery).
struct FastDiv {
    uint32_t d = 1, mul = 0, shr = 0;
    FastDiv() = default;
    __host__ explicit FastDiv(uint32_t divisor) : d(divisor) {
        if (d == 1) {
            mul = 0;
            shr = 0;
            return;
        }
        uint32_t l = 0;
        while ((1ull << l) < d) ++l;
        shr = l - 1;
        mul = static_cast<uint32_t>(((1ull << 32) * ((1ull << l) - d)) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(n, mul);
        return (t + ((n - t) >> 1)) >> shr;
    }
    __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
        q = div(n);
        r = n - q * d;
    }
};

// Implicit-GEMM view of one convolution pass. For every mode the GEMM is
//   D[m, j] = sum_kk A[m, kk] * B[j, kk]
//   Fwd  : m = output pixel (n,ho,wo), j = out channel k,  kk = (r,s,c)
//   Dgrad: m = input pixel  (n,h,w),   j = in channel c,   kk = (r,s,k)
//   Wgrad: m = out channel k,          j = (r,s,c),        kk = output pixel
struct ConvShape {
    int N, H, W, C, K, R, S, ph, pw, sh, sw, Ho, Wo;
    int M, Ncol, Kdim;
    FastDiv d_howo, d_wo, d_hw, d_w, d_c, d_k, d_s;
};

inline ConvShape make_shape(const ConvGeom& g, ConvMode mode) {
    ConvShape s{};
    s.N = g.n; s.H = g.h; s.W = g.w; s.C = g.c; s.K = g.k; s.R = g.r; s.S = g.s;
    s.ph = g.pad_h; s.pw = g.pad_w; s.sh = g.stride_h; s.sw = g.stride_w;
    s.Ho = (g.h + 2 * g.pad_h - g.r) / g.stride_h + 1;
    s.Wo = (g.w + 2 * g.pad_w - g.s) / g.stride_w + 1;
    const int P = g.n * s.Ho * s.Wo;
    if (mode == ConvMode::Fwd) {
        s.M = P; s.Ncol = g.k; s.Kdim = g.r * g.s * g.c;
    } else if (mode == ConvMode::Dgrad) {
        s.M = g.n * g.h * g.w; s.Ncol = g.c; s.Kdim = g.r * g.s * g.k;
    } else {
        s.M = g.k; s.Ncol = g.r * g.s * g.c; s.Kdim = P;
    }
    s.d_howo = FastDiv(static_cast<uint32_t>(s.Ho * s.Wo));
    s.d_wo = FastDiv(static_cast<uint32_t>(s.Wo));
    s.d_hw = FastDiv(static_cast<uint32_t>(g.h * g.w));
    s.d_w = FastDiv(static_cast<uint32_t>(g.w));
    s.d_c = FastDiv(static_cast<uint32_t>(g.c));
    s.d_k = FastDiv(static_cast<uint32_t>(g.k));
    s.d_s = FastDiv(static_cast<uint32_t>(g.s));
    return s;
}

// Strided dgrad, sub-pixel decomposition: input pixels (h, w) with
// h % sh == ph, w % sw == pw receive gradient only from filter taps
// r ≡ (ph + pad_h) (mod sh), s ≡ (pw + pad_w) (mod sw). Each phase is a dense
// implicit GEMM over its own pixel grid (Hq x Wq) and tap subset (tr x ts),
// with its weights packed as [C][tr][ts][K] at element offset woff.
struct DgradPhase {
    int ph, pw, r0, s0, tr, ts, bh, bw, Hq, Wq;
    size_t woff;
};

__host__ __device__ inline DgradPhase dgrad_phase(const ConvGeom& g, int ph, int pw) {
    DgradPhase d{};
    d.ph = ph;
    d.pw = pw;
    d.r0 = (ph + g.pad_h) % g.stride_h;
    d.s0 = (pw + g.pad_w) % g.stride_w;
    d.tr = d.r0 < g.r ? (g.r - 1 - d.r0) / g.stride_h + 1 : 0;
    d.ts = d.s0 < g.s ? (g.s - 1 - d.s0) / g.stride_w + 1 : 0;
    d.bh = (ph + g.pad_h - d.r0) / g.stride_h;
    d.bw = (pw + g.pad_w - d.s0) / g.stride_w;
    d.Hq = ph < g.h ? (g.h - ph + g.stride_h - 1) / g.stride_h : 0;
    d.Wq = pw < g.w ? (g.w - pw + g.stride_w - 1) / g.stride_w : 0;
    size_t off = 0;
    for (int q = 0; q < ph * g.stride_w + pw; ++q) {
        const int qh = q / g.stride_w, qw = q % g.stride_w;
        const int r0 = (qh + g.pad_h) % g.stride_h, s0 = (qw + g.pad_w) % g.stride_w;
        const int tr = r0 < g.r ? (g.r - 1 - r0) / g.stride_h + 1 : 0;
        const int ts = s0 < g.s ? (g.s - 1 - s0) / g.stride_w + 1 : 0;
        off += size_t(g.c) * g.k * tr * ts;
    }
    d.woff = off;
    return d;
}

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
    return __bfloat162float(v);
}

template <typename T>
__device__ __forceinline__ T from_f32(float v);
template <>
__device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
    return __float2bfloat16_rn(v);
}

inline int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}


// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains and must call pdl_wait() before touching
// anything the predecessor wrote.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace tcb
