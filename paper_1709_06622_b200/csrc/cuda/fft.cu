// FFT convolution family (stride 1, filters up to 8x8), the "fft" algorithm
// token of the reference catalog (/root/reference/proj/fixtures/alexnet_profile.csv).
//
// Overlap-save on 8x8 tiles: each tile of (8-R+1) x (8-S+1) outputs reads an
// 8x8 input patch. Per tile and channel the patch is real-FFT'd to 8x5
// complex bins (Hermitian half), held as two planes [bin][tile][Re C | Im C].
// Cross-correlation is X * conj(W) per bin; with real GEMMs this is
//     [Yr | Yi] = [Xr | Xi] * B^T,   B = [[Wr, Wi], [-Wi, Wr]]   (2K x 2C)
// i.e. 40 GEMMs [T x 2C] x [2C x 2K] on the tcgen05 kernel (plain-TMA mode)
// in bf16, or the FFMA kernel in fp32. The inverse real FFT keeps the first
// (8-R+1) x (8-S+1) outputs and applies the fused epilogue.
//   dgrad: the same algorithm on dy with the flipped, transposed filter.
//   wgrad: DW = sum_t X_t * conj(DY_t) per bin as a reduction GEMM over tiles
//          ([Re|Im] quadrants of [DYr|DYi]^T [Xr|Xi]), then an inverse FFT.
// The transforms are smem-free register DFTs (radix-8 matrices of the
// constant twiddles), one (tile, channel) per thread so NHWC accesses are
// coalesced across channels; they are HBM-bound.
#include <algorithm>

#include "common.cuh"

namespace tcb {
namespace {

constexpr int F = 8;          // FFT tile edge
constexpr int NB = F * (F / 2 + 1);  // 40 bins
constexpr int kBlock = 128;

inline int grid_of(size_t n) {
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>((n + kBlock - 1) / kBlock,
                                                                 size_t(num_sms()) * 64)));
}

__device__ __forceinline__ float cs(int k) {  // cos(2*pi*k/8)
    const float c[8] = {1.f, 0.70710678118654752f, 0.f, -0.70710678118654752f,
                        -1.f, -0.70710678118654752f, 0.f, 0.70710678118654752f};
    return c[k & 7];
}
__device__ __forceinline__ float sn(int k) {  // sin(2*pi*k/8)
    return cs(k - 2);
}

// Forward real 2-D DFT of an 8x8 patch -> re/im[u][v], u in [0,8), v in [0,5).
__device__ __forceinline__ void rfft8x8(const float (&x)[F][F], float (&re)[F][5], float (&im)[F][5]) {
    float rr[F][5], ri[F][5];
#pragma unroll
    for (int a = 0; a < F; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            float sr = 0.f, si = 0.f;
#pragma unroll
            for (int b = 0; b < F; ++b) {
                sr += x[a][b] * cs(v * b);
                si -= x[a][b] * sn(v * b);
            }
            rr[a][v] = sr;
            ri[a][v] = si;
        }
#pragma unroll
    for (int u = 0; u < F; ++u)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            float sr = 0.f, si = 0.f;
#pragma unroll
            for (int a = 0; a < F; ++a) {
                const float c = cs(u * a), s = -sn(u * a);  // e^{-i 2pi ua/8}
                sr += rr[a][v] * c - ri[a][v] * s;
                si += rr[a][v] * s + ri[a][v] * c;
            }
            re[u][v] = sr;
            im[u][v] = si;
        }
}

// Inverse: x[a][b] for a < OA, b < OB from the Hermitian half (scaled 1/64).
template <int OA, int OB>
__device__ __forceinline__ void irfft8x8(const float (&re)[F][5], const float (&im)[F][5],
                                         float (&x)[OA][OB]) {
    float cr[OA][5], ci[OA][5];  // inverse along u for the needed rows
#pragma unroll
    for (int a = 0; a < OA; ++a)
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            float sr = 0.f, si = 0.f;
#pragma unroll
            for (int u = 0; u < F; ++u) {
                const float c = cs(u * a), s = sn(u * a);
                sr += re[u][v] * c - im[u][v] * s;
                si += re[u][v] * s + im[u][v] * c;
            }
            cr[a][v] = sr;
            ci[a][v] = si;
        }
#pragma unroll
    for (int a = 0; a < OA; ++a)
#pragma unroll
        for (int b = 0; b < OB; ++b) {
            float s = cr[a][0] + cr[a][4] * ((b & 1) ? -1.f : 1.f);
#pragma unroll
            for (int v = 1; v < 4; ++v) s += 2.f * (cr[a][v] * cs(v * b) - ci[a][v] * sn(v * b));
            x[a][b] = s * (1.f / 64.f);
        }
}

struct FTiles {
    int n, h, w, c, k;  // source tensor and destination channels
    int r, s, ph, pw;   // filter and padding of this (possibly transposed) conv
    int ho, wo, oa, ob; // output extents, per-tile output size
    int th, tw;
    size_t T;
};

FTiles make_ftiles(int n, int h, int w, int c, int k, int r, int s, int ph, int pw) {
    FTiles t{};
    t.n = n; t.h = h; t.w = w; t.c = c; t.k = k; t.r = r; t.s = s; t.ph = ph; t.pw = pw;
    t.ho = h + 2 * ph - r + 1;
    t.wo = w + 2 * pw - s + 1;
    t.oa = F - r + 1;
    t.ob = F - s + 1;
    t.th = (t.ho + t.oa - 1) / t.oa;
    t.tw = (t.wo + t.ob - 1) / t.ob;
    t.T = size_t(n) * t.th * t.tw;
    return t;
}

__device__ __forceinline__ void tile_of(const FTiles& tl, size_t t, int& n, int& i, int& j) {
    j = int(t % tl.tw);
    i = int((t / tl.tw) % tl.th);
    n = int(t / (size_t(tl.tw) * tl.th));
}

// ------------------------------------------------ warp-cooperative transforms ---
// One block per (tile, 64-channel slice), 256 threads = 32 lane groups of 8:
// group g owns channel pair g of the slice, lane a of the group owns patch
// row a. The 8x8 patch x 64 channels is staged in shared memory by 16-byte
// coalesced loads; each lane runs the 8-point real FFT of its row in
// registers (radix 2: two 4-point DFTs + twiddles), then the 8-point complex
// FFT down each of the 5 Hermitian columns runs ACROSS the group's lanes with
// warp shuffles (decimation in frequency, 3 butterfly stages); lane a ends
// with frequency row bitrev(a). The 40 bins are re-staged in shared memory and
// leave as 128-byte coalesced rows of the [bin][tile][Re c | Im c] planes.
// Channel pairs travel as float2 through packed sm_100 fp32x2 arithmetic
// (FADD2 / FMUL2 / FFMA2: one instruction for both channels).
struct Cx {
    float2 r, i;
};

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float b) { return __fmul2_rn(a, f2(b)); }
__device__ __forceinline__ float2 fma2(float2 a, float b, float2 c) { return __ffma2_rn(a, f2(b), c); }

// z * (wr + i wi)
__device__ __forceinline__ Cx cmul(Cx z, float wr, float wi) {
    return {__ffma2_rn(z.r, f2(wr), __fmul2_rn(z.i, f2(-wi))), __ffma2_rn(z.r, f2(wi), __fmul2_rn(z.i, f2(wr)))};
}

// X[v], v = 0..4, of a real 8-point sequence (forward, e^{-2 pi i v b / 8}),
// radix 2: the 4-point DFTs of the even and odd samples plus the twiddles
__device__ __forceinline__ void rfft8(const float2 (&x)[8], Cx (&X)[5]) {
    const float s = 0.70710678118654752f;
    const float2 z = f2(0.f);
    const float2 e02p = add2(x[0], x[4]), e02m = sub2(x[0], x[4]), e13p = add2(x[2], x[6]), e13m = sub2(x[2], x[6]);
    const float2 o02p = add2(x[1], x[5]), o02m = sub2(x[1], x[5]), o13p = add2(x[3], x[7]), o13m = sub2(x[3], x[7]);
    const float2 E0 = add2(e02p, e13p), E2 = sub2(e02p, e13p);
    const float2 O0 = add2(o02p, o13p), O2 = sub2(o02p, o13p);
    // E1 = e02m - i e13m, O1 = o02m - i o13m, E3 = conj(E1), O3 = conj(O1)
    X[0] = {add2(E0, O0), z};
    // W8^1 O1 = (s - i s)(o02m - i o13m) = s (o02m - o13m) - i s (o02m + o13m)
    X[1] = {fma2(sub2(o02m, o13m), s, e02m), sub2(mul2(add2(o02m, o13m), -s), e13m)};
    X[2] = {E2, make_float2(-O2.x, -O2.y)};
    // W8^3 O3 = (-s - i s)(o02m + i o13m) = s (o13m - o02m) - i s (o02m + o13m)
    X[3] = {fma2(sub2(o13m, o02m), s, e02m), fma2(add2(o02m, o13m), -s, e13m)};
    X[4] = {sub2(E0, O0), z};
}

__device__ __forceinline__ float2 shfl2(float2 v, int m) {
    return make_float2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// Per-lane twiddles of the 3 decimation-in-frequency stages (span 4, 2, 1):
// the upper lane of a butterfly scales (partner - self) by W_{2h}^(a mod h).
struct LaneTw {
    float wr[3], wi[3];
    bool upper[3];
};

__device__ __forceinline__ LaneTw lane_twiddles(int a, float sign) {
    const float s = 0.70710678118654752f;
    LaneTw t;
    const int k4 = a & 3;
    t.upper[0] = a & 4;
    t.wr[0] = k4 == 0 ? 1.f : k4 == 1 ? s : k4 == 2 ? 0.f : -s;
    t.wi[0] = sign * (k4 == 0 ? 0.f : k4 == 2 ? 1.f : s);
    t.upper[1] = a & 2;
    t.wr[1] = (a & 1) ? 0.f : 1.f;
    t.wi[1] = (a & 1) ? sign : 0.f;
    t.upper[2] = a & 1;
    t.wr[2] = 1.f;
    t.wi[2] = 0.f;
    return t;
}

// 8-point complex FFT across the 8 lanes of a group (lane bits 0..2),
// decimation in frequency, unscaled, branch-free; lane a ends with bin bitrev(a).
__device__ __forceinline__ Cx lane_fft8(Cx v, const LaneTw& tw) {
#pragma unroll
    for (int st = 0; st < 3; ++st) {
        const int h = 4 >> st;
        const Cx p = {shfl2(v.r, h), shfl2(v.i, h)};
        if (tw.upper[st]) {
            v = cmul({sub2(p.r, v.r), sub2(p.i, v.i)}, tw.wr[st], tw.wi[st]);
        } else {
            v = {add2(v.r, p.r), add2(v.i, p.i)};
        }
    }
    return v;
}

__device__ __forceinline__ int bitrev3(int a) { return ((a & 1) << 2) | (a & 2) | ((a >> 2) & 1); }

template <typename T>
__device__ __forceinline__ float2 ld_pair(const T* p) {
    if constexpr (sizeof(T) == 2) return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p));
    else return *reinterpret_cast<const float2*>(p);
}
template <typename T>
__device__ __forceinline__ void st_pair(T* p, float2 v) {
    if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat162*>(p) = __floats2bfloat162_rn(v.x, v.y);
    else *reinterpret_cast<float2*>(p) = v;
}

// Forward transform of a patch: the source patch is rows a0..a0+7, cols
// b0..b0+7 of tensor src [n][hs][ws][c] with only rows < lim_a / cols < lim_b
// of the patch (and inside the tensor) taken, zero elsewhere.
template <typename T>
__global__ void __launch_bounds__(256) fft_fwd_smem_kernel(const T* __restrict__ src, T* __restrict__ out,
                                                           FTiles tl, int hs, int ws, int cs, int origin_scale_a,
                                                           int origin_scale_b, int off_a, int off_b, int lim_a,
                                                           int lim_b) {
    // row pads of 16 bytes keep the 8 lanes of a group (8 patch rows / 8
    // frequency rows) on different banks
    constexpr int PE = 16 / sizeof(T);
    constexpr int PROW = F * 64 + PE;  // patch row stride (elements)
    constexpr int BROW = 64 + PE;      // bin row stride; rows ordered [v][Re|Im][u]
    __shared__ __align__(16) T patch[F * PROW];
    __shared__ __align__(16) T bins[NB * 2 * BROW];
    const size_t t = blockIdx.x;
    const int c0 = blockIdx.y * 64;
    const int cw = min(64, cs - c0);
    int n, i, j;
    tile_of(tl, t, n, i, j);
    const int a0 = i * origin_scale_a - off_a, b0 = j * origin_scale_b - off_b;
    constexpr int VE = 16 / sizeof(T);
    const int vpp = cw / VE;
    for (int idx = threadIdx.x; idx < F * F * vpp; idx += blockDim.x) {
        const int v = idx % vpp, pix = idx / vpp;
        const int a = pix / F, b = pix % F;
        const int hh = a0 + a, ww = b0 + b;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (a < lim_a && b < lim_b && hh >= 0 && hh < hs && ww >= 0 && ww < ws)
            val = __ldg(reinterpret_cast<const uint4*>(src + ((size_t(n) * hs + hh) * ws + ww) * cs + c0 + v * VE));
        *reinterpret_cast<uint4*>(patch + a * PROW + b * 64 + v * VE) = val;
    }
    __syncthreads();
    const int g = threadIdx.x >> 3, a = threadIdx.x & 7;  // channel pair, patch row
    const bool live = 2 * g < cw;
    float2 row[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) row[b] = live ? ld_pair<T>(patch + a * PROW + b * 64 + 2 * g) : make_float2(0.f, 0.f);
    Cx X[5];
    rfft8(row, X);
    const LaneTw tw = lane_twiddles(a, -1.f);
#pragma unroll
    for (int v = 0; v < 5; ++v) X[v] = lane_fft8(X[v], tw);
    const int u = bitrev3(a);
    if (live) {
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            st_pair<T>(bins + ((v * 2 + 0) * F + u) * BROW + 2 * g, X[v].r);
            st_pair<T>(bins + ((v * 2 + 1) * F + u) * BROW + 2 * g, X[v].i);
        }
    }
    __syncthreads();
    const size_t plane = tl.T * 2 * size_t(cs);
    for (int idx = threadIdx.x; idx < NB * 2 * vpp; idx += blockDim.x) {
        const int q = idx % vpp, row = idx / vpp;  // row = (v * 2 + im) * 8 + u
        const int uu = row % F, vi = row / F, v = vi >> 1, im = vi & 1;
        *reinterpret_cast<uint4*>(out + (uu * 5 + v) * plane + t * 2 * cs + im * cs + c0 + q * VE) =
            *reinterpret_cast<const uint4*>(bins + row * BROW + q * VE);
    }
}

// Inverse transform + epilogue: Yf bins of one (tile, 64-channel slice) staged
// by coalesced rows, the inverse column FFT across each group's lanes
// (shuffles), the inverse real row FFT per lane, the valid oa x ob outputs
// re-staged and stored as coalesced channel rows with bias / residual / ReLU /
// ReLU-mask fused.
template <typename T>
__global__ void __launch_bounds__(256) fft_inv_smem_kernel(const T* __restrict__ Yf, T* __restrict__ y, FTiles tl,
                                                           const float* __restrict__ bias,
                                                           const T* __restrict__ residual,
                                                           const T* __restrict__ mask, int relu) {
    constexpr int PE = 16 / sizeof(T);
    constexpr int BROW = 64 + PE;      // bin rows ordered [v][Re|Im][u], 16-byte padded
    constexpr int OROW = F * 64 + 4;   // output patch row stride (floats)
    __shared__ __align__(16) T bins[NB * 2 * BROW];
    __shared__ __align__(16) float outs[F * OROW];
    const size_t t = blockIdx.x;
    const int c0 = blockIdx.y * 64;
    const int cw = min(64, tl.k - c0);
    int n, i, j;
    tile_of(tl, t, n, i, j);
    constexpr int VE = 16 / sizeof(T);
    const int vpp = cw / VE;
    const size_t plane = tl.T * 2 * size_t(tl.k);
    for (int idx = threadIdx.x; idx < NB * 2 * vpp; idx += blockDim.x) {
        const int q = idx % vpp, row = idx / vpp;
        const int uu = row % F, vi = row / F, v = vi >> 1, im = vi & 1;
        *reinterpret_cast<uint4*>(bins + row * BROW + q * VE) = __ldg(
            reinterpret_cast<const uint4*>(Yf + (uu * 5 + v) * plane + t * 2 * tl.k + im * tl.k + c0 + q * VE));
    }
    __syncthreads();
    const int g = threadIdx.x >> 3, a = threadIdx.x & 7;
    const bool live = 2 * g < cw;
    // lane a starts with frequency row u = a; the DIF inverse leaves row bitrev(a)
    {
        const LaneTw tw = lane_twiddles(a, 1.f);
        Cx Z[5];
#pragma unroll
        for (int v = 0; v < 5; ++v) {
            Z[v].r = live ? ld_pair<T>(bins + ((v * 2 + 0) * F + a) * BROW + 2 * g) : make_float2(0.f, 0.f);
            Z[v].i = live ? ld_pair<T>(bins + ((v * 2 + 1) * F + a) * BROW + 2 * g) : make_float2(0.f, 0.f);
            Z[v] = lane_fft8(Z[v], tw);
        }
        // inverse real row transform: x[b] = Re(Z0) + (-1)^b Re(Z4) + 2 sum_{v=1..3} Re(Z_v e^{+2 pi i v b/8})
        const int r = bitrev3(a);
        const float s = 0.70710678118654752f;
        const float cv[8] = {1.f, s, 0.f, -s, -1.f, -s, 0.f, s};
        const float2 p04 = add2(Z[0].r, Z[4].r), m04 = sub2(Z[0].r, Z[4].r);
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            float2 acc = (b & 1) ? m04 : p04;
#pragma unroll
            for (int v = 1; v < 4; ++v) {
                const float c = 2.f * cv[(v * b) & 7], sn = -2.f * cv[(v * b + 6) & 7];  // 2cos, -2sin
                acc = fma2(Z[v].r, c, acc);
                acc = fma2(Z[v].i, sn, acc);
            }
            if (live) *reinterpret_cast<float2*>(outs + r * OROW + b * 64 + 2 * g) = mul2(acc, 1.f / 64.f);
        }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < tl.oa * tl.ob * vpp; idx += blockDim.x) {
        const int v = idx % vpp, pix = idx / vpp;
        const int a2 = pix / tl.ob, b2 = pix % tl.ob;
        const int oh = i * tl.oa + a2, ow = j * tl.ob + b2;
        if (oh >= tl.ho || ow >= tl.wo) continue;
        const int c = c0 + v * VE;
        const size_t o = ((size_t(n) * tl.ho + oh) * tl.wo + ow) * tl.k + c;
        float val[VE];
#pragma unroll
        for (int q = 0; q < VE; ++q) val[q] = outs[a2 * OROW + b2 * 64 + v * VE + q];
        if (bias) {
#pragma unroll
            for (int q = 0; q < VE; ++q) val[q] += __ldg(bias + c + q);
        }
        if (residual) {
            const uint4 rv = __ldg(reinterpret_cast<const uint4*>(residual + o));
            const T* re = reinterpret_cast<const T*>(&rv);
#pragma unroll
            for (int q = 0; q < VE; ++q) val[q] += to_f32<T>(re[q]);
        }
        if (relu) {
#pragma unroll
            for (int q = 0; q < VE; ++q) val[q] = fmaxf(val[q], 0.f);
        }
        if (mask) {
            const uint4 mv = __ldg(reinterpret_cast<const uint4*>(mask + o));
            const T* me = reinterpret_cast<const T*>(&mv);
#pragma unroll
            for (int q = 0; q < VE; ++q)
                if (!(to_f32<T>(me[q]) > 0.f)) val[q] = 0.f;
        }
        uint4 ov;
        T* oe = reinterpret_cast<T*>(&ov);
#pragma unroll
        for (int q = 0; q < VE; ++q) oe[q] = from_f32<T>(val[q]);
        *reinterpret_cast<uint4*>(y + o) = ov;
    }
}

// Xf[bin][t][Re c | Im c]
template <typename T>
__global__ void fft_input_kernel(const T* __restrict__ x, T* __restrict__ Xf, FTiles tl) {
    const size_t total = tl.T * tl.c;
    const size_t plane = tl.T * 2 * tl.c;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % tl.c);
        const size_t t = idx / tl.c;
        int n, i, j;
        tile_of(tl, t, n, i, j);
        float p[F][F];
#pragma unroll
        for (int a = 0; a < F; ++a) {
            const int hh = i * tl.oa - tl.ph + a;
#pragma unroll
            for (int b = 0; b < F; ++b) {
                const int ww = j * tl.ob - tl.pw + b;
                p[a][b] = (hh >= 0 && hh < tl.h && ww >= 0 && ww < tl.w)
                              ? to_f32<T>(x[((size_t(n) * tl.h + hh) * tl.w + ww) * tl.c + c])
                              : 0.f;
            }
        }
        float re[F][5], im[F][5];
        rfft8x8(p, re, im);
#pragma unroll
        for (int u = 0; u < F; ++u)
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                T* row = Xf + (u * 5 + v) * plane + t * 2 * tl.c;
                row[c] = from_f32<T>(re[u][v]);
                row[tl.c + c] = from_f32<T>(im[u][v]);
            }
    }
}

// B[bin] = [[Wr, Wi], [-Wi, Wr]] (2K x 2C); flip_transpose for dgrad.
template <typename T>
__global__ void fft_filter_kernel(const T* __restrict__ w, T* __restrict__ Wf, FTiles tl,
                                  int flip_transpose) {
    const int K = tl.k, C = tl.c;
    const size_t total = size_t(K) * C;
    const size_t plane = size_t(2 * K) * 2 * C;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % C), k = int(idx / C);
        float p[F][F];
#pragma unroll
        for (int a = 0; a < F; ++a)
#pragma unroll
            for (int b = 0; b < F; ++b) {
                float v = 0.f;
                if (a < tl.r && b < tl.s)
                    v = flip_transpose
                            ? to_f32<T>(w[((size_t(c) * tl.r + (tl.r - 1 - a)) * tl.s + (tl.s - 1 - b)) * K + k])
                            : to_f32<T>(w[((size_t(k) * tl.r + a) * tl.s + b) * C + c]);
                p[a][b] = v;
            }
        float re[F][5], im[F][5];
        rfft8x8(p, re, im);
#pragma unroll
        for (int u = 0; u < F; ++u)
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                T* B = Wf + (u * 5 + v) * plane;
                B[size_t(k) * 2 * C + c] = from_f32<T>(re[u][v]);
                B[size_t(k) * 2 * C + C + c] = from_f32<T>(im[u][v]);
                B[size_t(K + k) * 2 * C + c] = from_f32<T>(-im[u][v]);
                B[size_t(K + k) * 2 * C + C + c] = from_f32<T>(re[u][v]);
            }
    }
}

// y = irfft(Yf) on the valid oa x ob outputs + epilogue.
template <typename T, int OA, int OB>
__global__ void fft_output_kernel(const T* __restrict__ Yf, T* __restrict__ y, FTiles tl,
                                  const float* __restrict__ bias, const T* __restrict__ residual,
                                  const T* __restrict__ mask, int relu) {
    const size_t total = tl.T * tl.k;
    const size_t plane = tl.T * 2 * tl.k;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int k = int(idx % tl.k);
        const size_t t = idx / tl.k;
        int n, i, j;
        tile_of(tl, t, n, i, j);
        float re[F][5], im[F][5];
#pragma unroll
        for (int u = 0; u < F; ++u)
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                const T* row = Yf + (u * 5 + v) * plane + t * 2 * tl.k;
                re[u][v] = to_f32<T>(row[k]);
                im[u][v] = to_f32<T>(row[tl.k + k]);
            }
        float out[OA][OB];
        irfft8x8<OA, OB>(re, im, out);
#pragma unroll
        for (int a = 0; a < OA; ++a) {
            const int oh = i * OA + a;
            if (oh >= tl.ho) continue;
#pragma unroll
            for (int b = 0; b < OB; ++b) {
                const int ow = j * OB + b;
                if (ow >= tl.wo) continue;
                const size_t o = ((size_t(n) * tl.ho + oh) * tl.wo + ow) * tl.k + k;
                float v = out[a][b];
                if (bias) v += bias[k];
                if (residual) v += to_f32<T>(residual[o]);
                if (relu) v = fmaxf(v, 0.f);
                if (mask && !(to_f32<T>(mask[o]) > 0.f)) v = 0.f;
                y[o] = from_f32<T>(v);
            }
        }
    }
}

// DYf[bin][t][Re k | Im k] of the oa x ob output-gradient tile (zero-padded).
template <typename T>
__global__ void fft_dy_kernel(const T* __restrict__ dy, T* __restrict__ DYf, FTiles tl) {
    const size_t total = tl.T * tl.k;
    const size_t plane = tl.T * 2 * tl.k;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int k = int(idx % tl.k);
        const size_t t = idx / tl.k;
        int n, i, j;
        tile_of(tl, t, n, i, j);
        float p[F][F];
#pragma unroll
        for (int a = 0; a < F; ++a)
#pragma unroll
            for (int b = 0; b < F; ++b) {
                const int oh = i * tl.oa + a, ow = j * tl.ob + b;
                p[a][b] = (a < tl.oa && b < tl.ob && oh < tl.ho && ow < tl.wo)
                              ? to_f32<T>(dy[((size_t(n) * tl.ho + oh) * tl.wo + ow) * tl.k + k])
                              : 0.f;
            }
        float re[F][5], im[F][5];
        rfft8x8(p, re, im);
#pragma unroll
        for (int u = 0; u < F; ++u)
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                T* row = DYf + (u * 5 + v) * plane + t * 2 * tl.k;
                row[k] = from_f32<T>(re[u][v]);
                row[tl.k + k] = from_f32<T>(im[u][v]);
            }
    }
}

// D[bin] = [DYr|DYi]^T [Xr|Xi] (2K x 2C, fp32) -> DW = X conj(DY) -> irfft -> dW[k][r][s][c]
__global__ void fft_dw_kernel(const float* __restrict__ D, float* __restrict__ dw, FTiles tl) {
    const int K = tl.k, C = tl.c;
    const size_t total = size_t(K) * C;
    const size_t plane = size_t(2 * K) * 2 * C;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % C), k = int(idx / C);
        float re[F][5], im[F][5];
#pragma unroll
        for (int u = 0; u < F; ++u)
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                const float* B = D + (u * 5 + v) * plane;
                const float q00 = B[size_t(k) * 2 * C + c], q01 = B[size_t(k) * 2 * C + C + c];
                const float q10 = B[size_t(K + k) * 2 * C + c], q11 = B[size_t(K + k) * 2 * C + C + c];
                re[u][v] = q00 + q11;
                im[u][v] = q01 - q10;
            }
        float out[F][F];
        irfft8x8<F, F>(re, im, out);
        for (int r = 0; r < tl.r; ++r)
            for (int s = 0; s < tl.s; ++s) dw[((size_t(k) * tl.r + r) * tl.s + s) * C + c] = out[r][s];
    }
}

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

struct FLayout {
    size_t x, y, w, d, gemm_ws, total;
};

ConvGeom gemm_geom(size_t T, int c2, int k2) { return ConvGeom{1, 1, static_cast<int>(T), c2, k2, 1, 1, 0, 0, 1, 1}; }

FLayout flayout(const FTiles& tl, size_t es, bool wgrad, DType dt) {
    FLayout L{};
    L.x = al(NB * tl.T * 2 * tl.c * es);
    L.y = al(NB * tl.T * 2 * tl.k * es);
    L.w = wgrad ? 0 : al(NB * size_t(2 * tl.k) * 2 * tl.c * es);
    L.d = wgrad ? al(NB * size_t(2 * tl.k) * 2 * tl.c * 4) : 0;
    const ConvGeom gg = gemm_geom(tl.T, 2 * tl.c, 2 * tl.k);
    L.gemm_ws = wgrad ? al(dt == DType::BF16 ? conv_tc_wgrad_batched_workspace(gg, NB)
                                             : conv_ffma_workspace(gg, ConvMode::Wgrad))
                      : 0;
    L.total = L.x + L.y + L.w + L.d + L.gemm_ws;
    return L;
}

#define FFT_DT(dt, T, ...)               \
    do {                                 \
        if ((dt) == DType::F32) {        \
            using T = float;             \
            __VA_ARGS__;                 \
        } else {                         \
            using T = __nv_bfloat16;     \
            __VA_ARGS__;                 \
        }                                \
    } while (0)

template <typename T>
cudaError_t launch_output(const FTiles& tl, const T* Yf, T* y, const Epilogue& ep, cudaStream_t st) {
    fft_inv_smem_kernel<T><<<dim3(static_cast<unsigned>(tl.T), (tl.k + 63) / 64), 256, 0, st>>>(
        Yf, y, tl, ep.bias, static_cast<const T*>(ep.residual), static_cast<const T*>(ep.mask), ep.relu ? 1 : 0);
    return cudaGetLastError();
}

// The per-thread register transform (kept for reference / A-B).
template <typename T>
cudaError_t launch_output_regs(const FTiles& tl, const T* Yf, T* y, const Epilogue& ep, cudaStream_t st) {
    const int g = grid_of(tl.T * tl.k);
    const float* b = ep.bias;
    const T* r = static_cast<const T*>(ep.residual);
    const T* m = static_cast<const T*>(ep.mask);
    const int relu = ep.relu ? 1 : 0;
#define FFT_OUT(OA, OB)                                                                       \
    if (tl.oa == OA && tl.ob == OB) {                                                         \
        fft_output_kernel<T, OA, OB><<<g, kBlock, 0, st>>>(Yf, y, tl, b, r, m, relu);         \
        return cudaGetLastError();                                                            \
    }
    FFT_OUT(6, 6) FFT_OUT(4, 4) FFT_OUT(2, 2) FFT_OUT(8, 2) FFT_OUT(2, 8) FFT_OUT(7, 7)
    FFT_OUT(5, 5) FFT_OUT(3, 3) FFT_OUT(8, 6) FFT_OUT(6, 8) FFT_OUT(8, 4) FFT_OUT(4, 8)
    FFT_OUT(6, 4) FFT_OUT(4, 6) FFT_OUT(1, 1) FFT_OUT(8, 8)
#undef FFT_OUT
    return cudaErrorNotSupported;
}

cudaError_t fft_conv(const FTiles& tl, DType dt, const void* src, const void* w, int flip,
                     const Epilogue& ep, void* out, void* ws, cudaStream_t st) {
    const size_t es = dtype_size(dt);
    const FLayout L = flayout(tl, es, false, dt);
    char* base = static_cast<char*>(ws);
    void* Xf = base;
    void* Yf = base + L.x;
    void* Wf = base + L.x + L.y;
    FFT_DT(dt, T, {
        fft_fwd_smem_kernel<T><<<dim3(static_cast<unsigned>(tl.T), (tl.c + 63) / 64), 256, 0, st>>>(
            static_cast<const T*>(src), static_cast<T*>(Xf), tl, tl.h, tl.w, tl.c, tl.oa, tl.ob, tl.ph, tl.pw, F, F);
        fft_filter_kernel<T><<<grid_of(size_t(tl.k) * tl.c), kBlock, 0, st>>>(
            static_cast<const T*>(w), static_cast<T*>(Wf), tl, flip);
    });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const ConvGeom gg = gemm_geom(tl.T, 2 * tl.c, 2 * tl.k);
    if (dt == DType::BF16) {
        // the 40 per-bin complex products (as real GEMMs) in one batched launch
        e = conv_tc_fwd_batched(gg, NB, Xf, Wf, Yf, st);
        if (e != cudaSuccess) return e;
    } else {
        for (int b = 0; b < NB; ++b) {
            const char* Xb = static_cast<const char*>(Xf) + b * tl.T * 2 * tl.c * es;
            const char* Wb = static_cast<const char*>(Wf) + b * size_t(2 * tl.k) * 2 * tl.c * es;
            char* Yb = static_cast<char*>(Yf) + b * tl.T * 2 * tl.k * es;
            Epilogue none;
            e = conv_ffma_fwd(gg, reinterpret_cast<const float*>(Xb), reinterpret_cast<const float*>(Wb), none,
                              reinterpret_cast<float*>(Yb), st);
            if (e != cudaSuccess) return e;
        }
    }
    FFT_DT(dt, T, { e = launch_output<T>(tl, static_cast<const T*>(Yf), static_cast<T*>(out), ep, st); });
    return e;
}

}  // namespace

bool fft_supported(const ConvGeom& g) {
    return g.stride_h == 1 && g.stride_w == 1 && g.r <= F && g.s <= F && (g.r > 1 || g.s > 1) &&
           g.pad_h >= 0 && g.pad_w >= 0 && g.pad_h <= g.r - 1 && g.pad_w <= g.s - 1 &&
           g.ho() >= 1 && g.wo() >= 1 && g.c % 8 == 0 && g.k % 8 == 0;
}

size_t fft_workspace(const ConvGeom& g, ConvMode mode) {
    // sized for bf16 and fp32 alike: the larger of the two layouts
    if (mode == ConvMode::Dgrad) {
        const FTiles tl = make_ftiles(g.n, g.ho(), g.wo(), g.k, g.c, g.r, g.s, g.r - 1 - g.pad_h,
                                      g.s - 1 - g.pad_w);
        return std::max(flayout(tl, 4, false, DType::F32).total, flayout(tl, 2, false, DType::BF16).total);
    }
    const FTiles tl = make_ftiles(g.n, g.h, g.w, g.c, g.k, g.r, g.s, g.pad_h, g.pad_w);
    const bool wg = mode == ConvMode::Wgrad;
    return std::max(flayout(tl, 4, wg, DType::F32).total, flayout(tl, 2, wg, DType::BF16).total);
}

cudaError_t fft_fwd(const ConvGeom& g, DType dt, const void* x, const void* w, const Epilogue& ep,
                    void* y, void* ws, cudaStream_t st) {
    if (!fft_supported(g) || !ws) return cudaErrorNotSupported;
    return fft_conv(make_ftiles(g.n, g.h, g.w, g.c, g.k, g.r, g.s, g.pad_h, g.pad_w), dt, x, w, 0,
                    ep, y, ws, st);
}

cudaError_t fft_dgrad(const ConvGeom& g, DType dt, const void* dy, const void* w,
                      const Epilogue& ep, void* dx, void* ws, cudaStream_t st) {
    if (!fft_supported(g) || !ws) return cudaErrorNotSupported;
    Epilogue e2 = ep;
    e2.bias = nullptr;
    e2.relu = false;
    return fft_conv(make_ftiles(g.n, g.ho(), g.wo(), g.k, g.c, g.r, g.s, g.r - 1 - g.pad_h,
                                g.s - 1 - g.pad_w),
                    dt, dy, w, 1, e2, dx, ws, st);
}

cudaError_t fft_wgrad(const ConvGeom& g, DType dt, const void* dy, const void* x, float* dw,
                      void* ws, cudaStream_t st) {
    if (!fft_supported(g) || !ws) return cudaErrorNotSupported;
    const FTiles tl = make_ftiles(g.n, g.h, g.w, g.c, g.k, g.r, g.s, g.pad_h, g.pad_w);
    const size_t es = dtype_size(dt);
    const FLayout L = flayout(tl, es, true, dt);
    char* base = static_cast<char*>(ws);
    void* Xf = base;
    void* DYf = base + L.x;
    float* D = reinterpret_cast<float*>(base + L.x + L.y);
    void* gws = base + L.x + L.y + L.d;
    FFT_DT(dt, T, {
        fft_fwd_smem_kernel<T><<<dim3(static_cast<unsigned>(tl.T), (tl.c + 63) / 64), 256, 0, st>>>(
            static_cast<const T*>(x), static_cast<T*>(Xf), tl, tl.h, tl.w, tl.c, tl.oa, tl.ob, tl.ph, tl.pw, F, F);
        // the output-gradient tile: oa x ob values at (i*oa, j*ob), zero-padded to 8x8
        fft_fwd_smem_kernel<T><<<dim3(static_cast<unsigned>(tl.T), (tl.k + 63) / 64), 256, 0, st>>>(
            static_cast<const T*>(dy), static_cast<T*>(DYf), tl, tl.ho, tl.wo, tl.k, tl.oa, tl.ob, 0, 0, tl.oa,
            tl.ob);
    });
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const ConvGeom gg = gemm_geom(tl.T, 2 * tl.c, 2 * tl.k);
    if (dt == DType::BF16) {
        e = conv_tc_wgrad_batched(gg, NB, DYf, Xf, D, gws, st);
        if (e != cudaSuccess) return e;
    } else {
        for (int b = 0; b < NB; ++b) {
            const char* Xb = static_cast<const char*>(Xf) + b * tl.T * 2 * tl.c * es;
            const char* Db = static_cast<const char*>(DYf) + b * tl.T * 2 * tl.k * es;
            float* Ob = D + b * size_t(2 * tl.k) * 2 * tl.c;
            e = conv_ffma_wgrad(gg, reinterpret_cast<const float*>(Db), reinterpret_cast<const float*>(Xb), Ob, gws,
                                st);
            if (e != cudaSuccess) return e;
        }
    }
    fft_dw_kernel<<<grid_of(size_t(tl.k) * tl.c), kBlock, 0, st>>>(D, dw, tl);
    return cudaGetLastError();
}

}  // namespace tcb
