// Winograd F(2x2, 3x3) convolution family (3x3 filters, stride 1), the
// "winograd" algorithm token of the reference catalog
// (/root/reference/proj/include/traincap/catalog.hpp:13).
//
//   fwd   : V = B^T d B (input tiles), U = G g G^T (filters),
//           M_xi = V_xi * U_xi^T for the 16 transform positions xi (16 GEMMs
//           [T x C] x [C x K] on the tcgen05 kernel in plain-TMA mode, or the
//           FFMA kernel in fp32 mode), Y = A^T M A with the fused epilogue
//           (bias, residual, ReLU / ReLU-mask).
//   dgrad : the forward algorithm on dy with the flipped, transposed filter
//           (pad' = 2 - pad), so the same kernels serve it.
//   wgrad : Z = A dY A^T (output-gradient tiles), dU_xi = Z_xi^T V_xi (16
//           reduction GEMMs over the tiles, deterministic split-K), then
//           dW = G^T dU G.
//
// The transforms are HBM-bound (roofline: bytes moved / HBM bandwidth): each
// thread owns 8 (bf16) or 4 (fp32) consecutive channels of one tile, so NHWC
// reads/writes are 16-byte vectors coalesced across the channel axis. The
// workspace (V, M/Z, U, dU) is what the planner's knapsack trades against
// time: 16 transformed planes per tensor.
#include <algorithm>

#include "common.cuh"

namespace tcb {
namespace {

constexpr int kBlock = 256;

template <typename T, int V>
struct alignas(16) Vec {
    T v[V];
};

inline int grid_of(size_t n) {
    return static_cast<int>(std::max<size_t>(1, std::min<size_t>((n + kBlock - 1) / kBlock,
                                                                 size_t(num_sms()) * 32)));
}

struct Tiles {
    int n, h, w, c;        // source tensor (x for fwd, dy for dgrad)
    int ho, wo, k;         // destination extents and channels
    int pad;
    int th, tw;            // tiles per image
    size_t T;              // total tiles
};

Tiles make_tiles(int n, int h, int w, int c, int k, int pad) {
    Tiles t{};
    t.n = n;
    t.h = h;
    t.w = w;
    t.c = c;
    t.k = k;
    t.pad = pad;
    t.ho = h + 2 * pad - 2;
    t.wo = w + 2 * pad - 2;
    t.th = (t.ho + 1) / 2;
    t.tw = (t.wo + 1) / 2;
    t.T = size_t(n) * t.th * t.tw;
    return t;
}

// ---------------------------------------------------------------- input ---
// V[xi][t][c] = (B^T d B)[xi], d = 4x4 input patch at (2i - pad, 2j - pad).
// Shared-memory-staged input transform (the path in use): one block per
// (image, tile row, channel slice of 128 bytes: 64 bf16 / 32 fp32 channels).
// The 4 input rows the tile row reads are staged once in shared memory as
// [row][padded column][channel] with the zero padding materialised (each
// input element leaves HBM once instead of once per overlapping patch), then
// every thread transforms one (tile, channel pair) patch out of shared memory
// — 16 values in registers instead of 16 x 8 — and stores the 16 planes; the
// lanes of a warp hold consecutive channel pairs, so every plane store is a
// contiguous 128-byte segment.
template <typename T>
__global__ void __launch_bounds__(256) wino_input_smem_kernel(const T* __restrict__ x, T* __restrict__ V,
                                                              Tiles tl, int cslice) {
    extern __shared__ __align__(16) uint8_t wsm_raw[];
    T* sm = reinterpret_cast<T*>(wsm_raw);
    constexpr int VE = 16 / sizeof(T);
    const int n = blockIdx.x / tl.th, i = blockIdx.x - n * tl.th;
    const int c0 = blockIdx.y * cslice;
    const int cw = min(cslice, tl.c - c0);
    const int Wp = 2 * tl.tw + 2;
    const int vpr = cw / VE;
    for (int idx = threadIdx.x; idx < 4 * Wp * vpr; idx += blockDim.x) {
        const int v = idx % vpr, rest = idx / vpr;
        const int u = rest % Wp, a = rest / Wp;
        const int hh = 2 * i - tl.pad + a, ww = u - tl.pad;
        uint4 val = make_uint4(0, 0, 0, 0);
        if (hh >= 0 && hh < tl.h && ww >= 0 && ww < tl.w)
            val = __ldg(reinterpret_cast<const uint4*>(x + ((size_t(n) * tl.h + hh) * tl.w + ww) * tl.c + c0 + v * VE));
        *reinterpret_cast<uint4*>(sm + (a * Wp + u) * cslice + v * VE) = val;
    }
    __syncthreads();
    const int pairs = cw / 2;
    const size_t plane = tl.T * tl.c;
    const size_t trow = (size_t(n) * tl.th + i) * tl.tw;
    // channel pairs as float2 through packed fp32x2 adds (FADD2: both channels at once)
    auto ld = [&](int a, int col, int pc) -> float2 {
        const T* q = sm + (a * Wp + col) * cslice + 2 * pc;
        if constexpr (sizeof(T) == 2) return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(q));
        else return *reinterpret_cast<const float2*>(q);
    };
    auto add = [](float2 x, float2 y) { return __fadd2_rn(x, y); };
    auto sub = [](float2 x, float2 y) { return __fadd2_rn(x, make_float2(-y.x, -y.y)); };
    for (int idx = threadIdx.x; idx < tl.tw * pairs; idx += blockDim.x) {
        const int pc = idx % pairs, j = idx / pairs;
        float2 d[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) d[a][b] = ld(a, 2 * j + b, pc);
        float2 r[4][4];  // B^T d
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            r[0][b] = sub(d[0][b], d[2][b]);
            r[1][b] = add(d[1][b], d[2][b]);
            r[2][b] = sub(d[2][b], d[1][b]);
            r[3][b] = sub(d[1][b], d[3][b]);
        }
        T* dst = V + (trow + j) * tl.c + c0 + 2 * pc;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float2 o[4] = {sub(r[a][0], r[a][2]), add(r[a][1], r[a][2]), sub(r[a][2], r[a][1]),
                                 sub(r[a][1], r[a][3])};
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                T* q = dst + (a * 4 + b) * plane;
                if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat162*>(q) = __floats2bfloat162_rn(o[b].x, o[b].y);
                else *reinterpret_cast<float2*>(q) = o[b];
            }
        }
    }
}

// Input transform launch: 128-byte channel slices, halved while the staged
// rows would exceed 48 KB (wide images).
template <typename T>
cudaError_t wino_input(const T* x, T* V, const Tiles& tl, cudaStream_t st) {
    constexpr int VE = 16 / sizeof(T);
    int cslice = 128 / static_cast<int>(sizeof(T));
    const int Wp = 2 * tl.tw + 2;
    while (cslice > VE && size_t(4) * Wp * cslice * sizeof(T) > 48 * 1024) cslice /= 2;
    if (tl.c % VE != 0) return cudaErrorInvalidValue;
    const size_t smem = size_t(4) * Wp * cslice * sizeof(T);
    if (smem > 48 * 1024) return cudaErrorInvalidValue;
    const dim3 grid(static_cast<unsigned>(size_t(tl.n) * tl.th), static_cast<unsigned>((tl.c + cslice - 1) / cslice));
    wino_input_smem_kernel<T><<<grid, 256, smem, st>>>(x, V, tl, cslice);
    return cudaGetLastError();
}

// --------------------------------------------------------------- filter ---
// U[xi][k][c] = (G g G^T)[xi]; flip_transpose: g = w[c][2-r][2-s][k] (dgrad).
template <typename T>
__global__ void wino_filter_kernel(const T* __restrict__ w, T* __restrict__ U, int K, int C,
                                   int flip_transpose) {
    const size_t total = size_t(K) * C;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % C), k = int(idx / C);
        float g[3][3];
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int s = 0; s < 3; ++s)
                g[r][s] = flip_transpose
                              ? to_f32<T>(w[((size_t(c) * 3 + (2 - r)) * 3 + (2 - s)) * K + k])
                              : to_f32<T>(w[((size_t(k) * 3 + r) * 3 + s) * C + c]);
        float t[4][3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            t[0][s] = g[0][s];
            t[1][s] = 0.5f * (g[0][s] + g[1][s] + g[2][s]);
            t[2][s] = 0.5f * (g[0][s] - g[1][s] + g[2][s]);
            t[3][s] = g[2][s];
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const float u[4] = {t[a][0], 0.5f * (t[a][0] + t[a][1] + t[a][2]),
                                0.5f * (t[a][0] - t[a][1] + t[a][2]), t[a][2]};
#pragma unroll
            for (int b = 0; b < 4; ++b) U[(a * 4 + b) * total + size_t(k) * C + c] = from_f32<T>(u[b]);
        }
    }
}

// --------------------------------------------------------------- output ---
// Y = A^T M A (2x2 per tile) + bias + residual, ReLU or ReLU-mask.
template <typename T, int VW>
__global__ void wino_output_kernel(const T* __restrict__ M, T* __restrict__ y, Tiles tl,
                                   const float* __restrict__ bias, const T* __restrict__ residual,
                                   const T* __restrict__ mask, int relu) {
    const int kg = tl.k / VW;
    const size_t total = tl.T * kg;
    const size_t plane = tl.T * tl.k;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int k = int(idx % kg) * VW;
        const size_t t = idx / kg;
        const int j = int(t % tl.tw);
        const int i = int((t / tl.tw) % tl.th);
        const int n = int(t / (size_t(tl.tw) * tl.th));
        float m[4][4][VW];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const Vec<T, VW> v = *reinterpret_cast<const Vec<T, VW>*>(M + (a * 4 + b) * plane + t * tl.k + k);
#pragma unroll
                for (int e = 0; e < VW; ++e) m[a][b][e] = to_f32<T>(v.v[e]);
            }
        // A^T m: rows (m0 + m1 + m2, m1 - m2 - m3)
        float r[2][4][VW];
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                r[0][b][e] = m[0][b][e] + m[1][b][e] + m[2][b][e];
                r[1][b][e] = m[1][b][e] - m[2][b][e] - m[3][b][e];
            }
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const int oh = 2 * i + a;
            if (oh >= tl.ho) continue;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int ow = 2 * j + b;
                if (ow >= tl.wo) continue;
                const size_t o = ((size_t(n) * tl.ho + oh) * tl.wo + ow) * tl.k + k;
                float v[VW];
#pragma unroll
                for (int e = 0; e < VW; ++e)
                    v[e] = b == 0 ? r[a][0][e] + r[a][1][e] + r[a][2][e]
                                  : r[a][1][e] - r[a][2][e] - r[a][3][e];
                if (bias) {
#pragma unroll
                    for (int e = 0; e < VW; ++e) v[e] += bias[k + e];
                }
                if (residual) {
                    const Vec<T, VW> rv = *reinterpret_cast<const Vec<T, VW>*>(residual + o);
#pragma unroll
                    for (int e = 0; e < VW; ++e) v[e] += to_f32<T>(rv.v[e]);
                }
                if (relu) {
#pragma unroll
                    for (int e = 0; e < VW; ++e) v[e] = fmaxf(v[e], 0.f);
                }
                if (mask) {
                    const Vec<T, VW> mv = *reinterpret_cast<const Vec<T, VW>*>(mask + o);
#pragma unroll
                    for (int e = 0; e < VW; ++e)
                        if (!(to_f32<T>(mv.v[e]) > 0.f)) v[e] = 0.f;
                }
                Vec<T, VW> out;
#pragma unroll
                for (int e = 0; e < VW; ++e) out.v[e] = from_f32<T>(v[e]);
                *reinterpret_cast<Vec<T, VW>*>(y + o) = out;
            }
        }
    }
}

// -------------------------------------------------------- wgrad helpers ---
// Z[xi][t][k] = (A dY A^T)[xi], dY = the tile's 2x2 output gradients (0 past the edge).
template <typename T, int VW>
__global__ void wino_dy_kernel(const T* __restrict__ dy, T* __restrict__ Z, Tiles tl) {
    const int kg = tl.k / VW;
    const size_t total = tl.T * kg;
    const size_t plane = tl.T * tl.k;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int k = int(idx % kg) * VW;
        const size_t t = idx / kg;
        const int j = int(t % tl.tw);
        const int i = int((t / tl.tw) % tl.th);
        const int n = int(t / (size_t(tl.tw) * tl.th));
        float g[2][2][VW];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int oh = 2 * i + a, ow = 2 * j + b;
                if (oh < tl.ho && ow < tl.wo) {
                    const Vec<T, VW> v = *reinterpret_cast<const Vec<T, VW>*>(
                        dy + ((size_t(n) * tl.ho + oh) * tl.wo + ow) * tl.k + k);
#pragma unroll
                    for (int e = 0; e < VW; ++e) g[a][b][e] = to_f32<T>(v.v[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < VW; ++e) g[a][b][e] = 0.f;
                }
            }
        // A = [[1,0],[1,1],[1,-1],[0,-1]]: (A g)[0]=g0, [1]=g0+g1, [2]=g0-g1, [3]=-g1
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            float row[2][VW];
#pragma unroll
            for (int b = 0; b < 2; ++b)
#pragma unroll
                for (int e = 0; e < VW; ++e)
                    row[b][e] = a == 0 ? g[0][b][e]
                                       : a == 1 ? g[0][b][e] + g[1][b][e]
                                                : a == 2 ? g[0][b][e] - g[1][b][e] : -g[1][b][e];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                Vec<T, VW> out;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const float v = b == 0 ? row[0][e]
                                           : b == 1 ? row[0][e] + row[1][e]
                                                    : b == 2 ? row[0][e] - row[1][e] : -row[1][e];
                    out.v[e] = from_f32<T>(v);
                }
                *reinterpret_cast<Vec<T, VW>*>(Z + (a * 4 + b) * plane + t * tl.k + k) = out;
            }
        }
    }
}

// dW[k][r][s][c] = (G^T dU G)[r][s]
__global__ void wino_dw_kernel(const float* __restrict__ dU, float* __restrict__ dw, int K, int C) {
    const size_t total = size_t(K) * C;
    for (size_t idx = blockIdx.x * size_t(blockDim.x) + threadIdx.x; idx < total;
         idx += size_t(gridDim.x) * blockDim.x) {
        const int c = int(idx % C), k = int(idx / C);
        float u[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) u[a][b] = dU[(a * 4 + b) * total + idx];
        // G^T = [[1,.5,.5,0],[0,.5,-.5,0],[0,.5,.5,1]]
        float t[3][4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            t[0][b] = u[0][b] + 0.5f * (u[1][b] + u[2][b]);
            t[1][b] = 0.5f * (u[1][b] - u[2][b]);
            t[2][b] = 0.5f * (u[1][b] + u[2][b]) + u[3][b];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const float o[3] = {t[r][0] + 0.5f * (t[r][1] + t[r][2]), 0.5f * (t[r][1] - t[r][2]),
                                0.5f * (t[r][1] + t[r][2]) + t[r][3]};
#pragma unroll
            for (int s = 0; s < 3; ++s) dw[((size_t(k) * 3 + r) * 3 + s) * C + c] = o[s];
        }
    }
}

// -------------------------------------------------------------- helpers ---
size_t al(size_t b) { return (b + 255) & ~size_t(255); }

struct WinoLayout {
    size_t v, m, u, du, gemm_ws, total;
};

WinoLayout layout_for(const Tiles& tl, size_t es, bool wgrad, const ConvGeom& gemm_g, DType dt) {
    WinoLayout L{};
    L.v = al(16 * tl.T * tl.c * es);
    L.m = al(16 * tl.T * tl.k * es);
    L.u = al(16 * size_t(tl.k) * tl.c * es);
    L.du = wgrad ? al(16 * size_t(tl.k) * tl.c * 4) : 0;
    L.gemm_ws = wgrad ? al(dt == DType::BF16 ? conv_tc_wgrad_batched_workspace(gemm_g, 16)
                                             : conv_ffma_workspace(gemm_g, ConvMode::Wgrad))
                      : 0;
    L.total = L.v + L.m + L.u + L.du + L.gemm_ws;
    return L;
}

// The per-position GEMM as a 1x1 "conv" over T pixels.
ConvGeom gemm_geom(size_t T, int c, int k) {
    return ConvGeom{1, 1, static_cast<int>(T), c, k, 1, 1, 0, 0, 1, 1};
}

#define WINO_DT(dt, T, VW, ...)                  \
    do {                                         \
        if ((dt) == DType::F32) {                \
            using T = float;                     \
            constexpr int VW = 4;                \
            __VA_ARGS__;                         \
        } else {                                 \
            using T = __nv_bfloat16;             \
            constexpr int VW = 8;                \
            __VA_ARGS__;                         \
        }                                        \
    } while (0)

// Shared by fwd (x, w) and dgrad (dy, flipped w^T).
cudaError_t wino_conv(const Tiles& tl, DType dt, const void* src, const void* w, int flip_transpose,
                      const Epilogue& ep, void* out, void* ws, cudaStream_t st) {
    const size_t es = dtype_size(dt);
    const ConvGeom gg = gemm_geom(tl.T, tl.c, tl.k);
    const WinoLayout L = layout_for(tl, es, false, gg, dt);
    char* base = static_cast<char*>(ws);
    void* V = base;
    void* M = base + L.v;
    void* U = base + L.v + L.m;
    cudaError_t e = cudaSuccess;
    WINO_DT(dt, T, VW, {
        e = wino_input<T>(static_cast<const T*>(src), static_cast<T*>(V), tl, st);
        if (e == cudaSuccess)
            wino_filter_kernel<T><<<grid_of(size_t(tl.k) * tl.c), kBlock, 0, st>>>(
                static_cast<const T*>(w), static_cast<T*>(U), tl.k, tl.c, flip_transpose);
    });
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (dt == DType::BF16) {
        // the 16 transform-position GEMMs in one batched tcgen05 launch
        e = conv_tc_fwd_batched(gg, 16, V, U, M, st);
        if (e != cudaSuccess) return e;
    } else {
        for (int xi = 0; xi < 16; ++xi) {
            const char* Vx = static_cast<const char*>(V) + xi * tl.T * tl.c * es;
            const char* Ux = static_cast<const char*>(U) + xi * size_t(tl.k) * tl.c * es;
            char* Mx = static_cast<char*>(M) + xi * tl.T * tl.k * es;
            Epilogue none;
            e = conv_ffma_fwd(gg, reinterpret_cast<const float*>(Vx), reinterpret_cast<const float*>(Ux), none,
                              reinterpret_cast<float*>(Mx), st);
            if (e != cudaSuccess) return e;
        }
    }
    WINO_DT(dt, T, VW, {
        wino_output_kernel<T, VW><<<grid_of(tl.T * tl.k / VW), kBlock, 0, st>>>(
            static_cast<const T*>(M), static_cast<T*>(out), tl, ep.bias,
            static_cast<const T*>(ep.residual), static_cast<const T*>(ep.mask), ep.relu ? 1 : 0);
    });
    return cudaGetLastError();
}

}  // namespace

bool winograd_supported(const ConvGeom& g) {
    return g.r == 3 && g.s == 3 && g.stride_h == 1 && g.stride_w == 1 && g.pad_h == g.pad_w &&
           g.pad_h >= 0 && g.pad_h <= 2 && g.ho() >= 1 && g.wo() >= 1 && g.c % 8 == 0 &&
           g.k % 8 == 0;
}

size_t winograd_workspace(const ConvGeom& g, ConvMode mode, DType dt) {
    const size_t es = dtype_size(dt);
    if (mode == ConvMode::Dgrad) {
        const Tiles tl = make_tiles(g.n, g.ho(), g.wo(), g.k, g.c, 2 - g.pad_h);
        return layout_for(tl, es, false, gemm_geom(tl.T, tl.c, tl.k), dt).total;
    }
    const Tiles tl = make_tiles(g.n, g.h, g.w, g.c, g.k, g.pad_h);
    return layout_for(tl, es, mode == ConvMode::Wgrad, gemm_geom(tl.T, tl.c, tl.k), dt).total;
}

cudaError_t winograd_fwd(const ConvGeom& g, DType dt, const void* x, const void* w,
                         const Epilogue& ep, void* y, void* ws, cudaStream_t st) {
    if (!winograd_supported(g) || !ws) return cudaErrorNotSupported;
    return wino_conv(make_tiles(g.n, g.h, g.w, g.c, g.k, g.pad_h), dt, x, w, 0, ep, y, ws, st);
}

cudaError_t winograd_dgrad(const ConvGeom& g, DType dt, const void* dy, const void* w,
                           const Epilogue& ep, void* dx, void* ws, cudaStream_t st) {
    if (!winograd_supported(g) || !ws) return cudaErrorNotSupported;
    // dx = conv(dy, flip(w)^T) with pad 2 - pad: input dy (Ho x Wo x K) -> H x W x C
    Epilogue e2 = ep;
    e2.bias = nullptr;
    e2.relu = false;
    return wino_conv(make_tiles(g.n, g.ho(), g.wo(), g.k, g.c, 2 - g.pad_h), dt, dy, w, 1, e2, dx,
                     ws, st);
}

cudaError_t winograd_wgrad(const ConvGeom& g, DType dt, const void* dy, const void* x, float* dw,
                           void* ws, cudaStream_t st) {
    if (!winograd_supported(g) || !ws) return cudaErrorNotSupported;
    const Tiles tl = make_tiles(g.n, g.h, g.w, g.c, g.k, g.pad_h);
    const size_t es = dtype_size(dt);
    const ConvGeom gg = gemm_geom(tl.T, tl.c, tl.k);
    const WinoLayout L = layout_for(tl, es, true, gg, dt);
    char* base = static_cast<char*>(ws);
    void* V = base;
    void* Z = base + L.v;
    float* dU = reinterpret_cast<float*>(base + L.v + L.m + L.u);
    void* gws = base + L.v + L.m + L.u + L.du;
    cudaError_t e = cudaSuccess;
    WINO_DT(dt, T, VW, {
        e = wino_input<T>(static_cast<const T*>(x), static_cast<T*>(V), tl, st);
        if (e == cudaSuccess)
            wino_dy_kernel<T, VW><<<grid_of(tl.T * tl.k / VW), kBlock, 0, st>>>(
                static_cast<const T*>(dy), static_cast<T*>(Z), tl);
    });
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (dt == DType::BF16) {
        // the 16 tile-reduction GEMMs in one batched launch (split-K over all of them)
        e = conv_tc_wgrad_batched(gg, 16, Z, V, dU, gws, st);
        if (e != cudaSuccess) return e;
    } else {
        for (int xi = 0; xi < 16; ++xi) {
            const char* Vx = static_cast<const char*>(V) + xi * tl.T * tl.c * es;
            const char* Zx = static_cast<const char*>(Z) + xi * tl.T * tl.k * es;
            float* dUx = dU + xi * size_t(tl.k) * tl.c;
            e = conv_ffma_wgrad(gg, reinterpret_cast<const float*>(Zx), reinterpret_cast<const float*>(Vx), dUx,
                                gws, st);
            if (e != cudaSuccess) return e;
        }
    }
    wino_dw_kernel<<<grid_of(size_t(tl.k) * tl.c), kBlock, 0, st>>>(dU, dw, tl.k, tl.c);
    return cudaGetLastError();
}

}  // namespace tcb
