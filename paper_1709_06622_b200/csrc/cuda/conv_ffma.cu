// FP32 FFMA implicit-GEMM convolution — the "fp32-FFMA mode" of the
// north-star tolerance split (1e-5 relative vs the CPU oracle). Same GEMM
// views as the tensor-core kernel (common.cuh::ConvShape), any channel
// count, SIMT 64x64 tiles, 4x4 outputs per thread, 16-deep k-steps through
// shared memory with a register-staged prefetch of the next k-step.
#include <algorithm>

#include "common.cuh"

namespace tcb {
namespace {

constexpr int TM = 64, TN = 64, TK = 16, kThreads = 256;

struct Params {
    ConvShape s;
    const float* a;
    const float* b;
    float* out;
    const float* bias;
    const float* residual;
    const float* mask;
    int relu;
    int splits, kb_per_split;
};

template <ConvMode MODE>
__device__ __forceinline__ float load_a(const Params& p, int m, int kk) {
    const ConvShape& s = p.s;
    if (m >= s.M || kk >= s.Kdim) return 0.f;
    if constexpr (MODE == ConvMode::Fwd) {
        uint32_t n, rem, ho, wo, rs, c, r, sx;
        s.d_howo.divmod(m, n, rem);
        s.d_wo.divmod(rem, ho, wo);
        s.d_c.divmod(kk, rs, c);
        s.d_s.divmod(rs, r, sx);
        const int hi = int(ho) * s.sh - s.ph + int(r), wi = int(wo) * s.sw - s.pw + int(sx);
        if (hi < 0 || hi >= s.H || wi < 0 || wi >= s.W) return 0.f;
        return __ldg(p.a + ((size_t(n) * s.H + hi) * s.W + wi) * s.C + c);
    } else if constexpr (MODE == ConvMode::Dgrad) {
        uint32_t n, rem, h, w, rs, k, r, sx;
        s.d_hw.divmod(m, n, rem);
        s.d_w.divmod(rem, h, w);
        s.d_k.divmod(kk, rs, k);
        s.d_s.divmod(rs, r, sx);
        int ho = int(h) + s.ph - int(r), wo = int(w) + s.pw - int(sx);
        if (ho < 0 || wo < 0 || ho % s.sh || wo % s.sw) return 0.f;
        ho /= s.sh;
        wo /= s.sw;
        if (ho >= s.Ho || wo >= s.Wo) return 0.f;
        return __ldg(p.a + ((size_t(n) * s.Ho + ho) * s.Wo + wo) * s.K + k);
    } else {
        return __ldg(p.a + size_t(kk) * s.K + m);  // dy[pixel][kout]
    }
}

template <ConvMode MODE>
__device__ __forceinline__ float load_b(const Params& p, int j, int kk) {
    const ConvShape& s = p.s;
    if (j >= s.Ncol || kk >= s.Kdim) return 0.f;
    if constexpr (MODE == ConvMode::Fwd) {
        return __ldg(p.b + size_t(j) * s.Kdim + kk);  // w[k][(r,s,c)]
    } else if constexpr (MODE == ConvMode::Dgrad) {
        uint32_t rs, k, r, sx;
        s.d_k.divmod(kk, rs, k);
        s.d_s.divmod(rs, r, sx);
        return __ldg(p.b + ((size_t(k) * s.R + r) * s.S + sx) * s.C + j);  // w[k][r][s][c=j]
    } else {
        uint32_t n, rem, ho, wo, rs, c, r, sx;
        s.d_howo.divmod(kk, n, rem);
        s.d_wo.divmod(rem, ho, wo);
        s.d_c.divmod(j, rs, c);
        s.d_s.divmod(rs, r, sx);
        const int hi = int(ho) * s.sh - s.ph + int(r), wi = int(wo) * s.sw - s.pw + int(sx);
        if (hi < 0 || hi >= s.H || wi < 0 || wi >= s.W) return 0.f;
        return __ldg(p.b + ((size_t(n) * s.H + hi) * s.W + wi) * s.C + c);
    }
}

// Thread->element maps chosen so a warp's loads walk the contiguous NHWC axis.
template <ConvMode MODE>
struct Maps {
    static constexpr bool a_k_fast = MODE != ConvMode::Wgrad;
    static constexpr bool b_k_fast = MODE == ConvMode::Fwd;
};

template <ConvMode MODE>
__global__ void __launch_bounds__(kThreads) conv_ffma_kernel(const __grid_constant__ Params p) {
    __shared__ float As[TK][TM + 4];
    __shared__ float Bs[TK][TN + 4];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
    const int split = blockIdx.z;
    const int kb_total = (p.s.Kdim + TK - 1) / TK;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(kb_total, kb0 + p.kb_per_split);
    const int tx = tid % 16, ty = tid / 16;

    float acc[4][4] = {};
    float ra[4], rb[4];
    auto fetch = [&](int kb) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * kThreads;
            int mm, ka, nn, kbb;
            if (Maps<MODE>::a_k_fast) { mm = idx / TK; ka = idx % TK; } else { ka = idx / TM; mm = idx % TM; }
            if (Maps<MODE>::b_k_fast) { nn = idx / TK; kbb = idx % TK; } else { kbb = idx / TN; nn = idx % TN; }
            ra[i] = load_a<MODE>(p, m0 + mm, kb * TK + ka);
            rb[i] = load_b<MODE>(p, n0 + nn, kb * TK + kbb);
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int idx = tid + i * kThreads;
            if (Maps<MODE>::a_k_fast) As[idx % TK][idx / TK] = ra[i]; else As[idx / TM][idx % TM] = ra[i];
            if (Maps<MODE>::b_k_fast) Bs[idx % TK][idx / TK] = rb[i]; else Bs[idx / TN][idx % TN] = rb[i];
        }
    };
    if (kb0 < kb1) fetch(kb0);
    for (int kb = kb0; kb < kb1; ++kb) {
        __syncthreads();
        stash();
        __syncthreads();
        if (kb + 1 < kb1) fetch(kb + 1);
#pragma unroll
        for (int k = 0; k < TK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                a[i] = As[k][ty + 16 * i];
                b[i] = Bs[k][tx + 16 * i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
    }

    const ConvShape& s = p.s;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= s.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= s.Ncol) continue;
            float v = acc[i][j];
            if constexpr (MODE == ConvMode::Wgrad) {
                p.out[(size_t(split) * s.M + m) * s.Ncol + n] = v;
            } else {
                const size_t o = size_t(m) * s.Ncol + n;
                if (p.bias) v += p.bias[n];
                if (p.residual) v += p.residual[o];
                if (p.relu) v = fmaxf(v, 0.f);
                if (p.mask && !(p.mask[o] > 0.f)) v = 0.f;
                p.out[o] = v;
            }
        }
    }
}

int wgrad_splits(const ConvShape& s, int& per) {
    const int kb_total = (s.Kdim + TK - 1) / TK;
    const int tiles = ((s.M + TM - 1) / TM) * ((s.Ncol + TN - 1) / TN);
    int want = std::max(1, (4 * num_sms() + tiles - 1) / tiles);
    want = std::min({want, std::max(1, kb_total / 8), 128});
    per = (kb_total + want - 1) / want;
    return (kb_total + per - 1) / per;
}

template <ConvMode MODE>
cudaError_t run(Params p, cudaStream_t st) {
    dim3 grid((p.s.M + TM - 1) / TM, (p.s.Ncol + TN - 1) / TN, p.splits);
    conv_ffma_kernel<MODE><<<grid, kThreads, 0, st>>>(p);
    return cudaGetLastError();
}

}  // namespace

size_t conv_ffma_workspace(const ConvGeom& g, ConvMode mode) {
    if (mode != ConvMode::Wgrad) return 0;
    const ConvShape s = make_shape(g, mode);
    int per = 0;
    const int sp = wgrad_splits(s, per);
    return sp > 1 ? size_t(sp) * s.M * s.Ncol * sizeof(float) : 0;
}

cudaError_t conv_ffma_fwd(const ConvGeom& g, const float* x, const float* w, const Epilogue& ep,
                          float* y, cudaStream_t st) {
    Params p{};
    p.s = make_shape(g, ConvMode::Fwd);
    p.a = x; p.b = w; p.out = y;
    p.bias = ep.bias;
    p.residual = static_cast<const float*>(ep.residual);
    p.relu = ep.relu;
    p.splits = 1;
    p.kb_per_split = (p.s.Kdim + TK - 1) / TK;
    return run<ConvMode::Fwd>(p, st);
}

cudaError_t conv_ffma_dgrad(const ConvGeom& g, const float* dy, const float* w,
                            const Epilogue& ep, float* dx, cudaStream_t st) {
    Params p{};
    p.s = make_shape(g, ConvMode::Dgrad);
    p.a = dy; p.b = w; p.out = dx;
    p.residual = static_cast<const float*>(ep.residual);
    p.mask = static_cast<const float*>(ep.mask);
    p.splits = 1;
    p.kb_per_split = (p.s.Kdim + TK - 1) / TK;
    return run<ConvMode::Dgrad>(p, st);
}

cudaError_t conv_ffma_wgrad(const ConvGeom& g, const float* dy, const float* x, float* dw,
                            void* workspace, cudaStream_t st) {
    Params p{};
    p.s = make_shape(g, ConvMode::Wgrad);
    p.a = dy; p.b = x;
    p.splits = wgrad_splits(p.s, p.kb_per_split);
    if (p.splits > 1 && !workspace) return cudaErrorInvalidValue;
    p.out = p.splits > 1 ? static_cast<float*>(workspace) : dw;
    cudaError_t e = run<ConvMode::Wgrad>(p, st);
    if (e != cudaSuccess || p.splits == 1) return e;
    return split_reduce(static_cast<float*>(workspace), p.splits, size_t(p.s.M) * p.s.Ncol, dw, st);
}

}  // namespace tcb
