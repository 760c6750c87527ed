// HBM-bound kernels of the step: synthetic fills, casts, the weight
// transpose dgrad needs, deterministic reductions (bias grads, split-K),
// pools, softmax cross-entropy and the fused momentum-SGD shard update.
//
// Arithmetic that the CPU oracle must reproduce bit-exactly (RNG fill,
// labels, SGD) uses explicitly rounded intrinsics (__fmul_rn/__fadd_rn) so
// nvcc cannot contract it into FMAs; oracle/numerics.c is compiled with
// -ffp-contract=off to match.
#include <algorithm>

#include "common.cuh"

namespace tcb {
namespace {

constexpr int kBlock = 256;

inline int grid_for(size_t n, int per_thread = 1) {
    size_t blocks = (n + size_t(kBlock) * per_thread - 1) / (size_t(kBlock) * per_thread);
    const size_t cap = size_t(num_sms()) * 16;
    return static_cast<int>(std::max<size_t>(1, std::min(blocks, cap)));
}

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t stream_base(uint64_t seed, uint64_t tag) {
    return splitmix64(seed ^ splitmix64(tag));
}

template <typename T>
__global__ void fill_uniform_kernel(T* p, size_t n, uint64_t base, float lo, float span) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t bits = splitmix64(base + i);
        const float u = static_cast<float>(bits >> 40) * (1.0f / 16777216.0f);
        p[i] = from_f32<T>(__fadd_rn(lo, __fmul_rn(span, u)));
    }
}

__global__ void fill_labels_kernel(int32_t* labels, int n, int classes, uint64_t base) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) labels[i] = static_cast<int32_t>(splitmix64(base + i) % uint64_t(classes));
}

template <typename S, typename D>
__global__ void cast_kernel(const S* src, D* dst, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        dst[i] = from_f32<D>(to_f32<S>(src[i]));
}

// [K][RS][C] -> [C][RS][K], 32x32 tiles through shared memory.
template <typename T>
__global__ void transpose_krsc_kernel(const T* __restrict__ w, T* __restrict__ wT, int K, int RS,
                                      int C) {
    __shared__ T tile[32][33];
    const int rs = blockIdx.z;
    const int c0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, c = c0 + threadIdx.x;
        if (k < K && c < C) tile[i][threadIdx.x] = w[(size_t(k) * RS + rs) * C + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, k = k0 + threadIdx.x;
        if (k < K && c < C) wT[(size_t(c) * RS + rs) * K + k] = tile[threadIdx.x][i];
    }
}

// w[K][R][S][C] -> per-phase packed dgrad operand [C][tr][ts][K] (see DgradPhase);
// one (r, s) tap per blockIdx.z, 32x32 (c, k) tiles through shared memory.
template <typename T>
__device__ __forceinline__ void pack_dgrad_block(const T* __restrict__ w, T* __restrict__ out,
                                                 const ConvGeom& g, int bx, int by, int bz) {
    __shared__ T tile[32][33];
    const int r = bz / g.s, s = bz % g.s;
    const int ph = ((r - g.pad_h) % g.stride_h + g.stride_h) % g.stride_h;
    const int pw = ((s - g.pad_w) % g.stride_w + g.stride_w) % g.stride_w;
    const DgradPhase d = dgrad_phase(g, ph, pw);
    // taps are stored flipped (ri' = tr - 1 - ri) so the dy operand walks forward
    const int ri = d.tr - 1 - (r - d.r0) / g.stride_h, si = d.ts - 1 - (s - d.s0) / g.stride_w;
    const int c0 = bx * 32, k0 = by * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int k = k0 + i, c = c0 + threadIdx.x;
        if (k < g.k && c < g.c) tile[i][threadIdx.x] = w[((size_t(k) * g.r + r) * g.s + s) * g.c + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, k = k0 + threadIdx.x;
        if (k < g.k && c < g.c)
            out[d.woff + ((size_t(c) * d.tr + ri) * d.ts + si) * g.k + k] = tile[threadIdx.x][i];
    }
}

template <typename T>
__global__ void pack_dgrad_kernel(const T* __restrict__ w, T* __restrict__ out, ConvGeom g) {
    pack_dgrad_block<T>(w, out, g, blockIdx.x, blockIdx.y, blockIdx.z);
}

// Every layer's dgrad packing in one launch: block b belongs to the job with
// the largest block_begin <= b.
__global__ void pack_dgrad_batched_kernel(const PackDgradJob* __restrict__ jobs, int njobs) {
    const int b = blockIdx.x;
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].block_begin <= b) lo = mid; else hi = mid - 1;
    }
    const PackDgradJob& j = jobs[lo];
    const int local = b - j.block_begin;
    const int gx = (j.g.c + 31) / 32, gy = (j.g.k + 31) / 32;
    pack_dgrad_block<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(j.w),
                                    static_cast<__nv_bfloat16*>(j.out), j.g, local % gx,
                                    (local / gx) % gy, local / (gx * gy));
}

template <typename T>
__global__ void column_partial_kernel(const T* __restrict__ in, float* __restrict__ part,
                                      int rows, int cols, int rows_per_chunk) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= cols) return;
    const int r0 = blockIdx.y * rows_per_chunk;
    const int r1 = min(rows, r0 + rows_per_chunk);
    float acc = 0.f;
    for (int r = r0; r < r1; ++r) acc += to_f32<T>(in[size_t(r) * cols + col]);
    part[size_t(blockIdx.y) * cols + col] = acc;
}

// Column sums (bias gradients) with 16-byte loads: thread = one 16-byte column
// group (V = 8 bf16 / 4 fp32) x one row lane; a block's rows are strided over
// its lanes, lanes reduced in shared memory, one fp32 partial row per block.
template <typename T>
__global__ void __launch_bounds__(256) column_partial_vec_kernel(const T* __restrict__ in, float* __restrict__ part,
                                                                 int rows, int cols, int rows_per_chunk) {
    constexpr int V = 16 / sizeof(T);
    __shared__ float red[2048];
    const int groups = cols / V;
    const int lanes = groups <= 256 ? 256 / groups : 1;
    const int r0 = blockIdx.x * rows_per_chunk;
    const int r1 = min(rows, r0 + rows_per_chunk);
    if (lanes > 1) {
        const int g = threadIdx.x % groups, lane = threadIdx.x / groups;
        float acc[V] = {};
        if (lane < lanes) {
            for (int r = r0 + lane; r < r1; r += lanes) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(in + size_t(r) * cols) + g);
                const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] += to_f32<T>(e[j]);
            }
#pragma unroll
            for (int j = 0; j < V; ++j) red[lane * cols + g * V + j] = acc[j];
        }
        __syncthreads();
        for (int c = threadIdx.x; c < cols; c += blockDim.x) {
            float t = 0.f;
            for (int l = 0; l < lanes; ++l) t += red[l * cols + c];
            part[size_t(blockIdx.x) * cols + c] = t;
        }
    } else {
        for (int g = threadIdx.x; g < groups; g += blockDim.x) {
            float acc[V] = {};
            for (int r = r0; r < r1; ++r) {
                const uint4 u = __ldg(reinterpret_cast<const uint4*>(in + size_t(r) * cols) + g);
                const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
                for (int j = 0; j < V; ++j) acc[j] += to_f32<T>(e[j]);
            }
#pragma unroll
            for (int j = 0; j < V; ++j) part[size_t(blockIdx.x) * cols + g * V + j] = acc[j];
        }
    }
}

__global__ void split_reduce_kernel(const float* __restrict__ parts, int splits, size_t n,
                                    float* __restrict__ out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int s = 0; s < splits; ++s) acc += parts[size_t(s) * n + i];
        out[i] = acc;
    }
}

__global__ void split_reduce4_kernel(const float4* __restrict__ parts, int splits, size_t n4,
                                     float4* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
         i += size_t(gridDim.x) * blockDim.x) {
        float4 acc = __ldcs(parts + i);
        for (int s0 = 1; s0 < splits; s0 += 8) {  // 8 loads in flight, adds in split order
            float4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j < splits) v[j] = __ldcs(parts + size_t(s0 + j) * n4 + i);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j < splits) {
                    acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w;
                }
        }
        out[i] = acc;
    }
}

// Many splits over few elements (early wgrad layers: up to 64 splits of a
// 64 x 576 tile): 8 split-groups per element run in parallel, group g summing
// splits g, g+8, ... in order, then the 8 group sums are added in order g = 0..7
// — a fixed tree, so the result is deterministic.
__global__ void __launch_bounds__(256) split_reduce4_tree_kernel(const float4* __restrict__ parts,
                                                                 int splits, size_t n4,
                                                                 float4* __restrict__ out) {
    __shared__ float4 part[8][32];
    pdl_wait();
    pdl_trigger();
    const int e = threadIdx.x & 31, g = threadIdx.x >> 5;
    const size_t i = blockIdx.x * size_t(32) + e;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < n4) {
        for (int s0 = g; s0 < splits; s0 += 64) {
            float4 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + 8 * j < splits) v[j] = __ldcs(parts + size_t(s0 + 8 * j) * n4 + i);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + 8 * j < splits) {
                    acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w;
                }
        }
    }
    part[g][e] = acc;
    __syncthreads();
    if (g == 0 && i < n4) {
#pragma unroll
        for (int k = 1; k < 8; ++k) {
            acc.x += part[k][e].x; acc.y += part[k][e].y; acc.z += part[k][e].z; acc.w += part[k][e].w;
        }
        out[i] = acc;
    }
}

// One PS shard: g' = g*scale + wd*w ; v = mom*v + g' ; w = w - lr*v ; wc = compute copy.
template <typename CT>
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                           float* __restrict__ v, CT* __restrict__ wc, size_t n, float lr,
                           float mom, float wd, float gscale) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const float wi = w[i];
        const float gi = __fadd_rn(__fmul_rn(g[i], gscale), __fmul_rn(wd, wi));
        const float vi = __fadd_rn(__fmul_rn(mom, v[i]), gi);
        const float wn = __fsub_rn(wi, __fmul_rn(lr, vi));
        v[i] = vi;
        w[i] = wn;
        if (wc) wc[i] = from_f32<CT>(wn);
    }
}

// Vectorised variant: 4 params per thread-iteration (n % 4 == 0, 16B-aligned).
template <typename CT>
__global__ void sgd4_kernel(float4* __restrict__ w, const float4* __restrict__ g,
                            float4* __restrict__ v, CT* __restrict__ wc, size_t n4, float lr,
                            float mom, float wd, float gscale) {
    pdl_wait();
    pdl_trigger();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n4;
         i += size_t(gridDim.x) * blockDim.x) {
        float4 wi = w[i], gi = g[i], vi = v[i];
        float* wp = &wi.x;
        float* gp = &gi.x;
        float* vp = &vi.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float gg = __fadd_rn(__fmul_rn(gp[j], gscale), __fmul_rn(wd, wp[j]));
            vp[j] = __fadd_rn(__fmul_rn(mom, vp[j]), gg);
            wp[j] = __fsub_rn(wp[j], __fmul_rn(lr, vp[j]));
        }
        v[i] = vi;
        w[i] = wi;
        if (wc) {
            if constexpr (sizeof(CT) == 2) {  // the four bf16 copies as one 8-byte store
                __align__(8) CT q[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) q[j] = from_f32<CT>(wp[j]);
                reinterpret_cast<uint2*>(wc)[i] = *reinterpret_cast<const uint2*>(q);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) wc[4 * i + j] = from_f32<CT>(wp[j]);
            }
        }
    }
}

template <typename T>
__global__ void pack_channels_kernel(const float* __restrict__ src, T* __restrict__ dst,
                                     size_t pixels, int cl, int cp) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < pixels * cp;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t px = i / cp;
        const int c = int(i % cp);
        dst[i] = from_f32<T>(c < cl ? src[px * cl + c] : 0.f);
    }
}

// uint8 pixels -> (u + 0.5) / 128 - 1 in (-1, 1), channel-padded to cp.
template <typename T>
__global__ void pack_channels_u8_kernel(const uint8_t* __restrict__ src, T* __restrict__ dst,
                                        size_t pixels, int cl, int cp) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < pixels * cp;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t px = i / cp;
        const int c = int(i % cp);
        dst[i] = from_f32<T>(c < cl ? __fsub_rn(__fmul_rn(float(src[px * cl + c]) + 0.5f, 0.0078125f), 1.f)
                                    : 0.f);
    }
}

// bf16, 8 padded channels (the RGB input): one pixel per thread, cl <= 8 bytes
// in, one 16-byte row out (same arithmetic as pack_channels_u8_kernel)
__global__ void pack_u8_bf16x8_kernel(const uint8_t* __restrict__ src, uint4* __restrict__ dst, size_t pixels,
                                      int cl) {
    pdl_wait();
    pdl_trigger();
    for (size_t px = blockIdx.x * size_t(blockDim.x) + threadIdx.x; px < pixels;
         px += size_t(gridDim.x) * blockDim.x) {
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c)
            v[c] = __float2bfloat16_rn(
                c < cl ? __fsub_rn(__fmul_rn(float(__ldg(src + px * cl + c)) + 0.5f, 0.0078125f), 1.f) : 0.f);
        dst[px] = *reinterpret_cast<const uint4*>(v);
    }
}

template <typename T>
__global__ void add_kernel(T* y, const T* x, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        y[i] = from_f32<T>(to_f32<T>(y[i]) + to_f32<T>(x[i]));
}

template <typename T>
__global__ void relu_mask_kernel(T* g, const T* act, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        if (!(to_f32<T>(act[i]) > 0.f)) g[i] = from_f32<T>(0.f);
}

// Max pool, NHWC; padded positions never win; ties keep the first (r, s) in scan order.
template <typename T>
__global__ void maxpool_fwd_kernel(const T* __restrict__ x, T* __restrict__ y,
                                   uint8_t* __restrict__ arg, int N, int H, int W, int C, int F,
                                   int S, int P, int Ho, int Wo) {
    const size_t total = size_t(N) * Ho * Wo * C;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        size_t t = i / C;
        const int wo = int(t % Wo);
        t /= Wo;
        const int ho = int(t % Ho);
        const int n = int(t / Ho);
        float best = -INFINITY;
        int best_idx = 0;
        for (int r = 0; r < F; ++r) {
            const int h = ho * S - P + r;
            if (h < 0 || h >= H) continue;
            for (int s = 0; s < F; ++s) {
                const int w = wo * S - P + s;
                if (w < 0 || w >= W) continue;
                const float v = to_f32<T>(x[((size_t(n) * H + h) * W + w) * C + c]);
                if (v > best) {
                    best = v;
                    best_idx = r * F + s;
                }
            }
        }
        y[i] = from_f32<T>(best);
        if (arg) arg[i] = static_cast<uint8_t>(best_idx);
    }
}

template <typename T>
__global__ void maxpool_bwd_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ arg,
                                   T* __restrict__ dx, int N, int H, int W, int C, int F, int S,
                                   int P, int Ho, int Wo, const T* __restrict__ ymask) {
    const size_t total = size_t(N) * H * W * C;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        size_t t = i / C;
        const int w = int(t % W);
        t /= W;
        const int h = int(t % H);
        const int n = int(t / H);
        // windows (ho, wo) with ho*S - P <= h <= ho*S - P + F - 1
        const int ho0 = max(0, (h + P - F + S) / S), ho1 = min(Ho - 1, (h + P) / S);
        const int wo0 = max(0, (w + P - F + S) / S), wo1 = min(Wo - 1, (w + P) / S);
        float acc = 0.f;
        for (int ho = ho0; ho <= ho1; ++ho) {
            const int r = h - (ho * S - P);
            if (r < 0 || r >= F) continue;
            for (int wo = wo0; wo <= wo1; ++wo) {
                const int s = w - (wo * S - P);
                if (s < 0 || s >= F) continue;
                const size_t o = ((size_t(n) * Ho + ho) * Wo + wo) * C + c;
                if (arg[o] == r * F + s && (!ymask || to_f32<T>(ymask[o]) > 0.f))
                    acc += to_f32<T>(dy[o]);
            }
        }
        dx[i] = from_f32<T>(acc);
    }
}

template <typename T>
__global__ void avgpool_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, int N, int HW,
                                   int C) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * C) return;
    const int n = i / C, c = i % C;
    float acc = 0.f;
    for (int p = 0; p < HW; ++p) acc += to_f32<T>(x[(size_t(n) * HW + p) * C + c]);
    y[i] = from_f32<T>(acc / float(HW));
}

template <typename T>
__global__ void avgpool_bwd_kernel(const T* __restrict__ dy, T* __restrict__ dx, int N, int HW,
                                   int C, const T* __restrict__ mask) {
    const size_t total = size_t(N) * HW * C;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int c = int(i % C);
        const int n = int(i / (size_t(HW) * C));
        float v = to_f32<T>(dy[size_t(n) * C + c]) / float(HW);
        if (mask && !(to_f32<T>(mask[i]) > 0.f)) v = 0.f;
        dx[i] = from_f32<T>(v);
    }
}

// bf16, C % 8 == 0: 8 channels per thread, 32-bit index math, fused ReLU mask.
__global__ void avgpool_bwd_vec_kernel(const __nv_bfloat16* __restrict__ dy,
                                       __nv_bfloat16* __restrict__ dx, int total8, int HW, int cg,
                                       const __nv_bfloat16* __restrict__ mask) {
    pdl_wait();
    pdl_trigger();
    const float inv = 1.f / float(HW);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total8; i += gridDim.x * blockDim.x) {
        const int ci = i % cg, n = i / (HW * cg);
        const uint4 g = reinterpret_cast<const uint4*>(dy)[n * cg + ci];
        const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&g);
        uint4 m = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);  // 1.0
        if (mask) m = reinterpret_cast<const uint4*>(mask)[i];
        const __nv_bfloat162* mh = reinterpret_cast<const __nv_bfloat162*>(&m);
        uint4 o;
        __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 a = __bfloat1622float2(gh[j]);
            const float2 k = __bfloat1622float2(mh[j]);
            oh[j] = __floats2bfloat162_rn(k.x > 0.f ? a.x * inv : 0.f, k.y > 0.f ? a.y * inv : 0.f);
        }
        reinterpret_cast<uint4*>(dx)[i] = o;
    }
}

// One block per row: softmax, per-row loss, gradient (p - onehot) / N.
template <typename T>
__global__ void softmax_xent_kernel(const T* __restrict__ logits, const int32_t* __restrict__ lab,
                                    T* __restrict__ dl, float* __restrict__ row_loss, int N,
                                    int K, int ld) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[32];
    const int n = blockIdx.x;
    const T* z = logits + size_t(n) * ld;
    float m = -INFINITY;
    for (int k = threadIdx.x; k < K; k += blockDim.x) m = fmaxf(m, to_f32<T>(z[k]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    m = red[0];
    __syncthreads();
    float s = 0.f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) s += expf(to_f32<T>(z[k]) - m);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    s = red[0];
    const int y = lab[n];
    const float inv_n = 1.0f / float(N);
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const float pk = expf(to_f32<T>(z[k]) - m) / s;
        dl[size_t(n) * ld + k] = from_f32<T>((pk - (k == y ? 1.f : 0.f)) * inv_n);
    }
    for (int k = K + threadIdx.x; k < ld; k += blockDim.x) dl[size_t(n) * ld + k] = from_f32<T>(0.f);
    if (threadIdx.x == 0) row_loss[n] = logf(s) + m - to_f32<T>(z[y]);
}

__global__ void mean_kernel(float* loss, const float* row_loss, int N) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < N; ++i) acc += row_loss[i];
        loss[0] = static_cast<float>(acc / N);
    }
}

}  // namespace

#define TCB_DT_SWITCH(dt, T, ...)                   \
    do {                                            \
        if ((dt) == DType::F32) {                   \
            using T = float;                        \
            __VA_ARGS__;                            \
        } else {                                    \
            using T = __nv_bfloat16;                \
            __VA_ARGS__;                            \
        }                                           \
    } while (0)

cudaError_t fill_uniform(DType dt, void* p, size_t n, uint64_t seed, uint64_t tag, float lo,
                         float hi, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const uint64_t base = stream_base(seed, tag);
    const float span = hi - lo;
    TCB_DT_SWITCH(dt, T, (fill_uniform_kernel<T><<<grid_for(n, 4), kBlock, 0, st>>>(
                              static_cast<T*>(p), n, base, lo, span)));
    return cudaGetLastError();
}

cudaError_t fill_labels(int32_t* labels, int n, int classes, uint64_t seed, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const uint64_t base = stream_base(seed, 0x4C4142454C53ull);
    fill_labels_kernel<<<(n + kBlock - 1) / kBlock, kBlock, 0, st>>>(labels, n, classes, base);
    return cudaGetLastError();
}

cudaError_t cast(DType src_t, const void* src, DType dst_t, void* dst, size_t n,
                 cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    TCB_DT_SWITCH(src_t, S, TCB_DT_SWITCH(dst_t, D, (cast_kernel<S, D><<<grid_for(n, 4), kBlock, 0, st>>>(
                                                        static_cast<const S*>(src), static_cast<D*>(dst), n))));
    return cudaGetLastError();
}

cudaError_t transpose_krsc(DType dt, const void* w, void* wT, int K, int R, int S, int C,
                           cudaStream_t st) {
    dim3 grid((C + 31) / 32, (K + 31) / 32, R * S), block(32, 8);
    TCB_DT_SWITCH(dt, T, (transpose_krsc_kernel<T><<<grid, block, 0, st>>>(
                              static_cast<const T*>(w), static_cast<T*>(wT), K, R * S, C)));
    return cudaGetLastError();
}

cudaError_t pack_dgrad_weights(DType dt, const void* w, void* packed, const ConvGeom& g,
                               cudaStream_t st) {
    dim3 grid((g.c + 31) / 32, (g.k + 31) / 32, g.r * g.s), block(32, 8);
    TCB_DT_SWITCH(dt, T, (pack_dgrad_kernel<T><<<grid, block, 0, st>>>(
                              static_cast<const T*>(w), static_cast<T*>(packed), g)));
    return cudaGetLastError();
}

int pack_dgrad_blocks(const ConvGeom& g) {
    return ((g.c + 31) / 32) * ((g.k + 31) / 32) * g.r * g.s;
}

cudaError_t pack_dgrad_weights_batched(const PackDgradJob* jobs, int njobs, int total_blocks,
                                       cudaStream_t st) {
    if (njobs == 0) return cudaSuccess;
    pack_dgrad_batched_kernel<<<total_blocks, dim3(32, 8), 0, st>>>(jobs, njobs);
    return cudaGetLastError();
}

size_t column_sum_workspace(int rows, int cols) {
    const int chunks = std::min(rows, 512);
    return size_t(chunks) * cols * sizeof(float);
}

cudaError_t column_sum(DType dt, const void* in, float* out, int rows, int cols, float* ws,
                       cudaStream_t st) {
    const int v = static_cast<int>(16 / dtype_size(dt));
    if (cols % v == 0 && cols <= 2048 * v && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
        // ~4 blocks per SM, each a contiguous row range (<= 512 chunks: the workspace bound)
        const int chunks = std::max(1, std::min({rows, 512, num_sms() * 4}));
        const int per = (rows + chunks - 1) / chunks;
        const int used = (rows + per - 1) / per;
        TCB_DT_SWITCH(dt, T, (column_partial_vec_kernel<T><<<used, 256, 0, st>>>(
                                  static_cast<const T*>(in), ws, rows, cols, per)));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        return split_reduce(ws, used, size_t(cols), out, st);
    }
    const int chunks = std::min(rows, 512);
    const int per = (rows + chunks - 1) / chunks;
    const int used = (rows + per - 1) / per;
    const int tpb = cols >= 128 ? 128 : 32 * ((cols + 31) / 32);
    dim3 grid((cols + tpb - 1) / tpb, used);
    TCB_DT_SWITCH(dt, T, (column_partial_kernel<T><<<grid, tpb, 0, st>>>(
                              static_cast<const T*>(in), ws, rows, cols, per)));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return split_reduce(ws, used, size_t(cols), out, st);
}

cudaError_t split_reduce(const float* parts, int splits, size_t n, float* out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = n % 4 == 0 && (reinterpret_cast<uintptr_t>(parts) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (vec && splits >= 16 && n / 4 < size_t(num_sms()) * 256 * 4)
        return launch_pdl(split_reduce4_tree_kernel, dim3(static_cast<int>((n / 4 + 31) / 32)), dim3(256), 0,
                          st, reinterpret_cast<const float4*>(parts), splits, n / 4,
                          reinterpret_cast<float4*>(out));
    else if (vec)
        return launch_pdl(split_reduce4_kernel, dim3(grid_for(n / 4, 2)), dim3(kBlock), 0, st,
                          reinterpret_cast<const float4*>(parts), splits, n / 4,
                          reinterpret_cast<float4*>(out));
    else
        split_reduce_kernel<<<grid_for(n), kBlock, 0, st>>>(parts, splits, n, out);
    return cudaGetLastError();
}

cudaError_t sgd_momentum(float* w, const float* g, float* v, DType cdt, void* wc, size_t n,
                         float lr, float mom, float wd, float gscale, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = n % 4 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(g) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(v) % 16 == 0;
    TCB_DT_SWITCH(cdt, CT, {
        if (vec)
            return launch_pdl(sgd4_kernel<CT>, dim3(grid_for(n / 4, 2)), dim3(kBlock), 0, st,
                              reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(g),
                              reinterpret_cast<float4*>(v), static_cast<CT*>(wc), n / 4, lr, mom, wd,
                              gscale);
        else
            sgd_kernel<CT><<<grid_for(n, 4), kBlock, 0, st>>>(w, g, v, static_cast<CT*>(wc), n, lr,
                                                              mom, wd, gscale);
    });
    return cudaGetLastError();
}

cudaError_t pack_channels_u8(DType dt, const uint8_t* src, void* dst, size_t pixels, int cl, int cp,
                             cudaStream_t st) {
    if (dt == DType::BF16 && cp == 8 && cl <= 8 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0)
        return launch_pdl(pack_u8_bf16x8_kernel, dim3(grid_for(pixels, 2)), dim3(kBlock), 0, st, src,
                          static_cast<uint4*>(dst), pixels, cl);
    TCB_DT_SWITCH(dt, T, (pack_channels_u8_kernel<T><<<grid_for(pixels * cp, 4), kBlock, 0, st>>>(
                              src, static_cast<T*>(dst), pixels, cl, cp)));
    return cudaGetLastError();
}

cudaError_t pack_channels(DType dt, const float* src, void* dst, size_t pixels, int cl, int cp,
                          cudaStream_t st) {
    TCB_DT_SWITCH(dt, T, (pack_channels_kernel<T><<<grid_for(pixels * cp, 4), kBlock, 0, st>>>(
                              src, static_cast<T*>(dst), pixels, cl, cp)));
    return cudaGetLastError();
}

cudaError_t add_inplace(DType dt, void* y, const void* x, size_t n, cudaStream_t st) {
    TCB_DT_SWITCH(dt, T, (add_kernel<T><<<grid_for(n, 4), kBlock, 0, st>>>(
                              static_cast<T*>(y), static_cast<const T*>(x), n)));
    return cudaGetLastError();
}

cudaError_t relu_mask_inplace(DType dt, void* g, const void* act, size_t n, cudaStream_t st) {
    TCB_DT_SWITCH(dt, T, (relu_mask_kernel<T><<<grid_for(n, 4), kBlock, 0, st>>>(
                              static_cast<T*>(g), static_cast<const T*>(act), n)));
    return cudaGetLastError();
}

namespace {

// 16-byte vector of V elements of T (V = 8 for bf16, 4 for fp32).
template <typename T, int V>
struct alignas(16) Vec {
    T v[V];
};

// Vectorised NHWC max pool: one block per output row (n, ho), one thread =
// V consecutive channels of one output pixel (32-bit index math only; the
// row is contiguous so loads and stores coalesce). argmax bytes stored V at a
// time. Same tie rule as the scalar kernel (first maximum in window order).
template <typename T, int V>
__global__ void __launch_bounds__(256) maxpool_fwd_vec_kernel(
    const T* __restrict__ x, T* __restrict__ y, uint8_t* __restrict__ arg, int N, int H, int W,
    int C, int F, int S, int P, int Ho, int Wo) {
    const int cg = C / V;
    const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
    const int h0 = ho * S - P;
    const T* xn = x + size_t(n) * H * W * C;
    const size_t orow = size_t(blockIdx.x) * Wo * C;
    for (int i = threadIdx.x; i < Wo * cg; i += blockDim.x) {
        const int wo = i / cg, c = (i - wo * cg) * V;
        const int w0 = wo * S - P;
        float best[V];
        uint8_t bi[V];
#pragma unroll
        for (int j = 0; j < V; ++j) {
            best[j] = -INFINITY;
            bi[j] = 0;
        }
        for (int r = 0; r < F; ++r) {
            const int h = h0 + r;
            if (h < 0 || h >= H) continue;
            for (int s = 0; s < F; ++s) {
                const int w = w0 + s;
                if (w < 0 || w >= W) continue;
                const Vec<T, V> in = *reinterpret_cast<const Vec<T, V>*>(xn + (h * W + w) * C + c);
#pragma unroll
                for (int j = 0; j < V; ++j) {
                    const float v = to_f32<T>(in.v[j]);
                    if (v > best[j]) {
                        best[j] = v;
                        bi[j] = static_cast<uint8_t>(r * F + s);
                    }
                }
            }
        }
        Vec<T, V> out;
#pragma unroll
        for (int j = 0; j < V; ++j) out.v[j] = from_f32<T>(best[j]);
        const size_t o = orow + size_t(wo) * C + c;
        *reinterpret_cast<Vec<T, V>*>(y + o) = out;
        if (arg) {
            Vec<uint8_t, V> a;
#pragma unroll
            for (int j = 0; j < V; ++j) a.v[j] = bi[j];
            *reinterpret_cast<Vec<uint8_t, V>*>(arg + o) = a;
        }
    }
}

// Gather-form backward, one block per input row (n, h), V channels per
// thread, optional fused ReLU mask of the pool input (dx *= [x > 0]).
template <typename T, int V>
__global__ void __launch_bounds__(256) maxpool_bwd_vec_kernel(
    const T* __restrict__ dy, const uint8_t* __restrict__ arg, T* __restrict__ dx,
    const T* __restrict__ ymask, int N, int H, int W, int C, int F, int S, int P, int Ho, int Wo) {
    const int cg = C / V;
    const int n = blockIdx.x / H, h = blockIdx.x - n * H;
    const int ho0 = max(0, (h + P - F + S) / S), ho1 = min(Ho - 1, (h + P) / S);
    const size_t nbase = size_t(n) * Ho * Wo * C;
    const size_t irow = size_t(blockIdx.x) * W * C;
    for (int i = threadIdx.x; i < W * cg; i += blockDim.x) {
        const int w = i / cg, c = (i - w * cg) * V;
        const int wo0 = max(0, (w + P - F + S) / S), wo1 = min(Wo - 1, (w + P) / S);
        float acc[V];
#pragma unroll
        for (int j = 0; j < V; ++j) acc[j] = 0.f;
        for (int ho = ho0; ho <= ho1; ++ho) {
            const int r = h - (ho * S - P);
            if (r < 0 || r >= F) continue;
            for (int wo = wo0; wo <= wo1; ++wo) {
                const int s = w - (wo * S - P);
                if (s < 0 || s >= F) continue;
                const size_t o = nbase + size_t(ho * Wo + wo) * C + c;
                const Vec<T, V> g = *reinterpret_cast<const Vec<T, V>*>(dy + o);
                const Vec<uint8_t, V> a = *reinterpret_cast<const Vec<uint8_t, V>*>(arg + o);
                const uint8_t want = static_cast<uint8_t>(r * F + s);
                if (ymask) {
                    const Vec<T, V> y = *reinterpret_cast<const Vec<T, V>*>(ymask + o);
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (a.v[j] == want && to_f32<T>(y.v[j]) > 0.f) acc[j] += to_f32<T>(g.v[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (a.v[j] == want) acc[j] += to_f32<T>(g.v[j]);
                }
            }
        }
        const size_t io = irow + size_t(w) * C + c;
        Vec<T, V> out;
#pragma unroll
        for (int j = 0; j < V; ++j) out.v[j] = from_f32<T>(acc[j]);
        *reinterpret_cast<Vec<T, V>*>(dx + io) = out;
    }
}

// bf16 specialisations, 8 channels per thread as 4 packed bf16x2 lanes:
// max / strict-greater via __hmax2 / __hgt2_mask (bit-identical to the
// scalar rule: first maximum in window order wins), argmax codes as 16-bit
// halves; backward matches argmax bytes with __vcmpeq4 and selects dy bits
// with the mask, accumulating in fp32 as the generic kernel does.
__global__ void __launch_bounds__(256) maxpool_fwd_bf16x8_kernel(
    const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ arg,
    int H, int W, int C, int F, int S, int P, int Ho, int Wo) {
    pdl_wait();
    pdl_trigger();
    const int cg = C / 8;
    const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
    const int h0 = ho * S - P;
    const __nv_bfloat16* xn = x + size_t(n) * H * W * C;
    const size_t orow = size_t(blockIdx.x) * Wo * C;
    for (int i = threadIdx.x; i < Wo * cg; i += blockDim.x) {
        const int wo = i / cg, c = (i - wo * cg) * 8;
        const int w0 = wo * S - P;
        __nv_bfloat162 best[4];
        uint32_t idx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            best[j] = __halves2bfloat162(__ushort_as_bfloat16(0xFF80u), __ushort_as_bfloat16(0xFF80u));
            idx[j] = 0;
        }
        for (int r = 0; r < F; ++r) {
            const int h = h0 + r;
            if (h < 0 || h >= H) continue;
            for (int sx = 0; sx < F; ++sx) {
                const int w = w0 + sx;
                if (w < 0 || w >= W) continue;
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(xn + (h * W + w) * C + c));
                const uint32_t code = static_cast<uint32_t>(r * F + sx) * 0x00010001u;
                const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&vw[j]);
                    const uint32_t gt = __hgt2_mask(b, best[j]);
                    best[j] = __hmax2(best[j], b);
                    idx[j] = (idx[j] & ~gt) | (code & gt);
                }
            }
        }
        const size_t o = orow + size_t(wo) * C + c;
        uint4 out;
        out.x = *reinterpret_cast<uint32_t*>(&best[0]);
        out.y = *reinterpret_cast<uint32_t*>(&best[1]);
        out.z = *reinterpret_cast<uint32_t*>(&best[2]);
        out.w = *reinterpret_cast<uint32_t*>(&best[3]);
        *reinterpret_cast<uint4*>(y + o) = out;
        if (arg)
            *reinterpret_cast<uint2*>(arg + o) =
                make_uint2(__byte_perm(idx[0], idx[1], 0x6420), __byte_perm(idx[2], idx[3], 0x6420));
    }
}

__global__ void __launch_bounds__(256) maxpool_bwd_bf16x8_kernel(
    const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
    __nv_bfloat16* __restrict__ dx, const __nv_bfloat16* __restrict__ ymask, int H, int W, int C,
    int F, int S, int P, int Ho, int Wo) {
    const int cg = C / 8;
    const int n = blockIdx.x / H, h = blockIdx.x - n * H;
    const int ho0 = max(0, (h + P - F + S) / S), ho1 = min(Ho - 1, (h + P) / S);
    const size_t nbase = size_t(n) * Ho * Wo * C;
    const size_t irow = size_t(blockIdx.x) * W * C;
    const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
    for (int i = threadIdx.x; i < W * cg; i += blockDim.x) {
        const int w = i / cg, c = (i - w * cg) * 8;
        const int wo0 = max(0, (w + P - F + S) / S), wo1 = min(Wo - 1, (w + P) / S);
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int ho = ho0; ho <= ho1; ++ho) {
            const int r = h - (ho * S - P);
            if (r < 0 || r >= F) continue;
            for (int wo = wo0; wo <= wo1; ++wo) {
                const int sx = w - (wo * S - P);
                if (sx < 0 || sx >= F) continue;
                const size_t o = nbase + size_t(ho * Wo + wo) * C + c;
                const uint4 g = __ldg(reinterpret_cast<const uint4*>(dy + o));
                const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o));
                const uint32_t want = static_cast<uint32_t>(r * F + sx) * 0x01010101u;
                const uint32_t lo = __vcmpeq4(a.x, want), hi = __vcmpeq4(a.y, want);
                uint32_t m[4] = {__byte_perm(lo, 0, 0x1100), __byte_perm(lo, 0, 0x3322),
                                 __byte_perm(hi, 0, 0x1100), __byte_perm(hi, 0, 0x3322)};
                if (ymask) {
                    const uint4 yv = __ldg(reinterpret_cast<const uint4*>(ymask + o));
                    const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        m[j] &= __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&yw[j]), zero2);
                }
                const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t sel = gw[j] & m[j];
                    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sel));
                    acc[2 * j] += f.x;
                    acc[2 * j + 1] += f.y;
                }
            }
        }
        uint4 out;
        uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
            ow[j] = *reinterpret_cast<const uint32_t*>(&b);
        }
        *reinterpret_cast<uint4*>(dx + irow + size_t(w) * C + c) = out;
    }
}

// The ResNet stem pool (3x3, stride 2, pad 1) backward, owner-computes: the
// thread of output window (ho, wo) writes input pixels (2ho + a, 2wo + b),
// a, b in {0, 1}, each fed by the windows (ho + dh, wo + dw) whose tap
// (a + 1 - 2dh, b + 1 - 2dw) lies in the filter — 9 (window, tap) pairs known
// at compile time, no index division per pixel. Windows are summed in
// (ho, wo) order, as in the generic kernel.
__device__ __forceinline__ void pool_window_add(float (&acc)[8], const uint4& g, const uint2& a,
                                                const uint32_t (&ypos)[4], bool use_y, int tap) {
    const uint32_t want = static_cast<uint32_t>(tap) * 0x01010101u;
    const uint32_t lo = __vcmpeq4(a.x, want), hi = __vcmpeq4(a.y, want);
    uint32_t m[4] = {__byte_perm(lo, 0, 0x1100), __byte_perm(lo, 0, 0x3322),
                     __byte_perm(hi, 0, 0x1100), __byte_perm(hi, 0, 0x3322)};
    const uint32_t gw[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t sel = gw[j] & m[j] & (use_y ? ypos[j] : 0xFFFFFFFFu);
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&sel));
        acc[2 * j] += f.x;
        acc[2 * j + 1] += f.y;
    }
}

// 3x3 / stride 2, pad P = 1 (ResNet / VGG-style stem pools) or 0 (Inception's
// reduction pools): the 9 window loads are unrolled with compile-time offsets
// and predicated, so a thread has all of them in flight at once (the generic
// kernel's runtime loop issued them one dependent iteration at a time:
// latency-bound at ~4 TB/s). Same tap order and tie rule (first maximum in
// row-major window order wins) as the generic one.
template <int P>
__global__ void __launch_bounds__(256) maxpool_fwd_k3s2_bf16_kernel(
    const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y, uint8_t* __restrict__ arg, int H, int W,
    int C, int Ho, int Wo) {
    pdl_wait();
    pdl_trigger();
    const int cg = C / 8;
    const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
    const int h0 = ho * 2 - P;
    const __nv_bfloat16* xn = x + size_t(n) * H * W * C;
    const size_t orow = size_t(blockIdx.x) * Wo * C;
    for (int i = threadIdx.x; i < Wo * cg; i += blockDim.x) {
        const int wo = i / cg, c = (i - wo * cg) * 8;
        const int w0 = wo * 2 - P;
        uint4 v[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const int h = h0 + t / 3, w = w0 + t % 3;
            v[t] = (h >= 0 && h < H && w >= 0 && w < W)
                       ? __ldg(reinterpret_cast<const uint4*>(xn + (size_t(h) * W + w) * C + c))
                       : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);  // -inf
        }
        __nv_bfloat162 best[4];
        uint32_t idx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            best[j] = __halves2bfloat162(__ushort_as_bfloat16(0xFF80u), __ushort_as_bfloat16(0xFF80u));
            idx[j] = 0;
        }
#pragma unroll
        for (int t = 0; t < 9; ++t) {
            const uint32_t code = static_cast<uint32_t>(t) * 0x00010001u;
            const uint32_t vw[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&vw[j]);
                const uint32_t gt = __hgt2_mask(b, best[j]);
                best[j] = __hmax2(best[j], b);
                idx[j] = (idx[j] & ~gt) | (code & gt);
            }
        }
        const size_t o = orow + size_t(wo) * C + c;
        uint4 out;
        out.x = *reinterpret_cast<uint32_t*>(&best[0]);
        out.y = *reinterpret_cast<uint32_t*>(&best[1]);
        out.z = *reinterpret_cast<uint32_t*>(&best[2]);
        out.w = *reinterpret_cast<uint32_t*>(&best[3]);
        *reinterpret_cast<uint4*>(y + o) = out;
        if (arg)
            *reinterpret_cast<uint2*>(arg + o) =
                make_uint2(__byte_perm(idx[0], idx[1], 0x6420), __byte_perm(idx[2], idx[3], 0x6420));
    }
}

// Owner (ob, wb) computes the 2x2 block of dx rows 2ob + ai, columns 2wb + bi
// from the pooled outputs whose windows cover it: rows ob + dh for dh in
// {0, 1} (P = 1) or {-1, 0} (P = 0), tap r = ai + P - 2 dh.
template <int P>
__global__ void __launch_bounds__(256) maxpool_bwd_k3s2_bf16_kernel(
    const __nv_bfloat16* __restrict__ dy, const uint8_t* __restrict__ arg,
    __nv_bfloat16* __restrict__ dx, const __nv_bfloat16* __restrict__ ymask, int H, int W, int C,
    int Ho, int Wo) {
    pdl_wait();
    pdl_trigger();
    constexpr int kD0 = P == 1 ? 0 : -1;
    const int cg = C / 8;
    const int OH = (H + 1) / 2, OW = (W + 1) / 2;
    const int n = blockIdx.x / OH, ho = blockIdx.x - n * OH;
    const size_t nbase = size_t(n) * Ho * Wo * C;
    const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
    const bool use_y = ymask != nullptr;
    for (int i = threadIdx.x; i < OW * cg; i += blockDim.x) {
        const int wo = i / cg, c = (i - wo * cg) * 8;
        uint4 g[2][2];
        uint2 a[2][2];
        uint32_t yp[2][2][4];
        bool ok[2][2];
#pragma unroll
        for (int dh = 0; dh < 2; ++dh)
#pragma unroll
            for (int dw = 0; dw < 2; ++dw) {
                const int ph = ho + dh + kD0, pw = wo + dw + kD0;
                ok[dh][dw] = ph >= 0 && ph < Ho && pw >= 0 && pw < Wo;
                g[dh][dw] = make_uint4(0, 0, 0, 0);
                a[dh][dw] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
#pragma unroll
                for (int j = 0; j < 4; ++j) yp[dh][dw][j] = 0;
                if (ok[dh][dw]) {
                    const size_t o = nbase + size_t(ph * Wo + pw) * C + c;
                    g[dh][dw] = __ldg(reinterpret_cast<const uint4*>(dy + o));
                    a[dh][dw] = __ldg(reinterpret_cast<const uint2*>(arg + o));
                    if (use_y) {
                        const uint4 yv = __ldg(reinterpret_cast<const uint4*>(ymask + o));
                        const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            yp[dh][dw][j] =
                                __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&yw[j]), zero2);
                    }
                }
            }
#pragma unroll
        for (int ai = 0; ai < 2; ++ai)
#pragma unroll
            for (int bi = 0; bi < 2; ++bi) {
                const int h = 2 * ho + ai, w = 2 * wo + bi;
                if (h >= H || w >= W) continue;
                float acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
                for (int dh = 0; dh < 2; ++dh)
#pragma unroll
                    for (int dw = 0; dw < 2; ++dw) {
                        const int r = ai + P - 2 * (dh + kD0), sx = bi + P - 2 * (dw + kD0);
                        if (r < 0 || sx < 0 || r > 2 || sx > 2) continue;  // compile-time after unrolling
                        pool_window_add(acc, g[dh][dw], a[dh][dw], yp[dh][dw], use_y, r * 3 + sx);
                    }
                uint4 out;
                uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * j], acc[2 * j + 1]);
                    ow[j] = *reinterpret_cast<const uint32_t*>(&b);
                }
                *reinterpret_cast<uint4*>(dx + ((size_t(n) * H + h) * W + w) * C + c) = out;
            }
    }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

cudaError_t maxpool_fwd(DType dt, const void* x, void* y, uint8_t* arg, int n, int h, int w,
                        int c, int f, int s, int p, cudaStream_t st) {
    const int ho = (h + 2 * p - f) / s + 1, wo = (w + 2 * p - f) / s + 1;
    const size_t total = size_t(n) * ho * wo * c;
    if (dt == DType::BF16 && c % 8 == 0 && aligned16(x) && aligned16(y) &&
        (!arg || (reinterpret_cast<uintptr_t>(arg) % 8) == 0) && size_t(h) * w * c < (size_t(1) << 31)) {
        if (f == 3 && s == 2 && (p == 0 || p == 1))
            return launch_pdl(p == 1 ? maxpool_fwd_k3s2_bf16_kernel<1> : maxpool_fwd_k3s2_bf16_kernel<0>,
                              dim3(n * ho), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(x),
                              static_cast<__nv_bfloat16*>(y), arg, h, w, c, ho, wo);
        return launch_pdl(maxpool_fwd_bf16x8_kernel, dim3(n * ho), dim3(256), 0, st,
                          static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), arg, h, w,
                          c, f, s, p, ho, wo);
    }
    TCB_DT_SWITCH(dt, T, {
        constexpr int V = 16 / sizeof(T);
        if (c % V == 0 && aligned16(x) && aligned16(y) && (!arg || (reinterpret_cast<uintptr_t>(arg) % V) == 0) &&
            size_t(h) * w * c < (size_t(1) << 31))
            maxpool_fwd_vec_kernel<T, V><<<n * ho, 256, 0, st>>>(
                static_cast<const T*>(x), static_cast<T*>(y), arg, n, h, w, c, f, s, p, ho, wo);
        else
            maxpool_fwd_kernel<T><<<grid_for(total, 2), kBlock, 0, st>>>(
                static_cast<const T*>(x), static_cast<T*>(y), arg, n, h, w, c, f, s, p, ho, wo);
    });
    return cudaGetLastError();
}

cudaError_t maxpool_bwd(DType dt, const void* dy, const uint8_t* arg, void* dx, int n, int h,
                        int w, int c, int f, int s, int p, cudaStream_t st, const void* ymask) {
    const int ho = (h + 2 * p - f) / s + 1, wo = (w + 2 * p - f) / s + 1;
    const size_t total = size_t(n) * h * w * c;
    if (dt == DType::BF16 && c % 8 == 0 && aligned16(dy) && aligned16(dx) &&
        (!ymask || aligned16(ymask)) && (reinterpret_cast<uintptr_t>(arg) % 8) == 0 &&
        size_t(ho) * wo * c < (size_t(1) << 31) && f == 3 && s == 2 && (p == 0 || p == 1)) {
        return launch_pdl(p == 1 ? maxpool_bwd_k3s2_bf16_kernel<1> : maxpool_bwd_k3s2_bf16_kernel<0>,
                          dim3(n * ((h + 1) / 2)), dim3(256), 0, st,
                          static_cast<const __nv_bfloat16*>(dy), arg, static_cast<__nv_bfloat16*>(dx),
                          static_cast<const __nv_bfloat16*>(ymask), h, w, c, ho, wo);
    }
    if (dt == DType::BF16 && c % 8 == 0 && aligned16(dy) && aligned16(dx) &&
        (!ymask || aligned16(ymask)) && (reinterpret_cast<uintptr_t>(arg) % 8) == 0 &&
        size_t(ho) * wo * c < (size_t(1) << 31)) {
        maxpool_bwd_bf16x8_kernel<<<n * h, 256, 0, st>>>(
            static_cast<const __nv_bfloat16*>(dy), arg, static_cast<__nv_bfloat16*>(dx),
            static_cast<const __nv_bfloat16*>(ymask), h, w, c, f, s, p, ho, wo);
        return cudaGetLastError();
    }
    TCB_DT_SWITCH(dt, T, {
        constexpr int V = 16 / sizeof(T);
        if (c % V == 0 && aligned16(dy) && aligned16(dx) && (!ymask || aligned16(ymask)) &&
            (reinterpret_cast<uintptr_t>(arg) % V) == 0 && size_t(ho) * wo * c < (size_t(1) << 31)) {
            maxpool_bwd_vec_kernel<T, V><<<n * h, 256, 0, st>>>(
                static_cast<const T*>(dy), arg, static_cast<T*>(dx), static_cast<const T*>(ymask), n,
                h, w, c, f, s, p, ho, wo);
        } else {
            maxpool_bwd_kernel<T><<<grid_for(total, 2), kBlock, 0, st>>>(
                static_cast<const T*>(dy), arg, static_cast<T*>(dx), n, h, w, c, f, s, p, ho, wo,
                static_cast<const T*>(ymask));
        }
    });
    return cudaGetLastError();
}

cudaError_t avgpool_global_fwd(DType dt, const void* x, void* y, int n, int hw, int c,
                               cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    TCB_DT_SWITCH(dt, T, (e = launch_pdl(avgpool_fwd_kernel<T>, dim3((n * c + kBlock - 1) / kBlock), dim3(kBlock),
                                        0, st, static_cast<const T*>(x), static_cast<T*>(y), n, hw, c)));
    return e;
}

cudaError_t avgpool_global_bwd(DType dt, const void* dy, void* dx, int n, int hw, int c,
                               cudaStream_t st, const void* mask) {
    const size_t total = size_t(n) * hw * c;
    if (dt == DType::BF16 && c % 8 == 0 && total / 8 < (size_t(1) << 31) && aligned16(dy) &&
        aligned16(dx) && (!mask || aligned16(mask))) {
        return launch_pdl(avgpool_bwd_vec_kernel, dim3(grid_for(total / 8, 2)), dim3(kBlock), 0, st,
                          static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx),
                          static_cast<int>(total / 8), hw, c / 8, static_cast<const __nv_bfloat16*>(mask));
    }
    TCB_DT_SWITCH(dt, T, (avgpool_bwd_kernel<T><<<grid_for(total, 2), kBlock, 0, st>>>(
                              static_cast<const T*>(dy), static_cast<T*>(dx), n, hw, c,
                              static_cast<const T*>(mask))));
    return cudaGetLastError();
}

cudaError_t softmax_xent(DType dt, const void* logits, const int32_t* labels, void* dlogits,
                         float* loss, int n, int classes, int ld, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    TCB_DT_SWITCH(dt, T, (e = launch_pdl(softmax_xent_kernel<T>, dim3(n), dim3(kBlock), 0, st,
                                        static_cast<const T*>(logits), labels, static_cast<T*>(dlogits),
                                        loss + 1, n, classes, ld)));
    if (e != cudaSuccess) return e;
    mean_kernel<<<1, 32, 0, st>>>(loss, loss + 1, n);
    return cudaGetLastError();
}

}  // namespace tcb
