// Tensor-core implicit-GEMM convolution for sm_100a (tcgen05 + TMEM + TMA).
//
// One warp-specialised, persistent kernel serves all three passes of a conv
// layer (GEMM views in common.cuh::ConvShape):
//
//   warps 0-3  producers. The activation operand (implicit im2col of NHWC x
//              for fwd, of dy for dgrad) is gathered in 16-byte chunks with
//              cp.async (zero-fill = padding / strides / ragged tiles) into
//              128B-swizzled K-major shared memory, several stages in flight
//              per thread. The weight operand is a plain row-major matrix
//              (w[K][R*S*C] for fwd, the per-phase packed w^T[C][taps*K] for
//              dgrad) and is fetched by one elected thread with a TMA tiled
//              load (SWIZZLE_128B, OOB -> 0) that completes on the same
//              mbarrier via expect_tx. For wgrad both operands are gathered
//              MN-major (pixels are the reduction axis).
//   warp  8    MMA issuer: one elected thread issues tcgen05.mma kind::f16
//              (bf16 x bf16 -> fp32, M=128, N=BN, K=16) into a double-buffered
//              TMEM accumulator; tcgen05.commit releases smem stages and
//              hands finished accumulators to the epilogue.
//   warps 4-7  epilogue: tcgen05.ld -> registers, fused bias + residual + ReLU
//              (fwd) or residual-grad + ReLU-mask (dgrad), bf16 stores; wgrad
//              writes fp32 split-K partials reduced in fixed order afterwards.
//
// Strided dgrad uses the sub-pixel decomposition (common.cuh::DgradPhase):
// stride^2 dense GEMMs over disjoint pixel phases, no zero-insertion waste.
#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"
#include "tma.cuh"

namespace tcb {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // bf16 elements per stage along the reduction
constexpr int kProducerThreads = 128;
constexpr int kEpilogueThreads = 256;  // warps 4-11
constexpr int kMmaWarp = 12;
constexpr int kThreads = kProducerThreads + kEpilogueThreads + 32;

// EPI: TMA epilogue (side inputs TMA-loaded into per-warp 64B-swizzled staging,
// outputs TMA-stored) for K-light layers whose time is the epilogue's HBM
// traffic; it trades ring stages for 64 KB of staging.
// EPI = side-input slots per epilogue warp: 0 (register epilogue), 2 (one chunk
// of lookahead) or 4 (BN >= 192: a warp's whole share of the tile prefetched at
// once, traded for ring stages — for 1-2 k-block layers).
// CTA2: a cluster pair runs M = 256 tiles with tcgen05 cta_group::2 — each CTA
// holds its 128 A rows and half of the B columns, so per-SM operand traffic
// drops by a third and more stages fit.
template <int BN, int EPI = 0, bool CTA2 = false>
struct Cfg {
    static constexpr int kABytes = BM * BK * 2;
    static constexpr int kBBytes = BN * BK * 2 / (CTA2 ? 2 : 1);  // this CTA's share
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages =
        CTA2 ? (EPI == 4 ? 2 : EPI == 2 ? (BN == 256 ? 4 : 6) : (BN == 512 ? 4 : BN == 256 ? 6 : 8))
             : EPI == 4 ? 2
             : EPI == 2 ? (BN == 256 ? 3 : BN == 192 ? 4 : BN == 128 ? 4 : 5)
                        : (BN == 384 ? 3 : BN == 256 ? 4 : BN == 192 ? 5 : BN == 128 ? 6 : 8);
    static constexpr int kRingBytes = kStages * kStageBytes;
    // EPI: slot = {in0/out, in1}, 32x32 bf16 each; register epilogue: one 32x32 bf16 staging tile
    static constexpr int kEpiWarpBytes = EPI == 0 ? 2048 : EPI * 2 * 2048;
    static constexpr int kEpiBytes = 8 * kEpiWarpBytes;
    // two accumulators (pow2); BN = 384 / 512 (wgrad double-N tiles, one unit per CTA):
    // one accumulator, two MMAs of N = BN / 2 per k-step
    static constexpr bool kDoubleN = BN == 384 || BN == 512;
    static constexpr uint32_t kTmemCols = BN == 192 || kDoubleN ? 512 : 2 * BN;
    static constexpr int kAccs = kDoubleN ? 1 : 2;
    static constexpr int kMmaN = kDoubleN ? BN / 2 : BN;
    static constexpr size_t kSmem = size_t(kRingBytes) + kEpiBytes + 1024 + 512;
};

struct Params {
    CUtensorMap tmap_a;      // activation operand when it is a plain matrix (1x1/s1/p0)
    CUtensorMap tmap_b;      // weight operand (fwd / dgrad) or x (plain wgrad)
    CUtensorMap tmap_out, tmap_res, tmap_mask;  // EPI: [M][Ncol] 32x32 boxes, SWIZZLE_64B
    ConvShape s;
    const __nv_bfloat16* a;  // fwd: x   dgrad: dy   wgrad: dy
    const __nv_bfloat16* b;  // wgrad: x (gathered)
    const __nv_bfloat16* wk; // dgrad TMA paths: the KRSC filters themselves (MN-major B)
    void* out;               // bf16 (fwd/dgrad) or fp32 partials [split][M][Ncol] (wgrad)
    const float* bias;
    const __nv_bfloat16* residual;
    const __nv_bfloat16* mask;
    int relu;
    int m_tiles, n_tiles, splits, kb_total, kb_per_split, num_tiles;
    int cta2;     // host decision: run as CTA pairs (num_tiles then counts pair units)
    int m_pairs;  // ceil(m_tiles / 2)
    // wgrad split-K reduced in-kernel: set when all units are co-resident (one
    // wave); partials in `out`, final sums to `dw`, 2 self-resetting counters per tile
    float* dw;
    int* counters;
    // dgrad phase
    DgradPhase ph;
    FastDiv d_hwq, d_wq, d_ts;
    // batched plain GEMMs (Winograd / FFT transform planes): `batch` independent
    // [M x Kdim] x [Ncol x Kdim]^T problems in contiguous planes; 3-D tensor maps
    // carry the plane index, outputs (and wgrad partials) are [split][batch][M][Ncol]
    int batch;
    // split-K forward (fc layers / K-deep plain GEMMs with few output tiles): fp32
    // partials [split][M][Ncol]; bias / residual / ReLU applied by fwd_split_reduce
    float* fwd_partial;
    int stage_epi;  // register epilogue stores through shared memory (whole sectors)
};

struct TileCoord {
    int split, mt, nt, kb_begin, kb_end, b;
};

template <bool CTA2 = false>
__device__ __forceinline__ TileCoord tile_coord(const Params& p, int t, uint32_t rank = 0) {
    TileCoord c;
    c.nt = t % p.n_tiles;
    const int rest = t / p.n_tiles;
    int outer;
    if constexpr (CTA2) {
        c.mt = 2 * (rest % p.m_pairs) + static_cast<int>(rank);
        outer = rest / p.m_pairs;
    } else {
        c.mt = rest % p.m_tiles;
        outer = rest / p.m_tiles;
    }
    c.b = outer % p.batch;
    c.split = outer / p.batch;
    c.kb_begin = c.split * p.kb_per_split;
    c.kb_end = min(p.kb_total, c.kb_begin + p.kb_per_split);
    return c;
}

// 128B swizzle: 16-byte chunk j of a 128-byte row r lands at chunk j ^ (r & 7).
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}

// Output / residual / mask row of GEMM row m. Dgrad phases scatter their rows
// over the stride lattice of dx.
template <ConvMode MODE>
__device__ __forceinline__ size_t out_row(const Params& p, int m) {
    if constexpr (MODE == ConvMode::Dgrad) {
        uint32_t n, rem, hq, wq;
        p.d_hwq.divmod(static_cast<uint32_t>(m), n, rem);
        p.d_wq.divmod(rem, hq, wq);
        const int h = static_cast<int>(hq) * p.s.sh + p.ph.ph;
        const int w = static_cast<int>(wq) * p.s.sw + p.ph.pw;
        return (size_t(n) * p.s.H + h) * p.s.W + w;
    } else {
        return static_cast<size_t>(m);
    }
}

// ------------------------------------------------------------ producers ----
// Activation operand of fwd / dgrad: one GEMM row (pixel) per thread.
template <ConvMode MODE>
__device__ __forceinline__ void gather_a_rows(const Params& p, int kb, uint32_t a_smem, int tid,
                                              int row_n, int row_hb, int row_wb, bool row_ok) {
    const ConvShape& s = p.s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int kk0 = kb * BK + j * 8;
        const void* src = p.a;
        uint32_t bytes = 0;
        if (row_ok && kk0 < s.Kdim) {
            if constexpr (MODE == ConvMode::Fwd) {
                uint32_t rs, c0, r, sx;
                s.d_c.divmod(static_cast<uint32_t>(kk0), rs, c0);
                s.d_s.divmod(rs, r, sx);
                const int hi = row_hb + static_cast<int>(r);
                const int wi = row_wb + static_cast<int>(sx);
                if (hi >= 0 && hi < s.H && wi >= 0 && wi < s.W) {
                    src = p.a + ((static_cast<size_t>(row_n) * s.H + hi) * s.W + wi) * s.C + c0;
                    bytes = 16;
                }
            } else {
                // packed dgrad taps are flipped: tap index t = (ri', si'),
                // ho = hq + bh - (tr - 1) + ri' = row_hb + ri'
                uint32_t t, k0, ri, si;
                s.d_k.divmod(static_cast<uint32_t>(kk0), t, k0);
                p.d_ts.divmod(t, ri, si);
                const int ho = row_hb + static_cast<int>(ri);
                const int wo = row_wb + static_cast<int>(si);
                if (ho >= 0 && ho < s.Ho && wo >= 0 && wo < s.Wo) {
                    src = p.a + ((static_cast<size_t>(row_n) * s.Ho + ho) * s.Wo + wo) * s.K + k0;
                    bytes = 16;
                }
            }
        }
        ptx::cp_async_16(a_smem + swz(tid, j), src, bytes);
    }
}

// Wgrad operands, both MN-major: smem row = pixel (the reduction index),
// 128 B = 64 consecutive M (or N) elements, 64-element blocks 8 KB apart.
// Per-thread constant part of the wgrad im2col column decode: with 128
// producer threads and BN/8 chunks per pixel row, thread t always loads
// column chunk t % (BN/8) of the tile.
struct WgradCol {
    int r, s, c0;
    bool ok;
};

// Pixel table entry of one stage: n*H, ho*sh - pad_h, wo*sw - pad_w (valid if nH >= 0).
__device__ __forceinline__ int4 wgrad_pixel(const ConvShape& s, int pix) {
    if (pix >= s.Kdim) return make_int4(-1, 0, 0, 0);
    uint32_t n, rem, ho, wo;
    s.d_howo.divmod(static_cast<uint32_t>(pix), n, rem);
    s.d_wo.divmod(rem, ho, wo);
    return make_int4(static_cast<int>(n) * s.H, static_cast<int>(ho) * s.sh - s.ph,
                     static_cast<int>(wo) * s.sw - s.pw, 0);
}

template <int BN>
__device__ __forceinline__ void gather_wgrad(const Params& p, const TileCoord& tc, int kb,
                                             uint32_t a_smem, uint32_t b_smem, int tid,
                                             const WgradCol& col, const int4* pixtab) {
    const ConvShape& s = p.s;
    const int P = s.Kdim;
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // A = dy: 64 pixels x 128 out-channels
        const int idx = tid + i * kProducerThreads;
        const int pl = idx >> 4, ck = idx & 15;
        const int pix = kb * BK + pl;
        const int k0 = tc.mt * BM + ck * 8;
        const bool ok = pix < P && k0 < s.K;
        const void* src = ok ? static_cast<const void*>(p.a + static_cast<size_t>(pix) * s.K + k0)
                             : static_cast<const void*>(p.a);
        ptx::cp_async_16(a_smem + (ck >> 3) * 8192u + swz(pl, ck & 7), src, ok ? 16u : 0u);
    }
    constexpr int kChunksPerRow = BN / 8;
    constexpr int kRowsPerPass = kProducerThreads / kChunksPerRow;
    const int cn = tid % kChunksPerRow;
#pragma unroll 4
    for (int i = 0; i < BN / 16; ++i) {  // B = im2col(x): 64 pixels x BN (r,s,c) columns
        const int pl = tid / kChunksPerRow + i * kRowsPerPass;
        const int4 px = pixtab[pl];
        const void* src = p.b;
        uint32_t bytes = 0;
        const int hi = px.y + col.r, wi = px.z + col.s;
        if (col.ok && px.x >= 0 && hi >= 0 && hi < s.H && wi >= 0 && wi < s.W) {
            src = p.b + ((static_cast<size_t>(px.x) + hi) * s.W + wi) * s.C + col.c0;
            bytes = 16;
        }
        ptx::cp_async_16(b_smem + (cn >> 3) * 8192u + swz(pl, cn & 7), src, bytes);
    }
}

// ------------------------------------------------------------- epilogue ----
__device__ __forceinline__ void unpack8(uint4 v, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 x = __bfloat1622float2(h[i]);
        f[2 * i] = x.x;
        f[2 * i + 1] = x.y;
    }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// Side inputs of one 32-column epilogue chunk (residual / ReLU-mask rows),
// loaded one chunk ahead so their HBM latency overlaps the TMEM load and math
// of the previous chunk.
struct SideIn {
    uint4 r[4];
    uint4 k[4];
};

// Flag templates: kX = the side input / option is present; kDyn = decide at run
// time instead (the general instantiation).
template <bool kRes, bool kMask, bool kDyn = false>
__device__ __forceinline__ void load_side(const Params& p, size_t row, int col0, bool valid,
                                          SideIn& f) {
    const bool has_res = kDyn ? p.residual != nullptr : kRes, has_mask = kDyn ? p.mask != nullptr : kMask;
    if (!valid || col0 + 32 > p.s.Ncol) return;  // tail chunks take the scalar path
    const size_t base = row * p.s.Ncol + col0;
    if (has_res) {
#pragma unroll
        for (int g = 0; g < 4; ++g) f.r[g] = __ldg(reinterpret_cast<const uint4*>(p.residual + base) + g);
    }
    if (has_mask) {
#pragma unroll
        for (int g = 0; g < 4; ++g) f.k[g] = __ldg(reinterpret_cast<const uint4*>(p.mask + base) + g);
    }
}

template <ConvMode MODE, bool kBias, bool kRes, bool kRelu, bool kMask, bool kDyn = false>
__device__ __forceinline__ void epilogue_chunk(const Params& p, const TileCoord& tc, int m,
                                               size_t row, int col0, const uint32_t (&acc)[32],
                                               const SideIn& side, uint8_t* stg = nullptr) {
    const bool has_bias = kDyn ? p.bias != nullptr : kBias, has_res = kDyn ? p.residual != nullptr : kRes;
    const bool has_relu = kDyn ? p.relu != 0 : kRelu, has_mask = kDyn ? p.mask != nullptr : kMask;
    const ConvShape& s = p.s;
    if (col0 >= s.Ncol) return;  // warp-uniform
    bool partial = MODE == ConvMode::Wgrad;
    if constexpr (kDyn && MODE == ConvMode::Fwd) partial = p.fwd_partial != nullptr;
    if (MODE != ConvMode::Wgrad && !partial && stg != nullptr && col0 + 32 <= s.Ncol) {
        // Staged store (whole warp, out-of-range rows included): the warp's 32 rows x
        // 64 B go through shared memory (16-byte units XOR-swizzled by row pair:
        // conflict-free both ways) and leave as 8 rows x 64 B per store instruction,
        // i.e. whole 32-byte sectors instead of 32 half-sector writes to 32 rows.
        const int lane = threadIdx.x & 31;
        const size_t base = (static_cast<size_t>(tc.b) * s.M + row) * s.Ncol + col0;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(acc[8 * g + i]);
            const int c = col0 + 8 * g;
            if (has_bias) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += __ldg(p.bias + c + i);
            }
            if (has_res) {
                float r[8];
                unpack8(side.r[g], r);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += r[i];
            }
            if (has_relu) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            if (has_mask) {
                float mk[8];
                unpack8(side.k[g], mk);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = mk[i] > 0.f ? v[i] : 0.f;
            }
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4)) = pack8(v);
        }
        __syncwarp();
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
        const int part = lane & 3;
        const int valid = m < s.M;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int r = it * 8 + (lane >> 2);
            const unsigned long long rb = __shfl_sync(0xffffffffu, static_cast<unsigned long long>(base), r);
            const int ok = __shfl_sync(0xffffffffu, valid, r);
            const uint4 val = *reinterpret_cast<const uint4*>(stg + r * 64 + ((part ^ ((r >> 1) & 3)) << 4));
            if (ok) *reinterpret_cast<uint4*>(out + rb + part * 8) = val;
        }
        __syncwarp();  // the next chunk reuses the staging rows
        return;
    }
    if (m >= s.M) return;
    if (partial) {
        float* out = (MODE == ConvMode::Wgrad ? static_cast<float*>(p.out) : p.fwd_partial) +
                     ((static_cast<size_t>(tc.split) * p.batch + tc.b) * s.M + m) * s.Ncol + col0;
        if (col0 + 32 <= s.Ncol) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                reinterpret_cast<float4*>(out)[i] =
                    make_float4(__uint_as_float(acc[4 * i]), __uint_as_float(acc[4 * i + 1]),
                                __uint_as_float(acc[4 * i + 2]), __uint_as_float(acc[4 * i + 3]));
        } else {
            for (int i = 0; i < 32 && col0 + i < s.Ncol; ++i) out[i] = __uint_as_float(acc[i]);
        }
    } else {
        const size_t base = (static_cast<size_t>(tc.b) * s.M + row) * s.Ncol + col0;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) + base;
        const bool full = col0 + 32 <= s.Ncol;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(acc[8 * g + i]);
            const int c = col0 + 8 * g;
            if (full) {
                if (has_bias) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] += __ldg(p.bias + c + i);
                }
                if (has_res) {
                    float r[8];
                    unpack8(side.r[g], r);
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] += r[i];
                }
                if (has_relu) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
                }
                if (has_mask) {
                    float mk[8];
                    unpack8(side.k[g], mk);
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[i] = mk[i] > 0.f ? v[i] : 0.f;
                }
                reinterpret_cast<uint4*>(out)[g] = pack8(v);
            } else {
                for (int i = 0; i < 8 && c + i < s.Ncol; ++i) {
                    float x = v[i];
                    if (has_bias) x += p.bias[c + i];
                    if (has_res) x += __bfloat162float(p.residual[base + 8 * g + i]);
                    if (has_relu) x = fmaxf(x, 0.f);
                    if (has_mask && !(__bfloat162float(p.mask[base + 8 * g + i]) > 0.f)) x = 0.f;
                    out[8 * g + i] = __float2bfloat16_rn(x);
                }
            }
        }
    }
}


// In-kernel split-K reduction of one wgrad tile, run by the 256 epilogue
// threads of every split's CTA once all splits of the tile have stored their
// partials (the units of one wave are co-resident, so waiting is safe). CTA
// `split` sums rows [split*per, ..) of the tile over splits 0..S-1 in order —
// the same fixed order as split_reduce, so results are deterministic.
template <int BN>
__device__ __forceinline__ void split_reduce_tile(const Params& p, const TileCoord& tc, int et) {
    const ConvShape& s = p.s;
    int* cnt = p.counters + 2 * (tc.mt * p.n_tiles + tc.nt);
    __threadfence();
    asm volatile("bar.sync 2, %0;" ::"n"(kEpilogueThreads) : "memory");
    if (et == 0) {
        atomicAdd(cnt, 1);
        while (*reinterpret_cast<volatile int*>(cnt) < p.splits) __nanosleep(100);
    }
    asm volatile("bar.sync 2, %0;" ::"n"(kEpilogueThreads) : "memory");
    __threadfence();
    const int rows = min(BM, s.M - tc.mt * BM), cols = min(BN, s.Ncol - tc.nt * BN);
    const int per = (rows + p.splits - 1) / p.splits;
    const int r0 = tc.split * per, r1 = min(rows, r0 + per);
    const size_t plane = size_t(s.M) * s.Ncol;
    if (s.Ncol % 4 == 0) {
        // float4 columns; up to 8 splits' loads in flight before the in-order adds
        const int cols4 = cols / 4;
        for (int i = et; i < (r1 - r0) * cols4; i += kEpilogueThreads) {
            const int rr = i / cols4, cc = (i - rr * cols4) * 4;
            const size_t o = size_t(tc.mt * BM + r0 + rr) * s.Ncol + tc.nt * BN + cc;
            const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(p.out) + o);
            const size_t plane4 = plane / 4;
            float4 acc = __ldcg(src);
            for (int k0 = 1; k0 < p.splits; k0 += 8) {
                float4 v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (k0 + j < p.splits) v[j] = __ldcg(src + (k0 + j) * plane4);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (k0 + j < p.splits) {
                        acc.x += v[j].x;
                        acc.y += v[j].y;
                        acc.z += v[j].z;
                        acc.w += v[j].w;
                    }
            }
            *reinterpret_cast<float4*>(p.dw + o) = acc;
        }
    } else {
        for (int i = et; i < (r1 - r0) * cols; i += kEpilogueThreads) {
            const int rr = i / cols, cc = i - rr * cols;
            const size_t o = size_t(tc.mt * BM + r0 + rr) * s.Ncol + tc.nt * BN + cc;
            const float* src = static_cast<const float*>(p.out) + o;
            float acc = __ldcg(src);
            for (int k = 1; k < p.splits; ++k) acc += __ldcg(src + k * plane);
            p.dw[o] = acc;
        }
    }
    asm volatile("bar.sync 2, %0;" ::"n"(kEpilogueThreads) : "memory");
    if (et == 0 && atomicAdd(cnt + 1, 1) == p.splits - 1) {
        cnt[0] = 0;
        cnt[1] = 0;
    }
}

// --------------------------------------------------------------- kernel ----
// Operand load modes.
//   kGather: the activation operand is gathered with cp.async by 128 producer
//            threads (any C % 8 == 0 geometry); weights by TMA (fwd/dgrad).
//   kPlain : 1x1 / stride 1 / no padding: every operand is a plain row-major
//            matrix fetched with 2-D TMA tiles by one thread.
//   kIm2col: the activation operand (x for fwd and wgrad, dy for dgrad) is an
//            im2col-mode TMA load (one instruction per 64-channel tap slice),
//            everything else 2-D TMA; one producer thread.
//   kIm2colC8: fwd with C == 8 (the padded RGB stem): eight 8-channel im2col
//            boxes per k-block (one per filter tap), each 128 pixels x 16 B,
//            landing as no-swizzle 8x16B core matrices (LBO 2 KB, SBO 128 B).
constexpr int kGather = 0, kPlain = 1, kIm2col = 2, kIm2colC8 = 3;

template <ConvMode MODE, int BN, int LOAD, int EPI, bool CTA2>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const __grid_constant__ Params p) {
    using C = Cfg<BN, EPI, CTA2>;
    const uint32_t rank = CTA2 ? ptx::cluster_ctarank() : 0u;  // 0 = the pair's MMA leader
    const int unit0 = CTA2 ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int ustride = CTA2 ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
    constexpr bool kTmaOnly = LOAD != kGather;
    constexpr bool kTmaB = MODE != ConvMode::Wgrad || kTmaOnly;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRingBytes + C::kEpiBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint64_t* side_bar = tempty + 2;  // EPI: [8 warps][2 * EPI slots]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(side_bar + 16 * EPI);
    // wgrad im2col pixel decode (gather mode), double-buffered; a stub elsewhere
    constexpr int kPixRows = MODE == ConvMode::Wgrad ? BK : 1;
    __shared__ int4 pixtab[2][kPixRows];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;

    if (tid == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            ptx::mbar_init(&full[i], kTmaOnly ? 1 : kProducerThreads + (kTmaB ? 1 : 0));
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], (CTA2 ? 2 : 1) * kEpilogueThreads);
        }
        for (int i = 0; i < 16 * EPI; ++i) ptx::mbar_init(&side_bar[i], 1);
        ptx::fence_mbarrier_init();
        if (kTmaB) ptx::tma_prefetch_desc(&p.tmap_b);
        if (kTmaOnly) ptx::tma_prefetch_desc(&p.tmap_a);
        if (EPI > 0) ptx::tma_prefetch_desc(&p.tmap_out);
    }
    if (warp == kMmaWarp) {
        if constexpr (CTA2) ptx::tmem_alloc_2sm<C::kTmemCols>(tmem_slot);
        else ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();  // peer barriers initialised before any remote signal
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // PDL: the prologue above overlapped the previous kernel's tail; nothing
    // it wrote is read before this point. Let the next kernel queue up early.
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t smem_base = ptx::smem_addr(smem);

    if (warp < 4 && kTmaOnly) {
        // ======================================= TMA-only producer ======
        if (tid == 0) {
            const ConvShape& s = p.s;
            int stage = 0;
            uint32_t phase = 0;
            for (int t = unit0; t < p.num_tiles; t += ustride) {
                const TileCoord tc = tile_coord<CTA2>(p, t, rank);
                // im2col base position of the tile's first GEMM row (fwd / dgrad)
                int bn = 0, bw = 0, bh = 0;
                if constexpr ((LOAD == kIm2col || LOAD == kIm2colC8) && MODE != ConvMode::Wgrad) {
                    uint32_t n, rem, a, b;
                    const uint32_t m0 = static_cast<uint32_t>(tc.mt * BM);
                    if constexpr (MODE == ConvMode::Fwd) {
                        s.d_howo.divmod(m0, n, rem);
                        s.d_wo.divmod(rem, a, b);
                        bh = static_cast<int>(a) * s.sh - s.ph;
                        bw = static_cast<int>(b) * s.sw - s.pw;
                    } else {
                        p.d_hwq.divmod(m0, n, rem);
                        p.d_wq.divmod(rem, a, b);
                        bh = static_cast<int>(a) + p.ph.bh - (p.ph.tr - 1);
                        bw = static_cast<int>(b) + p.ph.bw - (p.ph.ts - 1);
                    }
                    bn = static_cast<int>(n);
                }
                for (int kb = tc.kb_begin; kb < tc.kb_end; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    const uint32_t a_smem = smem_base + stage * C::kStageBytes;
                    const uint32_t b_smem = a_smem + C::kABytes;
                    // CTA pairs: both CTAs load their shares, completion bytes land on the
                    // leader's barrier, which expects the pair's total
                    const uint32_t bar_u = CTA2 ? ptx::leader_addr(ptx::smem_addr(&full[stage]))
                                                : ptx::smem_addr(&full[stage]);
                    if (!CTA2 || rank == 0)
                        ptx::mbar_arrive_expect_tx(&full[stage], (CTA2 ? 2 : 1) * C::kStageBytes);
                    auto ld2 = [&](uint32_t dst, const CUtensorMap* m, int c0, int c1) {
                        if (LOAD == kPlain && p.batch > 1) {  // plane index = third map dimension
                            if constexpr (CTA2) ptx::tma_load_3d_2sm(dst, m, bar_u, c0, c1, tc.b);
                            else ptx::tma_load_3d(dst, m, &full[stage], c0, c1, tc.b);
                        } else {
                            if constexpr (CTA2) ptx::tma_load_2d_2sm(dst, m, bar_u, c0, c1);
                            else ptx::tma_load_2d(dst, m, &full[stage], c0, c1);
                        }
                    };
                    auto ldi = [&](uint32_t dst, const CUtensorMap* m, int c, int w, int h, int n,
                                   uint16_t ow, uint16_t oh) {
                        if constexpr (CTA2) ptx::tma_load_im2col_4d_2sm(dst, m, bar_u, c, w, h, n, ow, oh);
                        else ptx::tma_load_im2col_4d(dst, m, &full[stage], c, w, h, n, ow, oh);
                    };
                    // B boxes of 64 N-elements: a pair's CTA takes its half
                    constexpr int kNB = CTA2 ? BN / 128 : BN / 64;
                    const int jb0 = CTA2 ? static_cast<int>(rank) * kNB : 0;
                    // tile column of this CTA's B box j (BN = 512: boxes 0-1 feed the first
                    // N = 256 MMA, 2-3 the second; each MMA takes 128 columns per CTA)
                    auto bcol = [&](int j) {
                        if constexpr (BN == 512) return (j >> 1) * 256 + static_cast<int>(rank) * 128 + (j & 1) * 64;
                        else return (jb0 + j) * 64;
                    };
                    if constexpr (MODE == ConvMode::Wgrad) {
                        // A = dy [P][K]: MN-major 64-channel x 64-pixel boxes (8 KB each)
                        ld2(a_smem, &p.tmap_a, tc.mt * BM, kb * BK);
                        ld2(a_smem + 8192, &p.tmap_a, tc.mt * BM + 64, kb * BK);
                        if constexpr (LOAD == kPlain) {
#pragma unroll
                            for (int j = 0; j < kNB; ++j)
                                ld2(b_smem + j * 8192, &p.tmap_b, tc.nt * BN + bcol(j), kb * BK);
                        } else {
                            // B = im2col(x): 64 pixels x 64 channels of one tap per box
                            const int4 px = wgrad_pixel(s, kb * BK);
                            const int pn = px.x >= 0 ? px.x / s.H : s.N;
#pragma unroll
                            for (int j = 0; j < kNB; ++j) {
                                int col0 = tc.nt * BN + bcol(j);
                                if (col0 >= s.Ncol) col0 = 0;  // padding columns: never stored
                                uint32_t rs, c0, r, sx;
                                s.d_c.divmod(static_cast<uint32_t>(col0), rs, c0);
                                s.d_s.divmod(rs, r, sx);
                                ldi(b_smem + j * 8192, &p.tmap_b, static_cast<int>(c0), px.z, px.y, pn,
                                    static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                            }
                        }
                    } else {
                        if constexpr (LOAD == kPlain) {
                            ld2(a_smem, &p.tmap_a, kb * BK, tc.mt * BM);
                        } else if constexpr (LOAD == kIm2colC8) {
                            const int taps = s.R * s.S;
#pragma unroll
                            for (int jj = 0; jj < 8; ++jj) {
                                int tap = kb * 8 + jj;
                                if (tap >= taps) tap = 0;  // K tail: B rows are zero there
                                uint32_t r, sx;
                                s.d_s.divmod(static_cast<uint32_t>(tap), r, sx);
                                ptx::tma_load_im2col_4d(a_smem + jj * 2048, &p.tmap_a, &full[stage], 0,
                                                        bw, bh, bn, static_cast<uint16_t>(sx),
                                                        static_cast<uint16_t>(r));
                            }
                        } else {
                            const uint32_t kk0 = static_cast<uint32_t>(kb * BK);
                            uint32_t tap, c0, r, sx;
                            if constexpr (MODE == ConvMode::Fwd) {
                                s.d_c.divmod(kk0, tap, c0);
                                s.d_s.divmod(tap, r, sx);
                            } else {
                                s.d_k.divmod(kk0, tap, c0);
                                p.d_ts.divmod(tap, r, sx);
                            }
                            ldi(a_smem, &p.tmap_a, static_cast<int>(c0), bw, bh, bn,
                                static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                        }
                        if constexpr (MODE == ConvMode::Dgrad) {
                            // B straight from w[K][R*S][C]: the k-block is filters k0..k0+63
                            // of one (flipped) phase tap; BN/64 channel boxes of 8 KB
                            uint32_t tap, k0, ri, si;
                            s.d_k.divmod(static_cast<uint32_t>(kb * BK), tap, k0);
                            p.d_ts.divmod(tap, ri, si);
                            const int rf = p.ph.r0 + (p.ph.tr - 1 - static_cast<int>(ri)) * s.sh;
                            const int sf = p.ph.s0 + (p.ph.ts - 1 - static_cast<int>(si)) * s.sw;
#pragma unroll
                            for (int j = 0; j < kNB; ++j) {
                                if constexpr (CTA2)
                                    ptx::tma_load_3d_2sm(b_smem + j * 8192, &p.tmap_b, bar_u,
                                                         tc.nt * BN + (jb0 + j) * 64, rf * s.S + sf,
                                                         static_cast<int>(k0));
                                else
                                    ptx::tma_load_3d(b_smem + j * 8192, &p.tmap_b, &full[stage],
                                                     tc.nt * BN + (jb0 + j) * 64, rf * s.S + sf,
                                                     static_cast<int>(k0));
                            }
                        } else {
                            // K-major weights: this CTA's BN / (1 + CTA2) rows
                            ld2(b_smem, &p.tmap_b, kb * BK, tc.nt * BN + (CTA2 ? static_cast<int>(rank) * BN / 2 : 0));
                        }
                    }
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp < 4) {
        // ================================================ producers ======
        int stage = 0;
        uint32_t phase = 0;
        int kb_seq = 0;
        for (int t = unit0; t < p.num_tiles; t += ustride) {
            const TileCoord tc = tile_coord<CTA2>(p, t, rank);
            int row_n = 0, row_hb = 0, row_wb = 0;
            bool row_ok = false;
            WgradCol col{0, 0, 0, false};
            if constexpr (MODE == ConvMode::Wgrad) {
                const int col0 = tc.nt * BN + (tid % (BN / 8)) * 8;
                col.ok = col0 < p.s.Ncol;
                if (col.ok) {
                    uint32_t rs, c0, r, sx;
                    p.s.d_c.divmod(static_cast<uint32_t>(col0), rs, c0);
                    p.s.d_s.divmod(rs, r, sx);
                    col = WgradCol{static_cast<int>(r), static_cast<int>(sx), static_cast<int>(c0), true};
                }
            } else {
                const int m = tc.mt * BM + tid;
                row_ok = m < p.s.M;
                if (row_ok) {
                    uint32_t n, rem, a, b;
                    if constexpr (MODE == ConvMode::Fwd) {
                        p.s.d_howo.divmod(static_cast<uint32_t>(m), n, rem);
                        p.s.d_wo.divmod(rem, a, b);
                        row_hb = static_cast<int>(a) * p.s.sh - p.s.ph;
                        row_wb = static_cast<int>(b) * p.s.sw - p.s.pw;
                    } else {
                        p.d_hwq.divmod(static_cast<uint32_t>(m), n, rem);
                        p.d_wq.divmod(rem, a, b);
                        row_hb = static_cast<int>(a) + p.ph.bh - (p.ph.tr - 1);
                        row_wb = static_cast<int>(b) + p.ph.bw - (p.ph.ts - 1);
                    }
                    row_n = static_cast<int>(n);
                }
            }
            for (int kb = tc.kb_begin; kb < tc.kb_end; ++kb, ++kb_seq) {
                int4* tab = pixtab[kb_seq & 1];
                if constexpr (MODE == ConvMode::Wgrad) {
                    // decode this stage's 64 pixels once, shared by all producers
                    if (tid < BK) tab[tid] = wgrad_pixel(p.s, kb * BK + tid);
                    asm volatile("bar.sync 1, %0;" ::"n"(kProducerThreads) : "memory");
                }
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t a_smem = smem_base + stage * C::kStageBytes;
                const uint32_t b_smem = a_smem + C::kABytes;
                if constexpr (kTmaB) {
                    if (tid == 0) {
                        ptx::mbar_arrive_expect_tx(&full[stage], C::kBBytes);
                        ptx::tma_load_2d(b_smem, &p.tmap_b, &full[stage], kb * BK, tc.nt * BN);
                    }
                    gather_a_rows<MODE>(p, kb, a_smem, tid, row_n, row_hb, row_wb, row_ok);
                } else {
                    gather_wgrad<BN>(p, tc, kb, a_smem, b_smem, tid, col, tab);
                }
                // arrives once this thread's copies of the stage have landed
                ptx::cp_async_mbar_arrive_noinc(&full[stage]);
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        ptx::cp_async_wait<0>();
    } else if (warp == kMmaWarp) {
        // =============================================== MMA issuer ======
        // (CTA pairs: the leader issues M = 256 MMAs over both CTAs' smem; the
        // follower's MMA warp only takes part in the TMEM alloc / dealloc)
        constexpr uint32_t kMN = MODE == ConvMode::Wgrad ? 1u : 0u;
        // dgrad with TMA operands reads B (the filters) MN-major
        constexpr bool kBmn = MODE == ConvMode::Wgrad || (MODE == ConvMode::Dgrad && kTmaOnly);
        constexpr uint32_t idesc = ptx::make_idesc(1, CTA2 ? 2 * BM : BM, C::kMmaN, kMN, kBmn ? 1u : 0u);
        if (!CTA2 || rank == 0) {
        int stage = 0;
        uint32_t phase = 0;
        int it = 0;
        for (int t = unit0; t < p.num_tiles; t += ustride, ++it) {
            const TileCoord tc = tile_coord<CTA2>(p, t, rank);
            const int acc = it % C::kAccs;
            const uint32_t acc_phase = (it / C::kAccs) & 1;
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = tc.kb_begin; kb < tc.kb_end; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                {
                    // warp-collective issue: all lanes run the loop, one elected lane
                    // issues each tcgen05 instruction (no divergent region per k-block)
                    const uint32_t a_addr = smem_base + stage * C::kStageBytes;
                    const uint32_t b_addr = a_addr + C::kABytes;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        uint64_t ad, bd;
                        if constexpr (MODE == ConvMode::Wgrad) {
                            ad = ptx::sw128_desc(a_addr + k * 2048, 8192, 1024);
                            bd = ptx::sw128_desc(b_addr + k * 2048, 8192, 1024);
                        } else if constexpr (LOAD == kIm2colC8) {
                            ad = ptx::interleave_desc(a_addr + k * 4096, 2048, 128);
                            bd = ptx::sw128_desc(b_addr + k * 32, 16, 1024);
                        } else if constexpr (kBmn) {
                            ad = ptx::sw128_desc(a_addr + k * 32, 16, 1024);
                            bd = ptx::sw128_desc(b_addr + k * 2048, 8192, 1024);
                        } else {
                            ad = ptx::sw128_desc(a_addr + k * 32, 16, 1024);
                            bd = ptx::sw128_desc(b_addr + k * 32, 16, 1024);
                        }
                        if constexpr (CTA2)
                            ptx::umma_f16_2sm_elect(d_tmem, ad, bd, idesc, (kb > tc.kb_begin || k > 0) ? 1u : 0u);
                        else
                            ptx::umma_f16_elect(d_tmem, ad, bd, idesc, (kb > tc.kb_begin || k > 0) ? 1u : 0u);
                        if constexpr (C::kDoubleN) {  // second N half: this CTA's upper B boxes
                            constexpr uint32_t kHalfB = (CTA2 ? BN / 128 : BN / 64) / 2 * 8192;
                            const uint64_t bd2 = ptx::sw128_desc(b_addr + kHalfB + k * 2048, 8192, 1024);
                            if constexpr (CTA2)
                                ptx::umma_f16_2sm_elect(d_tmem + C::kMmaN, ad, bd2, idesc,
                                                        (kb > tc.kb_begin || k > 0) ? 1u : 0u);
                            else
                                ptx::umma_f16_elect(d_tmem + C::kMmaN, ad, bd2, idesc,
                                                    (kb > tc.kb_begin || k > 0) ? 1u : 0u);
                        }
                    }
                    if constexpr (CTA2) ptx::umma_commit_2sm_elect(&empty[stage], 3);
                    else ptx::umma_commit_elect(&empty[stage]);
                }
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if constexpr (CTA2) ptx::umma_commit_2sm_elect(&tfull[acc], 3);
            else ptx::umma_commit_elect(&tfull[acc]);
        }
        }
    } else if constexpr (EPI > 0) {
        // ======================================== TMA epilogue (K-light) ======
        // Warp (quarter, half) owns rows quarter*32..+31 and half of the tile's
        // 32-column chunks. Per chunk: side inputs (residual / mask boxes, 32 x
        // 32 bf16, SWIZZLE_64B) arrive by TMA into a staging slot, the result
        // overwrites the first box in place and leaves by a TMA store. With at
        // most one side input a slot is one 2 KB box and a warp has 2 * EPI of
        // them: when that covers two tiles' shares the side inputs are double-
        // buffered by tile -- the next tile's boxes are requested while this
        // tile's chunks run instead of after its last store (these passes are
        // HBM-bound and a load latency per tile is a large share of them).
        const int quarter = warp & 3;
        const int half = (warp - 4) >> 2;
        const int lane = tid & 31;
        constexpr int kChunks = BN / 32, kHalfChunks = kChunks / 2;
        const int c_begin = half * kHalfChunks;
        uint8_t* ebuf = smem + C::kRingBytes + (warp - 4) * C::kEpiWarpBytes;
        const uint32_t ebuf_addr = ptx::smem_addr(ebuf);
        uint64_t* sbar = side_bar + (warp - 4) * 2 * EPI;
        // one instantiation per side-input / ReLU combination (no per-element flag tests)
        auto run = [&](auto res_c, auto mask_c, auto relu_c) {
            constexpr bool kRes = decltype(res_c)::value, kMask = decltype(mask_c)::value;
            constexpr bool kRelu = decltype(relu_c)::value;
            constexpr uint32_t side_bytes = (kRes ? 2048u : 0u) + (kMask ? 2048u : 0u);
            constexpr bool narrow_slots = side_bytes <= 2048u;
            const int nslots = narrow_slots ? 2 * EPI : EPI;
            const uint32_t sstride = narrow_slots ? 2048u : 4096u;
            constexpr uint32_t mask_off = kRes ? 2048u : 0u;
            const int ncol = p.s.Ncol;
            const int my_tiles = p.num_tiles > unit0 ? (p.num_tiles - unit0 + ustride - 1) / ustride : 0;
            // dbuf: side inputs double-buffered by tile (the next tile's boxes load while this tile's
            // chunks run); whole: one tile's boxes, loaded at tile start; else a ring of chunk slots
            const bool dbuf = side_bytes && nslots >= 2 * kHalfChunks;
            constexpr int kTrig = kHalfChunks > 1 ? 1 : 0;  // chunk of tile i that requests tile i + 1
            const bool whole = !dbuf && nslots >= kHalfChunks;
            auto load_tile = [&](int i) {  // lane 0
                const TileCoord tq = tile_coord<CTA2>(p, unit0 + i * ustride, rank);
                const int r0 = tq.mt * BM + quarter * 32;
                const int sbase = dbuf ? (i & 1) * kHalfChunks : 0;
                for (int k = 0; k < kHalfChunks && k < nslots; ++k) {
                    const uint32_t slot = static_cast<uint32_t>(sbase + k);
                    const int c0 = tq.nt * BN + (c_begin + k) * 32;
                    ptx::mbar_arrive_expect_tx(&sbar[slot], side_bytes);
                    if constexpr (kRes) ptx::tma_load_2d(ebuf_addr + slot * sstride, &p.tmap_res, &sbar[slot], c0, r0);
                    if constexpr (kMask)
                        ptx::tma_load_2d(ebuf_addr + slot * sstride + mask_off, &p.tmap_mask, &sbar[slot], c0, r0);
                }
            };
            if constexpr (!side_bytes) {
                // no side inputs: staging slots only hold outputs on their way to the TMA store
                constexpr bool kWhole = EPI >= kHalfChunks;
                const int c_end = c_begin + kHalfChunks;
                uint32_t seq = 0;
                int it = 0;
                for (int t = unit0; t < p.num_tiles; t += ustride, ++it) {
                    const TileCoord tc = tile_coord<CTA2>(p, t, rank);
                    const int acc = it % C::kAccs;
                    const uint32_t acc_phase = (it / C::kAccs) & 1;
                    const int row0 = tc.mt * BM + quarter * 32;
                    ptx::mbar_wait(&tfull[acc], acc_phase);
                    ptx::tc_fence_after();
        #pragma unroll 1
                    for (int c = c_begin; c < c_end; ++c, ++seq) {
                        const int col0 = tc.nt * BN + c * 32;
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                                    acc * BN + c * 32,
                                                v);
                        ptx::tmem_ld_wait();
                        const uint32_t slot = kWhole ? static_cast<uint32_t>(c - c_begin) : (seq & 1);
                        uint8_t* b0 = ebuf + slot * 4096;  // (4 KB slot pitch as with two side inputs)
                        if (lane == 0) {  // the store that last used this slot has read it
                            if constexpr (kWhole) ptx::bulk_wait_read<kHalfChunks - 1>();
                            else ptx::bulk_wait_read<1>();
                        }
                        __syncwarp();
                        if (col0 < ncol) {
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float x[8];
#pragma unroll
                                for (int i = 0; i < 8; ++i) x[i] = __uint_as_float(v[8 * g + i]);
                                const uint32_t off = lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4);
                                if (p.bias) {
                                    const int cb = col0 + 8 * g;
#pragma unroll
                                    for (int i = 0; i < 8; ++i)
                                        if (cb + i < ncol) x[i] += __ldg(p.bias + cb + i);
                                }
                                if constexpr (kRelu) {
#pragma unroll
                                    for (int i = 0; i < 8; ++i) x[i] = fmaxf(x[i], 0.f);
                                }
                                *reinterpret_cast<uint4*>(b0 + off) = pack8(x);
                            }
                            ptx::fence_proxy_async_smem();
                        }
                        __syncwarp();
                        if (lane == 0 && col0 < ncol) {
                            if (p.batch > 1) ptx::tma_store_3d(&p.tmap_out, ebuf_addr + slot * 4096, col0, row0, tc.b);
                            else ptx::tma_store_2d(&p.tmap_out, ebuf_addr + slot * 4096, col0, row0);
                            ptx::bulk_commit();
                        }
                    }
                    ptx::tc_fence_before();
                    if (CTA2 && rank != 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_addr(&tempty[acc]), 0));
                    else ptx::mbar_arrive(&tempty[acc]);
                }
                if (lane == 0) ptx::bulk_wait<0>();
            } else {
                uint32_t seq = 0;  // chunk sequence (ring mode)
                if (lane == 0 && side_bytes && (dbuf || whole) && my_tiles > 0) load_tile(0);
        #pragma unroll 1
                for (int i = 0; i < my_tiles; ++i) {
                    const TileCoord tc = tile_coord<CTA2>(p, unit0 + i * ustride, rank);
                    const int acc = i & 1;
                    const int row0 = tc.mt * BM + quarter * 32;
                    if (lane == 0 && side_bytes && whole && i > 0) {
                        ptx::bulk_wait_read<0>();  // the previous tile's stores have read every slot
                        load_tile(i);
                    }
                    ptx::mbar_wait(&tfull[acc], (i >> 1) & 1);
                    ptx::tc_fence_after();
        #pragma unroll 1
                    for (int k = 0; k < kHalfChunks; ++k, ++seq) {
                        const int c = c_begin + k;
                        const int col0 = tc.nt * BN + c * 32;
                        uint32_t slot;
                        if (dbuf) slot = static_cast<uint32_t>((i & 1) * kHalfChunks + k);
                        else if (whole) slot = static_cast<uint32_t>(k);
                        else slot = seq % static_cast<uint32_t>(nslots);
                        uint32_t v[32];
                        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 32, v);
                        ptx::tmem_ld_wait();
                        if (lane == 0) {
                            if (dbuf && k == kTrig && i + 1 < my_tiles) {
                                // tile i - 1's stores (slots of tile i + 1) have long been read
                                ptx::bulk_wait_read<kTrig>();
                                load_tile(i + 1);
                            } else if (side_bytes && !dbuf && !whole) {
                                // ring of nslots chunk slots: refill the previous chunk's slot one lap ahead
                                if (seq == 0) {
                                    for (uint32_t s2 = 0; s2 < static_cast<uint32_t>(nslots); ++s2) {
                                        const int qq = static_cast<int>(s2);
                                        const int ti = qq / kHalfChunks;
                                        if (ti >= my_tiles) break;
                                        const TileCoord tq = tile_coord<CTA2>(p, unit0 + ti * ustride, rank);
                                        const int c0 = tq.nt * BN + (c_begin + qq - ti * kHalfChunks) * 32;
                                        ptx::mbar_arrive_expect_tx(&sbar[s2], side_bytes);
                                        if constexpr (kRes)
                                            ptx::tma_load_2d(ebuf_addr + s2 * sstride, &p.tmap_res, &sbar[s2], c0, tq.mt * BM + quarter * 32);
                                        if constexpr (kMask)
                                            ptx::tma_load_2d(ebuf_addr + s2 * sstride + mask_off, &p.tmap_mask, &sbar[s2], c0,
                                                             tq.mt * BM + quarter * 32);
                                    }
                                } else {
                                    const int qn = static_cast<int>(seq) - 1 + nslots;
                                    const int ti = qn / kHalfChunks;
                                    if (ti < my_tiles) {
                                        ptx::bulk_wait_read<0>();
                                        const uint32_t s2 = (seq - 1) % static_cast<uint32_t>(nslots);
                                        const TileCoord tq = tile_coord<CTA2>(p, unit0 + ti * ustride, rank);
                                        const int c0 = tq.nt * BN + (c_begin + qn - ti * kHalfChunks) * 32;
                                        ptx::mbar_arrive_expect_tx(&sbar[s2], side_bytes);
                                        if constexpr (kRes)
                                            ptx::tma_load_2d(ebuf_addr + s2 * sstride, &p.tmap_res, &sbar[s2], c0, tq.mt * BM + quarter * 32);
                                        if constexpr (kMask)
                                            ptx::tma_load_2d(ebuf_addr + s2 * sstride + mask_off, &p.tmap_mask, &sbar[s2], c0,
                                                             tq.mt * BM + quarter * 32);
                                    }
                                }
                            }
                        }
                        uint8_t* b0 = ebuf + slot * sstride;
                        __syncwarp();
                        if (side_bytes) {
                            const uint32_t ph = dbuf ? (i >> 1) & 1 : whole ? i & 1 : (seq / nslots) & 1;
                            ptx::mbar_wait(&sbar[slot], ph);
                        }
                        if (col0 < ncol) {
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float x[8];
#pragma unroll
                                for (int e = 0; e < 8; ++e) x[e] = __uint_as_float(v[8 * g + e]);
                                const uint32_t off = lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4);
                                if (p.bias) {
                                    const int cb = col0 + 8 * g;
#pragma unroll
                                    for (int e = 0; e < 8; ++e)
                                        if (cb + e < ncol) x[e] += __ldg(p.bias + cb + e);
                                }
                                if constexpr (kRes) {
                                    float r[8];
                                    unpack8(*reinterpret_cast<const uint4*>(b0 + off), r);
#pragma unroll
                                    for (int e = 0; e < 8; ++e) x[e] += r[e];
                                }
                                if constexpr (kRelu) {
#pragma unroll
                                    for (int e = 0; e < 8; ++e) x[e] = fmaxf(x[e], 0.f);
                                }
                                if constexpr (kMask) {
                                    float mk[8];
                                    unpack8(*reinterpret_cast<const uint4*>(b0 + mask_off + off), mk);
#pragma unroll
                                    for (int e = 0; e < 8; ++e) x[e] = mk[e] > 0.f ? x[e] : 0.f;
                                }
                                *reinterpret_cast<uint4*>(b0 + off) = pack8(x);
                            }
                            ptx::fence_proxy_async_smem();
                        }
                        __syncwarp();
                        if (lane == 0) {
                            if (col0 < ncol) {
                                if (p.batch > 1)
                                    ptx::tma_store_3d(&p.tmap_out, ebuf_addr + slot * sstride, col0, row0, tc.b);
                                else
                                    ptx::tma_store_2d(&p.tmap_out, ebuf_addr + slot * sstride, col0, row0);
                            }
                            ptx::bulk_commit();  // (an empty group keeps the read-wait counts in step)
                        }
                    }
                    ptx::tc_fence_before();
                    if (CTA2 && rank != 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_addr(&tempty[acc]), 0));
                    else ptx::mbar_arrive(&tempty[acc]);
                }
                if (lane == 0) ptx::bulk_wait<0>();
            }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        const bool hr = p.residual != nullptr, hm = p.mask != nullptr, hu = p.relu != 0;
        if (hr && hm) { if (hu) run(T_{}, T_{}, T_{}); else run(T_{}, T_{}, F_{}); }
        else if (hr) { if (hu) run(T_{}, F_{}, T_{}); else run(T_{}, F_{}, F_{}); }
        else if (hm) { if (hu) run(F_{}, T_{}, T_{}); else run(F_{}, T_{}, F_{}); }
        else { if (hu) run(F_{}, F_{}, T_{}); else run(F_{}, F_{}, F_{}); }
    } else {
        // ================================================= epilogue ======
        // Two warps per TMEM lane quarter (a warp may only touch lanes
        // 32*(warp%4)..+31); each takes half of the tile's 32-column chunks.
        const int quarter = warp & 3;
        const int half = (warp - 4) >> 2;
        constexpr int kChunks = BN / 32, kHalfChunks = kChunks / 2;
        const int c_begin = half * kHalfChunks, c_end = c_begin + kHalfChunks;
        const int row = quarter * 32 + (tid & 31);
        uint8_t* const stg = (MODE != ConvMode::Wgrad && p.stage_epi) ? smem + C::kRingBytes + (warp - 4) * 2048
                                                                      : nullptr;
        auto run = [&](auto bias_c, auto res_c, auto relu_c, auto mask_c, auto dyn_c) {
            constexpr bool kBias = decltype(bias_c)::value, kRes = decltype(res_c)::value;
            constexpr bool kRelu = decltype(relu_c)::value, kMask = decltype(mask_c)::value;
            constexpr bool kDyn = decltype(dyn_c)::value;
            int it = 0;
            for (int t = unit0; t < p.num_tiles; t += ustride, ++it) {
                const TileCoord tc = tile_coord<CTA2>(p, t, rank);
                const int acc = it % C::kAccs;
                const uint32_t acc_phase = (it / C::kAccs) & 1;
                const int m = tc.mt * BM + row;
                const bool mvalid = m < p.s.M;
                const size_t orow = mvalid ? out_row<MODE>(p, m) : 0;
                // first chunk's residual / mask loads are in flight while the MMAs finish
                SideIn cur{}, nxt{};
                if constexpr (MODE != ConvMode::Wgrad)
                    load_side<kRes, kMask, kDyn>(p, orow, tc.nt * BN + c_begin * 32, mvalid, cur);
                ptx::mbar_wait(&tfull[acc], acc_phase);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int c = c_begin; c < c_end; ++c) {
                    if constexpr (MODE != ConvMode::Wgrad) {
                        if (c + 1 < c_end) load_side<kRes, kMask, kDyn>(p, orow, tc.nt * BN + (c + 1) * 32, mvalid, nxt);
                    }
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                                                acc * BN + c * 32,
                                            v);
                    ptx::tmem_ld_wait();
                    epilogue_chunk<MODE, kBias, kRes, kRelu, kMask, kDyn>(p, tc, m, orow, tc.nt * BN + c * 32, v, cur,
                                                                          stg);
                    cur = nxt;
                }
                ptx::tc_fence_before();
                if (CTA2 && rank != 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_addr(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
                if constexpr (MODE == ConvMode::Wgrad) {
                    if (p.counters) split_reduce_tile<BN>(p, tc, tid - kProducerThreads);
                }
            }
        };
        using T_ = std::true_type;
        using F_ = std::false_type;
        if constexpr (MODE == ConvMode::Wgrad) {
            run(F_{}, F_{}, F_{}, F_{}, F_{});
        } else {
            // one instantiation per side-input / ReLU combination the executor issues; bias
            // (fc layers, from_net convs) takes the run-time-checked general one
            const int f = (p.residual ? 1 : 0) | (p.relu ? 2 : 0) | (p.mask ? 4 : 0);
            if (p.bias || p.fwd_partial) run(F_{}, F_{}, F_{}, F_{}, T_{});
            else if (f == 0) run(F_{}, F_{}, F_{}, F_{}, F_{});
            else if (f == 2) run(F_{}, F_{}, T_{}, F_{}, F_{});
            else if (f == 3) run(F_{}, T_{}, T_{}, F_{}, F_{});
            else if (f == 4) run(F_{}, F_{}, F_{}, T_{}, F_{});
            else if (f == 5) run(F_{}, T_{}, F_{}, T_{}, F_{});
            else run(F_{}, F_{}, F_{}, F_{}, T_{});
        }
    }

    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();  // the leader's MMAs read the follower's smem
    else __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        if constexpr (CTA2) ptx::tmem_dealloc_2sm<C::kTmemCols>(tmem_base);
        else ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// Dgrad phases without any filter tap (e.g. odd pixels of a 1x1 stride-2
// conv): dx = residual_grad * mask (or 0).
__global__ void dgrad_empty_phase_kernel(const Params p) {
    pdl_wait();
    pdl_trigger();
    const int groups = p.s.Ncol / 8;  // C % 8 == 0 on the tensor-core path
    const size_t total = size_t(p.s.M) * groups;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total;
         i += size_t(gridDim.x) * blockDim.x) {
        const int m = static_cast<int>(i / groups);
        const int c = static_cast<int>(i % groups) * 8;
        const size_t o = out_row<ConvMode::Dgrad>(p, m) * p.s.Ncol + c;
        float v[8];
        if (p.residual) {
            unpack8(*reinterpret_cast<const uint4*>(p.residual + o), v);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f;
        }
        if (p.mask) {
            float mk[8];
            unpack8(*reinterpret_cast<const uint4*>(p.mask + o), mk);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = mk[j] > 0.f ? v[j] : 0.f;
        }
        *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + o) = pack8(v);
    }
}

// ------------------------------------------- explicit im2col (narrow C) ----
// A first layer sees 3 real channels padded to 8: the implicit GEMM would
// multiply 5/8 zeros and fetch 16-byte pixels through narrow im2col boxes.
// Instead the patch matrix is written out once, dropping the padding:
//   col[p][r * RW + s * CV + c] = x[n][oh*sh - ph + r][ow*sw - pw + s][c]
// (RW = S*CV rounded up to 8 so every filter row starts 16-byte aligned; the
// row pitch KC = R*RW rounded up to 64 keeps TMA rows 128-byte aligned; zero
// tails), and the conv becomes a plain TMA GEMM over K-dim KC (192 for the
// ResNet stem instead of 392). Weights are repacked to the same column order.
// Wgrad runs the plain GEMM on the same col (kept from the forward pass when
// the caller says so) and scatters back to [K][R][S][C].
struct NarrowPlan {
    bool use = false;
    int cv = 0, rw = 0, kc = 0, wp = 0;  // wp: input columns one output row spans
    size_t col_bytes = 0, smem = 0;
    ConvGeom g1{};  // the equivalent 1x1 conv over col
};

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

NarrowPlan narrow_plan(const ConvGeom& g) {
    NarrowPlan q;
    q.cv = g.c_valid > 0 && g.c_valid < g.c ? g.c_valid : g.c;
    q.rw = (g.s * q.cv + 7) / 8 * 8;
    q.kc = (g.r * q.rw + 63) / 64 * 64;
    const int ho = g.ho(), wo = g.wo();
    q.wp = (wo - 1) * g.stride_w + g.s;
    q.smem = size_t(g.r) * q.wp * q.cv * 2;
    q.use = g.c == 8 && q.cv < g.c && g.r * g.s > 1 && q.kc < g.r * g.s * g.c &&
            q.smem <= 48 * 1024 && q.kc <= 1024;
    if (!q.use) return q;
    q.col_bytes = size_t(g.n) * ho * wo * q.kc * 2;
    q.g1 = ConvGeom{g.n, ho, wo, q.kc, g.k, 1, 1, 0, 0, 1, 1};
    return q;
}

// One block per output row (n, oh): the R input rows it reads are staged in
// shared memory as [r][u][c] (u = input column + pad_w, only the CV real
// channels), so col element (ow, r, t = s*CV + c) is sm[(r*WP + ow*sw)*CV + t];
// the block's slice of col is contiguous and written in 16-byte chunks.
__global__ void __launch_bounds__(256) narrow_im2col_kernel(const __nv_bfloat16* __restrict__ x,
                                                            __nv_bfloat16* __restrict__ col,
                                                            ConvGeom g, int cv, int rw, int kc,
                                                            int wp, int ho, int wo) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __nv_bfloat16 sm[];
    const int n = blockIdx.x / ho, oh = blockIdx.x - n * ho;
    const int ih0 = oh * g.stride_h - g.pad_h;
    for (int i = threadIdx.x; i < g.r * wp; i += blockDim.x) {
        const int r = i / wp, u = i - r * wp;
        const int ih = ih0 + r, iw = u - g.pad_w;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (ih >= 0 && ih < g.h && iw >= 0 && iw < g.w)
            v = __ldg(reinterpret_cast<const uint4*>(x + ((size_t(n) * g.h + ih) * g.w + iw) * 8));
        const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
        for (int c = 0; c < cv; ++c) sm[i * cv + c] = e[c];
    }
    __syncthreads();
    const int span = g.s * cv, qpp = kc / 8;
    uint4* dst = reinterpret_cast<uint4*>(col + size_t(blockIdx.x) * wo * kc);
    if (qpp >= 16) {
        // wide col rows: one warp per output pixel, lane = chunk q (its (r, t0)
        // decode is per-lane constant)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
        int q_off[4], q_ok[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int q = lane + 32 * k;
            const int col0 = q * 8, r = col0 / rw, t0 = col0 - r * rw;
            q_ok[k] = q < qpp ? (r < g.r ? min(8, max(0, span - t0)) : 0) : -1;
            q_off[k] = r * wp * cv + t0;
        }
        for (int ow = warp; ow < wo; ow += nwarps) {
            const __nv_bfloat16* base = sm + ow * g.stride_w * cv;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (q_ok[k] < 0) break;
                __align__(16) __nv_bfloat16 v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = e < q_ok[k] ? base[q_off[k] + e] : __float2bfloat16(0.f);
                dst[size_t(ow) * qpp + lane + 32 * k] = *reinterpret_cast<const uint4*>(v);
            }
        }
        return;
    }
    // narrow col rows (KC < 128): thread = one chunk of one pixel, consecutive
    // threads on consecutive chunks, so every lane is busy and stores coalesce
    for (int i = threadIdx.x; i < wo * qpp; i += blockDim.x) {
        const int ow = i / qpp, q = i - ow * qpp;
        const int col0 = q * 8, r = col0 / rw, t0 = col0 - r * rw;
        const int ok = r < g.r ? min(8, max(0, span - t0)) : 0;
        const __nv_bfloat16* base = sm + ow * g.stride_w * cv + r * wp * cv + t0;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = e < ok ? base[e] : __float2bfloat16(0.f);
        dst[i] = *reinterpret_cast<const uint4*>(v);
    }
}

// w[K][R][S][C] -> wp[K][KC] (fwd operand, bf16)
__global__ void narrow_pack_weights(const __nv_bfloat16* __restrict__ w,
                                    __nv_bfloat16* __restrict__ wp, ConvGeom g, int cv, int rw,
                                    int kc) {
    pdl_wait();
    pdl_trigger();
    const int total = g.k * kc;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int k = i / kc, j = i - k * kc;
        const int r = j / rw, t = j - r * rw;
        const int s = t / cv, c = t - s * cv;
        wp[i] = (r < g.r && t < g.s * cv) ? w[((size_t(k) * g.r + r) * g.s + s) * g.c + c]
                                          : __float2bfloat16(0.f);
    }
}

// dwp[K][KC] (fp32) -> dw[K][R][S][C], zero on the padded channels
__global__ void narrow_scatter_grad(const float* __restrict__ dwp, float* __restrict__ dw,
                                    ConvGeom g, int cv, int rw, int kc) {
    pdl_wait();
    pdl_trigger();
    const int total = g.k * g.r * g.s * g.c;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int c = i % g.c;
        const int rest = i / g.c;
        const int s = rest % g.s, kr = rest / g.s;
        const int r = kr % g.r, k = kr / g.r;
        dw[i] = c < cv ? dwp[size_t(k) * kc + r * rw + s * cv + c] : 0.f;
    }
}

cudaError_t narrow_im2col(const ConvGeom& g, const NarrowPlan& q, const void* x, void* col,
                          cudaStream_t st) {
    const int ho = g.ho(), wo = g.wo();
    return launch_pdl(narrow_im2col_kernel, dim3(g.n * ho), dim3(256), q.smem, st,
                      static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(col), g, q.cv,
                      q.rw, q.kc, q.wp, ho, wo);
}

// ---------------------------------------------------------------- host ----
int g_sm_reserve = 0;  // SMs left free for concurrent communication kernels
int g_grid_cap = 0;    // > 0: at most this many CTAs (concurrent dgrad phases)
// programmatic dependent launch of the conv kernels ($TCB_PDL=0 disables)
const bool g_pdl = [] {
    const char* e = getenv("TCB_PDL");
    return !(e && e[0] == '0');
}();

// Tile width: the fewest padded columns among {256, 192} (ties -> 256) above
// 128 columns — e.g. Ncol = 576 (3x3x64 wgrad) runs as 3 x 192 instead of
// 3 x 256 with a quarter-empty last tile. 192 needs the TMA operand paths
// (the wgrad cp.async gather assumes 128 % (BN/8) == 0).
int pick_bn(int ncol, bool allow192 = true) {
    if (ncol <= 64) return 64;
    if (ncol <= 128) return 128;
    const int w256 = (ncol + 255) / 256 * 256 - ncol;
    const int w192 = (ncol + 191) / 192 * 192 - ncol;
    return allow192 && w192 < w256 ? 192 : 256;
}

struct SplitPlan {
    int splits, kb_per_split;
};

SplitPlan plan_splits(const ConvShape& s, int bn, bool pair = false, int batch = 1) {
    const int kb_total = (s.Kdim + BK - 1) / BK;
    const int m_tiles = (s.M + BM - 1) / BM;
    const int tiles = (pair ? (m_tiles + 1) / 2 : m_tiles) * ((s.Ncol + bn - 1) / bn) * batch;
    // one exact wave: splits * tiles <= #SMs (#pairs), so every CTA runs one equal
    // unit (no tail round) and the fp32 partials stay as few as the wave allows
    const int slots = (num_sms() - g_sm_reserve) / (pair ? 2 : 1);
    int want = std::max(1, slots / tiles);
    static const int min_kb = [] {  // keep >= this many k-blocks per split
        const char* e = getenv("TCB_SPLIT_MIN_KB");
        return e ? std::max(1, atoi(e)) : 4;
    }();
    want = std::min(want, std::max(1, kb_total / min_kb));
    want = std::min(want, 64);
    const int per = (kb_total + want - 1) / want;
    return {(kb_total + per - 1) / per, per};
}

// 1x1 filter, stride 1, no padding: every implicit-GEMM operand is a plain matrix.
bool plain_geometry(const ConvShape& s) {
    return s.R == 1 && s.S == 1 && s.ph == 0 && s.pw == 0 && s.sh == 1 && s.sw == 1;
}

// im2col TMA needs whole 64-channel slices of one tap per k-block and small
// bounding-box corners / tap offsets.
template <ConvMode MODE>
bool im2col_ok(const Params& p) {
    const ConvShape& s = p.s;
    const int ch = MODE == ConvMode::Dgrad ? s.K : s.C;
    if (ch % 64 != 0) return false;
    if (s.R > 16 || s.S > 16 || s.ph > 15 || s.pw > 15) return false;
    return true;
}

template <ConvMode MODE, int LOAD>
bool build_maps(Params& p, const void* a_matrix, const void* b_matrix, int bn) {
    const ConvShape& s = p.s;
    if (LOAD == kPlain && p.batch > 1) {
        // batched planes: [batch][rows][cols] bf16 with the plane as the third dimension
        if (MODE == ConvMode::Wgrad)
            return make_tmap_bf16_3d(&p.tmap_a, a_matrix, p.batch, s.Kdim, s.K, BK, 64) &&
                   make_tmap_bf16_3d(&p.tmap_b, b_matrix, p.batch, s.Kdim, s.C, BK, 64);
        if (MODE != ConvMode::Fwd) return false;
        return make_tmap_bf16_3d(&p.tmap_b, b_matrix, p.batch, s.Ncol, s.Kdim, bn, 64) &&
               make_tmap_bf16_3d(&p.tmap_a, a_matrix, p.batch, s.M, s.Kdim, BM, 64);
    }
    if (MODE == ConvMode::Wgrad) {
        if (LOAD == kGather) return true;
        // dy [P][K], MN-major 64 x 64 boxes
        if (!make_tmap_bf16_2d(&p.tmap_a, a_matrix, s.Kdim, s.K, BK, 64)) return false;
        if (LOAD == kPlain) return make_tmap_bf16_2d(&p.tmap_b, b_matrix, s.Kdim, s.C, BK, 64);
        return make_tmap_im2col_bf16(&p.tmap_b, b_matrix, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                     s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BK);
    }
    // weight operand: row-major [Ncol][Kdim] bf16, boxes of BN rows x 64 (fwd, gather
    // dgrad on packed w^T); TMA dgrad reads the KRSC filters as [K][R*S][C] boxes
    if (MODE == ConvMode::Dgrad && LOAD != kGather) {
        if (!make_tmap_filters_bf16(&p.tmap_b, p.wk, s.K, size_t(s.R) * s.S, s.C)) return false;
    } else if (!make_tmap_bf16_2d(&p.tmap_b, b_matrix, s.Ncol, s.Kdim, bn)) {
        return false;
    }
    if (LOAD == kPlain) return make_tmap_bf16_2d(&p.tmap_a, a_matrix, s.M, s.Kdim, BM);
    if (LOAD == kIm2colC8)
        return make_tmap_im2col_bf16(&p.tmap_a, a_matrix, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                     s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BM, 8);
    if (LOAD == kIm2col) {
        if (MODE == ConvMode::Fwd)
            return make_tmap_im2col_bf16(&p.tmap_a, a_matrix, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                         s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BM);
        // dgrad phase over dy: base positions lower .. lower + (Wq, Hq) - 1, stride 1
        const int lw = p.ph.bw - (p.ph.ts - 1), lh = p.ph.bh - (p.ph.tr - 1);
        return make_tmap_im2col_bf16(&p.tmap_a, a_matrix, s.N, s.Ho, s.Wo, s.K, lw, lh,
                                     lw + p.ph.Wq - s.Wo, lh + p.ph.Hq - s.Ho, 1, 1, BM);
    }
    return true;
}

// EPI output / side-input maps: [M][Ncol] bf16, 32-row x 32-column boxes.
bool build_epi_maps(Params& p) {
    const auto sw = CU_TENSOR_MAP_SWIZZLE_64B;
    if (p.batch > 1) {  // batched plain GEMMs (Winograd / FFT planes): [batch][M][Ncol], no side inputs
        if (p.residual || p.mask) return false;
        EncodeTiledFn fn = encode_tiled_fn();
        if (!fn) return false;
        const cuuint64_t dims[3] = {cuuint64_t(p.s.Ncol), cuuint64_t(p.s.M), cuuint64_t(p.batch)};
        const cuuint64_t strides[2] = {cuuint64_t(p.s.Ncol) * 2, cuuint64_t(p.s.M) * p.s.Ncol * 2};
        const cuuint32_t box[3] = {32, 32, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        return fn(&p.tmap_out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p.out, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (!make_tmap_bf16_2d(&p.tmap_out, p.out, p.s.M, p.s.Ncol, 32, 32, sw)) return false;
    if (p.residual && !make_tmap_bf16_2d(&p.tmap_res, p.residual, p.s.M, p.s.Ncol, 32, 32, sw))
        return false;
    if (p.mask && !make_tmap_bf16_2d(&p.tmap_mask, p.mask, p.s.M, p.s.Ncol, 32, 32, sw))
        return false;
    return true;
}

ConvTcLaunchInfo g_last_launch{};  // test hook: the configuration of the last conv_tc_kernel launch

template <ConvMode MODE, int BN, int LOAD, int EPI, bool CTA2 = false>
cudaError_t launch(Params& p, const void* a_matrix, const void* b_matrix, cudaStream_t st) {
    using C = Cfg<BN, EPI, CTA2>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(conv_tc_kernel<MODE, BN, LOAD, EPI, CTA2>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(C::kSmem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    // K-major weight boxes: a pair's CTA loads BN / 2 rows
    if (!build_maps<MODE, LOAD>(p, a_matrix, b_matrix, CTA2 ? BN / 2 : BN)) return cudaErrorInvalidValue;
    if (EPI > 0 && !build_epi_maps(p)) return cudaErrorInvalidValue;
    p.m_tiles = (p.s.M + BM - 1) / BM;
    p.m_pairs = (p.m_tiles + 1) / 2;
    p.n_tiles = (p.s.Ncol + BN - 1) / BN;
    p.kb_total = (p.s.Kdim + BK - 1) / BK;
    p.cta2 = CTA2 ? 1 : 0;
    if (MODE != ConvMode::Wgrad && !(MODE == ConvMode::Fwd && p.fwd_partial)) {
        p.splits = 1;
        p.kb_per_split = p.kb_total;
    }
    if (p.batch < 1) p.batch = 1;
    static const int stage_epi = [] {
        const char* e = getenv("TCB_EPI_STAGE");
        return e ? atoi(e) : 1;
    }();
    p.stage_epi = stage_epi;
    p.num_tiles = (CTA2 ? p.m_pairs : p.m_tiles) * p.n_tiles * p.batch * p.splits;
    const int sms = std::max(2, num_sms() - g_sm_reserve);
    const int cap = g_grid_cap > 0 ? std::min(g_grid_cap, sms) : sms;
    const int grid = CTA2 ? 2 * std::max(1, std::min(p.num_tiles, cap / 2)) : std::min(p.num_tiles, cap);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CTA2 ? 2 : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CTA2 ? 2 : 1;
    g_last_launch = ConvTcLaunchInfo{static_cast<int>(MODE), LOAD, BN, EPI, CTA2 ? 1 : 0, p.splits,
                                     p.num_tiles, grid, p.counters != nullptr ? 1 : 0, 0};
    return cudaLaunchKernelEx(&cfg, conv_tc_kernel<MODE, BN, LOAD, EPI, CTA2>, p);
}

// CTA pairs for K-heavy TMA-operand layers with at least two 128-row tiles
// ($TCB_CTA2=0 disables; $TCB_CTA2_KB = minimum k-blocks, default 9).
bool cta2_wanted(int load, int bn, int m_tiles, int kb_total) {
    static const int min_kb = [] {
        const char* e = getenv("TCB_CTA2");
        if (e && e[0] == '0') return 1 << 30;
        const char* k = getenv("TCB_CTA2_KB");
        return k ? atoi(k) : 9;
    }();
    return (load == kPlain || load == kIm2col) && (bn == 128 || bn == 256 || bn == 512) && m_tiles >= 2 &&
           kb_total >= min_kb;
}

int g_epi_kb = -1;  // TMA epilogue for 1x1 layers with at most this many k-blocks
int g_epi_kb_spatial = -1;  // ... and for spatial (im2col) layers

// The TMA epilogue needs the output rows contiguous (fwd; single-phase dgrad).
// Thresholds measured over whole steps (scripts/ab_epi_kb.sh): 1x1 layers lose
// past 12 k-blocks (ResNet-50's 1024-wide 1x1s), spatial ones gain up to 24
// (Inception-v3's 5x5 / 1x7 / 7x1 branches).
template <ConvMode MODE>
bool use_epi(const Params& p) {
    if (MODE == ConvMode::Wgrad || p.fwd_partial) return false;
    // batched plain GEMMs store through a 3-D map (no side inputs there)
    if (p.batch > 1 && (p.residual || p.mask)) return false;
    if (MODE == ConvMode::Dgrad && (p.s.sh != 1 || p.s.sw != 1)) return false;
    if (g_epi_kb < 0) {
        const char* e = getenv("TCB_CONV_EPI_KB");
        g_epi_kb = e ? atoi(e) : 12;
        const char* f = getenv("TCB_CONV_EPI_KB_SPATIAL");
        g_epi_kb_spatial = f ? atoi(f) : (e ? g_epi_kb : 24);
    }
    if (p.s.Ncol % 8 != 0) return false;
    const int kb = (p.s.Kdim + BK - 1) / BK;
    return kb <= (plain_geometry(p.s) ? g_epi_kb : g_epi_kb_spatial);
}

int wgrad_bn(const ConvShape& s);

template <ConvMode MODE, int LOAD>
cudaError_t dispatch_bn(Params& p, const void* a_matrix, const void* b_matrix, cudaStream_t st) {
    const int bn = MODE == ConvMode::Wgrad && LOAD != kGather ? wgrad_bn(p.s)
                                                              : pick_bn(p.s.Ncol, !(MODE == ConvMode::Wgrad && LOAD == kGather));
    if constexpr (MODE != ConvMode::Wgrad) {
        if (use_epi<MODE>(p)) {
            static const int deep_kb = [] {  // whole-share side-input prefetch up to this many k-blocks
                const char* e = getenv("TCB_EPI_DEEP_KB");
                return e ? atoi(e) : 2;
            }();
            const bool deep = (p.s.Kdim + BK - 1) / BK <= deep_kb;
            // CTA pairs keep the TMA epilogue ($TCB_CTA2_EPI: 1 pair + TMA epilogue (default),
            // 0 pairs take the register epilogue, -1 no pairs for TMA-epilogue layers)
            static const int cta2_epi = [] {
                const char* e = getenv("TCB_CTA2_EPI");
                return e ? atoi(e) : 1;
            }();
            if constexpr (LOAD == kPlain || LOAD == kIm2col) {
                if (cta2_epi >= 0 && (bn == 128 || bn == 256) &&
                    cta2_wanted(LOAD, bn, (p.s.M + BM - 1) / BM, (p.s.Kdim + BK - 1) / BK)) {
                    if (cta2_epi == 0) {
                        if (bn == 256) return launch<MODE, 256, LOAD, 0, true>(p, a_matrix, b_matrix, st);
                        return launch<MODE, 128, LOAD, 0, true>(p, a_matrix, b_matrix, st);
                    }
                    if (bn == 256) return launch<MODE, 256, LOAD, 2, true>(p, a_matrix, b_matrix, st);
                    return launch<MODE, 128, LOAD, 2, true>(p, a_matrix, b_matrix, st);
                }
            }
            switch (bn) {
                case 256:
                    return deep ? launch<MODE, 256, LOAD, 4>(p, a_matrix, b_matrix, st)
                                : launch<MODE, 256, LOAD, 2>(p, a_matrix, b_matrix, st);
                case 192:
                    return deep ? launch<MODE, 192, LOAD, 4>(p, a_matrix, b_matrix, st)
                                : launch<MODE, 192, LOAD, 2>(p, a_matrix, b_matrix, st);
                case 128: return launch<MODE, 128, LOAD, 2>(p, a_matrix, b_matrix, st);
                default: return launch<MODE, 64, LOAD, 2>(p, a_matrix, b_matrix, st);
            }
        }
    }
    if constexpr (LOAD == kPlain || LOAD == kIm2col) {
        const bool pair = MODE == ConvMode::Wgrad
                              ? p.cta2 != 0
                              : !p.fwd_partial && cta2_wanted(LOAD, bn, (p.s.M + BM - 1) / BM, (p.s.Kdim + BK - 1) / BK);
        if constexpr (MODE == ConvMode::Wgrad) {
            if (pair && bn == 512) return launch<MODE, 512, LOAD, 0, true>(p, a_matrix, b_matrix, st);
            if (!pair && bn == 384) return launch<MODE, 384, LOAD, 0, false>(p, a_matrix, b_matrix, st);
        }
        if (pair && bn == 256) return launch<MODE, 256, LOAD, 0, true>(p, a_matrix, b_matrix, st);
        if (pair && bn == 128) return launch<MODE, 128, LOAD, 0, true>(p, a_matrix, b_matrix, st);
    }
    switch (bn) {
        case 256: return launch<MODE, 256, LOAD, 0>(p, a_matrix, b_matrix, st);
        case 192:
            if constexpr (MODE == ConvMode::Wgrad && LOAD == kGather) return cudaErrorInvalidValue;
            else return launch<MODE, 192, LOAD, 0>(p, a_matrix, b_matrix, st);
        case 128: return launch<MODE, 128, LOAD, 0>(p, a_matrix, b_matrix, st);
        default: return launch<MODE, 64, LOAD, 0>(p, a_matrix, b_matrix, st);
    }
}


int g_force_gather = -1;  // test hook: 1 = always use the cp.async gather path

bool force_gather() {
    if (g_force_gather < 0) {
        const char* e = getenv("TCB_CONV_FORCE_GATHER");
        g_force_gather = (e && e[0] == '1') ? 1 : 0;
    }
    return g_force_gather == 1;
}

// Wgrad as CTA pairs (same operand-path rule as dispatch(), same tile width).
bool wgrad_pair(const ConvShape& s, int bn) {
    if (force_gather()) return false;
    const bool plain = plain_geometry(s);
    const bool im2col = s.C % 64 == 0 && s.R <= 16 && s.S <= 16 && s.ph <= 15 && s.pw <= 15;
    if (!plain && !im2col) return false;
    return cta2_wanted(plain ? kPlain : kIm2col, bn, (s.M + BM - 1) / BM, (s.Kdim + BK - 1) / BK);
}

// Wgrad tile width, consistent with the operand path dispatch() will pick.
// 512-column tiles for spatial (im2col) layers (two N = 256 MMAs per k-step into
// all of TMEM, CTA pairs only): a pair's CTA loads 16 KB of dy + 32 KB of x per
// k-block for twice the MMA work of a 256-column tile (16 + 16 KB) -- a quarter
// less L2 -> SM traffic per FLOP (ResNet-50 stage-4 3x3: 82.7 -> 77.3 us). 1x1
// layers measured slower (fewer tiles -> more splits: 38.9 -> 50.9 us).
// $TCB_WG512: 0 off, 1 when Ncol is a multiple of 512, 2 whenever Ncol >= 1024.
int wgrad_bn(const ConvShape& s) {
    const bool tma = !force_gather() &&
                     (plain_geometry(s) || (s.C % 64 == 0 && s.R <= 16 && s.S <= 16 && s.ph <= 15 &&
                                            s.pw <= 15));
    const int bn = pick_bn(s.Ncol, tma);
    static const int wg512 = [] {
        const char* e = getenv("TCB_WG512");
        return e ? atoi(e) : 1;
    }();
    if (tma && !plain_geometry(s) && bn == 256 && wg512 > 0 && (wg512 == 2 ? s.Ncol >= 1024 : s.Ncol % 512 == 0) &&
        cta2_wanted(plain_geometry(s) ? kPlain : kIm2col, 256, (s.M + BM - 1) / BM, (s.Kdim + BK - 1) / BK))
        return 512;
    // single-CTA spatial tiles of 2 x 192 columns where no pair forms (one 128-row M tile)
    if (tma && !plain_geometry(s) && bn == 192 && wg512 > 0 && s.Ncol % 384 == 0 &&
        !cta2_wanted(kIm2col, 192, (s.M + BM - 1) / BM, (s.Kdim + BK - 1) / BK))
        return 384;
    return bn;
}

template <ConvMode MODE>
cudaError_t dispatch(Params& p, const void* a_matrix, const void* b_matrix, cudaStream_t st) {
    if (!force_gather()) {
        const bool plain = MODE == ConvMode::Dgrad
                               ? plain_geometry(p.s) && p.ph.tr == 1 && p.ph.ts == 1
                               : plain_geometry(p.s);
        if (plain) return dispatch_bn<MODE, kPlain>(p, a_matrix, b_matrix, st);
        if (im2col_ok<MODE>(p)) return dispatch_bn<MODE, kIm2col>(p, a_matrix, b_matrix, st);
        if constexpr (MODE == ConvMode::Fwd) {
            if (p.s.C == 8 && p.s.R <= 16 && p.s.S <= 16 && p.s.ph <= 15 && p.s.pw <= 15)
                return dispatch_bn<MODE, kIm2colC8>(p, a_matrix, b_matrix, st);
        }
    }
    return dispatch_bn<MODE, kGather>(p, a_matrix, b_matrix, st);
}

// A fully connected layer (filter = the whole unpadded input map, 1x1 output)
// is the 1x1 conv over a 1x1 image of H*W*C channels: same memory (NHWC rows
// of x and KRSC rows of w are both [rows][H*W*C]), plain TMA operands.
bool fc_geometry(const ConvGeom& g) {
    return g.r == g.h && g.s == g.w && g.pad_h == 0 && g.pad_w == 0 && g.ho() == 1 && g.wo() == 1 &&
           (g.h > 1 || g.w > 1);
}

ConvGeom fc_as_1x1(const ConvGeom& g) {
    return fc_geometry(g) ? ConvGeom{g.n, 1, 1, g.h * g.w * g.c, g.k, 1, 1, 0, 0, 1, 1} : g;
}

// Split-K forward: a plain GEMM whose output tiles fill under half the SMs but
// whose reduction is deep (VGG fc6 at batch 64: 16 tiles x 392 k-blocks) runs
// `splits` k-ranges as separate units into fp32 partials, then one reduce pass
// adds them in fixed split order and applies bias / residual / ReLU.
// $TCB_FWD_SPLIT=0 disables.
SplitPlan fwd_split_plan(const ConvGeom& g0) {
    static const int enabled = [] {
        const char* e = getenv("TCB_FWD_SPLIT");
        return e ? atoi(e) : 1;
    }();
    const SplitPlan none{1, 0};
    if (!enabled || force_gather()) return none;
    const ConvGeom g = fc_as_1x1(g0);
    const ConvShape s = make_shape(g, ConvMode::Fwd);
    if (!plain_geometry(s) || s.Ncol % 8 != 0) return none;
    const int bn = pick_bn(s.Ncol);
    const int tiles = ((s.M + BM - 1) / BM) * ((s.Ncol + bn - 1) / bn);
    const int kb = (s.Kdim + BK - 1) / BK;
    const int slots = num_sms() - g_sm_reserve;
    if (2 * tiles > slots || kb < 16) return none;
    const int want = std::min({slots / tiles, kb / 4, 32});
    if (want < 2) return none;
    const int per = (kb + want - 1) / want;
    return {(kb + per - 1) / per, per};
}

// y[m][n] = act(sum_k parts[k][m][n] + bias[n] + residual[m][n]), 8 columns per
// thread (Ncol % 8 == 0), splits summed in index order (deterministic).
__global__ void fwd_split_reduce_kernel(const float* __restrict__ parts, int splits, int rows, int cols,
                                        const float* __restrict__ bias, const __nv_bfloat16* __restrict__ residual,
                                        int relu, __nv_bfloat16* __restrict__ y) {
    pdl_wait();
    pdl_trigger();
    const int c8 = cols / 8;
    const size_t n8 = size_t(rows) * c8;
    const size_t plane = size_t(rows) * cols;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n8; i += size_t(gridDim.x) * blockDim.x) {
        const size_t off = i * 8;
        const int col = static_cast<int>(i % c8) * 8;
        const float4* src = reinterpret_cast<const float4*>(parts + off);
        float4 a = __ldcs(src), b = __ldcs(src + 1);
        for (int k = 1; k < splits; ++k) {
            const float4* q = reinterpret_cast<const float4*>(parts + k * plane + off);
            const float4 u = __ldcs(q), v = __ldcs(q + 1);
            a.x += u.x; a.y += u.y; a.z += u.z; a.w += u.w;
            b.x += v.x; b.y += v.y; b.z += v.z; b.w += v.w;
        }
        float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        if (bias) {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += __ldg(bias + col + j);
        }
        if (residual) {
            float r[8];
            unpack8(__ldg(reinterpret_cast<const uint4*>(residual + off)), r);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] += r[j];
        }
        if (relu) {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j], 0.f);
        }
        *reinterpret_cast<uint4*>(y + off) = pack8(v);
    }
}

}  // namespace

void conv_tc_set_force_gather(int on) { g_force_gather = on ? 1 : 0; }
ConvTcLaunchInfo conv_tc_last_launch() { return g_last_launch; }
void conv_tc_note_launch(const ConvTcLaunchInfo& info) { g_last_launch = info; }
void conv_tc_set_epi_kb(int kb) { g_epi_kb = g_epi_kb_spatial = kb; }
void conv_tc_set_sm_reserve(int sms) { g_sm_reserve = std::max(0, sms); }

bool conv_tc_supported(const ConvGeom& g, ConvMode mode) {
    if (g.n < 1 || g.h < 1 || g.w < 1 || g.c < 1 || g.k < 1) return false;
    if (mode == ConvMode::Fwd) return g.c % 8 == 0;
    if (mode == ConvMode::Dgrad) return g.k % 8 == 0 && g.c % 8 == 0;
    return g.c % 8 == 0 && g.k % 8 == 0;
}

size_t conv_tc_workspace(const ConvGeom& g, ConvMode mode) {
    if (mode != ConvMode::Dgrad && conv_stem_applies(g)) return conv_stem_workspace(g);
    const NarrowPlan q = narrow_plan(g);
    if (q.use && mode == ConvMode::Fwd)
        return align256(q.col_bytes) + align256(size_t(g.k) * q.kc * 2);
    if (q.use && mode == ConvMode::Wgrad)
        return align256(q.col_bytes) + align256(size_t(g.k) * q.kc * 4) +
               conv_tc_workspace(q.g1, ConvMode::Wgrad);
    if (mode == ConvMode::Fwd) {
        const SplitPlan fs = fwd_split_plan(g);
        const ConvGeom g1 = fc_as_1x1(g);
        return fs.splits > 1 ? size_t(fs.splits) * g1.n * g1.h * g1.w * g1.k * sizeof(float) : 0;
    }
    if (mode != ConvMode::Wgrad) return 0;
    const ConvShape s = make_shape(g, mode);
    const int bn = wgrad_bn(s);
    const SplitPlan sp = plan_splits(s, bn, wgrad_pair(s, bn));
    const size_t im2col_ws = sp.splits > 1 ? size_t(sp.splits) * s.M * s.Ncol * sizeof(float) : 0;
    return std::max(im2col_ws, conv_win_wgrad_workspace(g));
}

bool conv_tc_narrow(const ConvGeom& g) { return conv_stem_applies(g) || narrow_plan(g).use; }

int conv_tc_launches(const ConvGeom& g, ConvMode mode, bool cols_ready, bool counters) {
    if (mode != ConvMode::Dgrad && conv_stem_applies(g)) return conv_stem_launches(g, mode, cols_ready);
    const NarrowPlan q = narrow_plan(g);
    if (mode == ConvMode::Fwd) return q.use ? 3 : (fwd_split_plan(g).splits > 1 ? 2 : 1);
    if (mode == ConvMode::Dgrad) return g.stride_h * g.stride_w;
    const ConvGeom& gw = q.use ? q.g1 : g;
    if (!q.use && !force_gather() && conv_win_wgrad_applies(g)) return conv_win_wgrad_launches(g);
    const ConvShape s = make_shape(gw, mode);
    const int bn = wgrad_bn(s);
    const bool pair = wgrad_pair(s, bn);
    const SplitPlan sp = plan_splits(s, bn, pair);
    const int tiles = (pair ? ((s.M + BM - 1) / BM + 1) / 2 * 2 : (s.M + BM - 1) / BM) * ((s.Ncol + bn - 1) / bn);
    const int split = (sp.splits > 1 && !(counters && tiles * sp.splits <= num_sms())) ? 2 : 1;
    return split + (q.use ? (cols_ready ? 1 : 2) : 0);
}

cudaError_t conv_tc_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep,
                        void* y, cudaStream_t st, void* workspace, bool x_ready) {
    if (workspace && conv_stem_applies(g)) return conv_stem_fwd(g, x, w, ep, y, workspace, st, x_ready);
    Params p{};
    const NarrowPlan q = narrow_plan(g);
    const void* a_matrix = x;
    const void* b_matrix = w;
    if (q.use && workspace) {
        char* ws = static_cast<char*>(workspace);
        cudaError_t e = narrow_im2col(g, q, x, ws, st);
        if (e != cudaSuccess) return e;
        auto* wp = reinterpret_cast<__nv_bfloat16*>(ws + align256(q.col_bytes));
        e = launch_pdl(narrow_pack_weights, dim3(std::max(1, std::min(g.k * q.kc / 256 + 1, 1024))), dim3(256),
                       0, st, static_cast<const __nv_bfloat16*>(w), wp, g, q.cv, q.rw, q.kc);
        if (e != cudaSuccess) return e;
        p.s = make_shape(q.g1, ConvMode::Fwd);
        a_matrix = ws;
        b_matrix = wp;
    } else {
        const SplitPlan fs = workspace ? fwd_split_plan(g) : SplitPlan{1, 0};
        if (fs.splits > 1) {
            const ConvGeom g1 = fc_as_1x1(g);
            p.s = make_shape(g1, ConvMode::Fwd);
            p.a = static_cast<const __nv_bfloat16*>(x);
            p.out = y;
            p.fwd_partial = static_cast<float*>(workspace);
            p.splits = fs.splits;
            p.kb_per_split = fs.kb_per_split;
            cudaError_t e = dispatch<ConvMode::Fwd>(p, x, w, st);
            if (e != cudaSuccess) return e;
            const int c8 = p.s.M * (g1.k / 8);
            return launch_pdl(fwd_split_reduce_kernel, dim3(std::max(1, std::min((c8 + 255) / 256, 4 * num_sms()))),
                              dim3(256), 0, st, static_cast<const float*>(workspace), fs.splits, p.s.M, g1.k,
                              ep.bias, static_cast<const __nv_bfloat16*>(ep.residual), ep.relu ? 1 : 0,
                              static_cast<__nv_bfloat16*>(y));
        }
        if (!force_gather() && conv_win_applies(g, ConvMode::Fwd)) return conv_win_fwd(g, x, w, ep, y, st);
        p.s = make_shape(g, ConvMode::Fwd);
    }
    p.a = static_cast<const __nv_bfloat16*>(a_matrix);
    p.out = y;
    p.bias = ep.bias;
    p.residual = static_cast<const __nv_bfloat16*>(ep.residual);
    p.relu = ep.relu ? 1 : 0;
    return dispatch<ConvMode::Fwd>(p, a_matrix, b_matrix, st);
}

// Batched plain GEMMs (Winograd's 16 / FFT's 40 transform-plane products in ONE
// launch): y[b] = x[b] * w[b]^T for b < batch, x[b] [M][Kdim], w[b] [Ncol][Kdim],
// y[b] [M][Ncol] bf16, g the 1x1 / stride-1 / unpadded "conv" of one plane.
cudaError_t conv_tc_fwd_batched(const ConvGeom& g, int batch, const void* x, const void* w, void* y,
                                cudaStream_t st) {
    Params p{};
    p.s = make_shape(g, ConvMode::Fwd);
    if (!plain_geometry(p.s) || batch < 1) return cudaErrorInvalidValue;
    p.batch = batch;
    p.a = static_cast<const __nv_bfloat16*>(x);
    p.out = y;
    return dispatch_bn<ConvMode::Fwd, kPlain>(p, x, w, st);
}

size_t conv_tc_wgrad_batched_workspace(const ConvGeom& g, int batch) {
    const ConvShape s = make_shape(g, ConvMode::Wgrad);
    const int bn = wgrad_bn(s);
    const SplitPlan sp = plan_splits(s, bn, wgrad_pair(s, bn), batch);
    return sp.splits > 1 ? size_t(sp.splits) * batch * s.M * s.Ncol * sizeof(float) : 0;
}

// dw[b] [Ncol=K][Kdim... ] = dy[b]^T x[b] summed over the plane's pixels, fp32,
// one launch (split-K over the batch's tiles) + one fixed-order reduction.
cudaError_t conv_tc_wgrad_batched(const ConvGeom& g, int batch, const void* dy, const void* x, float* dw,
                                  void* workspace, cudaStream_t st) {
    Params p{};
    p.s = make_shape(g, ConvMode::Wgrad);
    if (!plain_geometry(p.s) || batch < 1) return cudaErrorInvalidValue;
    const int bn = wgrad_bn(p.s);
    const bool pair = wgrad_pair(p.s, bn);
    p.cta2 = pair ? 1 : 0;
    const SplitPlan sp = plan_splits(p.s, bn, pair, batch);
    p.batch = batch;
    p.a = static_cast<const __nv_bfloat16*>(dy);
    p.b = static_cast<const __nv_bfloat16*>(x);
    p.splits = sp.splits;
    p.kb_per_split = sp.kb_per_split;
    p.out = sp.splits > 1 ? workspace : static_cast<void*>(dw);
    if (sp.splits > 1 && workspace == nullptr) return cudaErrorInvalidValue;
    cudaError_t e = dispatch_bn<ConvMode::Wgrad, kPlain>(p, dy, x, st);
    if (e != cudaSuccess || sp.splits == 1) return e;
    return split_reduce(static_cast<const float*>(workspace), sp.splits, size_t(batch) * p.s.M * p.s.Ncol, dw, st);
}

bool conv_tc_dgrad_needs_pack(const ConvGeom& g) {
    if (force_gather()) return true;
    const bool plain = g.r == 1 && g.s == 1 && g.pad_h == 0 && g.pad_w == 0 && g.stride_h == 1 &&
                       g.stride_w == 1;
    const bool im2col = g.k % 64 == 0 && g.r <= 16 && g.s <= 16 && g.pad_h <= 15 && g.pad_w <= 15;
    return !(plain || im2col);
}

// Strided dgrad phases run concurrently: phase i on its own stream (forked from /
// joined back into `st` by events, so it also captures into a CUDA graph) with
// CTAs in proportion to its work. $TCB_DGRAD_CONCURRENT: 0 never, 1 always,
// 2 (default) when no phase has two waves of tiles -- there sequential phases
// leave SMs idle (ResNet-50 stage 4, 98 tiles per phase: 101.5 -> 76.1 us with
// the ReLU mask); with many tiles per phase it measured neutral to slower
// (stage 2: 180 -> 201 us).
int g_dgrad_concurrent = -1;

struct PhaseStreams {
    cudaStream_t aux[3];
    cudaEvent_t fork, join[3];
    bool ok = false;
};

PhaseStreams& phase_streams() {  // one set per device, created on first use
    static PhaseStreams ps[16];
    static bool made[16] = {};
    static PhaseStreams none;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return none;
    if (!made[dev]) {
        made[dev] = true;
        PhaseStreams& q = ps[dev];
        bool ok = cudaEventCreateWithFlags(&q.fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; i < 3 && ok; ++i)
            ok = cudaStreamCreateWithFlags(&q.aux[i], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&q.join[i], cudaEventDisableTiming) == cudaSuccess;
        q.ok = ok;
    }
    return ps[dev];
}

cudaError_t conv_tc_dgrad(const ConvGeom& g, const void* dy, const void* w, const void* wTp,
                          const Epilogue& ep, void* dx, cudaStream_t st) {
    if (conv_tc_dgrad_needs_pack(g) && wTp == nullptr) return cudaErrorInvalidValue;
    if (!force_gather() && conv_win_applies(g, ConvMode::Dgrad)) return conv_win_dgrad(g, dy, w, ep, dx, st);
    if (g_dgrad_concurrent < 0) {
        const char* e = getenv("TCB_DGRAD_CONCURRENT");
        g_dgrad_concurrent = e ? atoi(e) : 2;
    }
    bool concurrent = g_dgrad_concurrent == 1;
    if (g_dgrad_concurrent == 2 && g.stride_h * g.stride_w > 1) {
        int most = 0;
        for (int ph = 0; ph < g.stride_h; ++ph)
            for (int pw = 0; pw < g.stride_w; ++pw) {
                const DgradPhase q = dgrad_phase(g, ph, pw);
                if (q.Hq > 0 && q.Wq > 0 && q.tr * q.ts > 0)
                    most = std::max(most, ((g.n * q.Hq * q.Wq + BM - 1) / BM) * ((g.c + 255) / 256));
            }
        concurrent = most > 0 && most < 2 * num_sms();
    }
    if (concurrent && g.stride_h * g.stride_w > 1 && g.stride_h * g.stride_w <= 4 &&
        wTp == nullptr && phase_streams().ok) {
        // work per phase ~ k-blocks + an epilogue share of 4 k-blocks per tile row
        int kb[4] = {0, 0, 0, 0}, np = 0, tot = 0;
        DgradPhase phs[4];
        for (int ph = 0; ph < g.stride_h; ++ph)
            for (int pw = 0; pw < g.stride_w; ++pw) {
                phs[np] = dgrad_phase(g, ph, pw);
                const DgradPhase& q = phs[np];
                kb[np] = (q.Hq > 0 && q.Wq > 0 && q.tr * q.ts > 0) ? q.tr * q.ts * ((g.k + BK - 1) / BK) + 4 : 0;
                tot += kb[np];
                ++np;
            }
        if (tot > 0) {
            PhaseStreams& S = phase_streams();
            cudaError_t e = cudaEventRecord(S.fork, st);
            if (e != cudaSuccess) return e;
            const int sms = num_sms() - g_sm_reserve;
            int used = 0;
            for (int i = 0; i < np; ++i) {
                cudaStream_t s_i = i == 0 ? st : S.aux[i - 1];
                if (i > 0 && (e = cudaStreamWaitEvent(s_i, S.fork, 0)) != cudaSuccess) return e;
                const DgradPhase& q = phs[i];
                if (q.Hq <= 0 || q.Wq <= 0) continue;
                Params p{};
                p.ph = q;
                p.s = make_shape(g, ConvMode::Dgrad);
                p.s.M = g.n * q.Hq * q.Wq;
                p.s.Kdim = q.tr * q.ts * g.k;
                p.d_hwq = FastDiv(static_cast<uint32_t>(q.Hq * q.Wq));
                p.d_wq = FastDiv(static_cast<uint32_t>(q.Wq));
                p.d_ts = FastDiv(static_cast<uint32_t>(std::max(q.ts, 1)));
                p.a = static_cast<const __nv_bfloat16*>(dy);
                p.wk = static_cast<const __nv_bfloat16*>(w);
                p.out = dx;
                p.residual = static_cast<const __nv_bfloat16*>(ep.residual);
                p.mask = static_cast<const __nv_bfloat16*>(ep.mask);
                if (p.s.Kdim == 0) {
                    if (ep.uncovered_zero && !ep.residual && !ep.mask) continue;
                    const size_t total = size_t(p.s.M) * (p.s.Ncol / 8);
                    const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 8192));
                    e = launch_pdl(dgrad_empty_phase_kernel, dim3(blocks), dim3(256), 0, s_i, p);
                } else {
                    g_grid_cap = i + 1 == np ? std::max(2, sms - used)
                                             : std::max(2, (sms * kb[i] / tot) & ~1);
                    used += g_grid_cap;
                    e = dispatch<ConvMode::Dgrad>(p, dy, nullptr, s_i);
                    g_grid_cap = 0;
                }
                if (e != cudaSuccess) return e;
            }
            for (int i = 1; i < np; ++i) {
                if ((e = cudaEventRecord(S.join[i - 1], S.aux[i - 1])) != cudaSuccess) return e;
                if ((e = cudaStreamWaitEvent(st, S.join[i - 1], 0)) != cudaSuccess) return e;
            }
            return cudaSuccess;
        }
    }
    for (int ph = 0; ph < g.stride_h; ++ph) {
        for (int pw = 0; pw < g.stride_w; ++pw) {
            Params p{};
            p.ph = dgrad_phase(g, ph, pw);
            if (p.ph.Hq <= 0 || p.ph.Wq <= 0) continue;
            p.s = make_shape(g, ConvMode::Dgrad);
            p.s.M = g.n * p.ph.Hq * p.ph.Wq;
            p.s.Kdim = p.ph.tr * p.ph.ts * g.k;
            p.d_hwq = FastDiv(static_cast<uint32_t>(p.ph.Hq * p.ph.Wq));
            p.d_wq = FastDiv(static_cast<uint32_t>(p.ph.Wq));
            p.d_ts = FastDiv(static_cast<uint32_t>(std::max(p.ph.ts, 1)));
            p.a = static_cast<const __nv_bfloat16*>(dy);
            p.wk = static_cast<const __nv_bfloat16*>(w);
            p.out = dx;
            p.residual = static_cast<const __nv_bfloat16*>(ep.residual);
            p.mask = static_cast<const __nv_bfloat16*>(ep.mask);
            cudaError_t e;
            if (p.s.Kdim == 0) {
                if (ep.uncovered_zero && !ep.residual && !ep.mask) continue;
                const size_t total = size_t(p.s.M) * (p.s.Ncol / 8);
                const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, 8192));
                e = launch_pdl(dgrad_empty_phase_kernel, dim3(blocks), dim3(256), 0, st, p);
            } else {
                e = dispatch<ConvMode::Dgrad>(
                    p, dy, wTp ? static_cast<const void*>(static_cast<const __nv_bfloat16*>(wTp) + p.ph.woff)
                               : nullptr,
                    st);
            }
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t conv_tc_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw,
                          void* workspace, cudaStream_t st, bool cols_ready, int* counters) {
    if (conv_stem_applies(g)) return conv_stem_wgrad(g, dy, x, dw, workspace, st, cols_ready);
    const NarrowPlan q = narrow_plan(g);
    if (q.use) {
        if (workspace == nullptr) return cudaErrorInvalidValue;
        char* ws = static_cast<char*>(workspace);
        cudaError_t e = cols_ready ? cudaSuccess : narrow_im2col(g, q, x, ws, st);
        if (e != cudaSuccess) return e;
        float* dwp = reinterpret_cast<float*>(ws + align256(q.col_bytes));
        void* rest = ws + align256(q.col_bytes) + align256(size_t(g.k) * q.kc * 4);
        if ((e = conv_tc_wgrad(q.g1, dy, ws, dwp, rest, st, false, counters)) != cudaSuccess)
            return e;
        const int total = g.k * g.r * g.s * g.c;
        return launch_pdl(narrow_scatter_grad, dim3(std::max(1, std::min(total / 256 + 1, 1024))), dim3(256), 0,
                          st, static_cast<const float*>(dwp), dw, g, q.cv, q.rw, q.kc);
    }
    if (!force_gather() && conv_win_wgrad_applies(g)) return conv_win_wgrad(g, dy, x, dw, workspace, st);
    Params p{};
    p.s = make_shape(g, ConvMode::Wgrad);
    const int bn0 = wgrad_bn(p.s);
    const bool pair = wgrad_pair(p.s, bn0);
    p.cta2 = pair ? 1 : 0;
    const SplitPlan sp = plan_splits(p.s, bn0, pair);
    p.a = static_cast<const __nv_bfloat16*>(dy);
    p.b = static_cast<const __nv_bfloat16*>(x);
    p.splits = sp.splits;
    p.kb_per_split = sp.kb_per_split;
    p.out = sp.splits > 1 ? workspace : static_cast<void*>(dw);
    if (sp.splits > 1 && workspace == nullptr) return cudaErrorInvalidValue;
    const int bn = wgrad_bn(p.s);
    const int tiles = ((p.s.M + BM - 1) / BM) * ((p.s.Ncol + bn - 1) / bn);
    const bool fused = counters && sp.splits > 1 && tiles * sp.splits <= num_sms();
    if (fused) {
        p.dw = dw;
        p.counters = counters;
    }
    cudaError_t e = dispatch<ConvMode::Wgrad>(p, dy, x, st);
    if (e != cudaSuccess || sp.splits == 1 || fused) return e;
    return split_reduce(static_cast<const float*>(workspace), sp.splits,
                        size_t(p.s.M) * p.s.Ncol, dw, st);
}

}  // namespace tcb
