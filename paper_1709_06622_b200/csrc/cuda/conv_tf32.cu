// TF32 tensor-core implicit-GEMM convolution (tcgen05.mma kind::tf32) — the
// "TF32 tensor-core mode" of the north-star tolerance split (2e-2 relative vs
// the CPU oracle): fp32 storage end to end (the reference's storage type,
// R:include/traincap/mem_model.hpp:10-11), tf32 multiplies, fp32 accumulate
// in TMEM. Same GEMM views as every other conv family (common.cuh::ConvShape).
//
// One output tile (128 x BN) per CTA, two CTAs per SM so one CTA's epilogue
// overlaps the other's main loop:
//   warps 0-3  producers: cp.async gathers (zero-fill = padding / strides /
//              ragged tiles) of both operands into 128B-swizzled shared
//              memory, one 128-byte row = 32 fp32 of the reduction (K-major)
//              or of the M/N axis (MN-major); then the epilogue (thread =
//              TMEM lane = output row).
//   warp  4    MMA issuer: one elected thread, 4 x (M=128, N=BN, K=8) per
//              32-deep k-block; tcgen05.commit frees the stage.
// Operand majors: fwd A (im2col x) and B (w[K][RSC]) K-major (SWIZZLE_128B);
// dgrad A (the flipped-tap im2col of dy) K-major, B (w[k][r][s][c..]) MN-major;
// wgrad A (dy[pixel][k..]) and B (im2col x[pixel][(r,s,c)..]) both MN-major.
// MN-major tf32 operands must use SWIZZLE_128B_BASE32B (32-byte granules).
// Strided dgrad runs the plain all-taps GEMM (non-lattice taps zero-filled).
// Wgrad splits the pixel reduction across CTAs and reduces the fp32 partials
// in fixed order afterwards (split_reduce), so results are deterministic.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"
#include "tma.cuh"

namespace tcb {
namespace {

constexpr int BM = 128;
constexpr int BKE = 32;  // fp32 elements of the reduction per stage (128 B rows)
constexpr int kProducerThreads = 128;
constexpr int kMmaWarp = 4;
constexpr int kThreads = kProducerThreads + 32;
constexpr uint32_t kMnBlock = 32 * 128;  // one MN-major 32-element block: 32 rows x 128 B

template <int BN>
struct Cfg {
    static constexpr int kABytes = BM * 128;
    static constexpr int kBBytes = BN * 128;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = BN == 128 ? 3 : 4;  // ~96 KB: two CTAs per SM
    static constexpr size_t kSmem = size_t(kStages) * kStageBytes + 1024 + 256;
};

struct Params {
    CUtensorMap tmap_a, tmap_b;  // TMA operand paths (one producer thread)
    int load;                    // kGather / kPlain / kIm2col
    ConvShape s;
    const float* a;  // fwd: x   dgrad: dy   wgrad: dy
    const float* b;  // fwd/dgrad: w   wgrad: x
    float* out;      // fwd: y  dgrad: dx  wgrad: dw or partials [split][M][Ncol]
    const float* bias;
    const float* residual;
    const float* mask;
    int relu;
    int m_tiles, n_tiles, kb_total, kb_per_split;
    // one k-block never crosses a filter tap (fwd: C % 32 == 0, dgrad: K % 32 == 0):
    // operand addresses are decoded once per k-block instead of per 16-B chunk
    int tap_aligned;
    // dgrad: one stride phase (common.cuh::DgradPhase) — rows m = (n, hq, wq),
    // reduction kk = (tap (ti, si), k); s.M / s.Kdim are the phase's GEMM sizes
    DgradPhase ph;
    FastDiv d_hwq, d_wq, d_ts;
};

// Operand loads: kGather = cp.async by 128 threads (any C, K % 4 == 0);
// kPlain = 1x1/s1/p0, every operand a plain matrix by 2-D TMA; kIm2col = the
// activation operand by im2col-mode TMA (one tap x 32 channels per k-block).
// kIm2colC4 = fwd with C == 4 (the padded RGB stem): eight one-tap boxes of
// 128 pixels x 16 B per k-block, landing as no-swizzle 8x16B core matrices.
constexpr int kGather = 0, kPlain = 1, kIm2col = 2, kIm2colC4 = 3;

// K-major rows (SWIZZLE_128B): 16-byte chunk j of row r lands at j ^ (r & 7).
__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ (row & 7u)) << 4);
}
// MN-major rows (SWIZZLE_128B_BASE32B): 32-byte granule g of row r lands at g ^ (r & 3).
__device__ __forceinline__ uint32_t swz_mn(uint32_t row, uint32_t chunk) {
    return row * 128u + ((chunk ^ ((row & 3u) << 1)) << 4);
}

template <ConvMode MODE, int BN, bool TMA>
__global__ void __launch_bounds__(kThreads, 2) conv_tf32_kernel(const __grid_constant__ Params p) {
    using C = Cfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* accfull = empty + C::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accfull + 1);
    constexpr int kPixRows = MODE == ConvMode::Wgrad ? BKE : 1;  // wgrad pixel decode table
    __shared__ int4 pixtab[2][kPixRows];

    const ConvShape& s = p.s;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int nt = blockIdx.x % p.n_tiles;
    const int mt = (blockIdx.x / p.n_tiles) % p.m_tiles;
    const int split = blockIdx.x / (p.n_tiles * p.m_tiles);
    const int kb_begin = split * p.kb_per_split;
    const int kb_end = min(p.kb_total, kb_begin + p.kb_per_split);
    const bool has_k = kb_end > kb_begin;  // false: a dgrad phase without filter taps

    if (tid == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            ptx::mbar_init(&full[i], TMA ? 1 : kProducerThreads);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(accfull, 1);
        ptx::fence_mbarrier_init();
    }
    if (warp == kMmaWarp) ptx::tmem_alloc<BN>(tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t smem_base = ptx::smem_addr(smem);

    if (warp < 4 && TMA) {
        // =========================================== TMA producer (1 thread) ======
        if (tid == 0 && has_k) {
            int bn = 0, bh = 0, bw = 0;  // im2col base of the tile's first GEMM row (fwd / dgrad)
            if (MODE != ConvMode::Wgrad && (p.load == kIm2col || p.load == kIm2colC4)) {
                uint32_t n, rem, a, b;
                const uint32_t m0 = static_cast<uint32_t>(mt * BM);
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
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = kb_begin; kb < kb_end; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t a_smem = smem_base + stage * C::kStageBytes;
                const uint32_t b_smem = a_smem + C::kABytes;
                uint64_t* bar = &full[stage];
                ptx::mbar_arrive_expect_tx(bar, C::kStageBytes);
                const int kk0 = kb * BKE;
                if constexpr (MODE == ConvMode::Fwd) {
                    if (p.load == kPlain) {
                        ptx::tma_load_2d(a_smem, &p.tmap_a, bar, kk0, mt * BM);
                    } else if (p.load == kIm2colC4) {
                        const int taps = s.R * s.S;
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            int tap = kb * 8 + jj;
                            if (tap >= taps) tap = 0;  // K tail: the B rows there are zero
                            uint32_t r, sx;
                            s.d_s.divmod(static_cast<uint32_t>(tap), r, sx);
                            ptx::tma_load_im2col_4d(a_smem + jj * 2048, &p.tmap_a, bar, 0, bw, bh, bn,
                                                    static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                        }
                    } else {
                        uint32_t tap, c0, r, sx;
                        s.d_c.divmod(static_cast<uint32_t>(kk0), tap, c0);
                        s.d_s.divmod(tap, r, sx);
                        ptx::tma_load_im2col_4d(a_smem, &p.tmap_a, bar, static_cast<int>(c0), bw, bh, bn,
                                                static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                    }
                    ptx::tma_load_2d(b_smem, &p.tmap_b, bar, kk0, nt * BN);
                } else if constexpr (MODE == ConvMode::Dgrad) {
                    // k-block = 32 filters k0.. of one phase tap; im2col offsets count the
                    // tap from the far corner (ho = base + r'), i.e. ti = tr - 1 - r'
                    uint32_t t, k0, rr, ss;
                    s.d_k.divmod(static_cast<uint32_t>(kk0), t, k0);
                    p.d_ts.divmod(t, rr, ss);
                    if (p.load == kPlain)
                        ptx::tma_load_2d(a_smem, &p.tmap_a, bar, static_cast<int>(k0), mt * BM);
                    else
                        ptx::tma_load_im2col_4d(a_smem, &p.tmap_a, bar, static_cast<int>(k0), bw, bh, bn,
                                                static_cast<uint16_t>(ss), static_cast<uint16_t>(rr));
                    const int rf = p.ph.r0 + (p.ph.tr - 1 - static_cast<int>(rr)) * s.sh;
                    const int sf = p.ph.s0 + (p.ph.ts - 1 - static_cast<int>(ss)) * s.sw;
#pragma unroll
                    for (int j = 0; j < BN / 32; ++j)
                        ptx::tma_load_3d(b_smem + j * kMnBlock, &p.tmap_b, bar, nt * BN + j * 32, rf * s.S + sf,
                                         static_cast<int>(k0));
                } else {
#pragma unroll
                    for (int j = 0; j < BM / 32; ++j)
                        ptx::tma_load_2d(a_smem + j * kMnBlock, &p.tmap_a, bar, mt * BM + j * 32, kk0);
                    if (p.load == kPlain) {
#pragma unroll
                        for (int j = 0; j < BN / 32; ++j)
                            ptx::tma_load_2d(b_smem + j * kMnBlock, &p.tmap_b, bar, nt * BN + j * 32, kk0);
                    } else {
                        uint32_t n, rem, ho, wo;
                        s.d_howo.divmod(static_cast<uint32_t>(kk0), n, rem);
                        s.d_wo.divmod(rem, ho, wo);
                        const int ph = static_cast<int>(ho) * s.sh - s.ph, pw = static_cast<int>(wo) * s.sw - s.pw;
#pragma unroll
                        for (int j = 0; j < BN / 32; ++j) {
                            int col0 = nt * BN + j * 32;
                            if (col0 >= s.Ncol) col0 = 0;  // padding columns: never stored
                            uint32_t tap, c0, r, sx;
                            s.d_c.divmod(static_cast<uint32_t>(col0), tap, c0);
                            s.d_s.divmod(tap, r, sx);
                            ptx::tma_load_im2col_4d(b_smem + j * kMnBlock, &p.tmap_b, bar, static_cast<int>(c0), pw,
                                                    ph, static_cast<int>(n), static_cast<uint16_t>(sx),
                                                    static_cast<uint16_t>(r));
                        }
                    }
                }
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }
    if (warp < 4 && !TMA) {
        // ================================================ producers ======
        constexpr int kCpr = BN / 4;                      // 16-B chunks per MN-major B row
        constexpr int kRowsPerPass = kProducerThreads / kCpr;
        // per-thread constant decode of the tile
        int row_n = 0, row_hb = 0, row_wb = 0;
        bool row_ok = false;                // fwd / dgrad: this thread's A row
        int col_r = 0, col_s = 0, col_c = 0;
        bool col_ok = false;                // wgrad: this thread's B column chunk
        if constexpr (MODE == ConvMode::Wgrad) {
            const int col = nt * BN + (tid % kCpr) * 4;
            col_ok = col < s.Ncol;
            if (col_ok) {
                uint32_t rs, c0, r, sx;
                s.d_c.divmod(static_cast<uint32_t>(col), rs, c0);
                s.d_s.divmod(rs, r, sx);
                col_r = static_cast<int>(r);
                col_s = static_cast<int>(sx);
                col_c = static_cast<int>(c0);
            }
        } else {
            const int m = mt * BM + tid;
            row_ok = m < s.M;
            if (row_ok) {
                uint32_t n, rem, a, b;
                if constexpr (MODE == ConvMode::Fwd) {
                    s.d_howo.divmod(static_cast<uint32_t>(m), n, rem);
                    s.d_wo.divmod(rem, a, b);
                    row_hb = static_cast<int>(a) * s.sh - s.ph;
                    row_wb = static_cast<int>(b) * s.sw - s.pw;
                } else {
                    // ho = hq + bh - ti for tap r = r0 + ti * sh (exact, no division)
                    p.d_hwq.divmod(static_cast<uint32_t>(m), n, rem);
                    p.d_wq.divmod(rem, a, b);
                    row_hb = static_cast<int>(a) + p.ph.bh;
                    row_wb = static_cast<int>(b) + p.ph.bw;
                }
                row_n = static_cast<int>(n);
            }
        }
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            int4* tab = pixtab[kb & 1];
            if constexpr (MODE == ConvMode::Wgrad) {
                // this k-block's 32 pixels decoded once, shared by all producers
                if (tid < BKE) {
                    const int pix = kb * BKE + tid;
                    int4 e = make_int4(-1, 0, 0, 0);
                    if (pix < s.Kdim) {
                        uint32_t n, rem, ho, wo;
                        s.d_howo.divmod(static_cast<uint32_t>(pix), n, rem);
                        s.d_wo.divmod(rem, ho, wo);
                        e = make_int4(static_cast<int>(n) * s.H, static_cast<int>(ho) * s.sh - s.ph,
                                      static_cast<int>(wo) * s.sw - s.pw, 0);
                    }
                    tab[tid] = e;
                }
                asm volatile("bar.sync 1, %0;" ::"n"(kProducerThreads) : "memory");
            }
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            const uint32_t a_smem = smem_base + stage * C::kStageBytes;
            const uint32_t b_smem = a_smem + C::kABytes;
            // ---- A
            if constexpr (MODE == ConvMode::Wgrad) {
                // dy[pixel][k]: 32 pixel rows x 128 channels, 4 MN blocks
                const int cq = tid & 31;
                const int k0 = mt * BM + cq * 4;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int rr = (tid >> 5) + 4 * i;
                    const int pix = kb * BKE + rr;
                    const bool ok = pix < s.Kdim && k0 < s.K;
                    const float* src = ok ? p.a + static_cast<size_t>(pix) * s.K + k0 : p.a;
                    ptx::cp_async_16(a_smem + (cq >> 3) * kMnBlock + swz_mn(rr, cq & 7), src, ok ? 16u : 0u);
                }
            } else {
                // one A row (output pixel for fwd, phase pixel for dgrad) per thread;
                // returns the row's source for reduction index kk0, or NULL (zero-fill)
                auto a_src = [&](int kk0) -> const float* {
                    if (!row_ok || kk0 >= s.Kdim) return nullptr;
                    if constexpr (MODE == ConvMode::Fwd) {
                        uint32_t rs, c0, r, sx;
                        s.d_c.divmod(static_cast<uint32_t>(kk0), rs, c0);
                        s.d_s.divmod(rs, r, sx);
                        const int hi = row_hb + static_cast<int>(r);
                        const int wi = row_wb + static_cast<int>(sx);
                        if (hi < 0 || hi >= s.H || wi < 0 || wi >= s.W) return nullptr;
                        return p.a + ((static_cast<size_t>(row_n) * s.H + hi) * s.W + wi) * s.C + c0;
                    } else {
                        uint32_t t, k0, ti, si;
                        s.d_k.divmod(static_cast<uint32_t>(kk0), t, k0);
                        p.d_ts.divmod(t, ti, si);
                        const int ho = row_hb - static_cast<int>(ti);
                        const int wo = row_wb - static_cast<int>(si);
                        if (ho < 0 || ho >= s.Ho || wo < 0 || wo >= s.Wo) return nullptr;
                        return p.a + ((static_cast<size_t>(row_n) * s.Ho + ho) * s.Wo + wo) * s.K + k0;
                    }
                };
                if (p.tap_aligned) {
                    const float* src = a_src(kb * BKE);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        ptx::cp_async_16(a_smem + swz(tid, j), src ? src + 4 * j : p.a, src ? 16u : 0u);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float* src = a_src(kb * BKE + 4 * j);
                        ptx::cp_async_16(a_smem + swz(tid, j), src ? src : p.a, src ? 16u : 0u);
                    }
                }
            }
            // ---- B
            if constexpr (MODE == ConvMode::Fwd) {
                // w[k][(r,s,c)]: BN filter rows, K-major
                const int cc = tid & 7;
                const int kk0 = kb * BKE + cc * 4;
#pragma unroll
                for (int i = 0; i < BN / 16; ++i) {
                    const int row = (tid >> 3) + 16 * i;
                    const int j = nt * BN + row;
                    const bool ok = j < s.Ncol && kk0 < s.Kdim;
                    const float* src = ok ? p.b + static_cast<size_t>(j) * s.Kdim + kk0 : p.b;
                    ptx::cp_async_16(b_smem + swz(row, cc), src, ok ? 16u : 0u);
                }
            } else {
                const int cq = tid % kCpr;
#pragma unroll
                for (int i = 0; i < BN / 16; ++i) {
                    const int rr = tid / kCpr + kRowsPerPass * i;
                    const int kk = kb * BKE + rr;
                    const float* src = p.b;
                    uint32_t bytes = 0;
                    if constexpr (MODE == ConvMode::Dgrad) {
                        // w[k][r][s][c..c+3]: reduction row (phase tap, k), channels along the row
                        const int c = nt * BN + cq * 4;
                        if (kk < s.Kdim && c < s.C) {
                            uint32_t t, k, ti, si;
                            s.d_k.divmod(static_cast<uint32_t>(kk), t, k);
                            p.d_ts.divmod(t, ti, si);
                            const int r = p.ph.r0 + static_cast<int>(ti) * s.sh;
                            const int sx = p.ph.s0 + static_cast<int>(si) * s.sw;
                            src = p.b + ((static_cast<size_t>(k) * s.R + r) * s.S + sx) * s.C + c;
                            bytes = 16;
                        }
                    } else {
                        // x[n][hi][wi][c..c+3] of pixel kk, column (r,s,c)
                        const int4 px = tab[rr];
                        const int hi = px.y + col_r, wi = px.z + col_s;
                        if (col_ok && px.x >= 0 && hi >= 0 && hi < s.H && wi >= 0 && wi < s.W) {
                            src = p.b + ((static_cast<size_t>(px.x) + hi) * s.W + wi) * s.C + col_c;
                            bytes = 16;
                        }
                    }
                    ptx::cp_async_16(b_smem + (cq >> 3) * kMnBlock + swz_mn(rr, cq & 7), src, bytes);
                }
            }
            ptx::cp_async_mbar_arrive_noinc(&full[stage]);
            if (++stage == C::kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
        ptx::cp_async_wait<0>();
    }
    if (warp < 4) {
        // ================================================= epilogue ======
        // Thread = TMEM lane = tile row. Each 32-column chunk is staged through a
        // warp-private 32x32 fp32 smem tile (the drained operand ring) and
        // leaves transposed: 8 lanes per row, 128-byte coalesced row segments
        // for the output and the residual / mask side inputs.
        if (has_k) {
            ptx::mbar_wait(accfull, 0);
            ptx::tc_fence_after();
        }
        const int lane = tid & 31;
        const int m = mt * BM + tid;
        // element offset of this thread's output row (-1: past the GEMM rows)
        long long orow = -1;
        if (m < s.M) {
            if constexpr (MODE == ConvMode::Dgrad) {
                uint32_t n, rem, hq, wq;
                p.d_hwq.divmod(static_cast<uint32_t>(m), n, rem);
                p.d_wq.divmod(rem, hq, wq);
                orow = ((static_cast<long long>(n) * s.H + hq * s.sh + p.ph.ph) * s.W + wq * s.sw + p.ph.pw) *
                       s.Ncol;
            } else if constexpr (MODE == ConvMode::Wgrad) {
                orow = (static_cast<long long>(split) * s.M + m) * s.Ncol;
            } else {
                orow = static_cast<long long>(m) * s.Ncol;
            }
        }
        float4* stage_tile = reinterpret_cast<float4*>(smem + warp * 4096);  // [32 rows][8 float4]
        const int sub = lane >> 3, cg = lane & 7;  // read-back: row sub + 4q, column group cg
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            const int col0 = nt * BN + c * 32;
            if (col0 >= s.Ncol) break;
            uint32_t v[32];
            if (has_k) {
                ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, v);
                ptx::tmem_ld_wait();
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0u;
            }
            __syncwarp();  // the previous chunk's read-back is done
#pragma unroll
            for (int g = 0; g < 8; ++g)
                stage_tile[lane * 8 + (g ^ (lane & 7))] =
                    make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3]));
            __syncwarp();
            const int col = col0 + cg * 4;
            const bool col_in = col < s.Ncol;  // Ncol % 4 == 0
            float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (MODE == ConvMode::Fwd && p.bias && col_in) b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col));
            long long rows[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) rows[q] = __shfl_sync(0xffffffffu, orow, sub + 4 * q);
            float4 r4[8], k4[8];
            if constexpr (MODE != ConvMode::Wgrad) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const bool ok = rows[q] >= 0 && col_in;
                    if (p.residual && ok) r4[q] = __ldg(reinterpret_cast<const float4*>(p.residual + rows[q] + col));
                    if (p.mask && ok) k4[q] = __ldg(reinterpret_cast<const float4*>(p.mask + rows[q] + col));
                }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int row = sub + 4 * q;
                if (rows[q] < 0 || !col_in) continue;
                float4 x = stage_tile[row * 8 + (cg ^ (row & 7))];
                if constexpr (MODE != ConvMode::Wgrad) {
                    x.x += b4.x; x.y += b4.y; x.z += b4.z; x.w += b4.w;
                    if (p.residual) { x.x += r4[q].x; x.y += r4[q].y; x.z += r4[q].z; x.w += r4[q].w; }
                    if (p.relu) {
                        x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f);
                        x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
                    }
                    if (p.mask) {
                        if (!(k4[q].x > 0.f)) x.x = 0.f;
                        if (!(k4[q].y > 0.f)) x.y = 0.f;
                        if (!(k4[q].z > 0.f)) x.z = 0.f;
                        if (!(k4[q].w > 0.f)) x.w = 0.f;
                    }
                }
                *reinterpret_cast<float4*>(p.out + rows[q] + col) = x;
            }
        }
    } else if (warp == kMmaWarp) {
        // =============================================== MMA issuer ======
        constexpr uint32_t kAmn = MODE == ConvMode::Wgrad ? 1u : 0u;
        constexpr uint32_t kBmn = MODE == ConvMode::Fwd ? 0u : 1u;
        constexpr uint32_t idesc = ptx::make_idesc(2 /*tf32*/, BM, BN, kAmn, kBmn);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb_begin; kb < kb_end; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t a_addr = smem_base + stage * C::kStageBytes;
                const uint32_t b_addr = a_addr + C::kABytes;
#pragma unroll
                for (int k = 0; k < BKE / 8; ++k) {
                    const uint64_t ad = kAmn ? ptx::sw128b32_desc(a_addr + k * 1024, kMnBlock, 512)
                                        : (TMA && p.load == kIm2colC4)
                                            ? ptx::interleave_desc(a_addr + k * 4096, 2048, 128)
                                            : ptx::sw128_desc(a_addr + k * 32, 16, 1024);
                    const uint64_t bd = kBmn ? ptx::sw128b32_desc(b_addr + k * 1024, kMnBlock, 512)
                                             : ptx::sw128_desc(b_addr + k * 32, 16, 1024);
                    ptx::umma_tf32(tmem_base, ad, bd, idesc, (kb > kb_begin || k > 0) ? 1u : 0u);
                }
                ptx::umma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == C::kStages) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (has_k && ptx::elect_one()) ptx::umma_commit(accfull);
        __syncwarp();
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<BN>(tmem_base);
    }
}

struct Plan {
    int bn, m_tiles, n_tiles, kb_total, kb_per_split, splits;
};

Plan make_plan(const ConvShape& s, ConvMode mode) {
    Plan pl{};
    pl.bn = s.Ncol <= 64 ? 64 : 128;
    pl.m_tiles = (s.M + BM - 1) / BM;
    pl.n_tiles = (s.Ncol + pl.bn - 1) / pl.bn;
    pl.kb_total = (s.Kdim + BKE - 1) / BKE;
    int want = 1;
    if (mode == ConvMode::Wgrad) {
        // fill two CTAs per SM with split-K units, each at least 8 k-blocks deep
        const int tiles = pl.m_tiles * pl.n_tiles;
        want = std::max(1, (2 * num_sms() + tiles - 1) / tiles);
        want = std::min({want, std::max(1, pl.kb_total / 8), 256});
    }
    pl.kb_per_split = std::max(1, (pl.kb_total + want - 1) / want);
    pl.splits = std::max(1, (pl.kb_total + pl.kb_per_split - 1) / pl.kb_per_split);
    return pl;
}

template <ConvMode MODE, int BN, bool TMA>
cudaError_t launch(const Params& p, int grid, cudaStream_t st) {
    auto kern = conv_tf32_kernel<MODE, BN, TMA>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(Cfg<BN>::kSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    kern<<<grid, kThreads, Cfg<BN>::kSmem, st>>>(p);
    return cudaGetLastError();
}

// $TCB_TF32_GATHER=1 / conv_tf32_set_force_gather: always the cp.async gather operands
int g_force_gather = [] {
    const char* e = getenv("TCB_TF32_GATHER");
    return e && e[0] == '1' ? 1 : 0;
}();
bool force_gather() { return g_force_gather != 0; }

bool plain_geometry(const ConvShape& s) {
    return s.R == 1 && s.S == 1 && s.ph == 0 && s.pw == 0 && s.sh == 1 && s.sw == 1;
}

// im2col TMA: whole 32-channel slices of one tap per k-block, small corners
bool im2col_geometry(const ConvShape& s, int channels) {
    return channels % BKE == 0 && s.R <= 16 && s.S <= 16 && s.ph <= 15 && s.pw <= 15;
}

template <ConvMode MODE>
int pick_load(const ConvShape& s) {
    if (force_gather()) return kGather;
    if (MODE == ConvMode::Dgrad && s.K % BKE != 0) return kGather;  // k-blocks within one tap
    if (plain_geometry(s)) return kPlain;
    if (MODE == ConvMode::Fwd && s.C == 4 && s.R <= 16 && s.S <= 16 && s.ph <= 15 && s.pw <= 15)
        return kIm2colC4;
    return im2col_geometry(s, MODE == ConvMode::Dgrad ? s.K : s.C) ? kIm2col : kGather;
}

template <ConvMode MODE>
bool build_maps(Params& p, int bn) {
    const ConvShape& s = p.s;
    const auto k_major = CU_TENSOR_MAP_SWIZZLE_128B, mn_major = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    if constexpr (MODE == ConvMode::Fwd) {
        const bool a = p.load == kPlain
                           ? make_tmap_f32_2d(&p.tmap_a, p.a, s.M, s.C, BM, k_major)
                       : p.load == kIm2colC4
                           ? make_tmap_im2col_f32(&p.tmap_a, p.a, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                                  s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BM,
                                                  CU_TENSOR_MAP_SWIZZLE_NONE, 4)
                           : make_tmap_im2col_f32(&p.tmap_a, p.a, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                                  s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BM, k_major);
        return a && make_tmap_f32_2d(&p.tmap_b, p.b, s.Ncol, s.Kdim, bn, k_major);
    } else if constexpr (MODE == ConvMode::Dgrad) {
        bool a;
        if (p.load == kPlain) {
            a = make_tmap_f32_2d(&p.tmap_a, p.a, s.M, s.K, BM, k_major);
        } else {
            const int lw = p.ph.bw - (p.ph.ts - 1), lh = p.ph.bh - (p.ph.tr - 1);
            a = make_tmap_im2col_f32(&p.tmap_a, p.a, s.N, s.Ho, s.Wo, s.K, lw, lh, lw + p.ph.Wq - s.Wo,
                                     lh + p.ph.Hq - s.Ho, 1, 1, BM, k_major);
        }
        return a && make_tmap_filters_f32(&p.tmap_b, p.b, s.K, size_t(s.R) * s.S, s.C);
    } else {
        const bool a = make_tmap_f32_2d(&p.tmap_a, p.a, s.Kdim, s.K, BKE, mn_major);
        return a && (p.load == kPlain
                         ? make_tmap_f32_2d(&p.tmap_b, p.b, s.Kdim, s.C, BKE, mn_major)
                         : make_tmap_im2col_f32(&p.tmap_b, p.b, s.N, s.H, s.W, s.C, -s.pw, -s.ph,
                                                s.pw - (s.S - 1), s.ph - (s.R - 1), s.sw, s.sh, BKE, mn_major));
    }
}

template <ConvMode MODE>
cudaError_t run(Params p, const Plan& pl, cudaStream_t st) {
    p.m_tiles = pl.m_tiles;
    p.n_tiles = pl.n_tiles;
    p.kb_total = pl.kb_total;
    p.kb_per_split = pl.kb_per_split;
    const int grid = pl.m_tiles * pl.n_tiles * pl.splits;
    p.load = p.s.Kdim > 0 ? pick_load<MODE>(p.s) : kGather;
    if (p.load != kGather && !build_maps<MODE>(p, pl.bn)) return cudaErrorInvalidValue;
    if (p.load != kGather)
        return pl.bn == 64 ? launch<MODE, 64, true>(p, grid, st) : launch<MODE, 128, true>(p, grid, st);
    return pl.bn == 64 ? launch<MODE, 64, false>(p, grid, st) : launch<MODE, 128, false>(p, grid, st);
}

}  // namespace

void conv_tf32_set_force_gather(int on) { g_force_gather = on ? 1 : 0; }

bool conv_tf32_supported(const ConvGeom& g) {
    return g.c % 4 == 0 && g.k % 4 == 0 && g.c > 0 && g.k > 0;
}

size_t conv_tf32_workspace(const ConvGeom& g, ConvMode mode) {
    if (mode != ConvMode::Wgrad) return 0;
    const ConvShape s = make_shape(g, mode);
    const Plan pl = make_plan(s, mode);
    return pl.splits > 1 ? size_t(pl.splits) * s.M * s.Ncol * sizeof(float) : 0;
}

cudaError_t conv_tf32_fwd(const ConvGeom& g, const float* x, const float* w, const Epilogue& ep,
                          float* y, cudaStream_t st) {
    if (!conv_tf32_supported(g)) return cudaErrorInvalidValue;
    Params p{};
    p.s = make_shape(g, ConvMode::Fwd);
    p.a = x;
    p.b = w;
    p.out = y;
    p.bias = ep.bias;
    p.residual = static_cast<const float*>(ep.residual);
    p.relu = ep.relu;
    p.tap_aligned = g.c % BKE == 0;
    return run<ConvMode::Fwd>(p, make_plan(p.s, ConvMode::Fwd), st);
}

cudaError_t conv_tf32_dgrad(const ConvGeom& g, const float* dy, const float* w,
                            const Epilogue& ep, float* dx, cudaStream_t st) {
    if (!conv_tf32_supported(g)) return cudaErrorInvalidValue;
    // one GEMM per stride phase: exact taps only, no zero-insertion waste
    Params p{};
    p.a = dy;
    p.b = w;
    p.out = dx;
    p.residual = static_cast<const float*>(ep.residual);
    p.mask = static_cast<const float*>(ep.mask);
    p.tap_aligned = g.k % BKE == 0;
    for (int ph = 0; ph < g.stride_h; ++ph) {
        for (int pw = 0; pw < g.stride_w; ++pw) {
            p.s = make_shape(g, ConvMode::Dgrad);
            p.ph = dgrad_phase(g, ph, pw);
            if (p.ph.Hq == 0 || p.ph.Wq == 0) continue;
            p.s.M = g.n * p.ph.Hq * p.ph.Wq;
            p.s.Kdim = p.ph.tr * p.ph.ts * g.k;  // 0: no taps, dx = residual * mask (or 0)
            p.d_hwq = FastDiv(static_cast<uint32_t>(p.ph.Hq * p.ph.Wq));
            p.d_wq = FastDiv(static_cast<uint32_t>(p.ph.Wq));
            p.d_ts = FastDiv(static_cast<uint32_t>(std::max(1, p.ph.ts)));
            cudaError_t e = run<ConvMode::Dgrad>(p, make_plan(p.s, ConvMode::Dgrad), st);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

cudaError_t conv_tf32_wgrad(const ConvGeom& g, const float* dy, const float* x, float* dw,
                            void* workspace, cudaStream_t st) {
    if (!conv_tf32_supported(g)) return cudaErrorInvalidValue;
    Params p{};
    p.s = make_shape(g, ConvMode::Wgrad);
    p.a = dy;
    p.b = x;
    const Plan pl = make_plan(p.s, ConvMode::Wgrad);
    if (pl.splits > 1 && !workspace) return cudaErrorInvalidValue;
    p.out = pl.splits > 1 ? static_cast<float*>(workspace) : dw;
    cudaError_t e = run<ConvMode::Wgrad>(p, pl, st);
    if (e != cudaSuccess || pl.splits == 1) return e;
    return split_reduce(static_cast<float*>(workspace), pl.splits, size_t(p.s.M) * p.s.Ncol, dw, st);
}

}  // namespace tcb
