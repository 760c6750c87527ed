// Window implicit-GEMM convolution for stride-1 R x S layers (sm_100a).
//
// The im2col TMA path (conv_tc.cu) brings one 128-pixel x 64-channel box per
// filter tap, so every input pixel crosses L2 -> SM R*S times; on the
// 56x56x64 and 28x28x128 3x3 layers that traffic, not the tensor pipe, sets
// the pace. Here the activation operand of a tile is loaded ONCE per 64-
// channel slice as a "window": whole padded input rows (a tiled 4-D TMA box
// {64 ch, Wp, WR rows, 1 image}, out-of-image rows / columns zero-filled).
// GEMM row m of a tile is flat position f0 + m of the padded output plane
// (row-major, Wp = Wo + S - 1 columns per row, the last S - 1 of each row are
// junk outputs that the epilogue drops), so filter tap (r, s) is the same
// window seen through a UMMA A descriptor shifted by r*Wp + s rows of 128 B.
// (Measured, scripts/probes/umma_shift_probe.cu: K-major SWIZZLE_128B
// descriptors at any 128-byte row offset of a TMA-swizzled buffer read
// correctly with base-offset 0 and at full MMA rate.)
//
//   warp 0 (1 thread) TMA producer: windows into a 2-4 stage ring; the weight
//                     operand per (tap, slice) into a B ring, or loaded once
//                     and kept resident when it fits (one N tile, <= 96 KB)
//   warp 12           MMA issuer: tcgen05.mma kind::f16, M = 128 (or 256 over
//                     a CTA pair: two images at the same flat offset, so both
//                     CTAs' windows share one A descriptor), N = BN, K = 16
//   warps 4-11        epilogue: tcgen05.ld, bias / residual / ReLU (fwd) or
//                     residual-grad / ReLU-mask (dgrad), bf16 stores of the
//                     valid rows; double-buffered TMEM accumulators
//
// Fwd: activation x, B = w[K][R*S*C] (K-major). Dgrad of a stride-1 conv is
// the same stencil over dy with flipped taps and padding R-1-pad: activation
// dy, B = the KRSC filters read MN-major ([K][R*S][C] boxes), no transpose.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tma.cuh"

namespace tcb {
namespace {

constexpr int BM = 128;
constexpr int kEpiThreads = 256;  // warps 4-11
constexpr int kMmaWarp = 12;
constexpr int kThreads = 13 * 32;
constexpr int kMaxWin = 4, kMaxB = 8;
constexpr size_t kSmemCap = 227 * 1024 - 2048;

struct WinParams {
    CUtensorMap tmap_win;  // activation [N][Ha][Wa][Ca] bf16, box {64, Wp, WR, 1}
    CUtensorMap tmap_b;    // fwd: w [Ncol][R*S*Ca] (K-major); dgrad: filters [Ca][R*S][Ncol]
    int n_img, Ho, Wo;     // GEMM output grid per image (fwd: y, dgrad: dx)
    int pad_h, pad_w;      // window padding (fwd: the conv's; dgrad: R-1-pad_h, S-1-pad_w)
    int R, S;              // taps of the stencil (dgrad: flipped)
    int Wp, tiles_img, slices;
    int rect, tw, th;      // rectangular tiles (wide images): th output rows x tw columns per tile
    FastDiv d_cb;          // column blocks per tile row (rect)
    int Ncol, n_tiles, units;
    uint32_t win_bytes, win_stride, b_bytes;
    int win_stages, b_stages;
    void* out;
    const float* bias;
    const __nv_bfloat16* residual;
    const __nv_bfloat16* mask;
    int relu;
    FastDiv d_wp, d_tiles, d_ntiles;
    unsigned long long* dbg;  // optional per-CTA role timing (tcb_conv_win_debug)
    uint32_t stg_off;         // epilogue staging tiles (8 x 2 KB) at this smem offset; 0 = direct stores
};

__device__ __forceinline__ long long clk(bool on) { return on ? clock64() : 0; }

struct Unit {
    int img, nt, row0, off0, f0, col0;
};

template <bool CTA2>
__device__ __forceinline__ Unit unit_of(const WinParams& p, int u, uint32_t rank) {
    Unit t;
    uint32_t rest, nt, g, j;
    p.d_ntiles.divmod(static_cast<uint32_t>(u), rest, nt);
    p.d_tiles.divmod(rest, g, j);
    t.nt = static_cast<int>(nt);
    t.img = CTA2 ? 2 * static_cast<int>(g) + static_cast<int>(rank) : static_cast<int>(g);
    if (p.rect) {  // window origin at the tile's (row, column) corner; GEMM rows start at its offset 0
        uint32_t rb, cb;
        p.d_cb.divmod(j, rb, cb);
        t.row0 = static_cast<int>(rb) * p.th;
        t.col0 = static_cast<int>(cb) * p.tw;
        t.off0 = 0;
        t.f0 = 0;
        return t;
    }
    t.f0 = static_cast<int>(j) * BM;
    uint32_t r0, o0;
    p.d_wp.divmod(static_cast<uint32_t>(t.f0), r0, o0);
    t.row0 = static_cast<int>(r0);
    t.off0 = static_cast<int>(o0);
    t.col0 = 0;
    return t;
}

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

// One 32-column accumulator chunk of one output row: fused epilogue + bf16 store
// (instantiated per bias / residual / ReLU / mask combination).
template <bool kBias, bool kRes, bool kRelu, bool kMask>
__device__ __forceinline__ void store_chunk(const WinParams& p, size_t orow, int col0, const uint32_t (&acc)[32]) {
    const size_t base = orow * p.Ncol + col0;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out) + base;
    if (col0 + 32 <= p.Ncol) {
        uint4 rv[4], mv[4];
        if constexpr (kRes) {
#pragma unroll
            for (int g = 0; g < 4; ++g) rv[g] = __ldg(reinterpret_cast<const uint4*>(p.residual + base) + g);
        }
        if constexpr (kMask) {
#pragma unroll
            for (int g = 0; g < 4; ++g) mv[g] = __ldg(reinterpret_cast<const uint4*>(p.mask + base) + g);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(acc[8 * g + i]);
            if constexpr (kBias) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += __ldg(p.bias + col0 + 8 * g + i);
            }
            if constexpr (kRes) {
                float r[8];
                unpack8(rv[g], r);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += r[i];
            }
            if constexpr (kRelu) {
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
            }
            if constexpr (kMask) {
                float mk[8];
                unpack8(mv[g], mk);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = mk[i] > 0.f ? v[i] : 0.f;
            }
            reinterpret_cast<uint4*>(out)[g] = pack8(v);
        }
    } else {
        for (int i = 0; i < 32 && col0 + i < p.Ncol; ++i) {
            float x = __uint_as_float(acc[i]);
            if constexpr (kBias) x += p.bias[col0 + i];
            if constexpr (kRes) x += __bfloat162float(p.residual[base + i]);
            if constexpr (kRelu) x = fmaxf(x, 0.f);
            if (kMask && !(__bfloat162float(p.mask[base + i]) > 0.f)) x = 0.f;
            out[i] = __float2bfloat16_rn(x);
        }
    }
}

// Whole-warp variant for full 32-column chunks (out-of-range rows included,
// `valid` masks them): the warp's 32 rows x 64 B are staged in shared memory
// (16-byte units XOR-swizzled by row pair, conflict-free both ways) and stored
// 8 rows x 64 B per instruction: whole 32-byte sectors instead of 32 half-sector
// writes to 32 rows.
template <bool kBias, bool kRes, bool kRelu, bool kMask>
__device__ __forceinline__ void store_chunk_staged(const WinParams& p, size_t orow, int col0, const uint32_t (&acc)[32],
                                                   bool valid, uint8_t* stg) {
    const int lane = threadIdx.x & 31;
    const size_t base = orow * p.Ncol + col0;
    uint4 rv[4] = {}, mv[4] = {};
    if (valid) {
        if constexpr (kRes) {
#pragma unroll
            for (int g = 0; g < 4; ++g) rv[g] = __ldg(reinterpret_cast<const uint4*>(p.residual + base) + g);
        }
        if constexpr (kMask) {
#pragma unroll
            for (int g = 0; g < 4; ++g) mv[g] = __ldg(reinterpret_cast<const uint4*>(p.mask + base) + g);
        }
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        float v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(acc[8 * g + i]);
        if constexpr (kBias) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += __ldg(p.bias + col0 + 8 * g + i);
        }
        if constexpr (kRes) {
            float r[8];
            unpack8(rv[g], r);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += r[i];
        }
        if constexpr (kRelu) {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = fmaxf(v[i], 0.f);
        }
        if constexpr (kMask) {
            float mk[8];
            unpack8(mv[g], mk);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = mk[i] > 0.f ? v[i] : 0.f;
        }
        *reinterpret_cast<uint4*>(stg + lane * 64 + ((g ^ ((lane >> 1) & 3)) << 4)) = pack8(v);
    }
    __syncwarp();
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
    const int part = lane & 3;
#pragma unroll
    for (int it = 0; it < 4; ++it) {
        const int r = it * 8 + (lane >> 2);
        const unsigned long long rb = __shfl_sync(0xffffffffu, static_cast<unsigned long long>(base), r);
        const int ok = __shfl_sync(0xffffffffu, valid ? 1 : 0, r);
        const uint4 val = *reinterpret_cast<const uint4*>(stg + r * 64 + ((part ^ ((r >> 1) & 3)) << 4));
        if (ok) *reinterpret_cast<uint4*>(out + rb + part * 8) = val;
    }
    __syncwarp();  // the next chunk reuses the staging rows
}

template <int BN, bool CTA2, bool BRES, bool DGRAD>
__global__ void __launch_bounds__(kThreads, 1) conv_win_kernel(const __grid_constant__ WinParams p) {
    // this CTA's share of the B tile per (tap, slice): K-major rows (fwd) or 64-channel
    // MN-major boxes (dgrad); a pair splits the N columns
    constexpr uint32_t kBBytes = BN * 64 * 2 / (CTA2 ? 2 : 1);
    constexpr int kNB = DGRAD ? (BN / (CTA2 ? 2 : 1)) / 64 : 1;  // dgrad boxes per B tile
    const uint32_t rank = CTA2 ? ptx::cluster_ctarank() : 0u;
    const int unit0 = CTA2 ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int ustride = CTA2 ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t wfull[kMaxWin], wempty[kMaxWin], bfull[kMaxB], bempty[kMaxB];
    __shared__ uint64_t tfull[2], tempty[2], bres_bar;
    __shared__ uint32_t tmem_slot;

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int taps = p.R * p.S;
    constexpr uint32_t kTmemCols = 2 * BN;

    if (tid == 0) {
        for (int i = 0; i < p.win_stages; ++i) {
            ptx::mbar_init(&wfull[i], 1);
            ptx::mbar_init(&wempty[i], 1);
        }
        for (int i = 0; i < p.b_stages; ++i) {
            ptx::mbar_init(&bfull[i], 1);
            ptx::mbar_init(&bempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], (CTA2 ? 2 : 1) * kEpiThreads);
        }
        ptx::mbar_init(&bres_bar, 1);
        ptx::fence_mbarrier_init();
        ptx::tma_prefetch_desc(&p.tmap_win);
        ptx::tma_prefetch_desc(&p.tmap_b);
    }
    if (warp == kMmaWarp) {
        if constexpr (CTA2) ptx::tmem_alloc_2sm<kTmemCols>(&tmem_slot);
        else ptx::tmem_alloc<kTmemCols>(&tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t smem_base = ptx::smem_addr(smem);
    const uint32_t b_base = smem_base + p.win_stages * p.win_stride;

    if (warp == 0) {
        // ================================================ TMA producer ======
        if (tid == 0) {
            auto leader = [&](uint64_t* bar) {
                return CTA2 ? ptx::leader_addr(ptx::smem_addr(bar)) : ptx::smem_addr(bar);
            };
            // B box(es) of stencil tap `tap` (window order) and channel slice cs
            auto load_b = [&](uint32_t dst, uint64_t* bar, int tap, int cs, int nt) {
                const uint32_t bar_u = leader(bar);
                if constexpr (DGRAD) {
                    const int ti = tap / p.S, tj = tap - ti * p.S;
                    const int ft = (p.R - 1 - ti) * p.S + (p.S - 1 - tj);  // flipped filter tap
                    const int c0 = nt * BN + (CTA2 ? static_cast<int>(rank) * (BN / 2) : 0);
#pragma unroll
                    for (int j = 0; j < kNB; ++j) {
                        if constexpr (CTA2) ptx::tma_load_3d_2sm(dst + j * 8192, &p.tmap_b, bar_u, c0 + j * 64, ft, cs * 64);
                        else ptx::tma_load_3d(dst + j * 8192, &p.tmap_b, bar, c0 + j * 64, ft, cs * 64);
                    }
                } else {
                    const int kk = tap * p.slices * 64 + cs * 64;
                    const int r0 = nt * BN + (CTA2 ? static_cast<int>(rank) * (BN / 2) : 0);
                    if constexpr (CTA2) ptx::tma_load_2d_2sm(dst, &p.tmap_b, bar_u, kk, r0);
                    else ptx::tma_load_2d(dst, &p.tmap_b, bar, kk, r0);
                }
            };
            if constexpr (BRES) {
                // the whole B operand of the (single) N tile, once
                if (!CTA2 || rank == 0)
                    ptx::mbar_arrive_expect_tx(&bres_bar, (CTA2 ? 2u : 1u) * kBBytes * taps * p.slices);
                for (int cs = 0; cs < p.slices; ++cs)
                    for (int tap = 0; tap < taps; ++tap)
                        load_b(b_base + (cs * taps + tap) * kBBytes, &bres_bar, tap, cs, 0);
            }
            int ws = 0, bs = 0;
            uint32_t wph = 0, bph = 0;
            long long t_w = 0, t_b = 0, t0 = clk(p.dbg != nullptr);
            for (int u = unit0; u < p.units; u += ustride) {
                const Unit t = unit_of<CTA2>(p, u, rank);
                for (int cs = 0; cs < p.slices; ++cs) {
                    long long a = clk(p.dbg != nullptr);
                    ptx::mbar_wait(&wempty[ws], wph ^ 1);
                    t_w += clk(p.dbg != nullptr) - a;
                    const uint32_t wdst = smem_base + ws * p.win_stride;
                    if (!CTA2 || rank == 0) ptx::mbar_arrive_expect_tx(&wfull[ws], (CTA2 ? 2u : 1u) * p.win_bytes);
                    if constexpr (CTA2)
                        ptx::tma_load_4d_2sm(wdst, &p.tmap_win, leader(&wfull[ws]), cs * 64, t.col0 - p.pad_w,
                                             t.row0 - p.pad_h, t.img);
                    else
                        ptx::tma_load_4d(wdst, &p.tmap_win, &wfull[ws], cs * 64, t.col0 - p.pad_w, t.row0 - p.pad_h,
                                         t.img);
                    if (++ws == p.win_stages) {
                        ws = 0;
                        wph ^= 1;
                    }
                    if constexpr (!BRES) {
                        for (int tap = 0; tap < taps; ++tap) {
                            long long b = clk(p.dbg != nullptr);
                            ptx::mbar_wait(&bempty[bs], bph ^ 1);
                            t_b += clk(p.dbg != nullptr) - b;
                            if (!CTA2 || rank == 0) ptx::mbar_arrive_expect_tx(&bfull[bs], (CTA2 ? 2u : 1u) * kBBytes);
                            load_b(b_base + bs * kBBytes, &bfull[bs], tap, cs, t.nt);
                            if (++bs == p.b_stages) {
                                bs = 0;
                                bph ^= 1;
                            }
                        }
                    }
                }
            }
            if (p.dbg) {
                unsigned long long* d = p.dbg + blockIdx.x * 8;
                d[0] = clk(p.dbg != nullptr) - t0;
                d[1] = t_w;
                d[2] = t_b;
            }
        }
    } else if (warp == kMmaWarp) {
        // =============================================== MMA issuer ======
        // one thread runs the whole issue loop: descriptors advance by plain
        // 64-bit adds of the 16-byte start-address field (taps: Wp*8 per filter
        // row, 8 per column; k steps: 2 for K-major, 128 for MN-major B)
        constexpr uint32_t idesc = ptx::make_idesc(1, CTA2 ? 2 * BM : BM, BN, 0u, DGRAD ? 1u : 0u);
        constexpr uint64_t kBStep = DGRAD ? 128 : 2;
        if (!CTA2 || rank == 0) {  // the whole warp runs the loop; one elected lane issues
            if constexpr (BRES) {
                ptx::mbar_wait(&bres_bar, 0);
                ptx::tc_fence_after();
            }
            int ws = 0, bs = 0, it = 0;
            uint32_t wph = 0, bph = 0;
            const uint64_t row_step = static_cast<uint64_t>(p.Wp) * 8;
            long long m_t = 0, m_w = 0, m_b = 0, m0 = clk(p.dbg != nullptr);
            for (int u = unit0; u < p.units; u += ustride, ++it) {
                const Unit t = unit_of<CTA2>(p, u, rank);
                const int acc = it & 1;
                long long a = clk(p.dbg != nullptr);
                ptx::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
                m_t += clk(p.dbg != nullptr) - a;
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                uint32_t accum = 0;
                for (int cs = 0; cs < p.slices; ++cs) {
                    a = clk(p.dbg != nullptr);
                    ptx::mbar_wait(&wfull[ws], wph);
                    m_w += clk(p.dbg != nullptr) - a;
                    const uint64_t a0 = ptx::sw128_desc(smem_base + ws * p.win_stride + t.off0 * 128, 16, 1024);
                    const uint64_t bres0 = BRES ? ptx::sw128_desc(b_base + cs * taps * kBBytes, DGRAD ? 8192 : 16, 1024) : 0;
                    uint64_t a_row = a0;
                    int tap = 0;
                    for (int ti = 0; ti < p.R; ++ti, a_row += row_step) {
                        uint64_t ad = a_row;
                        for (int tj = 0; tj < p.S; ++tj, ++tap, ad += 8) {
                            uint64_t bd;
                            if constexpr (BRES) {
                                bd = bres0 + static_cast<uint64_t>(tap) * (kBBytes >> 4);
                            } else {
                                long long b = clk(p.dbg != nullptr);
                                ptx::mbar_wait(&bfull[bs], bph);
                                m_b += clk(p.dbg != nullptr) - b;
                                bd = ptx::sw128_desc(b_base + bs * kBBytes, DGRAD ? 8192 : 16, 1024);
                            }
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                if constexpr (CTA2) ptx::umma_f16_2sm_elect(d_tmem, ad + 2 * k, bd + kBStep * k, idesc, accum);
                                else ptx::umma_f16_elect(d_tmem, ad + 2 * k, bd + kBStep * k, idesc, accum);
                                accum = 1;
                            }
                            if constexpr (!BRES) {
                                if constexpr (CTA2) ptx::umma_commit_2sm_elect(&bempty[bs], 3);
                                else ptx::umma_commit_elect(&bempty[bs]);
                                if (++bs == p.b_stages) {
                                    bs = 0;
                                    bph ^= 1;
                                }
                            }
                        }
                    }
                    if constexpr (CTA2) ptx::umma_commit_2sm_elect(&wempty[ws], 3);
                    else ptx::umma_commit_elect(&wempty[ws]);
                    if (++ws == p.win_stages) {
                        ws = 0;
                        wph ^= 1;
                    }
                }
                if constexpr (CTA2) ptx::umma_commit_2sm_elect(&tfull[acc], 3);
                else ptx::umma_commit_elect(&tfull[acc]);
            }
            if (p.dbg && (tid & 31) == 0) {
                unsigned long long* d = p.dbg + blockIdx.x * 8;
                d[3] = clk(p.dbg != nullptr) - m0;
                d[4] = m_t;
                d[5] = m_w;
                d[6] = m_b;
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ================================================= epilogue ======
        const int quarter = warp & 3;
        const int half = (warp - 4) >> 2;
        constexpr int kChunks = BN / 32, kHalf = kChunks / 2;
        const int row = quarter * 32 + (tid & 31);
        int it = 0;
        long long e_wait = 0, e_start = clk(p.dbg != nullptr);
        for (int u = unit0; u < p.units; u += ustride, ++it) {
            const Unit t = unit_of<CTA2>(p, u, rank);
            const int acc = it & 1;
            uint32_t ho, wq;
            p.d_wp.divmod(static_cast<uint32_t>(t.f0 + row), ho, wq);
            bool inside = true;
            if (p.rect) {  // (ho, wq) within the tile's window plane
                inside = static_cast<int>(ho) < p.th && static_cast<int>(wq) < p.tw;
                ho += t.row0;
                wq += t.col0;
            }
            const bool valid = inside && t.img < p.n_img && static_cast<int>(ho) < p.Ho && static_cast<int>(wq) < p.Wo;
            const size_t orow = (static_cast<size_t>(t.img) * p.Ho + ho) * p.Wo + wq;
            long long e0 = clk(p.dbg != nullptr);
            ptx::mbar_wait(&tfull[acc], (it >> 1) & 1);
            if (p.dbg && tid == 128) e_wait += clk(p.dbg != nullptr) - e0;
            ptx::tc_fence_after();
#pragma unroll 1
            for (int c = half * kHalf; c < (half + 1) * kHalf; ++c) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c * 32, v);
                ptx::tmem_ld_wait();
                const int col0 = t.nt * BN + c * 32;
                if (p.stg_off && col0 + 32 <= p.Ncol) {
                    uint8_t* stg = smem + p.stg_off + (warp - 4) * 2048;
                    const int f = (p.bias ? 1 : 0) | (p.residual ? 2 : 0) | (p.relu ? 4 : 0) | (p.mask ? 8 : 0);
                    switch (f) {
#define TCB_WIN_EPI(F) \
    case F: store_chunk_staged<(F & 1) != 0, (F & 2) != 0, (F & 4) != 0, (F & 8) != 0>(p, orow, col0, v, valid, stg); break;
                        TCB_WIN_EPI(0) TCB_WIN_EPI(1) TCB_WIN_EPI(2) TCB_WIN_EPI(3)
                        TCB_WIN_EPI(4) TCB_WIN_EPI(5) TCB_WIN_EPI(6) TCB_WIN_EPI(7)
                        TCB_WIN_EPI(8) TCB_WIN_EPI(9) TCB_WIN_EPI(10) TCB_WIN_EPI(11)
                        TCB_WIN_EPI(12) TCB_WIN_EPI(13) TCB_WIN_EPI(14) TCB_WIN_EPI(15)
#undef TCB_WIN_EPI
                    }
                } else if (valid && col0 < p.Ncol) {
                    const int f = (p.bias ? 1 : 0) | (p.residual ? 2 : 0) | (p.relu ? 4 : 0) | (p.mask ? 8 : 0);
                    switch (f) {
#define TCB_WIN_EPI(F) \
    case F: store_chunk<(F & 1) != 0, (F & 2) != 0, (F & 4) != 0, (F & 8) != 0>(p, orow, col0, v); break;
                        TCB_WIN_EPI(0) TCB_WIN_EPI(1) TCB_WIN_EPI(2) TCB_WIN_EPI(3)
                        TCB_WIN_EPI(4) TCB_WIN_EPI(5) TCB_WIN_EPI(6) TCB_WIN_EPI(7)
                        TCB_WIN_EPI(8) TCB_WIN_EPI(9) TCB_WIN_EPI(10) TCB_WIN_EPI(11)
                        TCB_WIN_EPI(12) TCB_WIN_EPI(13) TCB_WIN_EPI(14) TCB_WIN_EPI(15)
#undef TCB_WIN_EPI
                    }
                }
            }
            ptx::tc_fence_before();
            if (CTA2 && rank != 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_addr(&tempty[acc]), 0));
            else ptx::mbar_arrive(&tempty[acc]);
        }
        if (p.dbg && tid == 128) p.dbg[blockIdx.x * 8 + 7] = (static_cast<unsigned long long>(clk(p.dbg != nullptr) - e_start) << 32) |
                                                            static_cast<unsigned long long>(e_wait & 0xffffffff);
    }

    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();
    else __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        if constexpr (CTA2) ptx::tmem_dealloc_2sm<kTmemCols>(tmem_base);
        else ptx::tmem_dealloc<kTmemCols>(tmem_base);
    }
}

// ---------------------------------------------------------------- host ----
struct WinPlan {
    bool use = false;
    int Ha, Wa, Ca, Ho, Wo, pad_h, pad_w, R, S, Ncol;
    int Wp, WR, tiles_img, slices, bn, n_tiles;
    int rect = 0, tw = 0, th = 0, cblocks = 0;
    bool cta2, bres;
    uint32_t win_bytes, win_stride, b_bytes;
    int win_stages, b_stages;
    size_t smem;
    uint32_t stg_off = 0;
};

int g_win_mode = -1;  // $TCB_WIN: 0 off, 1 on (default, N = 64 tiles), 2 every applicable geometry
unsigned long long* g_win_dbg = nullptr;  // role timing buffer, 8 x u64 per CTA (diagnostics)

bool win_enabled() {
    if (g_win_mode < 0) {
        const char* e = getenv("TCB_WIN");
        g_win_mode = (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;
    }
    return g_win_mode >= 1;
}

// mode: 0 fwd (activation x), 1 dgrad (activation dy).
WinPlan win_plan(const ConvGeom& g, int mode) {
    WinPlan q;
    if (!win_enabled() || g.stride_h != 1 || g.stride_w != 1 || g.r * g.s < 2) return q;
    if (mode == 0) {
        q.Ha = g.h; q.Wa = g.w; q.Ca = g.c; q.Ncol = g.k;
        q.Ho = g.ho(); q.Wo = g.wo();
        q.pad_h = g.pad_h; q.pad_w = g.pad_w;
    } else {
        q.Ha = g.ho(); q.Wa = g.wo(); q.Ca = g.k; q.Ncol = g.c;
        q.Ho = g.h; q.Wo = g.w;
        q.pad_h = g.r - 1 - g.pad_h; q.pad_w = g.s - 1 - g.pad_w;
        if (q.pad_h < 0 || q.pad_w < 0) return q;
    }
    q.R = g.r; q.S = g.s;
    if (q.Ca % 64 != 0 || q.Ncol % 8 != 0 || q.pad_h > 15 || q.pad_w > 15) return q;
    q.Wp = q.Wo + q.S - 1;
    if (q.Wp <= 64) {
        // rows a 128-position tile can touch: positions [off0, off0 + 127 + (R-1)*Wp + S-1]
        q.WR = (q.Wp - 1 + BM - 1 + (q.R - 1) * q.Wp + q.S - 1) / q.Wp + 1;
        q.tiles_img = (q.Ho * q.Wp + BM - 1) / BM;
    } else {
        // wide rows ($TCB_WIN_RECT=0 keeps them on the im2col path): rectangular tiles of th
        // rows x tw columns, the window {tw + S - 1 columns, th + R - 1 rows} at the tile's
        // corner, GEMM rows = the window plane's first th rows (S - 1 junk columns each);
        // tw minimises the tile count (one 128-row MMA tile each), then the window size
        static const int env_rect = [] { const char* e = getenv("TCB_WIN_RECT"); return e ? atoi(e) : 1; }();
        if (env_rect == 0) return q;
        long best = -1;
        for (int tw = std::max(8, q.S); tw + q.S - 1 <= BM; ++tw) {
            const int wp = tw + q.S - 1, th = BM / wp;
            if (th < 1) break;
            const long tiles = long((q.Ho + th - 1) / th) * ((q.Wo + tw - 1) / tw);
            const long cost = tiles * 4096 + long(th + q.R - 1) * wp;
            if (best < 0 || cost < best) {
                best = cost;
                q.tw = tw;
                q.th = th;
            }
        }
        if (best < 0) return q;
        q.rect = 1;
        q.Wp = q.tw + q.S - 1;
        q.WR = q.th + q.R - 1;
        q.cblocks = (q.Wo + q.tw - 1) / q.tw;
        q.tiles_img = ((q.Ho + q.th - 1) / q.th) * q.cblocks;
    }
    q.win_bytes = static_cast<uint32_t>(q.WR) * q.Wp * 128;
    if (q.WR > 256 || q.Wp > 256 || q.win_bytes > 64 * 1024) return q;
    q.win_stride = (q.win_bytes + 1023) / 1024 * 1024;
    q.slices = q.Ca / 64;
    q.bn = q.Ncol <= 64 ? 64 : q.Ncol <= 128 ? 128 : 256;
    if (q.rect && q.bn != 64) return q;  // rectangular tiles: validated for 64-wide single-CTA tiles only
    // Measured (scripts/win_ab2.sh, bs256): the window wins where the im2col path's
    // 64-column tiles re-read each input pixel per tap at a low MMA width (ResNet
    // stage 1: fwd 117 -> 77 us, dgrad 130 -> 78 us); with 128/256-column tiles the
    // im2col path is already MMA-paced and the window's junk columns cost more
    // (stage 2: 66 vs 68 us, stage 3: 45 vs 54 us). $TCB_WIN=2 forces it on for every
    // applicable geometry (tests).
    if (q.bn != 64 && g_win_mode != 2) return q;
    q.n_tiles = (q.Ncol + q.bn - 1) / q.bn;
    // CTA pairs (two images per unit): N split in halves; dgrad halves must be whole
    // 64-channel MN-major boxes
    static const int env_cta2 = [] { const char* e = getenv("TCB_WIN_CTA2"); return e ? atoi(e) : -1; }();
    static const int env_bres = [] { const char* e = getenv("TCB_WIN_BRES"); return e ? atoi(e) : -1; }();
    static const int env_wst = [] { const char* e = getenv("TCB_WIN_WSTAGES"); return e ? atoi(e) : 0; }();
    static const int env_bst = [] { const char* e = getenv("TCB_WIN_BSTAGES"); return e ? atoi(e) : 0; }();
    // CTA pairs measured slower at N = 64 (stage 1 fwd: 107 vs 77 us single)
    q.cta2 = g.n >= 2 && q.bn >= 128 && env_cta2 != 0 && !q.rect;
    q.b_bytes = static_cast<uint32_t>(q.bn) * 64 * 2 / (q.cta2 ? 2 : 1);
    const size_t b_all = size_t(q.b_bytes) * q.R * q.S * q.slices;
    q.bres = q.n_tiles == 1 && b_all <= 96 * 1024 && env_bres != 0;
    const size_t b_ring = q.bres ? b_all : 0;
    q.b_stages = q.bres ? 1 : 0;
    // window stages first (>= 2), then B stages (>= 3) with what is left
    // epilogue staging tiles ($TCB_WIN_STAGE=1; off by default: the 16 KB cost a
    // window stage and stage-1 fwd / dgrad measured 75.4 -> 77.7 / 75.9 -> 78.4 us,
    // unlike the register epilogue of conv_tc.cu where it pays)
    static const int env_stage = [] { const char* e = getenv("TCB_WIN_STAGE"); return e ? atoi(e) : 0; }();
    const size_t stg = env_stage ? 8 * 2048 : 0;
    const size_t cap = kSmemCap - stg;
    for (q.win_stages = env_wst > 1 ? std::min(env_wst, kMaxWin) : kMaxWin; q.win_stages >= 2; --q.win_stages) {
        const size_t wbytes = size_t(q.win_stages) * q.win_stride;
        if (q.bres) {
            if (wbytes + b_ring + 1024 <= cap) break;
        } else {
            const size_t left = cap - std::min(cap, wbytes + 1024);
            const int bst = static_cast<int>(std::min<size_t>(env_bst > 2 ? std::min(env_bst, kMaxB) : kMaxB,
                                                              left / q.b_bytes));
            if (bst >= 3) {
                q.b_stages = bst;
                break;
            }
        }
    }
    if (q.win_stages < 2) return q;
    q.smem = size_t(q.win_stages) * q.win_stride + (q.bres ? b_ring : size_t(q.b_stages) * q.b_bytes) + 1024;
    q.stg_off = stg ? static_cast<uint32_t>(q.smem - 1024) : 0;
    q.smem += stg;
    q.use = true;
    return q;
}

template <int BN, bool CTA2, bool BRES, bool DGRAD>
cudaError_t launch_win(WinParams& p, const WinPlan& q, cudaStream_t st) {
    auto kern = conv_win_kernel<BN, CTA2, BRES, DGRAD>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(q.smem));
    if (e != cudaSuccess) return e;
    const int sms = num_sms();
    const int grid = CTA2 ? 2 * std::min(p.units, sms / 2) : std::min(p.units, sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = q.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CTA2 ? 2 : 1;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CTA2 ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <bool DGRAD>
cudaError_t dispatch_win(WinParams& p, const WinPlan& q, cudaStream_t st) {
#define TCB_WIN_CASE(BN)                                                              \
    if (q.bn == BN) {                                                                 \
        if (q.cta2) return q.bres ? launch_win<BN, true, true, DGRAD>(p, q, st)       \
                                  : launch_win<BN, true, false, DGRAD>(p, q, st);     \
        return q.bres ? launch_win<BN, false, true, DGRAD>(p, q, st)                  \
                      : launch_win<BN, false, false, DGRAD>(p, q, st);                \
    }
    TCB_WIN_CASE(64)
    TCB_WIN_CASE(128)
    TCB_WIN_CASE(256)
#undef TCB_WIN_CASE
    return cudaErrorInvalidValue;
}

cudaError_t run_win(const ConvGeom& g, const WinPlan& q, bool dgrad, const void* act, const void* b,
                    const Epilogue& ep, void* out, cudaStream_t st) {
    WinParams p{};
    if (!make_tmap_window_bf16(&p.tmap_win, act, g.n, q.Ha, q.Wa, q.Ca, q.Wp, q.WR)) return cudaErrorInvalidValue;
    if (dgrad) {
        if (!make_tmap_filters_bf16(&p.tmap_b, b, g.k, size_t(g.r) * g.s, g.c)) return cudaErrorInvalidValue;
    } else if (!make_tmap_bf16_2d(&p.tmap_b, b, q.Ncol, size_t(g.r) * g.s * g.c, q.cta2 ? q.bn / 2 : q.bn)) {
        return cudaErrorInvalidValue;
    }
    p.n_img = g.n;
    p.Ho = q.Ho;
    p.Wo = q.Wo;
    p.pad_h = q.pad_h;
    p.pad_w = q.pad_w;
    p.R = q.R;
    p.S = q.S;
    p.Wp = q.Wp;
    p.tiles_img = q.tiles_img;
    p.rect = q.rect;
    p.tw = q.tw;
    p.th = q.th;
    p.d_cb = FastDiv(static_cast<uint32_t>(std::max(q.cblocks, 1)));
    p.slices = q.slices;
    p.Ncol = q.Ncol;
    p.n_tiles = q.n_tiles;
    const int groups = q.cta2 ? (g.n + 1) / 2 : g.n;
    p.units = groups * q.tiles_img * q.n_tiles;
    p.win_bytes = q.win_bytes;
    p.win_stride = q.win_stride;
    p.b_bytes = q.b_bytes;
    p.win_stages = q.win_stages;
    p.stg_off = q.stg_off;
    p.b_stages = q.b_stages;
    p.out = out;
    p.bias = ep.bias;
    p.residual = static_cast<const __nv_bfloat16*>(ep.residual);
    p.mask = static_cast<const __nv_bfloat16*>(ep.mask);
    p.relu = ep.relu ? 1 : 0;
    p.d_wp = FastDiv(static_cast<uint32_t>(q.Wp));
    p.d_tiles = FastDiv(static_cast<uint32_t>(q.tiles_img));
    p.d_ntiles = FastDiv(static_cast<uint32_t>(q.n_tiles));
    p.dbg = g_win_dbg;
    conv_tc_note_launch(ConvTcLaunchInfo{dgrad ? 1 : 0, 4, q.bn, 0, q.cta2 ? 1 : 0, 1, p.units,
                                         q.cta2 ? 2 * std::min(p.units, num_sms() / 2) : std::min(p.units, num_sms()),
                                         0, q.bres ? 1 : 0});
    return dgrad ? dispatch_win<true>(p, q, st) : dispatch_win<false>(p, q, st);
}

// ============================================================ wgrad ======
//
// Window weight gradient for stride-1 R x S convs: the reduction runs over
// the positions of the padded output plane (flat f = ho * Wp + wq, junk
// columns wq >= Wo carry dy = 0 because the dy window reads them out of
// bounds). A k-block is P = 256 consecutive positions; per k-block one TMA
// window of x rows per 64-channel slice and one window of dy rows per
// 64-channel slice of K. The GEMM runs swapped: M = (tap, channel) of the
// filter gradient, N = K, both operands MN-major straight out of the windows.
// One M = 128 tile is TWO tap-slices: M block 0 at the first tap's row offset
// and M block 1 at the second's, i.e. the UMMA descriptor's leading byte
// offset is the distance between the two taps' shifted windows (measured:
// scripts/probes/umma_mn_probe.cu). Every CTA accumulates all M tiles of its
// contiguous range of k-blocks in TMEM (M tiles x K columns <= 512) and writes
// one fp32 partial [K][R][S][C]; a fixed-order split reduction sums them.
constexpr int kWgMaxStages = 4;

// positions per k-block: 256 (16 MMA K-steps, 2 stages) or 128 (8 K-steps, more stages in the
// same shared memory); $TCB_WIN_WG_POS
int wg_positions() {
    static const int v = [] {
        const char* e = getenv("TCB_WIN_WG_POS");
        return (e && atoi(e) == 128) ? 128 : 256;
    }();
    return v;
}

struct WgParams {
    CUtensorMap tmap_x;   // x [N][H][W][C], box {64, Wp, WRx, 1}
    CUtensorMap tmap_dy;  // dy [N][Ho][Wo][K], box {64, Wp, WRd, 1}
    int n_img, Ho, Wo, pad_h, pad_w, R, S, C, K;
    int Wp, kb_img, kb_total, kb_per_cta;
    int slices, kslices, nq, mtiles;
    int mt0, mt1;  // the M tiles (tap-slice pairs) this launch accumulates (tap groups)
    uint32_t xwin_bytes, dywin_bytes, stage_bytes;  // smem strides (1 KB aligned)
    uint32_t tx_bytes;                              // bytes the TMA boxes of one stage deliver
    int stages;
    float* partial;  // [gridDim.x][K][R][S][C]
    FastDiv d_wp, d_kbimg;
};

template <int BN, int kWP>
__global__ void __launch_bounds__(kThreads, 1) conv_win_wgrad_kernel(const __grid_constant__ WgParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kWgMaxStages], empty[kWgMaxStages], done;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int taps = p.R * p.S;
    const int kb0 = blockIdx.x * p.kb_per_cta;
    const int kb1 = min(p.kb_total, kb0 + p.kb_per_cta);
    if (tid == 0) {
        for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(&done, 1);
        ptx::fence_mbarrier_init();
        ptx::tma_prefetch_desc(&p.tmap_x);
        ptx::tma_prefetch_desc(&p.tmap_dy);
    }
    if (warp == kMmaWarp) ptx::tmem_alloc<512>(&tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t sbase = ptx::smem_addr(smem);

    if (warp == 0) {
        if (tid == 0) {  // ------------------------------------------ producer
            int st = 0;
            uint32_t ph = 0;
            for (int kb = kb0; kb < kb1; ++kb) {
                uint32_t img, j;
                p.d_kbimg.divmod(static_cast<uint32_t>(kb), img, j);
                uint32_t row0, off0;
                p.d_wp.divmod(j * kWP, row0, off0);
                ptx::mbar_wait(&empty[st], ph ^ 1);
                ptx::mbar_arrive_expect_tx(&full[st], p.tx_bytes);
                const uint32_t base = sbase + st * p.stage_bytes;
                for (int cs = 0; cs < p.slices; ++cs)
                    ptx::tma_load_4d(base + cs * p.xwin_bytes, &p.tmap_x, &full[st], cs * 64, -p.pad_w,
                                     static_cast<int>(row0) - p.pad_h, static_cast<int>(img));
                for (int ks = 0; ks < p.kslices; ++ks)
                    ptx::tma_load_4d(base + p.slices * p.xwin_bytes + ks * p.dywin_bytes, &p.tmap_dy, &full[st],
                                     ks * 64, 0, static_cast<int>(row0), static_cast<int>(img));
                if (++st == p.stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == kMmaWarp) {  // ------------------------------- MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc(1, 128, BN, 1u, 1u);
        int st = 0;
        uint32_t ph = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            uint32_t img, j;
            p.d_kbimg.divmod(static_cast<uint32_t>(kb), img, j);
            uint32_t row0, off0;
            p.d_wp.divmod(j * kWP, row0, off0);
            ptx::mbar_wait(&full[st], ph);
            ptx::tc_fence_after();
            const uint32_t base = sbase + st * p.stage_bytes;
            const uint32_t dyb = base + p.slices * p.xwin_bytes + off0 * 128;
            const uint64_t bd0 = ptx::sw128_desc(dyb, p.dywin_bytes, 1024);
            // tap-slice q (slice-major): address of its shifted window
            auto qaddr = [&](int q) {
                const int cs = q / taps, t = q - cs * taps;
                const int ti = t / p.S, tj = t - ti * p.S;
                return base + cs * p.xwin_bytes + (off0 + ti * p.Wp + tj) * 128;
            };
            for (int mt = p.mt0; mt < p.mt1; ++mt) {
                const int q0 = 2 * mt, q1 = min(2 * mt + 1, p.nq - 1);
                const uint32_t a0 = qaddr(q0);
                const uint64_t ad0 = ptx::sw128_desc(a0, qaddr(q1) - a0, 1024);
                const uint32_t first = kb > kb0 ? 1u : 0u;
                ptx::umma_f16_elect(tmem + (mt - p.mt0) * BN, ad0, bd0, idesc, first);
#pragma unroll
                for (int ks = 1; ks < kWP / 16; ++ks)  // compile-time descriptor offsets
                    ptx::umma_f16_elect(tmem + (mt - p.mt0) * BN, ad0 + ks * 128, bd0 + ks * 128, idesc, 1u);
            }
            ptx::umma_commit_elect(&empty[st]);
            if (++st == p.stages) {
                st = 0;
                ph ^= 1;
            }
        }
        ptx::umma_commit_elect(&done);
    } else if (warp >= 4) {  // ------------------------------------- epilogue
        const int quarter = warp & 3, half = (warp - 4) >> 2;
        const int lane = tid & 31;
        const int m = quarter * 32 + lane;  // row within an M tile
        float* part = p.partial + size_t(blockIdx.x) * p.K * taps * p.C;
        const bool any = kb1 > kb0;
        if (any) {
            ptx::mbar_wait(&done, 0);
            ptx::tc_fence_after();
        }
        for (int mt = p.mt0; mt < p.mt1; ++mt) {
            const int blk = m >> 6, q = 2 * mt + blk;
            const bool live = q < p.nq && !(blk == 1 && 2 * mt + 1 >= p.nq);
            const int cs = q / taps, t = q - cs * taps, c = cs * 64 + (m & 63);
#pragma unroll 1
            for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
                uint32_t v[32];
                if (any) {
                    ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + (mt - p.mt0) * BN + c0, v);
                    ptx::tmem_ld_wait();
                }
                if (!live) continue;
                for (int i = 0; i < 32 && c0 + i < p.K; ++i)
                    part[(size_t(c0 + i) * taps + t) * p.C + c] = any ? __uint_as_float(v[i]) : 0.f;
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

struct WgPlan {
    bool use = false;
    int Wp, WRx, WRd, slices, kslices, nq, mtiles, bn, kb_img, kb_total, grid, kb_per_cta, stages, groups, per_group;
    int wpos;
    uint32_t xwin, dywin, stage, tx;
    size_t smem, partial_bytes;
};

WgPlan wgrad_plan(const ConvGeom& g) {
    WgPlan q;
    if (!win_enabled() || g.stride_h != 1 || g.stride_w != 1 || g.r * g.s < 2) return q;
    if (g.c % 64 != 0 || g.k % 64 != 0 || g.pad_h > 15 || g.pad_w > 15) return q;
    const int Ho = g.ho(), Wo = g.wo();
    q.Wp = Wo + g.s - 1;
    if (q.Wp > 64 || q.Wp < 16) return q;
    q.slices = g.c / 64;
    q.kslices = g.k / 64;
    q.bn = g.k;
    // default: where the im2col path has 64-row tiles (K = 64). (K = 128 as three tap groups
    // measured 172 us against 100 us for the im2col path on ResNet stage 2: $TCB_WIN=2 only.)
    if (q.bn != 64 && g_win_mode != 2) return q;
    q.nq = g.r * g.s * q.slices;
    q.mtiles = (q.nq + 1) / 2;
    if (q.bn > 256) return q;
    // M tiles beyond 512 TMEM columns run as tap groups: one launch per group over the same
    // windows (balanced: ceil(mtiles / groups) tiles each)
    const int fit = 512 / q.bn;  // M tiles whose accumulators fit the 512 TMEM columns
    q.groups = (q.mtiles + fit - 1) / fit;
    q.per_group = (q.mtiles + q.groups - 1) / q.groups;  // balanced, <= fit
    if (q.groups > 3) return q;
    q.wpos = wg_positions();
    const int kWP = q.wpos;
    q.WRx = (q.Wp - 1 + kWP - 1 + (g.r - 1) * q.Wp + g.s - 1) / q.Wp + 1;
    q.WRd = (q.Wp - 1 + kWP - 1) / q.Wp + 1;
    if (q.WRx > 256) return q;
    q.xwin = (static_cast<uint32_t>(q.WRx) * q.Wp * 128 + 1023) / 1024 * 1024;
    q.dywin = (static_cast<uint32_t>(q.WRd) * q.Wp * 128 + 1023) / 1024 * 1024;
    q.stage = q.slices * q.xwin + q.kslices * q.dywin;
    q.tx = static_cast<uint32_t>(q.slices * q.WRx + q.kslices * q.WRd) * q.Wp * 128;
    if (size_t(q.stage) + 1024 > kSmemCap) return q;
    q.stages = static_cast<int>(std::min<size_t>(kWgMaxStages, (kSmemCap - 1024) / q.stage));
    q.smem = size_t(q.stages) * q.stage + 1024;
    q.kb_img = (Ho * q.Wp + kWP - 1) / kWP;
    q.kb_total = g.n * q.kb_img;
    q.grid = std::min(q.kb_total, num_sms());
    q.kb_per_cta = (q.kb_total + q.grid - 1) / q.grid;
    q.grid = (q.kb_total + q.kb_per_cta - 1) / q.kb_per_cta;
    q.partial_bytes = size_t(q.grid) * g.k * g.r * g.s * g.c * sizeof(float);
    q.use = true;
    return q;
}

template <int BN>
cudaError_t launch_wgrad(const WgParams& p, const WgPlan& q, cudaStream_t st) {
    auto kern = q.wpos == 128 ? conv_win_wgrad_kernel<BN, 128> : conv_win_wgrad_kernel<BN, 256>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(q.smem));
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(q.grid), dim3(kThreads), q.smem, st, p);
}

}  // namespace

bool conv_win_wgrad_applies(const ConvGeom& g) { return wgrad_plan(g).use; }
int conv_win_wgrad_launches(const ConvGeom& g) { return wgrad_plan(g).groups + 1; }

size_t conv_win_wgrad_workspace(const ConvGeom& g) {
    const WgPlan q = wgrad_plan(g);
    return q.use ? q.partial_bytes : 0;
}

cudaError_t conv_win_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw, void* workspace,
                           cudaStream_t st) {
    const WgPlan q = wgrad_plan(g);
    if (!q.use || workspace == nullptr) return cudaErrorInvalidValue;
    WgParams p{};
    if (!make_tmap_window_bf16(&p.tmap_x, x, g.n, g.h, g.w, g.c, q.Wp, q.WRx)) return cudaErrorInvalidValue;
    if (!make_tmap_window_bf16(&p.tmap_dy, dy, g.n, g.ho(), g.wo(), g.k, q.Wp, q.WRd)) return cudaErrorInvalidValue;
    p.n_img = g.n;
    p.Ho = g.ho();
    p.Wo = g.wo();
    p.pad_h = g.pad_h;
    p.pad_w = g.pad_w;
    p.R = g.r;
    p.S = g.s;
    p.C = g.c;
    p.K = g.k;
    p.Wp = q.Wp;
    p.kb_img = q.kb_img;
    p.kb_total = q.kb_total;
    p.kb_per_cta = q.kb_per_cta;
    p.slices = q.slices;
    p.kslices = q.kslices;
    p.nq = q.nq;
    p.mtiles = q.mtiles;
    p.mt0 = 0;
    p.mt1 = q.mtiles;
    p.xwin_bytes = q.xwin;
    p.dywin_bytes = q.dywin;
    p.stage_bytes = q.stage;
    p.tx_bytes = q.tx;
    p.stages = q.stages;
    p.partial = static_cast<float*>(workspace);
    p.d_wp = FastDiv(static_cast<uint32_t>(q.Wp));
    p.d_kbimg = FastDiv(static_cast<uint32_t>(q.kb_img));
    conv_tc_note_launch(ConvTcLaunchInfo{2, 4, q.bn, 0, 0, q.grid, q.kb_total, q.grid, 0, 0});
    cudaError_t e = cudaSuccess;
    for (int gi = 0; gi < q.groups && e == cudaSuccess; ++gi) {
        p.mt0 = gi * q.per_group;
        p.mt1 = std::min(q.mtiles, p.mt0 + q.per_group);
        switch (q.bn) {
            case 64: e = launch_wgrad<64>(p, q, st); break;
            case 128: e = launch_wgrad<128>(p, q, st); break;
            case 192: e = launch_wgrad<192>(p, q, st); break;
            case 256: e = launch_wgrad<256>(p, q, st); break;
            default: return cudaErrorInvalidValue;
        }
    }
    if (e != cudaSuccess) return e;
    return split_reduce(static_cast<const float*>(workspace), q.grid, size_t(g.k) * g.r * g.s * g.c, dw, st);
}

void conv_win_set_mode(int on) { g_win_mode = on < 0 ? -1 : on; }
void conv_win_set_debug(void* buf) { g_win_dbg = static_cast<unsigned long long*>(buf); }

bool conv_win_applies(const ConvGeom& g, ConvMode mode) {
    return mode != ConvMode::Wgrad && win_plan(g, mode == ConvMode::Fwd ? 0 : 1).use;
}

cudaError_t conv_win_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep, void* y,
                         cudaStream_t st) {
    const WinPlan q = win_plan(g, 0);
    if (!q.use) return cudaErrorInvalidValue;
    return run_win(g, q, false, x, w, ep, y, st);
}

cudaError_t conv_win_dgrad(const ConvGeom& g, const void* dy, const void* w, const Epilogue& ep, void* dx,
                           cudaStream_t st) {
    const WinPlan q = win_plan(g, 1);
    if (!q.use) return cudaErrorInvalidValue;
    return run_win(g, q, true, dy, w, ep, dx, st);
}

}  // namespace tcb
