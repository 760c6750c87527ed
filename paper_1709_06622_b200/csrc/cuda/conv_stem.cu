// Row-window convolution for the narrow RGB stem (sm_100a): ResNet's 7x7/2
// conv1, Inception's 3x3/2 -- stride-2 first layers over <= 4 real channels
// (R in {3, 5, 7, 11}, K in {32, 64, 128}).
//
// The explicit-im2col path (conv_tc.cu, narrow_plan) writes a 1.2 GB patch
// matrix for the ResNet-50 bs256 stem and reads it back twice (fwd GEMM and
// wgrad GEMM): 335 + 249 + 291 us of the 12 ms step, all HBM time. Here the
// patch matrix is never materialised. The input is stored once more as a
// "stem row" tensor x4[n][h][u][4] (4 bf16 channels = 8 bytes per pixel, the
// conv's left padding as zero columns u < pad_w, zero columns up to Wst, a
// multiple of 16 pixels), written by the executor's uint8 input preparation.
// Output pixel (ho, wo) reads, per filter row r, the 8 stored pixels
// u = 2wo .. 2wo + 7 of input row 2ho - pad_h + r: 32 contiguous bf16 = one
// K-chunk holding filter columns s = 0..7 (s >= S weighted by zero; S > 8
// takes nq = 2 chunks per filter row).
//
//   fwd   : per output row, the R stored rows (one TMA box of 16-pixel groups
//           each, no swizzle). Consecutive positions start 16 bytes apart, so
//           a no-swizzle K-major descriptor with LBO 16 / SBO 128 (8-row x
//           16-byte core matrices overlapping each other) IS the row's im2col
//           window: D[wo][k] = sum_r A_r * Wp_r^T, M = 128 rows (BW <= 128
//           valid), N = K, 2 MMAs per filter row with compile-time descriptor
//           offsets (the N = 64 MMAs are issue-bound), packed weights resident
//           (SW64); bias / ReLU epilogue through a swizzled staging tile and a
//           TMA store. Warp 0 TMA, warp 1 MMA, warps 2-9 epilogue from four
//           TMEM accumulators. Variants: CTA pairs ($TCB_STEM_CTA2) and the
//           following 3x3/2/1 max pool fused into the epilogue (config
//           fuse_stem_pool) -- both correct and both measured slower.
//   wgrad : D[(r, e)][k] = sum over positions of window^T * dy. The windows are
//           overlapping-row TMA boxes {32 el, BW, 1, 1} of a map whose row
//           stride (16 bytes) is smaller than its 64-byte inner extent, 64-byte
//           swizzled, used as MN-major A operands (4 filter rows per M = 128
//           tile, one box apart = the descriptor's leading byte offset); dy
//           boxes {K, BW} are the MN-major B. Two output rows per tile share
//           their R - 2 common input rows (9 boxes instead of 14 for 7x7).
//           Every CTA accumulates its contiguous range of rows in TMEM and
//           writes one fp32 partial; a fixed-order reduction sums the partials
//           and scatters into dw[K][R][S][C] (zero on padded c, s).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "ptx.cuh"
#include "tma.cuh"

namespace tcb {
namespace {

constexpr int kThreads = 10 * 32;  // warp 0 TMA, warp 1 MMA, warps 2-9 epilogue
constexpr int kMaxStages = 12;
constexpr uint32_t kRowStride = 2176;  // fwd row buffer: 17 groups of 16 pixels, or 128 positions + 2 chunks
constexpr size_t kSmemCap = 227 * 1024 - 2048;

// K-major / MN-major 64-byte swizzle descriptor (layout type 4).
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(4) << 61;  // SWIZZLE_64B
    return d;
}

struct StemParams {
    CUtensorMap tmap_x;   // fwd: x4 rows {64, Wst/16, H, N}, box {64, G, 1, 1} (no swizzle);
                          // wgrad: x4 windows {32, D1, H, N}, box {32, BW, 1, 1} (64-byte swizzle)
    CUtensorMap tmap_b;   // fwd: packed weights [K][T*32], box {32, K}; wgrad: dy {K, Wo, N*Ho}, box {min(K,64), BW, 1}
    CUtensorMap tmap_y;   // fwd: y {K, Wo, N*Ho}, box {min(K,64), BW, 1} (TMA store)
    int Ho, Wo, K, T, nq, chunk_step, sh, pad_h, BW, wtiles, tiles;
    uint32_t box_bytes, stage_bytes, b_bytes;
    int stages;
    // fwd
    int R, G, g_step;     // filter rows; 16-pixel groups per row box; groups per width tile
    uint32_t row_stride, stg_bytes;
    const float* bias;
    int relu;
    int dbg;              // diagnostics ($TCB_STEM_DBG): 1 no MMA, 2 no output stores, 4 no x loads
    // fused 3x3 / 2 / 1 max pool (conv_stem_fwd_pool_kernel)
    __nv_bfloat16* pool_y;
    uint8_t* pool_arg;
    int Po, Pw, pool_rows, pool_per_cta;
    // wgrad
    int mtiles, tiles_per_cta, dy_boxes, tr;  // tr: output rows per weight-gradient tile (1 or 2)
    uint32_t dy_box_bytes, xslots;
    float* partial;  // [grid][T*32][K]
    FastDiv d_wtiles, d_ho;
};

struct Tile {
    int n, ho, wo0;
};

__device__ __forceinline__ Tile tile_of(const StemParams& p, int u) {
    uint32_t row, wt, n, ho;
    p.d_wtiles.divmod(static_cast<uint32_t>(u), row, wt);
    p.d_ho.divmod(row, n, ho);
    return Tile{static_cast<int>(n), static_cast<int>(ho), static_cast<int>(wt) * p.BW};
}

// weight-gradient tile of tr whole output rows (one width tile per row)
__device__ __forceinline__ Tile row_tile(const StemParams& p, int u) {
    uint32_t n, ho;
    p.d_ho.divmod(static_cast<uint32_t>(u * p.tr), n, ho);
    return Tile{static_cast<int>(n), static_cast<int>(ho), 0};
}

__device__ __forceinline__ void load_x(const StemParams& p, uint32_t dst, uint64_t* bar, const Tile& t) {
    const int h0 = t.ho * p.sh - p.pad_h;
    for (int c = 0; c < p.T; ++c) {
        const int r = c / p.nq, q = c - r * p.nq;
        ptx::tma_load_4d(dst + c * p.box_bytes, &p.tmap_x, bar, 0, t.wo0 + q * p.chunk_step, h0 + r, t.n);
    }
}

__device__ __forceinline__ uint4 pack8f(const float (&f)[8]) {
    uint4 v;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return v;
}

// No-swizzle ("interleaved") K-major descriptor over a raw stem row: position m
// of the tile starts 16 bytes after position m - 1 (stride 2 x 4 channels x
// 2 bytes), so the 8-row x 16-byte core matrices along M are contiguous (SBO =
// 128) and the second 8-element K group of a row is the next row's first
// (LBO = 16): the overlapping windows are a descriptor, not a copy.
__device__ __forceinline__ uint64_t rows_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;  // LBO 16 B
    d |= static_cast<uint64_t>(8) << 32;  // SBO 128 B
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}

// 16-byte chunk j of staging row m under the TMA store's swizzle
__device__ __forceinline__ uint32_t stg_off(int m, int j, int row_bytes) {
    return row_bytes == 128 ? m * 128 + ((j ^ (m & 7)) << 4) : m * 64 + ((j ^ ((m >> 1) & 3)) << 4);
}

// CTA2: a cluster pair runs M = 256 MMAs (tcgen05 cta_group::2) over two consecutive tiles, one
// per CTA; each CTA holds its own A rows and half of the weight rows, so one MMA instruction
// serves two SMs ($TCB_STEM_CTA2=1; measured slower at N = 64, see stem_fwd host code).
template <int BN, int R, int NQ, bool CTA2 = false>
__global__ void __launch_bounds__(kThreads, 1) conv_stem_fwd_kernel(const __grid_constant__ StemParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kAcc = BN <= 64 ? 4 : 2;  // TMEM accumulators in flight
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull[kAcc], tempty[kAcc], bbar;
    __shared__ uint32_t tmem_slot;
    constexpr uint32_t kCols = kAcc * BN <= 64 ? 64 : kAcc * BN <= 128 ? 128 : 256;
    constexpr int kBox = BN >= 64 ? 64 : BN;          // output channels per store box
    constexpr int kRowB = kBox * 2;                   // staging row bytes (128 or 64)
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t rank = CTA2 ? ptx::cluster_ctarank() : 0u;
    const int unit0 = CTA2 ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int ustride = CTA2 ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
    const int units = CTA2 ? (p.tiles + 1) / 2 : p.tiles;
    constexpr uint32_t kBHalf = CTA2 ? 2u : 1u;  // this CTA's share of the weight rows
    if (tid == 0) {
        for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], (CTA2 ? 2 : 1) * 8 * 32);
        }
        ptx::mbar_init(&bbar, 1);
        ptx::fence_mbarrier_init();
        ptx::tma_prefetch_desc(&p.tmap_x);
        ptx::tma_prefetch_desc(&p.tmap_b);
        ptx::tma_prefetch_desc(&p.tmap_y);
    }
    if (warp == 1) {
        if constexpr (CTA2) ptx::tmem_alloc_2sm<kCols>(&tmem_slot);
        else ptx::tmem_alloc<kCols>(&tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t sbase = ptx::smem_addr(smem);
    const uint32_t bbase = sbase + p.stages * p.stage_bytes;
    const uint32_t bchunk = p.b_bytes / kBHalf;          // one filter row's weight slice in smem
    const uint32_t stg = bbase + p.T * p.b_bytes;  // 2 staging tiles of the output
    auto leader = [&](uint64_t* bar) {
        return CTA2 ? ptx::leader_addr(ptx::smem_addr(bar)) : ptx::smem_addr(bar);
    };

    if (warp == 0) {
        if (tid == 0) {  // ---------------------------------------- producer
            if (!CTA2 || rank == 0) ptx::mbar_arrive_expect_tx(&bbar, p.T * p.b_bytes);
            for (int c = 0; c < p.T; ++c) {
                if constexpr (CTA2)
                    ptx::tma_load_2d_2sm(bbase + c * bchunk, &p.tmap_b, leader(&bbar), c * 32,
                                         static_cast<int>(rank) * (BN / 2));
                else
                    ptx::tma_load_2d(bbase + c * bchunk, &p.tmap_b, &bbar, c * 32, 0);
            }
            int st = 0;
            uint32_t ph = 0;
            for (int u = unit0; u < units; u += ustride) {
                const int tile = CTA2 ? min(2 * u + static_cast<int>(rank), p.tiles - 1) : u;
                const Tile t = tile_of(p, tile);
                ptx::mbar_wait(&empty[st], ph ^ 1);
                const uint32_t dst = sbase + st * p.stage_bytes;
                const int h0 = t.ho * p.sh - p.pad_h, g0 = (t.wo0 / p.BW) * p.g_step;
                if (!CTA2 || rank == 0) ptx::mbar_arrive_expect_tx(&full[st], kBHalf * R * p.G * 128);
                for (int r = 0; r < R; ++r) {
                    if constexpr (CTA2)
                        ptx::tma_load_4d_2sm(dst + r * kRowStride, &p.tmap_x, leader(&full[st]), 0, g0, h0 + r, t.n);
                    else
                        ptx::tma_load_4d(dst + r * kRowStride, &p.tmap_x, &full[st], 0, g0, h0 + r, t.n);
                }
                if (++st == p.stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------------ MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc(1, CTA2 ? 256 : 128, BN, 0u, 0u);
        if (!CTA2 || rank == 0) {
        ptx::mbar_wait(&bbar, 0);
        ptx::tc_fence_after();
        int st = 0, it = 0;
        uint32_t ph = 0;
        for (int u = unit0; u < units; u += ustride, ++it) {
            const int acc = it % kAcc;
            ptx::mbar_wait(&tempty[acc], ((it / kAcc) & 1) ^ 1);
            ptx::mbar_wait(&full[st], ph);
            ptx::tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            // compile-time descriptor offsets: filter row r at r * kRowStride, chunk q 64 bytes on,
            // K step 32 bytes; packed weight chunk (r, q) BN * 64 bytes apart
            const uint64_t a0 = rows_desc(sbase + st * p.stage_bytes);
            const uint64_t b0 = sw64_desc(bbase, 16, 512);
#pragma unroll
            for (int r = 0; r < R; ++r) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const uint64_t ad = a0 + ((r * kRowStride + q * 64) >> 4);
                    const uint64_t bd = b0 + (((r * NQ + q) * (BN / kBHalf) * 64) >> 4);
                    if constexpr (CTA2) {
                        ptx::umma_f16_2sm_elect(d, ad, bd, idesc, (r | q) ? 1u : 0u);
                        ptx::umma_f16_2sm_elect(d, ad + 2, bd + 2, idesc, 1u);
                    } else {
                        ptx::umma_f16_elect(d, ad, bd, idesc, (r | q) ? 1u : 0u);
                        ptx::umma_f16_elect(d, ad + 2, bd + 2, idesc, 1u);
                    }
                }
            }
            if constexpr (CTA2) {
                ptx::umma_commit_2sm_elect(&empty[st], 3);
                ptx::umma_commit_2sm_elect(&tfull[acc], 3);
            } else {
                ptx::umma_commit_elect(&empty[st]);
                ptx::umma_commit_elect(&tfull[acc]);
            }
            if (++st == p.stages) {
                st = 0;
                ph ^= 1;
            }
        }
        }
        __syncwarp();
    } else {  // ------------------------------------------------------ epilogue
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const int row = quarter * 32 + (tid & 31);
        const bool store_lead = tid == 64;
        int it = 0;
        for (int u = unit0; u < units; u += ustride, ++it) {
            const int tile = CTA2 ? 2 * u + static_cast<int>(rank) : u;
            const bool live = tile < p.tiles;
            const Tile t = tile_of(p, live ? tile : p.tiles - 1);
            const int acc = it % kAcc;
            ptx::mbar_wait(&tfull[acc], (it / kAcc) & 1);
            ptx::tc_fence_after();
            constexpr int kChunks = (BN + 63) / 64;  // 32-column chunks per half
            uint32_t v[kChunks][32];
#pragma unroll
            for (int ch = 0; ch < kChunks; ++ch) {
                const int c0 = half * 32 + ch * 64;
                if (c0 < BN && !(p.dbg & 8)) ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c0, v[ch]);
            }
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            if (CTA2 && rank != 0) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_addr(&tempty[acc]), 0));
            else ptx::mbar_arrive(&tempty[acc]);
            // staging tile acc is free once the store issued two tiles ago has read it
            if (store_lead) ptx::bulk_wait_read<1>();
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const uint32_t sb = stg + (it & 1) * p.stg_bytes;
            if (row < p.BW && live && !(p.dbg & 2)) {
#pragma unroll
                for (int ch = 0; ch < kChunks; ++ch) {
                    const int c0 = half * 32 + ch * 64;
                    if (c0 >= BN) break;
                    const int box = c0 / kBox, j0 = (c0 % kBox) / 8;
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        float f[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            float x = __uint_as_float(v[ch][8 * g + i]);
                            if (p.bias) x += __ldg(p.bias + c0 + 8 * g + i);
                            f[i] = p.relu ? fmaxf(x, 0.f) : x;
                        }
                        const uint4 w = pack8f(f);
                        const uint32_t a = sb + box * (p.BW * kRowB) + stg_off(row, j0 + g, kRowB);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w.x), "r"(w.y),
                                     "r"(w.z), "r"(w.w)
                                     : "memory");
                    }
                }
            }
            ptx::fence_proxy_async_smem();
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (store_lead && live && !(p.dbg & 2)) {
                for (int b = 0; b < (BN + kBox - 1) / kBox; ++b)
                    asm volatile(
                        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                            &p.tmap_y),
                        "r"(sb + b * (p.BW * kRowB)), "r"(b * kBox), "r"(t.wo0), "r"(t.n * p.Ho + t.ho)
                        : "memory");
                ptx::bulk_commit();
            }
        }
        if (store_lead) ptx::bulk_wait<0>();
    }
    ptx::tc_fence_before();
    if constexpr (CTA2) ptx::cluster_sync();  // the leader's MMAs read the follower's smem
    else __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (CTA2) ptx::tmem_dealloc_2sm<kCols>(tmem);
        else ptx::tmem_dealloc<kCols>(tmem);
    }
}

// Stem rows a CTA computes for its contiguous range of pooled rows [q, q1) (flattened
// (image, pooled row)): pooled row p reads stem rows 2p-1..2p+1, rows are emitted once in
// increasing order (the first pooled row of a range recomputes its row 2p-1, which the
// neighbouring CTA also writes -- the same values), and the emission of row min(2p+1, Ho-1)
// completes pooled row p.
struct PoolSeq {
    int q, q1, k, last;
    __device__ PoolSeq(int q0, int qe) : q(q0), q1(qe), k(0), last(-1) {}
    __device__ bool next(const StemParams& p, int& n, int& ho, int& done_q) {
        while (q < q1) {
            const int img = q / p.Po, pr = q - img * p.Po;
            const int hlast = min(2 * pr + 1, p.Ho - 1);
            while (k < 3) {
                const int h = 2 * pr - 1 + k;
                ++k;
                if (h < 0 || h >= p.Ho) continue;
                const int flat = img * p.Ho + h;
                if (flat <= last) continue;
                last = flat;
                n = img;
                ho = h;
                done_q = h == hlast ? q : -1;
                if (h == hlast) {
                    ++q;
                    k = 0;
                }
                return true;
            }
            ++q;
            k = 0;
        }
        return false;
    }
};

// The stem forward fused with the 3x3 / stride 2 / pad 1 max pool that follows it (ResNet):
// the ReLU'd stem rows pass through four swizzled staging tiles on their way to the TMA
// store, and whenever a row completes a pooled row the epilogue warps pool the three staged
// rows straight from shared memory -- the separate pool kernel's 411 MB re-read of the stem
// output is gone. Same max / first-maximum tie rule / argmax code as maxpool_fwd. BN = 64,
// one width tile per row.
template <int R>
__global__ void __launch_bounds__(kThreads, 1) conv_stem_fwd_pool_kernel(const __grid_constant__ StemParams p) {
    constexpr int BN = 64;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kAcc = 4;
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages], tfull[kAcc], tempty[kAcc], bbar;
    __shared__ uint32_t tmem_slot;
    constexpr uint32_t kCols = kAcc * BN;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int q0 = blockIdx.x * p.pool_per_cta, q1 = min(p.pool_rows, q0 + p.pool_per_cta);
    if (tid == 0) {
        for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < kAcc; ++i) {
            ptx::mbar_init(&tfull[i], 1);
            ptx::mbar_init(&tempty[i], 8 * 32);
        }
        ptx::mbar_init(&bbar, 1);
        ptx::fence_mbarrier_init();
        ptx::tma_prefetch_desc(&p.tmap_x);
        ptx::tma_prefetch_desc(&p.tmap_b);
        ptx::tma_prefetch_desc(&p.tmap_y);
    }
    if (warp == 1) ptx::tmem_alloc<kCols>(&tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t sbase = ptx::smem_addr(smem);
    const uint32_t bbase = sbase + p.stages * p.stage_bytes;
    const uint32_t stg = bbase + R * p.b_bytes;  // 4 staging tiles: the TMA store and the pool both read them

    if (warp == 0) {
        if (tid == 0) {  // ---------------------------------------- producer
            ptx::mbar_arrive_expect_tx(&bbar, R * p.b_bytes);
            for (int c = 0; c < R; ++c) ptx::tma_load_2d(bbase + c * p.b_bytes, &p.tmap_b, &bbar, c * 32, 0);
            int st = 0;
            uint32_t ph = 0;
            PoolSeq seq(q0, q1);
            int n, ho, dq;
            while (seq.next(p, n, ho, dq)) {
                ptx::mbar_wait(&empty[st], ph ^ 1);
                const uint32_t dst = sbase + st * p.stage_bytes;
                const int h0 = ho * p.sh - p.pad_h;
                ptx::mbar_arrive_expect_tx(&full[st], R * p.G * 128);
                for (int r = 0; r < R; ++r)
                    ptx::tma_load_4d(dst + r * kRowStride, &p.tmap_x, &full[st], 0, 0, h0 + r, n);
                if (++st == p.stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------------ MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc(1, 128, BN, 0u, 0u);
        ptx::mbar_wait(&bbar, 0);
        ptx::tc_fence_after();
        int st = 0, it = 0;
        uint32_t ph = 0;
        PoolSeq seq(q0, q1);
        int n, ho, dq;
        while (seq.next(p, n, ho, dq)) {
            const int acc = it % kAcc;
            ptx::mbar_wait(&tempty[acc], ((it / kAcc) & 1) ^ 1);
            ptx::mbar_wait(&full[st], ph);
            ptx::tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            const uint64_t a0 = rows_desc(sbase + st * p.stage_bytes);
            const uint64_t b0 = sw64_desc(bbase, 16, 512);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint64_t ad = a0 + ((r * kRowStride) >> 4);
                const uint64_t bd = b0 + ((r * BN * 64) >> 4);
                ptx::umma_f16_elect(d, ad, bd, idesc, r ? 1u : 0u);
                ptx::umma_f16_elect(d, ad + 2, bd + 2, idesc, 1u);
            }
            ptx::umma_commit_elect(&empty[st]);
            ptx::umma_commit_elect(&tfull[acc]);
            if (++st == p.stages) {
                st = 0;
                ph ^= 1;
            }
            ++it;
        }
        __syncwarp();
    } else {  // ------------------------------------------------------ epilogue
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const int row = quarter * 32 + (tid & 31);
        const int et = tid - 64;  // 0..255
        const bool store_lead = et == 0;
        int it = 0;
        PoolSeq seq(q0, q1);
        int n, ho, dq;
        while (seq.next(p, n, ho, dq)) {
            const int acc = it % kAcc;
            ptx::mbar_wait(&tfull[acc], (it / kAcc) & 1);
            ptx::tc_fence_after();
            uint32_t v[32];
            ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + half * 32, v);
            ptx::tmem_ld_wait();
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
            // staging tile it & 3 is free once the store issued four rows ago has read it
            if (store_lead) ptx::bulk_wait_read<3>();
            asm volatile("bar.sync 1, 256;" ::: "memory");
            const uint32_t sb = stg + (it & 3) * p.stg_bytes;
            if (row < p.BW) {
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    float f[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float x = __uint_as_float(v[8 * g + i]);
                        if (p.bias) x += __ldg(p.bias + half * 32 + 8 * g + i);
                        f[i] = p.relu ? fmaxf(x, 0.f) : x;
                    }
                    const uint4 w = pack8f(f);
                    const uint32_t a = sb + stg_off(row, half * 4 + g, 128);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w.x), "r"(w.y), "r"(w.z),
                                 "r"(w.w)
                                 : "memory");
                }
            }
            ptx::fence_proxy_async_smem();
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (store_lead) {
                asm volatile(
                    "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                        &p.tmap_y),
                    "r"(sb), "r"(0), "r"(0), "r"(n * p.Ho + ho)
                    : "memory");
                ptx::bulk_commit();
            }
            if (dq >= 0) {
                // pooled row pr of image n from staged stem rows 2pr-1 .. 2pr+1 (tiles it - (ho - h))
                const int pr = dq - n * p.Po;
                const size_t obase = (size_t(n) * p.Po + pr) * p.Pw * BN;
                for (int item = et; item < p.Pw * 8; item += 256) {
                    const int pw = item >> 3, cg = item & 7;
                    __nv_bfloat162 best[4];
                    uint32_t idx[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        best[j] = __halves2bfloat162(__ushort_as_bfloat16(0xFF80u), __ushort_as_bfloat16(0xFF80u));
                        idx[j] = 0;
                    }
#pragma unroll
                    for (int t = 0; t < 9; ++t) {
                        const int h = 2 * pr - 1 + t / 3, w = 2 * pw - 1 + t % 3;
                        if (h < 0 || h >= p.Ho || w < 0 || w >= p.Wo) continue;
                        const uint32_t tile = stg + ((it - (ho - h)) & 3) * p.stg_bytes;
                        uint4 vv;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(vv.x), "=r"(vv.y), "=r"(vv.z), "=r"(vv.w)
                                     : "r"(tile + stg_off(w, cg, 128)));
                        const uint32_t code = static_cast<uint32_t>(t) * 0x00010001u;
                        const uint32_t vw[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162*>(&vw[j]);
                            const uint32_t gt = __hgt2_mask(b, best[j]);
                            best[j] = __hmax2(best[j], b);
                            idx[j] = (idx[j] & ~gt) | (code & gt);
                        }
                    }
                    const size_t o = obase + size_t(pw) * BN + cg * 8;
                    uint4 out;
                    out.x = *reinterpret_cast<uint32_t*>(&best[0]);
                    out.y = *reinterpret_cast<uint32_t*>(&best[1]);
                    out.z = *reinterpret_cast<uint32_t*>(&best[2]);
                    out.w = *reinterpret_cast<uint32_t*>(&best[3]);
                    *reinterpret_cast<uint4*>(p.pool_y + o) = out;
                    *reinterpret_cast<uint2*>(p.pool_arg + o) =
                        make_uint2(__byte_perm(idx[0], idx[1], 0x6420), __byte_perm(idx[2], idx[3], 0x6420));
                }
            }
            ++it;
        }
        if (store_lead) ptx::bulk_wait<0>();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<kCols>(tmem);
    }
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1) conv_stem_wgrad_kernel(const __grid_constant__ StemParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages], done;
    __shared__ uint32_t tmem_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int u0 = blockIdx.x * p.tiles_per_cta;
    const int u1 = min(p.tiles, u0 + p.tiles_per_cta);
    if (tid == 0) {
        for (int i = 0; i < p.stages; ++i) {
            ptx::mbar_init(&full[i], 1);
            ptx::mbar_init(&empty[i], 1);
        }
        ptx::mbar_init(&done, 1);
        ptx::fence_mbarrier_init();
        ptx::tma_prefetch_desc(&p.tmap_x);
        ptx::tma_prefetch_desc(&p.tmap_b);
    }
    if (warp == 1) ptx::tmem_alloc<512>(&tmem_slot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_slot;
    ptx::griddep_wait();
    ptx::griddep_launch_dependents();
    const uint32_t sbase = ptx::smem_addr(smem);
    const uint32_t xslots = p.xslots;

    if (warp == 0) {
        if (tid == 0) {  // ---------------------------------------- producer
            int st = 0;
            uint32_t ph = 0;
            for (int u = u0; u < u1; ++u) {
                const Tile t = p.tr == 1 ? tile_of(p, u) : row_tile(p, u);
                ptx::mbar_wait(&empty[st], ph ^ 1);
                const int nbox = p.tr == 1 ? p.T : p.T + p.sh * (p.tr - 1);
                ptx::mbar_arrive_expect_tx(&full[st], nbox * p.box_bytes + p.tr * p.dy_boxes * p.dy_box_bytes);
                const uint32_t base = sbase + st * p.stage_bytes;
                if (p.tr == 1) {
                    load_x(p, base, &full[st], t);
                } else {  // nq = 1: the R + sh (tr - 1) input rows the tile's output rows share
                    const int h0 = t.ho * p.sh - p.pad_h;
                    for (int c = 0; c < nbox; ++c)
                        ptx::tma_load_4d(base + c * p.box_bytes, &p.tmap_x, &full[st], 0, t.wo0, h0 + c, t.n);
                }
                for (int r = 0; r < p.tr; ++r)
                    for (int j = 0; j < p.dy_boxes; ++j)
                        ptx::tma_load_3d(base + xslots + (r * p.dy_boxes + j) * p.dy_box_bytes, &p.tmap_b,
                                         &full[st], j * 64, t.wo0, t.n * p.Ho + t.ho + r);
                if (++st == p.stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------------ MMA issuer
        constexpr uint32_t idesc = ptx::make_idesc(1, 128, BN, 1u, 1u);
        // dy rows: BN * 2 bytes; 128-byte swizzle (64-channel boxes, LBO apart) or 64-byte (BN = 32)
        constexpr bool kDy128 = BN >= 64;
        constexpr uint32_t kDyRow = kDy128 ? 128 : 64;
        const int ksteps = p.BW / 16;
        int st = 0;
        uint32_t ph = 0;
        for (int u = u0; u < u1; ++u) {
            ptx::mbar_wait(&full[st], ph);
            ptx::tc_fence_after();
            const uint32_t base = sbase + st * p.stage_bytes;
            for (int r = 0; r < p.tr; ++r) {  // output row r of the tile: input rows from box sh * r
                const uint32_t dyb = base + xslots + r * p.dy_boxes * p.dy_box_bytes;
                const uint64_t bd0 = kDy128 ? ptx::sw128_desc(dyb, p.dy_box_bytes, 8 * kDyRow)
                                            : sw64_desc(dyb, p.dy_box_bytes, 8 * kDyRow);
                for (int mt = 0; mt < p.mtiles; ++mt) {
                    const uint64_t ad0 = sw64_desc(base + (r * p.sh + mt * 4) * p.box_bytes, p.box_bytes, 512);
                    const uint32_t acc0 = (u > u0 || r > 0) ? 1u : 0u;
#pragma unroll
                    for (int ks = 0; ks < 8; ++ks) {  // compile-time descriptor offsets, BW / 16 <= 8 steps
                        if (ks >= ksteps) break;
                        ptx::umma_f16_elect(tmem + mt * BN, ad0 + ks * 64, bd0 + ks * (16 * kDyRow >> 4), idesc,
                                            ks > 0 ? 1u : acc0);
                    }
                }
            }
            ptx::umma_commit_elect(&empty[st]);
            if (++st == p.stages) {
                st = 0;
                ph ^= 1;
            }
        }
        ptx::umma_commit_elect(&done);
        __syncwarp();
    } else if (warp < 6) {  // ----------------------------------------- epilogue
        const int quarter = warp & 3;
        const int m = quarter * 32 + (tid & 31);
        const bool any = u1 > u0;
        const int rows = p.T * 32;
        float* part = p.partial + size_t(blockIdx.x) * rows * p.K;
        if (any) {
            ptx::mbar_wait(&done, 0);
            ptx::tc_fence_after();
        }
        for (int mt = 0; mt < p.mtiles; ++mt) {
            const int grow = mt * 128 + m;
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t v[32];
                if (any) {
                    ptx::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + mt * BN + c0, v);
                    ptx::tmem_ld_wait();
                }
                if (grow >= rows) continue;
                float4* dst = reinterpret_cast<float4*>(part + size_t(grow) * p.K + c0);
#pragma unroll
                for (int g = 0; g < 8; ++g)
                    dst[g] = any ? make_float4(__uint_as_float(v[4 * g]), __uint_as_float(v[4 * g + 1]),
                                               __uint_as_float(v[4 * g + 2]), __uint_as_float(v[4 * g + 3]))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<512>(tmem);
    }
}

// x [N][H][W][C] (C = 8, cv real) -> x4 [N][H][Wst][4], zero columns around
__global__ void stem_pack_kernel(const uint4* __restrict__ x, uint2* __restrict__ x4, int H, int W, int Wst,
                                 int pad_w, int cv, size_t total) {
    pdl_wait();
    pdl_trigger();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int u = static_cast<int>(i % Wst);
        const size_t row = i / Wst;
        const int w = u - pad_w;
        uint2 v = make_uint2(0, 0);
        if (w >= 0 && w < W) {
            const uint4 p = __ldg(x + row * W + w);
            v = make_uint2(p.x, p.y);
            if (cv < 4) v.y &= cv < 3 ? 0u : 0xFFFFu;  // channels >= cv are zero already; keep it exact
            if (cv < 2) v.x &= 0xFFFFu;
        }
        x4[i] = v;
    }
}

// uint8 RGB pixels -> (u + 0.5) / 128 - 1 (the executor's input preparation,
// pack_channels_u8) written straight into x4 (zero padding columns) and, when
// x8 is given, into the 8-channel activation as well: the stem input costs one
// pass over the uint8 batch instead of a pack plus a repack.
__global__ void stem_pack_u8_kernel(const uint8_t* __restrict__ src, uint2* __restrict__ x4,
                                    uint4* __restrict__ x8, int W, int Wst, int pad_w, int cl, size_t total) {
    pdl_wait();
    pdl_trigger();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const int u = static_cast<int>(i % Wst);
        const size_t row = i / Wst;
        const int w = u - pad_w;
        __align__(16) __nv_bfloat16 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = __float2bfloat16(0.f);
        if (w >= 0 && w < W) {
            const uint8_t* px = src + (row * W + w) * cl;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < cl) v[c] = __float2bfloat16_rn(__fsub_rn(__fmul_rn(float(__ldg(px + c)) + 0.5f, 0.0078125f), 1.f));
            if (x8) x8[row * W + w] = *reinterpret_cast<const uint4*>(v);
        }
        x4[i] = *reinterpret_cast<const uint2*>(v);
    }
}

// w [K][R][S][C] -> wp [K][T][32]: chunk (r, q), element e = s_local * 4 + c
__global__ void stem_pack_weights(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wp, int K,
                                  int R, int S, int C, int cv, int nq) {
    pdl_wait();
    pdl_trigger();
    const int T = R * nq, total = K * T * 32;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int e = i & 31, kt = i >> 5;
        const int t = kt % T, k = kt / T;
        const int r = t / nq, q = t - r * nq;
        const int s = q * 8 + (e >> 2), c = e & 3;
        wp[i] = (s < S && c < cv) ? w[((size_t(k) * R + r) * S + s) * C + c] : __float2bfloat16(0.f);
    }
}

// dw[k][r][s][c] = sum over the grid's partials [g][(r, q, e)][K], zero where c >= cv
__global__ void stem_reduce_scatter(const float* __restrict__ part, int parts, float* __restrict__ dw, int K,
                                    int R, int S, int C, int cv, int nq) {
    pdl_wait();
    pdl_trigger();
    const int total = K * R * S * C;
    const size_t pstride = size_t(R) * nq * 32 * K;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int c = i % C, rest = i / C;
        const int s = rest % S, kr = rest / S;
        const int r = kr % R, k = kr / R;
        float acc = 0.f;
        if (c < cv) {
            const size_t row = (size_t(r) * nq + s / 8) * 32 + (s % 8) * 4 + c;
            const float* src = part + row * K + k;
            for (int g = 0; g < parts; ++g) acc += __ldg(src + g * pstride);
        }
        dw[i] = acc;
    }
}

struct StemPlan {
    bool use = false;
    int cv, nq, T, Wst, D1, BW, wtiles, tiles, Ho, Wo, chunk_step;
    uint32_t box_bytes, b_bytes, stage_bytes, row_stride, stg_bytes;
    int stages, G, g_step;
    size_t smem, x4_bytes, wp_bytes;
    // wgrad
    int mtiles, dy_boxes, grid_wg, tiles_per_cta, wg_stages, tr, wg_tiles;
    uint32_t dy_box_bytes, wg_stage_bytes, xslots;
    size_t wg_smem, partial_bytes;
};

int g_stem_mode = -1;  // $TCB_STEM: 0 off (explicit im2col), 1 on

bool stem_enabled() {
    if (g_stem_mode < 0) {
        const char* e = getenv("TCB_STEM");
        g_stem_mode = (e && e[0] == '0') ? 0 : 1;
    }
    return g_stem_mode == 1;
}

size_t a256(size_t b) { return (b + 255) & ~size_t(255); }

StemPlan stem_plan(const ConvGeom& g) {
    StemPlan q;
    if (!stem_enabled()) return q;
    q.cv = g.c_valid > 0 ? g.c_valid : g.c;
    // stride 2: consecutive output positions 16 bytes apart in a 4-channel row (the forward
    // descriptor's core-matrix row pitch)
    if (g.c != 8 || q.cv > 4 || g.r * g.s < 2 || g.stride_w != 2) return q;
    if (g.k != 32 && g.k != 64 && g.k != 128) return q;  // N of both GEMMs; dy boxes of 32 or 64 channels
    q.nq = (g.s + 7) / 8;
    q.chunk_step = 8 / g.stride_w;
    q.T = g.r * q.nq;
    q.Ho = g.ho();
    q.Wo = g.wo();
    q.Wst = std::max(g.w + g.pad_w, (q.Wo - 1) * g.stride_w + 8 * q.nq);
    q.Wst = (q.Wst + 15) / 16 * 16;  // whole 16-pixel (128-byte) groups per stored row
    q.D1 = (q.Wst - 8) / g.stride_w + 1;
    q.BW = std::min((std::min(q.Wo, 128) + 15) / 16 * 16, 128);
    q.wtiles = (q.Wo + q.BW - 1) / q.BW;
    q.tiles = g.n * q.Ho * q.wtiles;
    q.box_bytes = static_cast<uint32_t>(q.BW) * 64;
    q.b_bytes = static_cast<uint32_t>(g.k) * 64;
    q.x4_bytes = size_t(g.n) * g.h * q.Wst * 8;
    q.wp_bytes = size_t(g.k) * q.T * 64;
    // fwd: per stage the R stored rows a width tile reads (G 16-pixel groups each, row buffers
    // long enough for the M = 128 descriptor's last window), packed weights resident, two
    // output staging tiles for the TMA store
    q.G = ((q.BW - 1) * 2 + 8 * q.nq + 15) / 16;
    q.g_step = q.BW / 8;
    q.row_stride = kRowStride;
    if (static_cast<uint32_t>(std::max(q.G * 128, 16 * 128 + 64 * q.nq)) > kRowStride) return q;
    // compiled (R, chunks) variants of the forward kernel
    if (!((g.r == 7 && q.nq == 1) || (g.r == 3 && q.nq == 1) || (g.r == 5 && q.nq == 1) || (g.r == 11 && q.nq == 2)))
        return q;
    q.stage_bytes = (g.r * q.row_stride + 1023) / 1024 * 1024;
    q.stg_bytes = (static_cast<uint32_t>(q.BW) * g.k * 2 + 1023) / 1024 * 1024;
    const size_t fixed = size_t(q.T) * q.b_bytes + 2 * size_t(q.stg_bytes) + 1024;
    for (q.stages = kMaxStages; q.stages >= 2; --q.stages)
        if (size_t(q.stages) * q.stage_bytes + fixed <= kSmemCap) break;
    if (q.stages < 2) return q;
    q.smem = size_t(q.stages) * q.stage_bytes + fixed;
    // wgrad: M tiles of 4 chunks; dy boxes of 64 channels (128-byte rows) or one 32-channel box
    q.mtiles = (q.T + 3) / 4;
    if (q.mtiles * g.k > 512 || (g.k != 32 && g.k % 64 != 0)) return q;
    q.dy_boxes = g.k >= 64 ? g.k / 64 : 1;
    q.dy_box_bytes = static_cast<uint32_t>(q.BW) * (g.k >= 64 ? 128 : 64);
    // two output rows per tile share R - stride of their R input rows: 9 boxes instead of 14 for
    // the ResNet stem ($TCB_STEM_WG_ROWS=1 keeps one row per tile)
    static const int env_rows = [] { const char* e = getenv("TCB_STEM_WG_ROWS"); return e ? atoi(e) : 2; }();
    for (q.tr = (env_rows >= 2 && q.wtiles == 1 && q.nq == 1 && q.Ho % 2 == 0) ? 2 : 1; q.tr >= 1; --q.tr) {
        q.xslots = static_cast<uint32_t>(q.mtiles * 4 + g.stride_h * (q.tr - 1)) * q.box_bytes;
        q.wg_stage_bytes = (q.xslots + q.tr * q.dy_boxes * q.dy_box_bytes + 1023) / 1024 * 1024;
        for (q.wg_stages = kMaxStages; q.wg_stages >= 2; --q.wg_stages)
            if (size_t(q.wg_stages) * q.wg_stage_bytes + 1024 <= kSmemCap) break;
        if (q.wg_stages >= 2) break;
    }
    if (q.tr < 1) return q;
    q.wg_smem = size_t(q.wg_stages) * q.wg_stage_bytes + 1024;
    q.wg_tiles = q.tiles / q.tr;
    q.grid_wg = std::min(q.wg_tiles, num_sms());
    q.tiles_per_cta = (q.wg_tiles + q.grid_wg - 1) / q.grid_wg;
    q.grid_wg = (q.wg_tiles + q.tiles_per_cta - 1) / q.tiles_per_cta;
    q.partial_bytes = size_t(q.grid_wg) * q.T * 32 * g.k * sizeof(float);
    q.use = true;
    return q;
}

bool make_x4_map(CUtensorMap* m, const void* x4, const ConvGeom& g, const StemPlan& q) {
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return false;
    const cuuint64_t dims[4] = {32, cuuint64_t(q.D1), cuuint64_t(g.h), cuuint64_t(g.n)};
    const cuuint64_t strides[3] = {cuuint64_t(g.stride_w) * 8, cuuint64_t(q.Wst) * 8, cuuint64_t(q.Wst) * 8 * g.h};
    const cuuint32_t box[4] = {32, cuuint32_t(q.BW), 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x4), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void fill_common(StemParams& p, const ConvGeom& g, const StemPlan& q) {
    p.Ho = q.Ho;
    p.Wo = q.Wo;
    p.K = g.k;
    p.T = q.T;
    p.nq = q.nq;
    p.chunk_step = q.chunk_step;
    p.sh = g.stride_h;
    p.pad_h = g.pad_h;
    p.BW = q.BW;
    p.wtiles = q.wtiles;
    p.tiles = q.tiles;
    p.box_bytes = q.box_bytes;
    p.d_wtiles = FastDiv(static_cast<uint32_t>(q.wtiles));
    p.d_ho = FastDiv(static_cast<uint32_t>(q.Ho));
}

template <typename K>
cudaError_t launch_pair(K kern, dim3 grid, size_t smem, cudaStream_t st, const StemParams& p) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

template <typename K>
cudaError_t launch_big(K kern, dim3 grid, size_t smem, cudaStream_t st, const StemParams& p) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, grid, dim3(kThreads), smem, st, p);
}

cudaError_t stem_pack(const ConvGeom& g, const StemPlan& q, const void* x, void* x4, cudaStream_t st) {
    const size_t total = size_t(g.n) * g.h * q.Wst;
    const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, size_t(num_sms()) * 16));
    return launch_pdl(stem_pack_kernel, dim3(grid), dim3(256), 0, st, static_cast<const uint4*>(x),
                      static_cast<uint2*>(x4), g.h, g.w, q.Wst, g.pad_w, q.cv, total);
}

}  // namespace

bool conv_stem_applies(const ConvGeom& g) { return stem_plan(g).use; }

bool conv_stem_pool_fusable(const ConvGeom& g) {
    static const int env_cta2 = [] { const char* e = getenv("TCB_STEM_CTA2"); return e ? atoi(e) : 0; }();
    const StemPlan q = stem_plan(g);
    return q.use && g.k == 64 && q.wtiles == 1 && q.nq == 1 && (g.r == 3 || g.r == 5 || g.r == 7) && env_cta2 == 0;
}

cudaError_t conv_stem_pack_input(const ConvGeom& g, const void* x, void* workspace, cudaStream_t st) {
    const StemPlan q = stem_plan(g);
    if (!q.use || workspace == nullptr) return cudaErrorInvalidValue;
    return stem_pack(g, q, x, workspace, st);
}

cudaError_t conv_stem_pack_u8(const ConvGeom& g, const uint8_t* src, int cl, void* x8, void* workspace,
                              cudaStream_t st) {
    const StemPlan q = stem_plan(g);
    if (!q.use || workspace == nullptr || cl < 1 || cl > q.cv) return cudaErrorInvalidValue;
    const size_t total = size_t(g.n) * g.h * q.Wst;
    const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, size_t(num_sms()) * 16));
    return launch_pdl(stem_pack_u8_kernel, dim3(grid), dim3(256), 0, st, src, static_cast<uint2*>(workspace),
                      static_cast<uint4*>(x8), g.w, q.Wst, g.pad_w, cl, total);
}
void conv_stem_set_mode(int on) { g_stem_mode = on < 0 ? -1 : (on ? 1 : 0); }

size_t conv_stem_workspace(const ConvGeom& g) {
    const StemPlan q = stem_plan(g);
    if (!q.use) return 0;
    return a256(q.x4_bytes) + std::max(a256(q.wp_bytes), a256(q.partial_bytes));
}

int conv_stem_launches(const ConvGeom& g, ConvMode mode, bool x_ready) {
    (void)g;
    if (mode == ConvMode::Fwd) return x_ready ? 2 : 3;
    return x_ready ? 2 : 3;
}

cudaError_t conv_stem_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep, void* y,
                          void* workspace, cudaStream_t st, bool x_ready) {
    const StemPlan q = stem_plan(g);
    if (!q.use || workspace == nullptr || ep.residual || ep.mask) return cudaErrorInvalidValue;
    char* ws = static_cast<char*>(workspace);
    void* x4 = ws;
    auto* wp = reinterpret_cast<__nv_bfloat16*>(ws + a256(q.x4_bytes));
    cudaError_t e = x_ready ? cudaSuccess : stem_pack(g, q, x, x4, st);
    if (e != cudaSuccess) return e;
    const int wtotal = g.k * q.T * 32;
    e = launch_pdl(stem_pack_weights, dim3(std::max(1, std::min(wtotal / 256 + 1, 512))), dim3(256), 0, st,
                   static_cast<const __nv_bfloat16*>(w), wp, g.k, g.r, g.s, g.c, q.cv, q.nq);
    if (e != cudaSuccess) return e;
    StemParams p{};
    EncodeTiledFn fn = encode_tiled_fn();
    if (!fn) return cudaErrorInvalidValue;
    {  // stored rows in 16-pixel groups, no swizzle
        const cuuint64_t dims[4] = {64, cuuint64_t(q.Wst / 16), cuuint64_t(g.h), cuuint64_t(g.n)};
        const cuuint64_t strides[3] = {128, cuuint64_t(q.Wst) * 8, cuuint64_t(q.Wst) * 8 * g.h};
        const cuuint32_t box[4] = {64, cuuint32_t(q.G), 1, 1};
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        if (fn(&p.tmap_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x4, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {  // y [N*Ho][Wo][K] stores, 64-channel (128-byte swizzle) or 32-channel (64-byte) boxes
        const cuuint64_t dims[3] = {cuuint64_t(g.k), cuuint64_t(q.Wo), cuuint64_t(g.n) * q.Ho};
        const cuuint64_t strides[2] = {cuuint64_t(g.k) * 2, cuuint64_t(q.Wo) * g.k * 2};
        const cuuint32_t box[3] = {cuuint32_t(std::min(g.k, 64)), cuuint32_t(q.BW), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (fn(&p.tmap_y, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, g.k >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    // CTA pairs ($TCB_STEM_CTA2=1): M = 256 MMAs over two output rows, half the weight rows per
    // CTA. Correct, but measured 0.37 vs 0.22 ms for the ResNet stem (N = 64 pairs lose, as in
    // conv_win), so off by default.
    static const int env_cta2 = [] { const char* e = getenv("TCB_STEM_CTA2"); return e ? atoi(e) : 0; }();
    const bool cta2 = env_cta2 != 0 && q.tiles >= 2;
    if (!make_tmap_bf16_2d(&p.tmap_b, wp, g.k, size_t(q.T) * 32, cta2 ? g.k / 2 : g.k, 32,
                           CU_TENSOR_MAP_SWIZZLE_64B))
        return cudaErrorInvalidValue;
    fill_common(p, g, q);
    p.stage_bytes = q.stage_bytes;
    p.b_bytes = q.b_bytes;
    p.stages = q.stages;
    p.R = g.r;
    p.G = q.G;
    p.g_step = q.g_step;
    p.row_stride = q.row_stride;
    p.stg_bytes = q.stg_bytes;
    p.bias = ep.bias;
    p.relu = ep.relu ? 1 : 0;
    static const int env_dbg = [] { const char* e = getenv("TCB_STEM_DBG"); return e ? atoi(e) : 0; }();
    p.dbg = env_dbg;
    if (ep.pool_y) {  // fused 3x3 / 2 / 1 max pool
        if (g.k != 64 || q.wtiles != 1 || q.nq != 1 || !ep.pool_arg || cta2) return cudaErrorInvalidValue;
        p.pool_y = static_cast<__nv_bfloat16*>(ep.pool_y);
        p.pool_arg = ep.pool_arg;
        p.Po = (q.Ho - 1) / 2 + 1;
        p.Pw = (q.Wo - 1) / 2 + 1;
        p.pool_rows = g.n * p.Po;
        const size_t psmem = size_t(q.stages) * q.stage_bytes + size_t(q.T) * q.b_bytes + 4 * size_t(q.stg_bytes) + 1024;
        int stages = q.stages;
        size_t smem = psmem;
        while (smem > kSmemCap && stages > 2) {
            --stages;
            smem = size_t(stages) * q.stage_bytes + size_t(q.T) * q.b_bytes + 4 * size_t(q.stg_bytes) + 1024;
        }
        if (smem > kSmemCap) return cudaErrorInvalidValue;
        p.stages = stages;
        const int pgrid = std::min(p.pool_rows, num_sms());
        p.pool_per_cta = (p.pool_rows + pgrid - 1) / pgrid;
        const int grid2 = (p.pool_rows + p.pool_per_cta - 1) / p.pool_per_cta;
        conv_tc_note_launch(ConvTcLaunchInfo{0, 5, g.k, 4, 0, 1, p.pool_rows, grid2, 0, 1});
        switch (g.r) {
            case 7: return launch_big(conv_stem_fwd_pool_kernel<7>, dim3(grid2), smem, st, p);
            case 5: return launch_big(conv_stem_fwd_pool_kernel<5>, dim3(grid2), smem, st, p);
            case 3: return launch_big(conv_stem_fwd_pool_kernel<3>, dim3(grid2), smem, st, p);
            default: return cudaErrorInvalidValue;
        }
    }
    const int grid = cta2 ? 2 * std::min((q.tiles + 1) / 2, num_sms() / 2) : std::min(q.tiles, num_sms());
    conv_tc_note_launch(ConvTcLaunchInfo{0, 5, g.k, 0, cta2 ? 1 : 0, 1, q.tiles, grid, 0, 1});
#define TCB_STEM_FWD(BN, R, NQ)                                                                         \
    if (g.k == BN && g.r == R && q.nq == NQ)                                                           \
        return cta2 ? launch_pair(conv_stem_fwd_kernel<BN, R, NQ, true>, dim3(grid), q.smem, st, p)   \
                    : launch_big(conv_stem_fwd_kernel<BN, R, NQ>, dim3(grid), q.smem, st, p);
#define TCB_STEM_FWD_R(R, NQ) TCB_STEM_FWD(32, R, NQ) TCB_STEM_FWD(64, R, NQ) TCB_STEM_FWD(128, R, NQ)
    TCB_STEM_FWD_R(7, 1)
    TCB_STEM_FWD_R(3, 1)
    TCB_STEM_FWD_R(5, 1)
    TCB_STEM_FWD_R(11, 2)
#undef TCB_STEM_FWD_R
#undef TCB_STEM_FWD
    return cudaErrorInvalidValue;
}

cudaError_t conv_stem_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw, void* workspace,
                            cudaStream_t st, bool x_ready) {
    const StemPlan q = stem_plan(g);
    if (!q.use || workspace == nullptr) return cudaErrorInvalidValue;
    char* ws = static_cast<char*>(workspace);
    void* x4 = ws;
    float* part = reinterpret_cast<float*>(ws + a256(q.x4_bytes));
    cudaError_t e = x_ready ? cudaSuccess : stem_pack(g, q, x, x4, st);
    if (e != cudaSuccess) return e;
    StemParams p{};
    if (!make_x4_map(&p.tmap_x, x4, g, q)) return cudaErrorInvalidValue;
    {
        EncodeTiledFn fn = encode_tiled_fn();
        if (!fn) return cudaErrorInvalidValue;
        const cuuint64_t dims[3] = {cuuint64_t(g.k), cuuint64_t(q.Wo), cuuint64_t(g.n) * q.Ho};
        const cuuint64_t strides[2] = {cuuint64_t(g.k) * 2, cuuint64_t(q.Wo) * g.k * 2};
        const cuuint32_t box[3] = {cuuint32_t(std::min(g.k, 64)), cuuint32_t(q.BW), 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (fn(&p.tmap_b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(dy), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, g.k >= 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    fill_common(p, g, q);
    p.stage_bytes = q.wg_stage_bytes;
    p.stages = q.wg_stages;
    p.mtiles = q.mtiles;
    p.tiles_per_cta = q.tiles_per_cta;
    p.dy_boxes = q.dy_boxes;
    p.dy_box_bytes = q.dy_box_bytes;
    p.tr = q.tr;
    p.xslots = q.xslots;
    p.tiles = q.wg_tiles;
    p.partial = part;
    conv_tc_note_launch(ConvTcLaunchInfo{2, 5, g.k, 0, 0, q.grid_wg, q.tiles, q.grid_wg, 0, 0});
    switch (g.k) {
        case 32: e = launch_big(conv_stem_wgrad_kernel<32>, dim3(q.grid_wg), q.wg_smem, st, p); break;
        case 64: e = launch_big(conv_stem_wgrad_kernel<64>, dim3(q.grid_wg), q.wg_smem, st, p); break;
        case 128: e = launch_big(conv_stem_wgrad_kernel<128>, dim3(q.grid_wg), q.wg_smem, st, p); break;
        default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    const int total = g.k * g.r * g.s * g.c;
    return launch_pdl(stem_reduce_scatter, dim3(std::max(1, std::min((total + 255) / 256, 1024))), dim3(256), 0, st,
                      static_cast<const float*>(part), q.grid_wg, dw, g.k, g.r, g.s, g.c, q.cv, q.nq);
}

}  // namespace tcb
