// Probe: tcgen05.mma issue cost for short-N tiles (M = 128, N = 64, K = 16,
// 48-cycle tensor floor) under different issue styles, 14 MMAs per "tile"
// (7 filter rows x 2 K-steps, as the stem), a stage index that rotates per tile:
//   0 warp-collective elect per MMA, offsets from a runtime loop
//   1 warp-collective elect per MMA, unrolled compile-time offsets
//   2 one lane issues (divergent branch), unrolled
//   3 one elect per PAIR of MMAs (one asm block, +2 K-step adds inside)
//   4 one elect per 14 MMAs (one asm block, immediate offsets)
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1709_06622_b200/csrc/cuda
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tcb;

__device__ __forceinline__ uint64_t rdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(8) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    return d;
}
__device__ __forceinline__ uint64_t s64desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(32) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(4) << 61;
    return d;
}

__device__ __forceinline__ void mma_raw(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_pair_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a2, b2;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "add.s64 a2, %1, 2;\n\tadd.s64 b2, %2, 2;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

// 7 rows x 2 K-steps, A rows 136 x 16 B apart, B chunks 256 x 16 B apart
__device__ __forceinline__ void mma_tile14_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
#define MMA_RK(AO, BO, P) \
    "add.s64 a2, %1, " #AO ";\n\tadd.s64 b2, %2, " #BO ";\n\t@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, " P ";\n\t"
    asm volatile(
        "{\n\t.reg .pred e, f, t;\n\t.reg .b64 a2, b2;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 f, 0, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        MMA_RK(0, 0, "f") MMA_RK(2, 2, "t")
        MMA_RK(136, 256, "t") MMA_RK(138, 258, "t")
        MMA_RK(272, 512, "t") MMA_RK(274, 514, "t")
        MMA_RK(408, 768, "t") MMA_RK(410, 770, "t")
        MMA_RK(544, 1024, "t") MMA_RK(546, 1026, "t")
        MMA_RK(680, 1280, "t") MMA_RK(682, 1282, "t")
        MMA_RK(816, 1536, "t") MMA_RK(818, 1538, "t")
        "}" ::"r"(d), "l"(a), "l"(b), "r"(idesc)
        : "memory");
#undef MMA_RK
}

__global__ void __launch_bounds__(128, 1) probe(int mode, long long* cyc, int tiles, int nr) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 180 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_mbarrier_init();
    }
    if (tid < 32) ptx::tmem_alloc<256>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t sbase = ptx::smem_addr(sm);
    const uint32_t bbase = sbase + 128 * 1024;
    constexpr uint32_t idesc = ptx::make_idesc(1, 128, 64, 0, 0);
    if (tid < 32) {
        long long t0 = clock64();
        int st = 0;
        for (int u = 0; u < tiles; ++u) {
            const uint32_t d = tmem + (u & 1) * 64;
            const uint64_t a0 = rdesc(sbase + st * 16384);
            const uint64_t b0 = s64desc(bbase);
            if (mode == 0) {
                for (int r = 0; r < nr; ++r) {
                    ptx::umma_f16_elect(d, a0 + r * 136, b0 + r * 256, idesc, r ? 1u : 0u);
                    ptx::umma_f16_elect(d, a0 + r * 136 + 2, b0 + r * 256 + 2, idesc, 1u);
                }
            } else if (mode == 1) {
#pragma unroll
                for (int r = 0; r < 7; ++r) {
                    ptx::umma_f16_elect(d, a0 + r * 136, b0 + r * 256, idesc, r ? 1u : 0u);
                    ptx::umma_f16_elect(d, a0 + r * 136 + 2, b0 + r * 256 + 2, idesc, 1u);
                }
            } else if (mode == 2) {
                if (tid == 0) {
#pragma unroll
                    for (int r = 0; r < 7; ++r) {
                        mma_raw(d, a0 + r * 136, b0 + r * 256, idesc, r ? 1u : 0u);
                        mma_raw(d, a0 + r * 136 + 2, b0 + r * 256 + 2, idesc, 1u);
                    }
                }
                __syncwarp();
            } else if (mode == 3) {
#pragma unroll
                for (int r = 0; r < 7; ++r) mma_pair_elect(d, a0 + r * 136, b0 + r * 256, idesc, r ? 1u : 0u);
            } else {
                mma_tile14_elect(d, a0, b0, idesc);
            }
            ptx::umma_commit_elect(&bar[u & 1]);
            if (++st == 6) st = 0;
        }
        ptx::umma_commit_elect(&bar[3]);
        ptx::mbar_wait(&bar[3], 0);
        long long t1 = clock64();
        if (tid == 0) *cyc = t1 - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (tid < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<256>(tmem);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int tiles = 2000;
    for (int mode = 0; mode < 5; ++mode) {
        probe<<<1, 128, 200 * 1024>>>(mode, d, tiles, 7);
        cudaError_t e = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d: %7.1f cycles per 14-MMA tile (%5.1f per MMA) %s\n", mode, double(cyc) / tiles,
               double(cyc) / tiles / 14, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
