// Probe: tcgen05.mma (kind::f16, M = 128, K = 16) issue throughput for the
// shared-memory operand layouts the stem kernels can use: 128- / 64-byte
// swizzled K-major, the canonical no-swizzle layout, and the overlapping
// no-swizzle view of a raw stride-2 stem row (LBO 16, SBO 128).
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1709_06622_b200/csrc/cuda
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tcb;

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

struct Cfg {
    const char* name;
    uint32_t a_lbo, a_sbo, a_lay, a_kstep;  // kstep: bytes between the two K=16 steps of one 32-element chunk
    uint32_t b_lbo, b_sbo, b_lay, b_kstep;
    uint32_t a_major, b_major;
    uint32_t a_off = 0;  // start offset of A (row-shifted views)
};

template <int N>
__global__ void __launch_bounds__(384, 1) probe(Cfg c, long long* cyc, int iters, int spin) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, never;
    __shared__ uint32_t tslot;
    __shared__ volatile int stop;
    const int tid = threadIdx.x;
    for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&never, 1);
        stop = 0;
        ptx::fence_mbarrier_init();
    }
    if (tid < 32) ptx::tmem_alloc<256>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t a0 = ptx::smem_addr(sm), b0 = a0 + 64 * 1024;
    const uint32_t idesc = ptx::make_idesc(1, 128, N, c.a_major, c.b_major);
    if (tid < 32) {
        const uint64_t ad = desc(a0 + c.a_off, c.a_lbo, c.a_sbo, c.a_lay), bd = desc(b0, c.b_lbo, c.b_sbo, c.b_lay);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t aoff = (k >> 1) * (2048 >> 4) + (k & 1) * (c.a_kstep >> 4);
                const uint64_t boff = (k >> 1) * (2048 >> 4) + (k & 1) * (c.b_kstep >> 4);
                ptx::umma_f16_elect(tmem, ad + aoff, bd + boff, idesc, (it | k) ? 1u : 0u);
            }
        }
        ptx::umma_commit_elect(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (tid == 0) *cyc = t1 - t0;
        if (tid == 0) stop = 1;
    } else if (spin && tid >= 128) {  // 8 warps polling an mbarrier like idle epilogue warps
        while (!stop) {
            if (spin == 1) ptx::mbar_try_wait(&never, 0);
            else __nanosleep(200);
        }
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
    const Cfg cfgs[] = {
        {"A sw128 K / B sw128 K", 16, 1024, 2, 32, 16, 1024, 2, 32, 0, 0},
        {"A sw64 K  / B sw64 K ", 16, 512, 4, 32, 16, 512, 4, 32, 0, 0},
        {"A sw32 K  / B sw32 K ", 16, 256, 6, 0, 16, 256, 6, 0, 0, 0},
        {"A none std/ B sw64 K ", 128, 256, 0, 256, 16, 512, 4, 32, 0, 0},
        {"A none ovl/ B sw64 K ", 16, 128, 0, 32, 16, 512, 4, 32, 0, 0},
        {"A none ovl/ B sw128 K", 16, 128, 0, 32, 16, 1024, 2, 32, 0, 0},
        {"A sw64 MN / B sw128 MN", 1024, 512, 4, 1024, 8192, 1024, 2, 2048, 1, 1},
        {"A sw32 MN ovl32/ B sw128 MN", 32, 256, 6, 512, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN / B sw128 MN", 8192, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN lbo128 / B MN", 128, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN lbo256 / B MN", 256, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN lbo7424 / B MN", 7424, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN lbo7552 / B MN", 7552, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN lbo1024 / B MN", 1024, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1},
        {"A sw128 MN off128 / B MN", 7424, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1, 128},
        {"A sw128 MN off384 / B MN", 7424, 1024, 2, 2048, 8192, 1024, 2, 2048, 1, 1, 384},
        {"A sw128 K off128 / B K", 16, 1024, 2, 32, 16, 1024, 2, 32, 0, 0, 128},
        {"A sw128 K off896 / B K", 16, 1024, 2, 32, 16, 1024, 2, 32, 0, 0, 896},
    };
    const int iters = 2000;
    for (int spin : {0, 1, 2})
    for (const Cfg& c : cfgs) {
        if (spin && c.a_major == 0 && c.a_lay != 2) continue;
        for (int n : {64}) {
            auto k = n == 64 ? probe<64> : probe<128>;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            k<<<1, 384, 200 * 1024>>>(c, d, iters, spin);
            cudaError_t e = cudaDeviceSynchronize();
            long long cyc = 0;
            cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
            printf("spin%d %-30s N=%3d  %6.1f cycles/MMA  %s\n", spin, c.name, n, double(cyc) / (iters * 8.0),
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
    return 0;
}
