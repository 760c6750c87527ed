// Probe: cost of short tcgen05.mma groups (the stem's 14 MMAs per output
// tile) -- per-group commits, accumulator switches, accumulate=0 restarts.
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

// mode bits: 1 commit per group, 2 switch accumulator per group (4 buffers), 4 accumulate=0 at group start,
// 8 second commit per group, 16 interleave A (LBO 16 / SBO 128) instead of sw128
__global__ void __launch_bounds__(128, 1) probe(int mode, int group, long long* cyc, int groups) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[8];
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_mbarrier_init();
    }
    if (tid < 32) ptx::tmem_alloc<256>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t a0 = ptx::smem_addr(sm), b0 = a0 + 64 * 1024;
    const uint32_t idesc = ptx::make_idesc(1, 128, 64, 0, 0);
    if (tid < 32) {
        const uint64_t ad = (mode & 16) ? desc(a0, 16, 128, 0) : desc(a0, 16, 1024, 2);
        const uint64_t bd = desc(b0, 16, 512, 4);
        long long t0 = clock64();
        for (int g = 0; g < groups; ++g) {
            const uint32_t d = tmem + ((mode & 2) ? (g & 3) * 64 : 0);
            for (int k = 0; k < group; ++k)
                ptx::umma_f16_elect(d, ad + (k >> 1) * (2176 >> 4) + (k & 1) * 2, bd + (k >> 1) * 256 + (k & 1) * 2,
                                    idesc, ((mode & 4) && k == 0) ? 0u : 1u);
            if (mode & 1) ptx::umma_commit_elect(&bar[g & 3]);
            if (mode & 8) ptx::umma_commit_elect(&bar[4 + (g & 3)]);
        }
        ptx::umma_commit_elect(&bar[7]);
        ptx::mbar_wait(&bar[7], 0);
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
    const int groups = 2000;
    for (int mode : {0, 1, 2, 4, 6, 7, 9, 15, 16, 31}) {
        probe<<<1, 128, 200 * 1024>>>(mode, 14, d, groups);
        cudaError_t e = cudaDeviceSynchronize();
        long long cyc = 0;
        cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %2d: %7.1f cycles per 14-MMA group (%5.1f per MMA) %s\n", mode, double(cyc) / groups,
               double(cyc) / groups / 14, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
