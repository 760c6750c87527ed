// Probe: MN-major SWIZZLE_128B A operand over a TMA-style swizzled "window"
// of 128-byte rows (row = pixel = reduction index k, 64 channels along the
// row), with the two 64-element M blocks at DIFFERENT row offsets (LBO = the
// offset difference): one M = 128 tile = two filter taps of a wgrad.
//   D[m][n] = sum_k A[m][k] B[n][k],  A[m][k] = win[k + o(m/64)][m%64],
//   B[n][k] = dy[k][n] (MN-major, 64 n per row)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tcb;

constexpr int kRows = 192;

__global__ void probe(const uint16_t* Wg, const uint16_t* Bg, float* out, int o0, int o1, int iters, long long* cyc,
                      int kmajor) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* W = sm;
    uint8_t* B = sm + kRows * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < kRows * 8; i += 128) {
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(W + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(Wg)[i];
    }
    for (int i = tid; i < 16 * 8; i += 128) {
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(B + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(Bg)[i];
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbarrier_init();
    }
    if (tid < 32) ptx::tmem_alloc<64>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    constexpr uint32_t idesc = ptx::make_idesc(1, 128, 64, 1, 1);
    const long long t0 = clock64();
    if (tid < 32) {
        const uint32_t a = ptx::smem_addr(W) + o0 * 128;
        const uint64_t ad = ptx::sw128_desc(a, static_cast<uint32_t>((o1 - o0) * 128), 1024);
        const uint64_t bd = ptx::sw128_desc(ptx::smem_addr(B), 8192, 1024);
        constexpr uint32_t idesc_k = ptx::make_idesc(1, 128, 64, 0, 0);
        for (int it = 0; it < iters; ++it)
            for (int ks = 0; ks < 8; ++ks) {
                if (kmajor)
                    ptx::umma_f16_elect(tmem, ptx::sw128_desc(a + (ks & 3) * 32, 16, 1024),
                                        ptx::sw128_desc(ptx::smem_addr(B) + (ks & 3) * 32, 16, 1024), idesc_k, it | ks);
                else
                    ptx::umma_f16_elect(tmem, ad + (ks & 3) * 128 * (iters > 1), bd + (ks & 3) * 0, idesc, it | ks);
            }
        if (ptx::elect_one()) ptx::umma_commit(&bar);
        __syncwarp();
    }
    ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_after();
    if (tid == 0 && cyc) *cyc = clock64() - t0;
    uint32_t v[32];
    for (int c = 0; c < 64; c += 32) {
        ptx::tmem_ld_32x32b_x32(tmem + ((static_cast<uint32_t>(tid & ~31)) << 16) + c, v);
        ptx::tmem_ld_wait();
        for (int j = 0; j < 32; ++j) out[tid * 64 + c + j] = __uint_as_float(v[j]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (tid < 32) ptx::tmem_dealloc<64>(tmem);
}

static float bf(uint16_t h) {
    uint32_t u = uint32_t(h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    std::vector<uint16_t> W(kRows * 64), B(16 * 64);
    srand(7);
    for (auto& x : W) x = uint16_t(0x3c00 + rand() % 256 - 128) ^ (rand() & 1 ? 0x8000 : 0);
    for (auto& x : B) x = uint16_t(0x3c00 + rand() % 256 - 128) ^ (rand() & 1 ? 0x8000 : 0);
    uint16_t *dW, *dB;
    float* dO;
    cudaMalloc(&dW, W.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dW, W.data(), W.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int cases[][2] = {{0, 8}, {3, 4}, {5, 63}, {1, 2}, {2, 60}};
    int rc = 0;
    for (auto& cs : cases) {
        probe<<<1, 128, 64 * 1024>>>(dW, dB, dO, cs[0], cs[1], 1, nullptr, 0);
        if (cudaDeviceSynchronize() != cudaSuccess) { printf("CUDA error\n"); return 1; }
        std::vector<float> O(128 * 64);
        cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
        double worst = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 64; ++n) {
                double ref = 0;
                const int o = m < 64 ? cs[0] : cs[1];
                for (int k = 0; k < 16; ++k) ref += double(bf(W[(k + o) * 64 + m % 64])) * bf(B[k * 64 + n]);
                worst = std::max(worst, std::fabs(O[m * 64 + n] - ref) / (std::fabs(ref) + 1.0));
            }
        printf("o0=%d o1=%d (LBO %d B): %s (max rel err %.3g)\n", cs[0], cs[1], (cs[1] - cs[0]) * 128,
               worst < 1e-3 ? "ok" : "BAD", worst);
        rc |= worst >= 1e-3;
    }
    long long* dC;
    cudaMalloc(&dC, 8);
    for (int km = 0; km < 2; ++km) {
        probe<<<148, 128, 64 * 1024>>>(dW, dB, dO, 3, 4, 2048, dC, km);
        cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, dC, 8, cudaMemcpyDeviceToHost);
        printf("%s A/B, M=128 N=64: %.2f cycles per MMA\n", km ? "K-major" : "MN-major", c / (2048.0 * 8));
    }
    return rc;
}
