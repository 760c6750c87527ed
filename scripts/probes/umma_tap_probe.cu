// Probe: can a K-major SWIZZLE_128B UMMA A-operand descriptor start at any
// 128-byte row of a TMA-style swizzled window (row-shifted "tap" views of one
// input window, the basis of a window implicit-GEMM conv), and at what cost?
//   correctness: D = A[o : o+128] * B^T for o = 0..7, base-offset field 0 or
//                (addr >> 7) & 7
//   throughput : cycles per M=128 x N x K=16 MMA at row offsets 0 / 1 / 3 / 8
// Build: nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_1709_06622_b200/csrc/cuda
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tcb;

constexpr int kRows = 300;

template <int N>
__global__ void __launch_bounds__(416, 1) probe(const uint16_t* Ag, const uint16_t* Bg, float* out,
                                                long long* cyc, int iters, int single_lane) {
    extern __shared__ __align__(1024) uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = sm;
    uint8_t* B = sm + kRows * 128;
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < kRows * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(A + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(Ag)[i];
    }
    for (int i = tid; i < N * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(B + r * 128 + ((c ^ (r & 7)) << 4)) = reinterpret_cast<const uint4*>(Bg)[i];
    }
    ptx::fence_proxy_async_smem();
    if (tid == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_mbarrier_init();
    }
    constexpr uint32_t kCols = N <= 32 ? 64 : N <= 64 ? 128 : N <= 128 ? 256 : 512;
    if (tid < 32) ptx::tmem_alloc<kCols>(&tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    const uint32_t a0 = ptx::smem_addr(A), b0 = ptx::smem_addr(B);
    constexpr uint32_t idesc = ptx::make_idesc(1, 128, N, 0, 0);
    uint32_t phase = 0;
    auto run = [&](int o, int mode, int reps) {
        if (tid < 32) {
            if (ptx::elect_one()) {
                for (int it = 0; it < reps; ++it) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t aa = a0 + o * 128 + k * 32;
                        uint64_t ad = ptx::sw128_desc(aa, 16, 1024);
                        if (mode) ad |= static_cast<uint64_t>((aa >> 7) & 7) << 49;
                        const uint64_t bd = ptx::sw128_desc(b0 + k * 32, 16, 1024);
                        ptx::umma_f16(tmem, ad, bd, idesc, (it > 0 || k > 0) ? 1u : 0u);
                    }
                }
                ptx::umma_commit(&bar);
            }
            __syncwarp();
        }
        ptx::mbar_wait(&bar, phase);
        phase ^= 1;
        ptx::tc_fence_after();
    };
    if (blockIdx.x == 0) {
        for (int mode = 0; mode < 2; ++mode) {
            for (int o = 0; o < 8; ++o) {
                run(o, mode, 1);
                const int row = tid;  // warp w reads lanes 32w..32w+31
                for (int c = 0; c < N && tid < 128; c += 32) {
                    uint32_t v[32];
                    ptx::tmem_ld_32x32b_x32(tmem + ((static_cast<uint32_t>(tid & ~31)) << 16) + c, v);
                    ptx::tmem_ld_wait();
                    for (int j = 0; j < 32; ++j)
                        out[((size_t(mode) * 8 + o) * 128 + row) * N + c + j] = __uint_as_float(v[j]);
                }
                ptx::tc_fence_before();
                __syncthreads();
                ptx::tc_fence_after();
            }
        }
    }
    // q0: 3x3 taps of a Wp=30 window; q1: + tcgen05.commit after every tap;
    // q2: + another warp streaming cp.async.bulk copies (64 KB per round) into
    // smem meanwhile; q3: both
    __shared__ uint64_t dummy, cpbar, spin;
    __shared__ volatile int done;
    if (tid == 0) {
        ptx::mbar_init(&dummy, 1);
        ptx::mbar_init(&cpbar, 1);
        ptx::mbar_init(&spin, 1);
        ptx::fence_mbarrier_init();
    }
    __syncthreads();
    uint32_t cph = 0, sph = 0;
    for (int q = 0; q < 4; ++q) {
        if (tid == 0) done = 0;
        __syncthreads();
        const long long t0 = clock64();
        if (tid < 32) {
            // q0: loop inside elect_one (the old shape); q1: whole warp runs the loop,
            // each MMA an asm with its own elect.sync; q2: whole warp, the 4 MMAs of a
            // tap in one asm block; q3: q2 with descriptors advanced by 64-bit adds
            for (int it = 0; it < iters / 9; ++it) {
                const uint32_t d = tmem + (it & 1) * N;
                const int off0 = (it * 37) % 30;
                if (q == 0) {
                    if (ptx::elect_one()) {
                        for (int tap = 0; tap < 9; ++tap) {
                            const int ti = tap / 3, tj = tap % 3;
                            const int o = off0 + ti * 30 + tj;
                            const uint32_t bb = b0 + (tap % 2) * 8192;
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                ptx::umma_f16(d, ptx::sw128_desc(a0 + o * 128 + k * 32, 16, 1024),
                                              ptx::sw128_desc(bb + k * 32, 16, 1024), idesc, (tap == 0 && k == 0) ? 0u : 1u);
                        }
                        ptx::umma_commit(&dummy);
                    }
                    __syncwarp();
                } else if (q == 1) {
                    for (int tap = 0; tap < 9; ++tap) {
                        const int ti = tap / 3, tj = tap % 3;
                        const int o = off0 + ti * 30 + tj;
                        const uint32_t bb = b0 + (tap % 2) * 8192;
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const uint64_t ad = ptx::sw128_desc(a0 + o * 128 + k * 32, 16, 1024);
                            const uint64_t bd = ptx::sw128_desc(bb + k * 32, 16, 1024);
                            asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                                         ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((tap == 0 && k == 0) ? 0u : 1u) : "memory");
                        }
                    }
                    if (ptx::elect_one()) ptx::umma_commit(&dummy);
                    __syncwarp();
                } else {
                    uint64_t arow = ptx::sw128_desc(a0 + off0 * 128, 16, 1024);
                    const uint64_t bdesc0 = ptx::sw128_desc(b0, 16, 1024);
                    for (int tap = 0; tap < 9; ++tap) {
                        const int ti = tap / 3, tj = tap % 3;
                        const uint64_t ad = q == 2 ? ptx::sw128_desc(a0 + (off0 + ti * 30 + tj) * 128, 16, 1024)
                                                   : arow + static_cast<uint64_t>(ti * 30 + tj) * 8;
                        const uint64_t bd = bdesc0 + static_cast<uint64_t>(tap % 2) * 512;
                        asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, 1;\n\t"
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, 1;\n\t"
                                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, 1;\n\t}"
                                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(tap == 0 ? 0u : 1u),
                                       "l"(ad + 2), "l"(bd + 2), "l"(ad + 4), "l"(bd + 4), "l"(ad + 6), "l"(bd + 6) : "memory");
                    }
                    if (ptx::elect_one()) ptx::umma_commit(&dummy);
                    __syncwarp();
                }
            }
            if (ptx::elect_one()) ptx::umma_commit(&bar);
            __syncwarp();
        } else if (tid >= 128 && false) {
            // 9 warps spin on an mbarrier that completes only when the MMAs are done
            ptx::mbar_wait(&spin, sph);
        } else if (tid < 64 && false) {
            if (tid == 32) {
                const uint32_t dst = ptx::smem_addr(B) + N * 128;  // scratch after B
                while (!done) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ptx::smem_addr(&cpbar)), "r"(65536u) : "memory");
                    for (int j = 0; j < 4; ++j)
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(dst + j * 16384), "l"(Ag + (blockIdx.x % 4) * 8192 * 0), "r"(16384u), "r"(ptx::smem_addr(&cpbar)) : "memory");
                    ptx::mbar_wait(&cpbar, cph);
                    cph ^= 1;
                }
            }
        }
        if (tid < 32) {
            ptx::mbar_wait(&bar, phase);
            phase ^= 1;
            if (tid == 0) {
                done = 1;
                if (q & 2) ptx::mbar_arrive(&spin);
            }
        }
        if (q & 2) sph ^= 1;
        const long long t1 = clock64();
        if (tid == 0) cyc[blockIdx.x * 4 + q] = t1 - t0;
        __syncthreads();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (tid < 32) ptx::tmem_dealloc<kCols>(tmem);
}

static float bf2f(uint16_t h) {
    uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

template <int N>
int test(int iters) {
    std::vector<uint16_t> A(kRows * 64), B(N * 64);
    srand(1234 + N);
    // PROBE_DATA: 0 = narrow-exponent values (default), 1 = normal-like values with
    // full random mantissas and signs, 2 = zeros
    const int mode = getenv("PROBE_DATA") ? atoi(getenv("PROBE_DATA")) : 0;
    auto gen = [&]() -> uint16_t {
        if (mode == 2) return 0;
        if (mode == 1) {
            const uint16_t sign = (rand() & 1) << 15;
            const uint16_t expo = static_cast<uint16_t>(120 + rand() % 8) << 7;  // 2^-7 .. 2^0
            return sign | expo | static_cast<uint16_t>(rand() & 0x7f);
        }
        return static_cast<uint16_t>(0x3c00 + (rand() % 256) - 128) & 0xffff;
    };
    for (auto& v : A) v = gen();
    for (auto& v : B) v = gen();
    for (size_t i = 0; i < A.size(); i += 3) A[i] ^= 0x8000;
    uint16_t *dA, *dB;
    float* dO;
    long long* dC;
    const int blocks = 148;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dO, size_t(2) * 8 * 128 * N * 4);
    cudaMalloc(&dC, blocks * 4 * sizeof(long long));
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    const size_t smem = getenv("PROBE_SMEM") ? atoi(getenv("PROBE_SMEM")) * 1024 : 1024 + kRows * 128 + 16384 + N * 128 + 65536;
    cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int single = getenv("PROBE_SINGLE") ? 1 : 0;
    if (getenv("PROBE_PDL")) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(blocks);
        cfg.blockDim = dim3(416);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, probe<N>, (const uint16_t*)dA, (const uint16_t*)dB, dO, dC, iters, single);
    } else {
        probe<N><<<blocks, 416, smem>>>(dA, dB, dO, dC, iters, single);
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d CUDA error %s\n", N, cudaGetErrorString(e));
        return 1;
    }
    std::vector<float> O(size_t(2) * 8 * 128 * N);
    std::vector<long long> C(blocks * 4);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
    for (int mode = 0; mode < 2; ++mode) {
        printf("N=%d base_offset=%s:", N, mode ? "addr" : "0   ");
        for (int o = 0; o < 8; ++o) {
            double worst = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < N; ++n) {
                    double ref = 0;
                    for (int k = 0; k < 64; ++k) ref += double(bf2f(A[(o + m) * 64 + k])) * bf2f(B[n * 64 + k]);
                    const double got = O[((size_t(mode) * 8 + o) * 128 + m) * N + n];
                    worst = std::max(worst, std::fabs(got - ref) / (std::fabs(ref) + 1.0));
                }
            printf(" o%d:%s", o, worst < 1e-3 ? "ok" : "BAD");
        }
        printf("\n");
    }
    const char* names[4] = {"elect_one loop", "warp loop, asm elect per MMA", "warp loop, 4 MMAs per asm", "4 MMAs per asm, desc adds"};
    for (int q = 0; q < 4; ++q) {
        double s = 0;
        for (int b = 0; b < blocks; ++b) s += C[b * 4 + q];
        s /= blocks;
        printf("N=%d %s: %.2f cycles per MMA (ideal %d)\n", N, names[q], s / ((iters / 9) * 9 * 4.0), N / 2);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dO); cudaFree(dC);
    return 0;
}

int main() {
    int rc = 0;
    const int it64 = getenv("PROBE_ITERS") ? atoi(getenv("PROBE_ITERS")) : 4096;
    rc |= test<64>(it64);
    rc |= test<128>(4096);
    rc |= test<256>(2043);
    return rc;
}
