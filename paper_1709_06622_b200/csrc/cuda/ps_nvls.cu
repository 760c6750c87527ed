// Parameter-server step fused into one kernel over NVSwitch multicast (NVLS):
// reduce-scatter + momentum SGD + all-gather of a = PS shard of the flat
// parameter buffer (PAPER steps 5-7: push ΔW, update, pull W).
//
// Every GPU's fp32 gradient buffer and bf16 compute-weight buffer are bound to
// multicast objects (torch symmetric memory does the allocation / handle
// exchange). For its shard, each rank
//   g  = multimem.ld_reduce.add.f32 [grad_mc + i]    (the switch sums all GPUs' copies)
//   v  = mu*v + (g/G + wd*w);  w -= lr*v             (same rounding as sgd4_kernel)
//   multimem.st [wc_mc + i] = bf16(w)                (the switch writes every GPU)
// so the aggregation traffic never materialises a reduce-scattered copy and
// the refreshed weights reach all GPUs in the same pass. The reduced gradient
// is also written back to the local shard (same observable state as the NCCL
// reduce-scatter path). Cross-GPU ordering uses a signal-pad barrier before
// (all gradients written) and after (all weights delivered) the update.
#include <cuda_bf16.h>

#include "common.cuh"

namespace tcb {
namespace {

__device__ __forceinline__ float4 mc_ld_reduce_add_v4(const float* mc) {
    float4 r;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(mc)
                 : "memory");
    return r;
}

__device__ __forceinline__ void mc_st_v2(void* mc, uint32_t a, uint32_t b) {
    asm volatile("multimem.st.relaxed.sys.global.v2.f32 [%0], {%1, %2};" ::"l"(mc), "f"(__uint_as_float(a)),
                 "f"(__uint_as_float(b))
                 : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

template <int U>
__global__ void __launch_bounds__(256) ps_nvls_update_kernel(const float* __restrict__ grad_mc,
                                                             float* __restrict__ grad,
                                                             float4* __restrict__ w,
                                                             float4* __restrict__ v, char* wc_mc,
                                                             size_t begin, size_t n4, float lr,
                                                             float mom, float wd, float gscale) {
    // U independent 16-byte multicast reductions in flight per thread
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i0 < n4; i0 += U * stride) {
        float4 gi[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + u * stride;
            if (i < n4) gi[u] = mc_ld_reduce_add_v4(grad_mc + begin + 4 * i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = i0 + u * stride;
            if (i >= n4) break;
            const size_t e = begin + 4 * i;  // element index in the flat buffer
            reinterpret_cast<float4*>(grad + e)[0] = gi[u];
            float4 wi = w[e / 4], vi = v[e / 4];
            float* wp = &wi.x;
            float* gp = &gi[u].x;
            float* vp = &vi.x;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float gg = __fadd_rn(__fmul_rn(gp[j], gscale), __fmul_rn(wd, wp[j]));
                vp[j] = __fadd_rn(__fmul_rn(mom, vp[j]), gg);
                wp[j] = __fsub_rn(wp[j], __fmul_rn(lr, vp[j]));
            }
            v[e / 4] = vi;
            w[e / 4] = wi;
            mc_st_v2(wc_mc + e * 2, pack_bf16x2(wp[0], wp[1]), pack_bf16x2(wp[2], wp[3]));
        }
    }
}

// Microbenchmark halves of the fused kernel (scripts/nvls_bench.py):
// mode 1 = multicast reduce only (into the local shard), 2 = multicast store only.
__global__ void __launch_bounds__(256) nvls_probe_kernel(int mode, const float* __restrict__ grad_mc,
                                                         float* __restrict__ grad, const float* __restrict__ w,
                                                         char* wc_mc, size_t begin, size_t n4) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i0 < n4; i0 += 4 * stride) {
        if (mode == 1) {
            float4 g[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * stride < n4) g[u] = mc_ld_reduce_add_v4(grad_mc + begin + 4 * (i0 + u * stride));
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * stride < n4) reinterpret_cast<float4*>(grad + begin)[i0 + u * stride] = g[u];
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t i = i0 + u * stride;
                if (i >= n4) break;
                const float4 x = reinterpret_cast<const float4*>(w + begin)[i];
                mc_st_v2(wc_mc + (begin + 4 * i) * 2, pack_bf16x2(x.x, x.y), pack_bf16x2(x.z, x.w));
            }
        }
    }
}

// All-GPU barrier on the signal pads (P2P-mapped, one u32 slot per peer).
// Epochs are counted on the device so the kernel replays inside CUDA graphs.
// The wait is bounded: a peer that does not arrive within timeout_ns (a rank
// that stalled or died) sets *err = 1 and the barrier gives up instead of
// hanging the GPU; the host reports TCB_ERR_NCCL at its next health check.
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void nvls_barrier_kernel(uint32_t* const* __restrict__ pads, uint32_t* __restrict__ epoch,
                                    int slot0, int rank, int world, uint32_t* __restrict__ err,
                                    uint64_t timeout_ns) {
    __shared__ uint32_t e;
    if (threadIdx.x == 0) {
        e = *epoch + 1;
        *epoch = e;
    }
    __syncthreads();
    const int p = threadIdx.x;
    if (p < world) {
        __threadfence_system();  // this GPU's earlier writes (previous kernels) before the signal
        uint32_t* to = pads[p] + slot0 + rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(to), "r"(e) : "memory");
        const uint32_t* from = pads[rank] + slot0 + p;
        uint32_t got = 0;
        const uint64_t t0 = globaltimer_ns();
        for (uint32_t spin = 0;; ++spin) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(got) : "l"(from) : "memory");
            if (static_cast<int32_t>(got - e) >= 0) break;
            if ((spin & 1023) == 1023) {
                if (*reinterpret_cast<volatile uint32_t*>(err) != 0) break;  // another lane timed out
                if (globaltimer_ns() - t0 > timeout_ns) {
                    atomicExch(err, 1u);
                    break;
                }
            }
        }
    }
    __syncthreads();
}

}  // namespace

cudaError_t nvls_barrier(uint32_t* const* pads_dev, uint32_t* epoch_dev, int slot0, int rank, int world,
                         cudaStream_t st, uint32_t* err_dev, uint64_t timeout_ns) {
    if (world > 32 || err_dev == nullptr) return cudaErrorInvalidValue;
    nvls_barrier_kernel<<<1, 32, 0, st>>>(pads_dev, epoch_dev, slot0, rank, world, err_dev, timeout_ns);
    return cudaGetLastError();
}

cudaError_t ps_nvls_update(const float* grad_mc, float* grad, float* w, float* v, void* wc_mc, size_t begin,
                           size_t n, float lr, float mom, float wd, float gscale, cudaStream_t st) {
    if (n % 4 || begin % 4) return cudaErrorInvalidValue;
    const size_t n4 = n / 4;
    constexpr int kU = 4;
    const int grid = static_cast<int>(std::min<size_t>((n4 + 256 * kU - 1) / (256 * kU), size_t(num_sms()) * 4));
    if (grid == 0) return cudaSuccess;
    ps_nvls_update_kernel<kU><<<grid, 256, 0, st>>>(grad_mc, grad, reinterpret_cast<float4*>(w),
                                                reinterpret_cast<float4*>(v), static_cast<char*>(wc_mc),
                                                begin, n4, lr, mom, wd, gscale);
    return cudaGetLastError();
}

cudaError_t nvls_probe(int mode, const float* grad_mc, float* grad, const float* w, void* wc_mc, size_t begin,
                       size_t n, cudaStream_t st) {
    if (n % 4 || begin % 4) return cudaErrorInvalidValue;
    const size_t n4 = n / 4;
    const int grid = static_cast<int>(std::min<size_t>((n4 + 1023) / 1024, size_t(num_sms()) * 4));
    if (grid == 0) return cudaSuccess;
    nvls_probe_kernel<<<grid, 256, 0, st>>>(mode, grad_mc, grad, w, static_cast<char*>(wc_mc), begin, n4);
    return cudaGetLastError();
}

}  // namespace tcb
