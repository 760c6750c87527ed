// extern "C" surface of libtcb.so for single-op use (include/tcb.h): conv
// plans over the three algorithm families and two precisions, pools, loss,
// fills, the fused SGD shard update. No exception crosses the boundary;
// failures return a negative status and set a thread-local message.
#include <cstring>
#include <new>
#include <string>

#include <cuda_runtime.h>

#include "runtime.h"
#include "tcb.h"
#include "tcb/kernels.h"

namespace tcb {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TCB_OK;
    return fail(e == cudaErrorNotSupported ? TCB_ERR_UNSUPPORTED : TCB_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

ConvGeom to_geom(const tcb_conv_geom& g) {
    return ConvGeom{g.n, g.h, g.w, g.c, g.k, g.r, g.s, g.pad_h, g.pad_w, g.stride_h, g.stride_w};
}

bool geom_valid(const ConvGeom& g, std::string* why) {
    if (g.n < 1 || g.h < 1 || g.w < 1 || g.c < 1 || g.k < 1 || g.r < 1 || g.s < 1) {
        *why = "geometry extents must be >= 1";
        return false;
    }
    if (g.pad_h < 0 || g.pad_w < 0 || g.stride_h < 1 || g.stride_w < 1) {
        *why = "padding must be >= 0 and stride >= 1";
        return false;
    }
    if (g.h + 2 * g.pad_h < g.r || g.w + 2 * g.pad_w < g.s) {
        *why = "filter exceeds padded input, output shape collapses";
        return false;
    }
    return true;
}

static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

ConvPlanLayout conv_plan_layout(const ConvGeom& g, int algo, int prec) {
    ConvPlanLayout L{};
    const size_t P = size_t(g.n) * g.ho() * g.wo();
    const DType dt = prec == TCB_PREC_BF16 ? DType::BF16 : DType::F32;
    if (algo == TCB_ALGO_GEMM) {
        L.wgrad = prec == TCB_PREC_BF16   ? std::max(conv_tc_workspace(g, ConvMode::Wgrad),
                                                     conv_tc_workspace(g, ConvMode::Fwd))
                  : prec == TCB_PREC_TF32 ? conv_tf32_workspace(g, ConvMode::Wgrad)
                                          : conv_ffma_workspace(g, ConvMode::Wgrad);
        L.wT = prec == TCB_PREC_BF16 ? size_t(g.k) * g.r * g.s * g.c * 2 : 0;
    } else if (algo == TCB_ALGO_WINOGRAD) {
        L.wgrad = std::max({winograd_workspace(g, ConvMode::Fwd, dt),
                            winograd_workspace(g, ConvMode::Dgrad, dt),
                            winograd_workspace(g, ConvMode::Wgrad, dt)});
    } else {
        L.wgrad = std::max({fft_workspace(g, ConvMode::Fwd), fft_workspace(g, ConvMode::Dgrad),
                            fft_workspace(g, ConvMode::Wgrad)});
    }
    L.colsum = column_sum_workspace(static_cast<int>(P), g.k);
    L.counters = algo == TCB_ALGO_GEMM && prec == TCB_PREC_BF16 ? conv_tc_counter_ints() * sizeof(int) : 0;
    L.off_wT = align256(L.wgrad);
    L.off_colsum = L.off_wT + align256(L.wT);
    L.off_counters = L.off_colsum + align256(L.colsum);
    L.total = L.off_counters + align256(L.counters);
    return L;
}

bool algo_applies(const ConvGeom& g, int algo, int prec) {
    if (algo == TCB_ALGO_GEMM)
        return prec == TCB_PREC_FFMA_FP32 || (prec == TCB_PREC_TF32 && conv_tf32_supported(g)) ||
               (prec == TCB_PREC_BF16 && conv_tc_supported(g, ConvMode::Fwd) &&
                conv_tc_supported(g, ConvMode::Wgrad) && conv_tc_supported(g, ConvMode::Dgrad));
    // Winograd / FFT run fp32 SIMT transforms: no tensor-core (TF32) variant
    if (prec == TCB_PREC_TF32) return false;
    if (algo == TCB_ALGO_WINOGRAD) return winograd_supported(g);
    if (algo == TCB_ALGO_FFT) return fft_supported(g);
    return false;
}

}  // namespace tcb

using namespace tcb;

struct tcb_conv_plan {
    ConvGeom g;
    int algo, prec;
    ConvPlanLayout layout;
};

#define TCB_API extern "C" __attribute__((visibility("default")))

#define TCB_GUARD_BEGIN try {
#define TCB_GUARD_END                                                  \
    }                                                                  \
    catch (const std::bad_alloc&) {                                    \
        return fail(TCB_ERR_OOM, "host allocation failed");            \
    }                                                                  \
    catch (const std::exception& e) {                                  \
        return fail(TCB_ERR_INTERNAL, e.what());                       \
    }

TCB_API const char* tcb_last_error(void) { return g_last_error.c_str(); }
TCB_API const char* tcb_version(void) { return "tcb 0.1 (sm_100a)"; }

TCB_API int tcb_device_count(int* count) {
    if (!count) return fail(TCB_ERR_INVALID, "count is NULL");
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return check_cuda(e, "cudaGetDeviceCount");
    }
    return TCB_OK;
}

TCB_API int tcb_device_init(int device) { return check_cuda(cudaSetDevice(device), "cudaSetDevice"); }

TCB_API int tcb_conv_out_hw(const tcb_conv_geom* g, int* ho, int* wo) {
    if (!g || !ho || !wo) return fail(TCB_ERR_INVALID, "NULL argument");
    std::string why;
    const ConvGeom cg = to_geom(*g);
    if (!geom_valid(cg, &why)) return fail(TCB_ERR_INVALID, why);
    *ho = cg.ho();
    *wo = cg.wo();
    return TCB_OK;
}

TCB_API int tcb_conv_plan_create(const tcb_conv_geom* g, int algo, int prec, tcb_conv_plan** plan,
                                 size_t* workspace_bytes) {
    TCB_GUARD_BEGIN
    if (!g || !plan) return fail(TCB_ERR_INVALID, "NULL argument");
    const ConvGeom cg = to_geom(*g);
    std::string why;
    if (!geom_valid(cg, &why)) return fail(TCB_ERR_INVALID, why);
    if (algo < 0 || algo > 2 || prec < 0 || prec > 2) return fail(TCB_ERR_INVALID, "bad algo/prec");
    if (!algo_applies(cg, algo, prec))
        return fail(TCB_ERR_UNSUPPORTED, "algorithm/precision does not apply to this geometry");
    auto* p = new tcb_conv_plan{cg, algo, prec, conv_plan_layout(cg, algo, prec)};
    *plan = p;
    if (workspace_bytes) *workspace_bytes = p->layout.total;
    return TCB_OK;
    TCB_GUARD_END
}

// Narrow inputs: only the first c_valid of the C channels can be non-zero (the
// rest is bf16 channel padding). Lets first layers take the explicit-im2col /
// row-window stem paths, as the executor does; the workspace size can grow.
TCB_API int tcb_conv_plan_set_valid_channels(tcb_conv_plan* plan, int c_valid, size_t* workspace_bytes) {
    TCB_GUARD_BEGIN
    if (!plan) return fail(TCB_ERR_INVALID, "NULL argument");
    if (c_valid < 0 || c_valid > plan->g.c) return fail(TCB_ERR_INVALID, "c_valid must be in [0, C]");
    plan->g.c_valid = c_valid;
    plan->layout = conv_plan_layout(plan->g, plan->algo, plan->prec);
    if (workspace_bytes) *workspace_bytes = plan->layout.total;
    return TCB_OK;
    TCB_GUARD_END
}

TCB_API int tcb_conv_plan_destroy(tcb_conv_plan* plan) {
    delete plan;
    return TCB_OK;
}

TCB_API int tcb_conv_fwd(const tcb_conv_plan* plan, const void* x, const void* w,
                         const float* bias, const void* residual, int relu, void* y,
                         void* workspace, void* stream) {
    if (!plan || !x || !w || !y) return fail(TCB_ERR_INVALID, "NULL argument");
    auto st = static_cast<cudaStream_t>(stream);
    Epilogue ep;
    ep.bias = bias;
    ep.residual = residual;
    ep.relu = relu != 0;
    const DType dt = plan->prec == TCB_PREC_BF16 ? DType::BF16 : DType::F32;
    cudaError_t e;
    switch (plan->algo) {
        case TCB_ALGO_GEMM:
            e = plan->prec == TCB_PREC_BF16 ? conv_tc_fwd(plan->g, x, w, ep, y, st,
                                                          plan->g.c_valid > 0 || (!conv_tc_narrow(plan->g) &&
                                                                                  conv_tc_workspace(plan->g, ConvMode::Fwd))
                                                              ? workspace
                                                              : nullptr)
                : plan->prec == TCB_PREC_TF32
                    ? conv_tf32_fwd(plan->g, static_cast<const float*>(x),
                                    static_cast<const float*>(w), ep, static_cast<float*>(y), st)
                    : conv_ffma_fwd(plan->g, static_cast<const float*>(x),
                                    static_cast<const float*>(w), ep, static_cast<float*>(y), st);
            break;
        case TCB_ALGO_WINOGRAD: e = winograd_fwd(plan->g, dt, x, w, ep, y, workspace, st); break;
        default: e = fft_fwd(plan->g, dt, x, w, ep, y, workspace, st); break;
    }
    return check_cuda(e, "conv_fwd");
}

TCB_API int tcb_conv_dgrad(const tcb_conv_plan* plan, const void* dy, const void* w,
                           const void* residual_grad, const void* mask_act, void* dx,
                           void* workspace, void* stream) {
    if (!plan || !dy || !w || !dx) return fail(TCB_ERR_INVALID, "NULL argument");
    auto st = static_cast<cudaStream_t>(stream);
    Epilogue ep;
    ep.residual = residual_grad;
    ep.mask = mask_act;
    const DType dt = plan->prec == TCB_PREC_BF16 ? DType::BF16 : DType::F32;
    cudaError_t e;
    switch (plan->algo) {
        case TCB_ALGO_GEMM:
            if (plan->prec == TCB_PREC_BF16) {
                if (!workspace) return fail(TCB_ERR_INVALID, "bf16 dgrad needs the plan workspace");
                void* wT = nullptr;
                e = cudaSuccess;
                if (conv_tc_dgrad_needs_pack(plan->g)) {
                    wT = static_cast<char*>(workspace) + plan->layout.off_wT;
                    e = pack_dgrad_weights(DType::BF16, w, wT, plan->g, st);
                }
                if (e == cudaSuccess) e = conv_tc_dgrad(plan->g, dy, w, wT, ep, dx, st);
            } else if (plan->prec == TCB_PREC_TF32) {
                e = conv_tf32_dgrad(plan->g, static_cast<const float*>(dy),
                                    static_cast<const float*>(w), ep, static_cast<float*>(dx), st);
            } else {
                e = conv_ffma_dgrad(plan->g, static_cast<const float*>(dy),
                                    static_cast<const float*>(w), ep, static_cast<float*>(dx), st);
            }
            break;
        case TCB_ALGO_WINOGRAD: e = winograd_dgrad(plan->g, dt, dy, w, ep, dx, workspace, st); break;
        default: e = fft_dgrad(plan->g, dt, dy, w, ep, dx, workspace, st); break;
    }
    return check_cuda(e, "conv_dgrad");
}

TCB_API int tcb_conv_wgrad(const tcb_conv_plan* plan, const void* dy, const void* x, float* dw,
                           float* db, void* workspace, void* stream) {
    if (!plan || !dy || !x || !dw) return fail(TCB_ERR_INVALID, "NULL argument");
    auto st = static_cast<cudaStream_t>(stream);
    const DType dt = plan->prec == TCB_PREC_BF16 ? DType::BF16 : DType::F32;
    cudaError_t e;
    switch (plan->algo) {
        case TCB_ALGO_GEMM:
            e = plan->prec == TCB_PREC_BF16
                    ? conv_tc_wgrad(plan->g, dy, x, dw, workspace, st, false,
                                    workspace ? reinterpret_cast<int*>(static_cast<char*>(workspace) +
                                                                       plan->layout.off_counters)
                                              : nullptr)
                : plan->prec == TCB_PREC_TF32
                    ? conv_tf32_wgrad(plan->g, static_cast<const float*>(dy),
                                      static_cast<const float*>(x), dw, workspace, st)
                    : conv_ffma_wgrad(plan->g, static_cast<const float*>(dy),
                                      static_cast<const float*>(x), dw, workspace, st);
            break;
        case TCB_ALGO_WINOGRAD: e = winograd_wgrad(plan->g, dt, dy, x, dw, workspace, st); break;
        default: e = fft_wgrad(plan->g, dt, dy, x, dw, workspace, st); break;
    }
    if (e == cudaSuccess && db) {
        const int P = plan->g.n * plan->g.ho() * plan->g.wo();
        float* ws = reinterpret_cast<float*>(static_cast<char*>(workspace) + plan->layout.off_colsum);
        if (!workspace) return fail(TCB_ERR_INVALID, "bias gradient needs the plan workspace");
        e = column_sum(dt, dy, db, P, plan->g.k, ws, st);
    }
    return check_cuda(e, "conv_wgrad");
}

static DType dt_of(int d) { return d == TCB_DT_BF16 ? DType::BF16 : DType::F32; }

TCB_API int tcb_maxpool_fwd(int dtype, const void* x, void* y, uint8_t* argmax, int n, int h,
                            int w, int c, int f, int stride, int pad, void* stream) {
    if (f < 1 || f > 15 || stride < 1 || pad < 0) return fail(TCB_ERR_INVALID, "bad pool window");
    return check_cuda(maxpool_fwd(dt_of(dtype), x, y, argmax, n, h, w, c, f, stride, pad,
                                  static_cast<cudaStream_t>(stream)),
                      "maxpool_fwd");
}

TCB_API int tcb_maxpool_relu_bwd(int dtype, const void* dy, const uint8_t* argmax, const void* y,
                                 void* dx, int n, int h, int w, int c, int f, int stride, int pad,
                                 void* stream) {
    if (!y) return fail(TCB_ERR_INVALID, "maxpool_relu_bwd needs the pool output y");
    return check_cuda(maxpool_bwd(dt_of(dtype), dy, argmax, dx, n, h, w, c, f, stride, pad,
                                  static_cast<cudaStream_t>(stream), y),
                      "maxpool_relu_bwd");
}

TCB_API int tcb_avgpool2d_fwd(int dtype, const void* x, void* y, int n, int h, int w, int c, int f, int stride,
                              int pad, void* stream) {
    if (f < 1 || stride < 1 || pad < 0) return fail(TCB_ERR_INVALID, "bad pool window");
    if (!avgpool2d_supported(dt_of(dtype), c)) return fail(TCB_ERR_UNSUPPORTED, "channels must fill 16-byte vectors");
    return check_cuda(avgpool2d_fwd(dt_of(dtype), x, y, n, h, w, c, f, stride, pad, static_cast<cudaStream_t>(stream)),
                      "avgpool2d_fwd");
}

TCB_API int tcb_avgpool2d_bwd(int dtype, const void* dy, const void* mask_act, void* dx, int n, int h, int w,
                              int c, int f, int stride, int pad, void* stream) {
    if (f < 1 || stride < 1 || pad < 0) return fail(TCB_ERR_INVALID, "bad pool window");
    if (!avgpool2d_supported(dt_of(dtype), c)) return fail(TCB_ERR_UNSUPPORTED, "channels must fill 16-byte vectors");
    return check_cuda(avgpool2d_bwd(dt_of(dtype), dy, dx, n, h, w, c, f, stride, pad,
                                    static_cast<cudaStream_t>(stream), mask_act),
                      "avgpool2d_bwd");
}

TCB_API int tcb_slice_copy(int dtype, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                           size_t rows, void* stream) {
    if ((!src || !dst) && rows && width) return fail(TCB_ERR_INVALID, "NULL argument");
    if (width < 0 || size_t(width) > src_pitch || size_t(width) > dst_pitch)
        return fail(TCB_ERR_INVALID, "width exceeds a pitch");
    return check_cuda(slice_copy(dt_of(dtype), src, src_pitch, dst, dst_pitch, width, rows,
                                 static_cast<cudaStream_t>(stream)),
                      "slice_copy");
}

TCB_API int tcb_maxpool_bwd(int dtype, const void* dy, const uint8_t* argmax, void* dx, int n,
                            int h, int w, int c, int f, int stride, int pad, void* stream) {
    return check_cuda(maxpool_bwd(dt_of(dtype), dy, argmax, dx, n, h, w, c, f, stride, pad,
                                  static_cast<cudaStream_t>(stream)),
                      "maxpool_bwd");
}

TCB_API int tcb_avgpool_global_fwd(int dtype, const void* x, void* y, int n, int hw, int c,
                                   void* stream) {
    return check_cuda(avgpool_global_fwd(dt_of(dtype), x, y, n, hw, c,
                                         static_cast<cudaStream_t>(stream)),
                      "avgpool_fwd");
}

TCB_API int tcb_avgpool_global_bwd(int dtype, const void* dy, void* dx, int n, int hw, int c,
                                   void* stream) {
    return check_cuda(avgpool_global_bwd(dt_of(dtype), dy, dx, n, hw, c,
                                         static_cast<cudaStream_t>(stream)),
                      "avgpool_bwd");
}

TCB_API int tcb_softmax_xent(int dtype, const void* logits, const int32_t* labels, void* dlogits,
                             float* loss, int n, int classes, void* stream) {
    return check_cuda(softmax_xent(dt_of(dtype), logits, labels, dlogits, loss, n, classes, classes,
                                   static_cast<cudaStream_t>(stream)),
                      "softmax_xent");
}

TCB_API int tcb_fill_uniform(int dtype, void* p, size_t n, uint64_t seed, uint64_t tag, float lo,
                             float hi, void* stream) {
    return check_cuda(fill_uniform(dt_of(dtype), p, n, seed, tag, lo, hi,
                                   static_cast<cudaStream_t>(stream)),
                      "fill_uniform");
}

TCB_API int tcb_fill_labels(int32_t* labels, int n, int classes, uint64_t seed, void* stream) {
    if (classes < 1) return fail(TCB_ERR_INVALID, "classes must be >= 1");
    return check_cuda(fill_labels(labels, n, classes, seed, static_cast<cudaStream_t>(stream)),
                      "fill_labels");
}

TCB_API int tcb_cast(int src_dtype, const void* src, int dst_dtype, void* dst, size_t n,
                     void* stream) {
    return check_cuda(cast(dt_of(src_dtype), src, dt_of(dst_dtype), dst, n,
                           static_cast<cudaStream_t>(stream)),
                      "cast");
}

TCB_API int tcb_ps_nvls_update(const float* grad_mc, float* grad, float* w, float* v, void* wcompute_mc,
                               size_t begin, size_t n, float lr, float momentum, float weight_decay,
                               float grad_scale, void* stream) {
    if (!grad_mc || !grad || !w || !v || !wcompute_mc) return fail(TCB_ERR_INVALID, "NULL argument");
    return check_cuda(ps_nvls_update(grad_mc, grad, w, v, wcompute_mc, begin, n, lr, momentum, weight_decay,
                                     grad_scale, static_cast<cudaStream_t>(stream)),
                      "ps_nvls_update");
}

TCB_API int tcb_nvls_barrier(void* const* signal_pads_dev, uint32_t* epoch_dev, int rank, int world,
                             int slot0, uint32_t* err_dev, uint64_t timeout_ns, void* stream) {
    if (!signal_pads_dev || !epoch_dev || !err_dev) return fail(TCB_ERR_INVALID, "NULL argument");
    return check_cuda(nvls_barrier(reinterpret_cast<uint32_t* const*>(signal_pads_dev), epoch_dev, slot0, rank,
                                   world, static_cast<cudaStream_t>(stream), err_dev, timeout_ns),
                      "nvls_barrier");
}

TCB_API int tcb_nvls_probe(int mode, const float* grad_mc, float* grad, const float* w, void* wcompute_mc,
                           size_t begin, size_t n, void* stream) {
    return check_cuda(nvls_probe(mode, grad_mc, grad, w, wcompute_mc, begin, n, static_cast<cudaStream_t>(stream)),
                      "nvls_probe");
}

TCB_API int tcb_sgd_momentum(float* w, const float* grad, float* v, int compute_dtype,
                             void* w_compute, size_t n, float lr, float momentum,
                             float weight_decay, float grad_scale, void* stream) {
    if (!w || !grad || !v) return fail(TCB_ERR_INVALID, "NULL argument");
    return check_cuda(sgd_momentum(w, grad, v, dt_of(compute_dtype), w_compute, n, lr, momentum,
                                   weight_decay, grad_scale, static_cast<cudaStream_t>(stream)),
                      "sgd_momentum");
}

TCB_API void tcb_free(void* p) { std::free(p); }

// Diagnostics: per-CTA role timing of the window conv kernel into a device
// buffer of 8 x u64 per CTA (producer total / window-slot wait / B-slot wait,
// MMA total / accumulator wait / window wait / B wait, epilogue total<<32|wait),
// or nullptr to switch it off.
TCB_API int tcb_conv_win_debug(void* dev_buffer) {
    conv_win_set_debug(dev_buffer);
    return TCB_OK;
}

TCB_API int tcb_conv_last_launch_info(int* out10) {
    if (!out10) return fail(TCB_ERR_INVALID, "NULL argument");
    const ConvTcLaunchInfo i = conv_tc_last_launch();
    const int v[10] = {i.mode, i.load, i.bn, i.epi, i.cta2, i.splits, i.units, i.grid, i.fused_reduce, i.b_resident};
    for (int k = 0; k < 10; ++k) out10[k] = v[k];
    return TCB_OK;
}

// 1 (default): row-window stem kernels for narrow even-stride first layers;
// 0: the explicit-im2col GEMM path for them (A/B comparisons, tests).
TCB_API int tcb_set_conv_stem(int on) {
    conv_stem_set_mode(on);
    return TCB_OK;
}

TCB_API int tcb_set_conv_operand_path(int mode) {
    if (mode < 0 || mode > 4)
        return fail(TCB_ERR_INVALID, "mode must be 0 (auto), 1 (gather), 2 (register epilogue), 3 (auto "
                                     "without the window path) or 4 (window path wherever it applies)");
    conv_tc_set_force_gather(mode == 1);
    conv_tf32_set_force_gather(mode == 1);
    conv_tc_set_epi_kb(mode == 2 ? 0 : -1);
    conv_win_set_mode(mode == 3 ? 0 : mode == 4 ? 2 : -1);
    return TCB_OK;
}
