/*
 * tcb.h — C-ABI of the B200 training-step library (libtcb.so).
 *
 * The reference (arXiv 1709.06622 `traincap`, /root/reference/proj) has no
 * device code and no FFI: its hot path enters through the C++ planner's
 * measurement boundary — per-layer conv cost rows (`CostEntry`,
 * /root/reference/proj/include/traincap/catalog.hpp:19-27), the step trace
 * (`StepTrace`, /root/reference/proj/include/traincap/io.hpp:23-26) and the
 * parameter-server sizing inputs (`ClusterSpec`,
 * /root/reference/proj/include/traincap/scale_plan.hpp:39-44). Every entry
 * point below produces or consumes one of those quantities; the comment on
 * each names the reference interface it feeds. INTEGRATION.md shows the
 * bindings a maintainer adds on the reference side.
 *
 * Conventions
 *   - plain pointers + sizes; device pointers are caller-owned CUDA device
 *     memory; `stream` is a cudaStream_t passed as void*.
 *   - every call returns TCB_OK (0) or a negative status; the message of the
 *     last failure on the calling thread is tcb_last_error().
 *   - handles are not thread-safe: one host thread per GPU.
 *   - tensors are NHWC; conv weights are KRSC ([out][fh][fw][in]).
 *   - dtype of activations/weights follows the plan precision:
 *       TCB_PREC_FFMA_FP32 -> float (SIMT FFMA),
 *       TCB_PREC_TF32      -> float (tcgen05 kind::tf32 GEMM convs; C, K % 4 == 0;
 *                             Winograd / FFT have no TF32 plan: UNSUPPORTED),
 *       TCB_PREC_BF16      -> bf16 (uint16_t bits).
 *     Weight gradients are always fp32 (they land in the PS flat buffer).
 */
#ifndef TCB_H_
#define TCB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TCB_OK = 0,
    TCB_ERR_INVALID = -1,     /* bad argument (maps to traincap::DomainError)   */
    TCB_ERR_UNSUPPORTED = -2, /* algorithm/precision not applicable to geometry */
    TCB_ERR_CUDA = -3,        /* CUDA runtime failure                           */
    TCB_ERR_NCCL = -4,        /* NCCL failure                                   */
    TCB_ERR_OOM = -5,         /* workspace does not fit: infeasible CostEntry   */
    TCB_ERR_INTERNAL = -6
};

typedef enum { TCB_ALGO_GEMM = 0, TCB_ALGO_WINOGRAD = 1, TCB_ALGO_FFT = 2 } tcb_algo;
typedef enum { TCB_PREC_FFMA_FP32 = 0, TCB_PREC_TF32 = 1, TCB_PREC_BF16 = 2 } tcb_prec;
typedef enum { TCB_DT_F32 = 0, TCB_DT_BF16 = 1 } tcb_dtype;

/* One convolution (geometry of Eq 1, generalised to rectangular filters). */
typedef struct tcb_conv_geom {
    int n, h, w, c;         /* input  N x H x W x C                      */
    int k, r, s;            /* K filters of R x S                        */
    int pad_h, pad_w;       /* symmetric zero padding                    */
    int stride_h, stride_w; /* strides                                   */
} tcb_conv_geom;

typedef struct tcb_conv_plan tcb_conv_plan;

/* ---------------------------------------------------------------- status -- */
const char* tcb_last_error(void);
const char* tcb_version(void);
int tcb_device_count(int* count);
int tcb_device_init(int device);

/* Output spatial size, Eq 1: floor((in - f + 2p)/s) + 1
 * (traincap::propagate_shapes, /root/reference/proj/src/net_model.cpp:80-99). */
int tcb_conv_out_hw(const tcb_conv_geom* g, int* ho, int* wo);

/* ------------------------------------------------------------ conv plans -- */
/* Builds a plan for (geometry, algorithm, precision). Returns
 * TCB_ERR_UNSUPPORTED when the algorithm does not apply (e.g. Winograd on a
 * non-3x3/stride-1 layer) so the profiler omits that CostEntry, matching the
 * catalog's "absent algorithm is a value" rule
 * (/root/reference/proj/include/traincap/catalog.hpp:60-62).
 * *workspace_bytes receives the plan's scratch need; the profiler records it
 * as CostEntry::memory_bits = 8 * workspace_bytes. The workspace must be
 * zero-filled once before its first use (it holds self-resetting split-K
 * counters); it can then be reused across calls without clearing. */
int tcb_conv_plan_create(const tcb_conv_geom* g, int algo, int prec, tcb_conv_plan** plan,
                         size_t* workspace_bytes);
/* Only the first c_valid of C input channels can be non-zero (bf16 channel
 * padding of a narrow first layer): enables the explicit-im2col and row-window
 * stem paths; *workspace_bytes is updated (it can grow). */
int tcb_conv_plan_set_valid_channels(tcb_conv_plan* plan, int c_valid, size_t* workspace_bytes);
int tcb_conv_plan_destroy(tcb_conv_plan* plan);
/* Operand-load path of the tensor-core GEMM conv: 0 = automatic (2-D TMA for
 * 1x1/stride-1 layers, im2col-mode TMA when channels % 64 == 0, cp.async
 * gather otherwise; TMA-store epilogue on K-light layers), 1 = force the
 * cp.async gather path, 2 = automatic loads with the register epilogue
 * everywhere (A/B testing). */
/* Row-window stem kernels for narrow even-stride first layers: 1 on (default), 0 the
 * explicit-im2col path, -1 from $TCB_STEM. */
int tcb_set_conv_stem(int on);
int tcb_set_conv_operand_path(int mode); /* 0 auto, 1 gather, 2 register epilogue, 3 auto w/o window,
                                           4 window wherever it applies */
/* Test hook: the configuration of the last bf16 tensor-core conv kernel launch
 * on this process: {mode (0 fwd / 1 dgrad / 2 wgrad), operand path (0 cp.async
 * gather, 1 2-D TMA, 2 im2col TMA, 3 8-channel im2col TMA, 4 window), tile N,
 * TMA-epilogue slots, CTA pair, split-K factor, work units, grid CTAs, in-kernel
 * split reduce, weight operand resident in shared memory}. */
int tcb_conv_last_launch_info(int* out10);
/* Diagnostics: per-CTA role timing of the window conv kernel (8 x u64 per CTA)
 * written to a device buffer on each launch; NULL switches it off. */
int tcb_conv_win_debug(void* dev_buffer);

/* y = act(conv(x, w) + bias + residual); bias (fp32, K) and residual (same
 * dtype/shape as y) may be NULL; relu != 0 applies max(0, .). */
int tcb_conv_fwd(const tcb_conv_plan* plan, const void* x, const void* w, const float* bias,
                 const void* residual, int relu, void* y, void* workspace, void* stream);

/* dx = (conv^T(dy, w) + residual_grad) * [mask_act > 0]; residual_grad and
 * mask_act (activation whose ReLU is undone) may be NULL. */
int tcb_conv_dgrad(const tcb_conv_plan* plan, const void* dy, const void* w,
                   const void* residual_grad, const void* mask_act, void* dx, void* workspace,
                   void* stream);

/* dw = sum_{n,ho,wo} dy (x) x  (fp32, KRSC) and db = sum dy (fp32, K; may be
 * NULL). Deterministic (fixed-order split reduction, no float atomics). */
int tcb_conv_wgrad(const tcb_conv_plan* plan, const void* dy, const void* x, float* dw,
                   float* db, void* workspace, void* stream);

/* --------------------------------------------------------- other layers -- */
/* max pool (pooling layers of the chain: depth preserved, Eq 1 geometry). */
int tcb_maxpool_fwd(int dtype, const void* x, void* y, uint8_t* argmax, int n, int h, int w,
                    int c, int f, int stride, int pad, void* stream);
int tcb_maxpool_bwd(int dtype, const void* dy, const uint8_t* argmax, void* dx, int n, int h,
                    int w, int c, int f, int stride, int pad, void* stream);
/* Backward of maxpool(relu(x)) in one pass: y is the pool output; windows
 * with y <= 0 route no gradient (y equals the ReLU'd input at the argmax). */
int tcb_maxpool_relu_bwd(int dtype, const void* dy, const uint8_t* argmax, const void* y, void* dx,
                         int n, int h, int w, int c, int f, int stride, int pad, void* stream);
int tcb_avgpool_global_fwd(int dtype, const void* x, void* y, int n, int hw, int c, void* stream);
/* Windowed average pool (Inception's branch pool), padding counted (/ f*f);
 * c must fill 16-byte vectors (8 bf16 / 4 fp32). The backward optionally
 * fuses the ReLU mask of the pool input (mask_act may be NULL). */
int tcb_avgpool2d_fwd(int dtype, const void* x, void* y, int n, int h, int w, int c, int f, int stride,
                      int pad, void* stream);
int tcb_avgpool2d_bwd(int dtype, const void* dy, const void* mask_act, void* dx, int n, int h, int w, int c,
                      int f, int stride, int pad, void* stream);
/* rows x width elements between row-pitched buffers: channel concat of NHWC
 * tensors (forward) and the split of its gradient (backward). */
int tcb_slice_copy(int dtype, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                   size_t rows, void* stream);
int tcb_avgpool_global_bwd(int dtype, const void* dy, void* dx, int n, int hw, int c,
                           void* stream);
/* mean softmax cross-entropy over n rows of `classes` logits; writes
 * dlogits = (softmax - onehot)/n and the mean loss (device float). */
int tcb_softmax_xent(int dtype, const void* logits, const int32_t* labels, void* dlogits,
                     float* loss, int n, int classes, void* stream);

/* ------------------------------------------------------ synthetic inputs -- */
/* Counter-based uniform fill, identical stream on CPU (oracle) and GPU:
 * u = splitmix64(seed ^ tag*0x9E3779B97F4A7C15 ^ i) -> 24-bit -> [lo, hi). */
int tcb_fill_uniform(int dtype, void* p, size_t n, uint64_t seed, uint64_t tag, float lo,
                     float hi, void* stream);
int tcb_fill_labels(int32_t* labels, int n, int classes, uint64_t seed, void* stream);
int tcb_cast(int src_dtype, const void* src, int dst_dtype, void* dst, size_t n, void* stream);

/* ----------------------------------------------------- parameter update -- */
/* Fused momentum SGD on one PS shard (paper step 6):
 *   g' = grad*grad_scale + weight_decay*w;  v = momentum*v + g';  w -= lr*v
 * and refreshes the compute-dtype copy (w_compute, may be NULL). */
int tcb_sgd_momentum(float* w, const float* grad, float* v, int compute_dtype, void* w_compute,
                     size_t n, float lr, float momentum, float weight_decay, float grad_scale,
                     void* stream);

/* Fused PS step of one shard over NVSwitch multicast (what the trainer's
 * NVLS path launches): grad_mc / wcompute_mc are multicast addresses of the
 * fp32 gradient and bf16 weight buffers, grad / w / v this GPU's buffers;
 * elements [begin, begin + n), n and begin multiples of 4. */
int tcb_ps_nvls_update(const float* grad_mc, float* grad, float* w, float* v, void* wcompute_mc,
                       size_t begin, size_t n, float lr, float momentum, float weight_decay,
                       float grad_scale, void* stream);
/* All-GPU barrier on P2P-mapped signal pads (slots slot0 + rank); epoch_dev
 * is a zero-initialised device u32 per rank. The wait is bounded: a peer that
 * does not arrive within timeout_ns sets *err_dev = 1 and the kernel returns
 * (failure detection instead of a hung GPU). */
int tcb_nvls_barrier(void* const* signal_pads_dev, uint32_t* epoch_dev, int rank, int world, int slot0,
                     uint32_t* err_dev, uint64_t timeout_ns, void* stream);
/* Microbenchmark halves of tcb_ps_nvls_update: mode 1 = multicast reduce only,
 * 2 = multicast store only. */
int tcb_nvls_probe(int mode, const float* grad_mc, float* grad, const float* w, void* wcompute_mc,
                   size_t begin, size_t n, void* stream);

/* ------------------------------------------------------------ profiler -- */
/* Measures every (conv layer, algorithm, mini-batch) on this GPU and returns
 * the reference's cost catalog: rows of traincap::CostEntry
 * (/root/reference/proj/include/traincap/catalog.hpp:19-27) as CSV in the
 * reference's format (time_seconds = median fwd+dgrad+wgrad, memory_bits =
 * 8 * workspace bytes; inapplicable algorithms produce no row). Request and
 * reply are JSON (see csrc/runtime/profiler.cpp); free the reply with tcb_free. */
int tcb_profile_catalog(const char* request_json, char** reply_out);

/* ------------------------------------------------------------- trainer -- */
/* A whole data-parallel training step on one GPU: fwd chain -> loss ->
 * bwd (dgrad + wgrad into the flat PS gradient buffer) -> PS aggregation
 * (reduce-scatter over NCCL when world > 1) -> fused momentum SGD on the
 * owned shard -> all-gather of updated weights. Model and options are a JSON
 * document (see paper_1709_06622_b200/models.py). */
typedef struct tcb_trainer tcb_trainer;

int tcb_trainer_create(const char* config_json, tcb_trainer** out);
/* The step's exact HBM layout for a model config, without a GPU or any
 * allocation: JSON {"arena_bytes", "algorithm_workspace_bytes",
 * "resident_bytes" (arena minus conv workspaces: activations, gradients,
 * fan-in temporaries, parameters, momentum, staging), "param_padded", ...}
 * (free with tcb_free). The planner's memory model for branched graphs. */
int tcb_trainer_layout(const char* config_json, char** json_out);
int tcb_trainer_destroy(tcb_trainer* t);
/* NCCL unique id for rank 0 to broadcast (128 bytes). */
int tcb_nccl_unique_id(uint8_t* id128);
/* Join a world of `world` ranks (one process per GPU). world == 1 needs no id. */
int tcb_trainer_join(tcb_trainer* t, int rank, int world, const uint8_t* id128);
/* NVSwitch-multicast parameter-server step (after join, before the first
 * step; bf16, PS shards = GPUs): the flat fp32 gradient buffer and the bf16
 * compute-weight buffer (param_padded elements each, see describe) live in
 * caller-allocated symmetric memory bound to multicast objects (e.g. torch
 * symmetric memory). `grad`/`wcompute` are this GPU's buffers, `*_mc` their
 * multicast addresses, `signal_pads_dev` a device array of the world's
 * P2P-mapped signal pads of signal_pad_bytes each (the barrier uses the slots
 * min(2048, words - world) .. + world - 1; pads under 256 + world words are
 * rejected). A peer that never reaches the barrier is reported by
 * tcb_trainer_health / tcb_trainer_loss as TCB_ERR_NCCL instead of hanging.
 * Each step then runs barrier -> one kernel (multimem reduce of the own
 * shard + momentum SGD + multimem store of the bf16 weights) -> barrier,
 * replacing NCCL reduce-scatter / SGD / all-gather. */
int tcb_trainer_attach_nvls(tcb_trainer* t, void* grad, const void* grad_mc, void* wcompute,
                            void* wcompute_mc, void* const* signal_pads_dev, size_t signal_pad_bytes);
/* Asynchronous PS (config "ps_async": the aggregation + update of step s runs
 * on the trainer's own stream behind step s+1, which computes with weights
 * one update old — the paper's asynchronous policy): over
 * NVLS the second bf16 weight buffer is caller-provided too. */
int tcb_trainer_attach_nvls_async(tcb_trainer* t, void* wcompute2, void* wcompute2_mc);
/* Makes `stream` wait for every update issued so far (asynchronous PS; no-op
 * otherwise). */
int tcb_trainer_finish(tcb_trainer* t, void* stream);
/* Loads a mini-batch from HOST memory (NHWC fp32 images, int32 labels). NULL
 * images = keep the device-resident synthetic batch. */
int tcb_trainer_set_batch(tcb_trainer* t, const float* host_images, const int32_t* host_labels,
                          void* stream);
/* Pipelined input (the paper's steps 2-4 hidden behind compute): copies a
 * host batch (pinned for overlap) into one of two device staging slots on the
 * trainer's own copy stream and returns; the next tcb_trainer_step consumes
 * the oldest staged batch (waiting on its copy, converting it on the device).
 * format: TCB_INPUT_F32 (NHWC fp32) or TCB_INPUT_U8 (NHWC uint8 pixels u,
 * x = (u + 0.5) / 128 - 1). At most two batches may be staged ahead. */
enum { TCB_INPUT_F32 = 0, TCB_INPUT_U8 = 1 };
int tcb_trainer_stage_batch(tcb_trainer* t, const void* host_images, int format,
                            const int32_t* host_labels);
int tcb_trainer_step(tcb_trainer* t, void* stream);
int tcb_trainer_loss(tcb_trainer* t, float* loss_host, void* stream);
/* Failure detection (synchronises `stream`): NCCL asynchronous errors (the
 * communicators are aborted, never left hanging) and the NVLS barrier's bounded
 * wait ($TCB_NVLS_TIMEOUT_MS, default 10 s). TCB_ERR_NCCL once a peer failed;
 * the trainer stays failed. tcb_trainer_step polls the NCCL half (no sync) and
 * tcb_trainer_loss runs the whole check. */
int tcb_trainer_health(tcb_trainer* t, void* stream);
/* Per-phase device times of the last timed step (ms): fwd, bwd, reduce-scatter,
 * sgd, all-gather — the StepTrace the Lemma-1 estimate consumes. */
int tcb_trainer_phase_times(tcb_trainer* t, float* ms5);
int tcb_trainer_enable_timing(tcb_trainer* t, int on);
/* Paper steps 3-4 of the last staged batch consumed while timing was on:
 * {host-to-device copy ms on the copy stream, on-device preparation ms}
 * (-1 where none was timed). */
int tcb_trainer_data_times(tcb_trainer* t, float* ms2);
/* Introspection for tests: JSON description of the layer table, flat-buffer
 * layout (per-layer offsets) and shard table; caller frees with tcb_free. */
int tcb_trainer_describe(tcb_trainer* t, char** json_out);
/* Device pointers of named tensors ("param", "grad", "momentum", "act:<i>",
 * "dact:<i>", "input", "labels", "logits", "wcompute"). */
int tcb_trainer_tensor(tcb_trainer* t, const char* name, void** ptr, size_t* bytes);
/* Per-conv-pass CUDA events inside a real step (fwd, dgrad, wgrad of every conv
 * layer) -> per-layer CostEntry times under real cache state; JSON list, free
 * with tcb_free. */
int tcb_trainer_enable_layer_timing(tcb_trainer* t, int on);
int tcb_trainer_layer_times(tcb_trainer* t, char** json_out);
/* Count of kernels launched by the last step (for the bench's gpu_launches). */
int tcb_trainer_launch_count(tcb_trainer* t, int* count);
void tcb_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* TCB_H_ */
