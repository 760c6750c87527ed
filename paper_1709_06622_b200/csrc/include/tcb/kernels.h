// Host-side declarations of every kernel launcher in csrc/cuda/*.cu. The
// runtime (csrc/runtime) calls only these; all take a cudaStream_t and return
// cudaError_t from the launch (asynchronous errors surface at the next sync).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tcb {

struct ConvGeom {
    int n, h, w, c, k, r, s, pad_h, pad_w, stride_h, stride_w;
    // channels of x that can be non-zero (the rest are bf16 channel padding,
    // always zero); 0 = all c. Lets narrow first layers drop the padding.
    int c_valid = 0;
    int ho() const { return (h + 2 * pad_h - r) / stride_h + 1; }
    int wo() const { return (w + 2 * pad_w - s) / stride_w + 1; }
};

enum class ConvMode { Fwd = 0, Dgrad = 1, Wgrad = 2 };
enum class DType { F32 = 0, BF16 = 1 };

inline size_t dtype_size(DType t) { return t == DType::F32 ? 4 : 2; }

// Epilogue options shared by fwd / dgrad.
struct Epilogue {
    const float* bias = nullptr;     // [Ncol] fp32, fwd only
    const void* residual = nullptr;  // same dtype/shape as the output, added before act
    const void* mask = nullptr;      // dgrad: multiply by [mask > 0]
    bool relu = false;               // fwd: max(0, .)
    // dgrad: dx pixels no filter tap reaches (stride phases without taps, e.g. the
    // odd pixels of a 1x1 stride-2 conv) already hold 0 -- skip writing them
    // (only without residual / mask)
    bool uncovered_zero = false;
    // fwd of a row-window stem (conv_stem.cu): also max-pool the ReLU'd output 3x3 / stride 2 /
    // pad 1 into pool_y ([N][Ho/2][Wo/2][K]) and its argmax (uint8, maxpool_fwd's encoding)
    void* pool_y = nullptr;
    uint8_t* pool_arg = nullptr;
};

// ---- tensor-core implicit GEMM (tcgen05 / TMEM), bf16 in, fp32 accumulate ----
// Requirements: C % 8 == 0 (fwd/wgrad), K % 8 == 0 (dgrad/wgrad).
// wTp (dgrad) is w packed per stride phase by pack_dgrad_weights.
// Narrow-input convs (c_valid * R * S far below C * R * S, e.g. the 3-channel
// stem) run as a plain GEMM over an explicit im2col in `workspace`; without a
// workspace they take the implicit im2col path.
size_t conv_tc_workspace(const ConvGeom& g, ConvMode mode);
int conv_tc_launches(const ConvGeom& g, ConvMode mode, bool cols_ready = false,
                     bool counters = false);  // kernels per call (fwd: cols_ready = stem input packed)
cudaError_t conv_tc_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep,
                        void* y, cudaStream_t st, void* workspace = nullptr, bool x_ready = false);
// Dgrad reads the KRSC filters `w` directly (MN-major TMA boxes) whenever its
// operands load by TMA; only gather-path geometries (conv_tc_dgrad_needs_pack)
// need `wT` = pack_dgrad_weights(w), otherwise it may be NULL.
bool conv_tc_dgrad_needs_pack(const ConvGeom& g);
cudaError_t conv_tc_dgrad(const ConvGeom& g, const void* dy, const void* w, const void* wT,
                          const Epilogue& ep, void* dx, cudaStream_t st);
// cols_ready: `workspace` still holds the forward pass's explicit im2col of x
// (narrow layers; the trainer gives them a dedicated workspace for the step).
// counters: a dedicated, zero-initialised int buffer of at least
// conv_tc_counter_ints() entries (self-resetting, reusable across calls, not
// shared with concurrent launches). With it, split-K partials are reduced
// inside the GEMM kernel; without it a separate split_reduce pass runs.
cudaError_t conv_tc_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw,
                          void* workspace, cudaStream_t st, bool cols_ready = false,
                          int* counters = nullptr);
inline constexpr int conv_tc_counter_ints() { return 2 * 1024; }
bool conv_tc_narrow(const ConvGeom& g);
// Batched plain GEMMs on the tcgen05 kernel (one launch for all planes): g is
// the 1x1 / stride-1 / unpadded conv of one plane; planes are contiguous.
cudaError_t conv_tc_fwd_batched(const ConvGeom& g, int batch, const void* x, const void* w, void* y,
                                cudaStream_t st);
size_t conv_tc_wgrad_batched_workspace(const ConvGeom& g, int batch);
cudaError_t conv_tc_wgrad_batched(const ConvGeom& g, int batch, const void* dy, const void* x, float* dw,
                                  void* workspace, cudaStream_t st);
bool conv_tc_supported(const ConvGeom& g, ConvMode mode);
// 1: always use the cp.async gather operand path (tests / A-B comparisons);
// 0: pick plain-TMA / im2col-TMA / gather per geometry.
void conv_tc_set_force_gather(int on);
// Test hook: configuration of the most recent conv_tc_kernel launch (mode,
// operand path 0 gather / 1 plain TMA / 2 im2col TMA / 3 8-channel im2col,
// tile width, TMA-epilogue slots, CTA pair, split-K factor, work units, grid,
// in-kernel split reduction).
struct ConvTcLaunchInfo {
    int mode, load, bn, epi, cta2, splits, units, grid, fused_reduce, b_resident;
};
ConvTcLaunchInfo conv_tc_last_launch();
void conv_tc_note_launch(const ConvTcLaunchInfo& info);

// Window implicit GEMM (conv_win.cu): stride-1 R x S convs whose activation
// operand has whole 64-channel slices; one TMA window of padded input rows per
// tile and slice, every tap a shifted UMMA descriptor into it (fwd, and the
// stride-1 dgrad over dy with flipped taps). Operand path 4 in ConvTcLaunchInfo.
bool conv_win_applies(const ConvGeom& g, ConvMode mode);
cudaError_t conv_win_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep, void* y,
                         cudaStream_t st);
cudaError_t conv_win_dgrad(const ConvGeom& g, const void* dy, const void* w, const Epilogue& ep, void* dx,
                           cudaStream_t st);
void conv_win_set_mode(int on);  // 0 off, 1 on (N = 64 tiles), 2 all applicable, -1 from $TCB_WIN
// Window weight gradient (stride-1 R x S, C and K multiples of 64, M tiles x K
// <= 512 TMEM columns): per-CTA fp32 partials in `workspace`, then a split reduction.
bool conv_win_wgrad_applies(const ConvGeom& g);
size_t conv_win_wgrad_workspace(const ConvGeom& g);
int conv_win_wgrad_launches(const ConvGeom& g);  // tap-group launches + the split reduction
cudaError_t conv_win_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw, void* workspace,
                           cudaStream_t st);
void conv_win_set_debug(void* buf);
// Row-window stem (conv_stem.cu): even-stride first layers over <= 4 real
// channels of an 8-channel input (ResNet 7x7/2, Inception 3x3/2). The input is
// repacked once to 4-channel rows with zero padding columns in `workspace`
// (kept for the weight gradient: x_ready), and one overlapping-row TMA box per
// filter row is the GEMM A tile of a whole output row; no patch matrix.
// Operand path 5 in ConvTcLaunchInfo.
bool conv_stem_applies(const ConvGeom& g);
size_t conv_stem_workspace(const ConvGeom& g);
int conv_stem_launches(const ConvGeom& g, ConvMode mode, bool x_ready);
cudaError_t conv_stem_fwd(const ConvGeom& g, const void* x, const void* w, const Epilogue& ep, void* y,
                          void* workspace, cudaStream_t st, bool x_ready = false);
// The 4-channel rows at the head of the stem workspace, from the 8-channel
// activation x, or straight from uint8 pixels (cl channels per pixel) with the
// executor's input normalisation, also writing the 8-channel activation x8
// when it is not NULL.
cudaError_t conv_stem_pack_input(const ConvGeom& g, const void* x, void* workspace, cudaStream_t st);
cudaError_t conv_stem_pack_u8(const ConvGeom& g, const uint8_t* src, int cl, void* x8, void* workspace,
                              cudaStream_t st);
cudaError_t conv_stem_wgrad(const ConvGeom& g, const void* dy, const void* x, float* dw, void* workspace,
                            cudaStream_t st, bool x_ready);
// the stem forward can also produce the following 3x3 / 2 / 1 max pool (Epilogue::pool_y)
bool conv_stem_pool_fusable(const ConvGeom& g);
void conv_stem_set_mode(int on);  // 0 off (explicit im2col path), 1 on, -1 from $TCB_STEM
  // diagnostics: per-CTA role timing (8 x u64 per CTA) or nullptr
// TMA epilogue for layers with at most `kb` 64-deep k-blocks (0 = never,
// -1 = default: $TCB_CONV_EPI_KB or 8).
void conv_tc_set_epi_kb(int kb);
// Persistent conv kernels use at most #SMs - sms CTAs (SMs kept free for
// communication kernels running concurrently).
void conv_tc_set_sm_reserve(int sms);

// ---- FP32 FFMA implicit GEMM (parity mode) ----
size_t conv_ffma_workspace(const ConvGeom& g, ConvMode mode);
cudaError_t conv_ffma_fwd(const ConvGeom& g, const float* x, const float* w, const Epilogue& ep,
                          float* y, cudaStream_t st);
cudaError_t conv_ffma_dgrad(const ConvGeom& g, const float* dy, const float* w,
                            const Epilogue& ep, float* dx, cudaStream_t st);
cudaError_t conv_ffma_wgrad(const ConvGeom& g, const float* dy, const float* x, float* dw,
                            void* workspace, cudaStream_t st);

// ---- TF32 tensor-core implicit GEMM (tcgen05 kind::tf32; fp32 storage) ----
// Requirements: C % 4 == 0 and K % 4 == 0 (16-byte fp32 chunks).
bool conv_tf32_supported(const ConvGeom& g);
// 1: always the cp.async gather operands; 0: 2-D / im2col TMA where the geometry
// allows (also $TCB_TF32_GATHER=1)
void conv_tf32_set_force_gather(int on);
size_t conv_tf32_workspace(const ConvGeom& g, ConvMode mode);
cudaError_t conv_tf32_fwd(const ConvGeom& g, const float* x, const float* w, const Epilogue& ep,
                          float* y, cudaStream_t st);
cudaError_t conv_tf32_dgrad(const ConvGeom& g, const float* dy, const float* w,
                            const Epilogue& ep, float* dx, cudaStream_t st);
cudaError_t conv_tf32_wgrad(const ConvGeom& g, const float* dy, const float* x, float* dw,
                            void* workspace, cudaStream_t st);

// ---- parameter-server step over NVSwitch multicast (ps_nvls.cu) ----
// Barrier across `world` GPUs on P2P-mapped signal pads (device array of
// per-rank pad pointers; slots slot0 .. slot0 + world - 1 are used);
// `epoch_dev` is a zero-initialised per-rank device counter.
cudaError_t nvls_barrier(uint32_t* const* pads_dev, uint32_t* epoch_dev, int slot0, int rank, int world,
                         cudaStream_t st, uint32_t* err_dev, uint64_t timeout_ns);
// Fused reduce-scatter + momentum SGD + all-gather of elements [begin, begin+n)
// of the flat buffer: grad_mc / wc_mc are multicast addresses of the fp32
// gradient and bf16 compute-weight buffers; grad, w, v are local.
cudaError_t ps_nvls_update(const float* grad_mc, float* grad, float* w, float* v, void* wc_mc, size_t begin,
                           size_t n, float lr, float mom, float wd, float gscale, cudaStream_t st);
// microbenchmark halves of ps_nvls_update: 1 = multicast reduce only, 2 = multicast store only
cudaError_t nvls_probe(int mode, const float* grad_mc, float* grad, const float* w, void* wc_mc, size_t begin,
                       size_t n, cudaStream_t st);

// ---- graph operators for branched networks (graph_ops.cu) ----
// rows x width elements from src (row pitch src_pitch) to dst (row pitch
// dst_pitch): concat forward / backward as channel-slice copies
cudaError_t slice_copy(DType dt, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                       size_t rows, cudaStream_t st);
// the same copy times [mask > 0] (bf16, 16-byte aligned rows; mask rows at dst_pitch): a concat
// input's gradient with its producer's ReLU in one pass
bool slice_copy_mask_supported(DType dt, const void* src, size_t src_pitch, const void* dst, size_t dst_pitch,
                               int width, const void* mask);
cudaError_t slice_copy_mask(DType dt, const void* src, size_t src_pitch, void* dst, size_t dst_pitch, int width,
                            size_t rows, const void* mask, cudaStream_t st);
// windowed average pool, padding counted (/ f*f); c % (16 B / element) == 0
bool avgpool2d_supported(DType dt, int c);
cudaError_t avgpool2d_fwd(DType dt, const void* x, void* y, int n, int h, int w, int c, int f, int s, int p,
                          cudaStream_t st);
// dx = [mask > 0] * (sum of the covering windows' dy / f^2); mask may be NULL
// residual (may alias dx): added before the mask — accumulating fan-in gradients in place
cudaError_t avgpool2d_bwd(DType dt, const void* dy, void* dx, int n, int h, int w, int c, int f, int s, int p,
                          cudaStream_t st, const void* mask = nullptr, const void* residual = nullptr);

// ---- Winograd F(2x2,3x3) (3x3, stride 1) ----
size_t winograd_workspace(const ConvGeom& g, ConvMode mode, DType dt);
bool winograd_supported(const ConvGeom& g);
cudaError_t winograd_fwd(const ConvGeom& g, DType dt, const void* x, const void* w,
                         const Epilogue& ep, void* y, void* ws, cudaStream_t st);
cudaError_t winograd_dgrad(const ConvGeom& g, DType dt, const void* dy, const void* w,
                           const Epilogue& ep, void* dx, void* ws, cudaStream_t st);
cudaError_t winograd_wgrad(const ConvGeom& g, DType dt, const void* dy, const void* x, float* dw,
                           void* ws, cudaStream_t st);

// ---- FFT convolution (stride 1) ----
size_t fft_workspace(const ConvGeom& g, ConvMode mode);
bool fft_supported(const ConvGeom& g);
cudaError_t fft_fwd(const ConvGeom& g, DType dt, const void* x, const void* w, const Epilogue& ep,
                    void* y, void* ws, cudaStream_t st);
cudaError_t fft_dgrad(const ConvGeom& g, DType dt, const void* dy, const void* w,
                      const Epilogue& ep, void* dx, void* ws, cudaStream_t st);
cudaError_t fft_wgrad(const ConvGeom& g, DType dt, const void* dy, const void* x, float* dw,
                      void* ws, cudaStream_t st);

// ---- elementwise / layout / reductions ----
cudaError_t fill_uniform(DType dt, void* p, size_t n, uint64_t seed, uint64_t tag, float lo,
                         float hi, cudaStream_t st);
cudaError_t fill_labels(int32_t* labels, int n, int classes, uint64_t seed, cudaStream_t st);
cudaError_t cast(DType src_t, const void* src, DType dst_t, void* dst, size_t n, cudaStream_t st);
// [K][R][S][C] -> [C][R][S][K]
cudaError_t transpose_krsc(DType dt, const void* w, void* wT, int K, int R, int S, int C,
                           cudaStream_t st);
// [K][R][S][C] -> per stride-phase packed [C][taps_r][taps_s][K] blocks (the dgrad
// B operand of conv_tc_dgrad; same total size as w; plain transpose at stride 1).
cudaError_t pack_dgrad_weights(DType dt, const void* w, void* packed, const ConvGeom& g,
                               cudaStream_t st);
// All bf16 dgrad packings of a network in one launch (job table in device memory).
struct PackDgradJob {
    const void* w;
    void* out;
    ConvGeom g;
    int block_begin;  // prefix sum of pack_dgrad_blocks over earlier jobs
};
int pack_dgrad_blocks(const ConvGeom& g);
cudaError_t pack_dgrad_weights_batched(const PackDgradJob* jobs, int njobs, int total_blocks,
                                       cudaStream_t st);
// out[j] = sum_i in[i][j] (rows x cols, fp32 result), deterministic.
cudaError_t column_sum(DType dt, const void* in, float* out, int rows, int cols, float* ws,
                       cudaStream_t st);
size_t column_sum_workspace(int rows, int cols);
// out[i] = sum_s parts[s][i] (fixed order)
cudaError_t split_reduce(const float* parts, int splits, size_t n, float* out, cudaStream_t st);
cudaError_t sgd_momentum(float* w, const float* g, float* v, DType cdt, void* wc, size_t n,
                         float lr, float mom, float wd, float gscale, cudaStream_t st);
// dst[px][c] = c < cl ? src[px][c] : 0 for c < cp (fp32 src, dst in dt): channel padding.
// uint8 NHWC pixels u -> (u + 0.5) / 128 - 1, channel-padded (staged host batches)
cudaError_t pack_channels_u8(DType dt, const uint8_t* src, void* dst, size_t pixels, int cl, int cp,
                             cudaStream_t st);
cudaError_t pack_channels(DType dt, const float* src, void* dst, size_t pixels, int cl, int cp,
                          cudaStream_t st);
cudaError_t add_inplace(DType dt, void* y, const void* x, size_t n, cudaStream_t st);
cudaError_t relu_mask_inplace(DType dt, void* g, const void* act, size_t n, cudaStream_t st);

cudaError_t maxpool_fwd(DType dt, const void* x, void* y, uint8_t* arg, int n, int h, int w,
                        int c, int f, int s, int p, cudaStream_t st);
// ymask (may be NULL): the pool OUTPUT y; windows with y <= 0 route no
// gradient. That is the fused ReLU backward of a ReLU'd pool input x: every
// window whose argmax is x[p] has y = x[p], so [x[p] > 0] == [y > 0] — and y
// is a quarter of x's size.
cudaError_t maxpool_bwd(DType dt, const void* dy, const uint8_t* arg, void* dx, int n, int h,
                        int w, int c, int f, int s, int p, cudaStream_t st,
                        const void* ymask = nullptr);
cudaError_t avgpool_global_fwd(DType dt, const void* x, void* y, int n, int hw, int c,
                               cudaStream_t st);
cudaError_t avgpool_global_bwd(DType dt, const void* dy, void* dx, int n, int hw, int c,
                               cudaStream_t st, const void* mask = nullptr);
// logits rows are `ld` apart (ld >= classes; padded columns get zero gradient)
cudaError_t softmax_xent(DType dt, const void* logits, const int32_t* labels, void* dlogits,
                         float* loss, int n, int classes, int ld, cudaStream_t st);

}  // namespace tcb
