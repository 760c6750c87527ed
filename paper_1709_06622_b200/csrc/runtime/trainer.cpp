// The data-parallel training step on one B200 (one process per GPU):
//
//   paper step 5  GPU processing : fwd chain -> softmax-xent -> bwd (dgrad +
//                                  wgrad straight into the flat PS gradient buffer)
//   paper step 7  distributed update : PS aggregation — ncclReduceScatter of
//                                  the flat fp32 gradient (N_ps = G) or grouped
//                                  ncclReduce to N_ps < G shard owners
//   paper step 6  parameter update : fused momentum-SGD on the owned shard,
//                                  refreshing the compute-dtype copy
//   paper step 1  parameter refresh : ncclAllGather (or per-owner broadcast)
//                                  of the updated compute-dtype weights
// (/root/reference/PAPER.md:229-238). Per-phase CUDA-event times form the
// StepTrace the reference's Lemma 1 consumes
// (/root/reference/proj/include/traincap/io.hpp:23-26).
//
// Memory: one cudaMalloc'ed HBM arena holds activations, gradients, flat
// parameter/gradient/momentum buffers and workspaces (bump-allocated,
// 256-byte aligned). The layer-to-PS-shard assignment: the
// parameters of conv layers 1..q (fc layers are convs spanning the whole
// spatial map) are flattened in layer order, [K][R][S][C] weights then bias,
// each segment 64-element aligned; the buffer is padded to G*64 elements and
// rank r owns [r*P/G, (r+1)*P/G).
#include <array>
#include <chrono>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <sstream>
#include <vector>

#include <cuda_runtime.h>
#include <json.hpp>
#include <nccl.h>

#include "runtime.h"
#include "tcb.h"
#include "tcb/kernels.h"

namespace tcb {
namespace {

using json = nlohmann::json;

constexpr size_t kAlign = 256;
constexpr size_t kParamAlign = 64;  // elements

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

enum class Op { Input, Conv, MaxPool, AvgPool, Loss, Concat };

struct Node {
    Op op = Op::Input;
    std::string name;
    int in = -1, residual = -1;
    // output tensor NHWC (c = allocated channels, c_logical = semantic channels)
    int n = 0, h = 0, w = 0, c = 0, c_logical = 0;
    // conv
    ConvGeom g{};
    bool bias = false, relu = false, need_dgrad = true;
    int conv_index = 0;
    size_t woff = 0, boff = 0, wcount = 0;  // flat param offsets (elements)
    size_t bcomp = 0;                        // offset in the compact fp32 bias copies
    float init_scale = 0.f;
    std::string algo = "gemm";
    int algo_id = 0;  // TCB_ALGO_*
    // pool (avgpool: f == 0 -> global average)
    int f = 0, s = 0, p = 0;
    // concat: inputs and their channel offsets in this tensor
    std::vector<int> ins, coff;
    // arena offsets (bytes)
    size_t act = 0, grad = 0, argmax = 0, wT = 0;
    size_t nws = 0;  // narrow (explicit im2col) layers: own workspace, col kept fwd -> wgrad
    bool narrow = false;
    bool pack_wT = false;  // bf16 dgrad on the gather path needs the packed w^T
    // backward plan for this node's OUTPUT tensor
    int final_writer = -1;              // consumer node that writes G[this] last
    std::vector<int> compute_from;      // consumers with a computed contribution
    std::vector<int> alias_from;        // consumers whose G[out] adds via the residual path
    std::map<int, size_t> tmp;          // consumer -> temp buffer offset (non-final computed)
    // non-final GEMM-conv consumers accumulate into one buffer through their
    // dgrad epilogue's residual input (in place), instead of a temp each plus
    // separate add passes at the final writer (Inception's 3-4 way fan-out)
    std::vector<int> chain;
    size_t acc = 0;
    int acc_written = 0;                // per step
    int grad_alias = -1;                // G[this] is G[grad_alias] (no copy)
};

struct Phase {
    cudaEvent_t e[6]{};
};

}  // namespace
}  // namespace tcb

using namespace tcb;

struct tcb_trainer {
    json cfg;
    DType dt = DType::BF16;
    bool bf16 = true;
    bool tf32 = false;  // fp32 storage, GEMM convs on tcgen05 kind::tf32
    int cpad = 8;       // channel padding of the tensor-core layouts (16-byte rows)
    int batch = 0, classes = 0;
    uint64_t seed = 20260810;
    float lr = 0.01f, momentum = 0.9f, weight_decay = 0.f;
    std::vector<Node> nodes;
    int logits = -1;

    // distributed
    int rank = 0, world = 1, n_ps = 0;
    ncclComm_t comm = nullptr;
    size_t param_count = 0;   // logical (unpadded) parameter elements
    size_t param_padded = 0;  // padded to world * kParamAlign
    size_t shard = 0;

    // arena
    void* arena = nullptr;
    size_t arena_bytes = 0;
    size_t algorithm_ws_bytes = 0;  // conv workspaces inside the arena (depend on the algorithms)
    size_t off_param = 0, off_grad = 0, off_mom = 0, off_wc = 0, off_ws = 0, off_colsum = 0;
    size_t off_labels = 0, off_loss = 0, off_input_f32 = 0;
    // staged host batches (pipelined H2D): two slots filled on a copy stream,
    // consumed in order by the next steps
    size_t off_stage[2] = {0, 0}, off_stage_labels[2] = {0, 0}, stage_bytes = 0;
    int stage_format[2] = {0, 0};
    uint64_t stage_w = 0, stage_r = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t staged[2]{}, consumed[2]{};
    // paper steps 3-4 measured into the StepTrace (timing mode): the staged
    // batch's host-to-device copy on the copy stream, its on-device preparation
    // (uint8 -> compute dtype, channel padding) on the step stream
    cudaEvent_t ev_h2d[2]{}, ev_prep[2]{};
    bool h2d_timed = false, prep_timed = false;
    bool consumed_recorded[2] = {false, false};
    size_t ws_bytes = 0, colsum_bytes = 0;
    size_t off_pack_jobs = 0;  // device table of the batched dgrad weight packing
    size_t off_counters = 0;   // split-K counters of the in-kernel wgrad reduction
    // Overlapped PS aggregation (N_ps = G): shard s is reduced to its owner on
    // the comm stream as soon as backward has written every gradient in it
    bool overlap = false;                   // config "overlap_comm" (measured: see DESIGN §6)
    cudaStream_t comm_stream = nullptr;
    // the overlapped shard reduces run on their own communicator limited to a
    // few CTAs, so they steal almost no SMs from the persistent conv kernels
    ncclComm_t comm_bg = nullptr;
    int comm_bg_ctas = 8;                   // config "overlap_ctas"
    std::vector<cudaEvent_t> ev_ready;      // per shard
    cudaEvent_t ev_comm_done = nullptr, ev_bwd_start = nullptr;
    std::map<int, std::vector<int>> shard_trigger;  // node index -> shards it completes
    bool fused_split_reduce = false;  // config "fused_split_reduce" / $TCB_FUSED_SPLIT_REDUCE
    // row-window stem conv reading the input (conv_stem.cu), -1 if none: every
    // write of the input activation also refreshes its 4-channel rows in the
    // layer's workspace, so the step never repacks them
    int stem_node = -1;
    // max pool node whose forward the stem kernel produces (3x3 / 2 / 1 right after a ReLU'd
    // stem that feeds nothing else; config "fuse_stem_pool"), -1 if none. Off by default:
    // bit-identical, but the epilogue pooling made the stem kernel 0.32 ms against 0.15 +
    // 0.12 ms for the stem and the separate pool kernel (ResNet-50 bs256)
    int fused_pool = -1;
    // CUDA graph of the step (config "cuda_graph", $TCB_GRAPH)
    bool use_graph = true;
    int eager_steps = 0, graph_launches = 0;
    cudaGraphExec_t graph_exec = nullptr;
    cudaStream_t graph_stream = nullptr;
    cudaEvent_t graph_in = nullptr, graph_out = nullptr;
    int pack_njobs = 0, pack_blocks = 0;
    bool pack_jobs_ready = false;

    cudaStream_t stream = nullptr;  // stream of the last step call
    bool timing = false;
    Phase ph;
    float phase_ms[5] = {0, 0, 0, 0, 0};
    int launches = 0;
    bool initialized = false;
    // per-conv-pass CUDA events inside a real step: [node][fwd0,fwd1,dgrad0,dgrad1,wgrad0,wgrad1]
    bool layer_timing = false;
    std::vector<std::array<cudaEvent_t, 6>> lev;
    cudaStream_t lev_stream = nullptr;

    // per-layer weight gradient on its own stream, concurrent with the layer's data
    // gradient and joined before the next layer (config / $TCB_BWD_CONCURRENT)
    cudaStream_t wg_stream = nullptr;
    cudaEvent_t wg_fork = nullptr, wg_join = nullptr;

    bool overlap_active() const {
        return overlap && world > 1 && (n_ps <= 0 || n_ps >= world) && comm_stream != nullptr;
    }
    void mark(size_t node, int slot, cudaStream_t st) {
        if (layer_timing) cudaEventRecord(lev[node][slot], st);
    }

    template <typename T = void>
    T* at(size_t off) const {
        return reinterpret_cast<T*>(static_cast<char*>(arena) + off);
    }

    // NVLS parameter-server path (tcb_trainer_attach_nvls): the fp32 gradient
    // and bf16 compute-weight buffers live in caller-provided symmetric memory
    // bound to NVSwitch multicast objects; RS + SGD + AG is one kernel.
    bool nvls = false;
    float* ext_grad = nullptr;
    const float* grad_mc = nullptr;
    void* ext_wc = nullptr;
    void* wc_mc = nullptr;
    uint32_t* const* pads_dev = nullptr;
    uint32_t* nvls_epoch = nullptr;  // [0] barrier epoch, [1] barrier timeout flag
    int nvls_slot0 = 2048;           // first signal-pad slot of the PS barrier
    uint64_t nvls_timeout_ns = 10ull * 1000 * 1000 * 1000;  // $TCB_NVLS_TIMEOUT_MS
    // failure detection: a collective that failed, or a barrier that
    // timed out, poisons the trainer; every later call reports it
    std::string failed;
    float* grad_ptr() const { return ext_grad ? ext_grad : at<float>(off_grad); }
    void* wc_ptr() const {
        if (async_ps) return wc_buf(wc_rd);
        return ext_wc ? ext_wc : at(off_wc);
    }

    // Asynchronous PS (config "ps_async"): the aggregation +
    // update of step s runs on its own stream, hidden behind step s+1, which
    // computes with the weights one update old (staleness 1). Double-buffered
    // bf16 weights: W_j lives in buffer j % 2; step s reads W_max(s-1,0) while
    // update s writes W_s+1 into the other buffer.
    bool async_ps = false;
    size_t off_wc2 = 0;
    void* ext_wc2 = nullptr;
    void* wc2_mc = nullptr;
    int wc_rd = 0;
    long long step_idx = 0;
    // fp32 biases the forward reads, refreshed from a bf16 weight buffer after
    // every update whenever the local fp32 master is not the source of truth
    // (world > 1: only the owned shard of it is current; asynchronous PS: the
    // step reads the weights one update old). One copy per weight buffer.
    bool bias_from_wc = false;
    size_t bias_total = 0, off_biasc[2] = {0, 0};
    cudaStream_t ps_stream = nullptr;
    cudaEvent_t ev_bwd_done = nullptr, ev_upd[2] = {nullptr, nullptr};
    void* wc_buf(int i) const {
        if (i == 0) return ext_wc ? ext_wc : at(off_wc);
        return ext_wc2 ? ext_wc2 : at(off_wc2);
    }
    void* wc_mc_buf(int i) const { return i == 0 ? wc_mc : wc2_mc; }
};

namespace tcb {
namespace {

#define TRY_CUDA(expr)                                           \
    do {                                                         \
        cudaError_t e__ = (expr);                                \
        if (e__ != cudaSuccess) return check_cuda(e__, #expr);   \
    } while (0)
#define TRY_NCCL(expr)                                                                    \
    do {                                                                                  \
        ncclResult_t r__ = (expr);                                                        \
        if (r__ != ncclSuccess)                                                           \
            return fail(TCB_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r__)); \
    } while (0)
#define TRY(expr)                     \
    do {                              \
        int rc__ = (expr);            \
        if (rc__ != TCB_OK) return rc__; \
    } while (0)

// --------------------------------------------------------------- build ----
int build_graph(tcb_trainer* t) {
    const json& cfg = t->cfg;
    const std::string prec = cfg.value("precision", std::string("bf16"));
    if (prec != "bf16" && prec != "tf32" && prec != "ffma")
        throw std::runtime_error("precision must be bf16, tf32 or ffma, got " + prec);
    t->bf16 = prec == "bf16";
    t->tf32 = prec == "tf32";
    t->cpad = t->bf16 ? 8 : t->tf32 ? 4 : 1;
    t->dt = t->bf16 ? DType::BF16 : DType::F32;
    t->batch = cfg.at("batch").get<int>();
    t->classes = cfg.at("classes").get<int>();
    t->seed = cfg.value("seed", uint64_t(20260810));
    t->overlap = t->cfg.value("overlap_comm", false);
    t->async_ps = cfg.value("ps_async", false);
    {
        const char* e = std::getenv("TCB_GRAPH");
        t->use_graph = t->cfg.value("cuda_graph", !(e && e[0] == '0')) && !t->async_ps;
    }
    t->comm_bg_ctas = t->cfg.value("overlap_ctas", 8);
    {
        const char* e = std::getenv("TCB_FUSED_SPLIT_REDUCE");
        t->fused_split_reduce = cfg.value("fused_split_reduce", e != nullptr && e[0] == '1');
    }
    t->lr = cfg.value("lr", 0.01f);
    t->momentum = cfg.value("momentum", 0.9f);
    t->weight_decay = cfg.value("weight_decay", 0.f);
    t->n_ps = cfg.value("n_ps", 0);
    t->world = cfg.value("world", 1);  // layout planning before join (join overrides)

    std::map<std::string, int> by_name;
    // bf16: conv outputs narrower than 64 channels, and those read by a spatial
    // (R*S > 1) conv with K % 64 != 0, get K rounded up to 64 allocated channels,
    // so their consumers meet the im2col-TMA operand path (whole 64-channel
    // slices) instead of the cp.async gather; the extra channels are zero
    // filters and stay exactly 0. Not for tensors that feed a channel concat.
    const bool pad_narrow = t->bf16 && cfg.value("pad_narrow_channels", true);
    std::set<std::string> concat_inputs, spatial_inputs;
    for (const json& L : cfg.at("layers")) {
        const std::string lop = L.value("op", std::string());
        if (lop == "concat")
            for (const json& nm : L.at("in")) concat_inputs.insert(nm.get<std::string>());
        if (lop == "conv" && L.value("r", 1) * L.value("s", L.value("r", 1)) > 1 && L.contains("in"))
            spatial_inputs.insert(L.at("in").get<std::string>());
    }
    int conv_idx = 0;
    for (const json& L : cfg.at("layers")) {
        Node nd;
        nd.name = L.at("name").get<std::string>();
        const std::string op = L.at("op").get<std::string>();
        auto src = [&](const char* key) -> int {
            if (!L.contains(key) || L.at(key).is_null()) return -1;
            auto it = by_name.find(L.at(key).get<std::string>());
            if (it == by_name.end()) throw std::runtime_error("unknown tensor " + L.at(key).dump());
            return it->second;
        };
        if (op == "input") {
            nd.op = Op::Input;
            nd.n = t->batch;
            nd.h = L.at("h").get<int>();
            nd.w = L.at("w").get<int>();
            nd.c_logical = L.at("c").get<int>();
            nd.c = static_cast<int>(round_up(nd.c_logical, t->cpad));
        } else if (op == "conv") {
            nd.op = Op::Conv;
            nd.in = src("in");
            nd.residual = src("residual");
            const Node& x = t->nodes.at(nd.in);
            // tensor-core paths: output channels padded to a multiple of 8 (bf16) / 4
            // (tf32) — 16-byte NHWC rows; padded filters are zero, so padded channels
            // stay exactly 0.
            const int k_logical = L.at("k").get<int>();
            const bool widen = pad_narrow && !concat_inputs.count(nd.name) &&
                               (k_logical < 64 || (k_logical % 64 != 0 && spatial_inputs.count(nd.name)));
            const int k_alloc = static_cast<int>(round_up(k_logical, widen ? 64 : t->cpad));
            nd.g = ConvGeom{x.n, x.h, x.w, x.c, k_alloc, L.at("r").get<int>(),
                            L.value("s", L.at("r").get<int>()), L.value("pad_h", L.value("pad", 0)),
                            L.value("pad_w", L.value("pad", 0)), L.value("stride_h", L.value("stride", 1)),
                            L.value("stride_w", L.value("stride", 1))};
            if (x.c_logical < x.c) nd.g.c_valid = x.c_logical;  // zero channel padding
            nd.bias = L.value("bias", false);
            nd.relu = L.value("relu", false);
            nd.algo = L.value("algo", std::string("gemm"));
            nd.n = x.n;
            nd.h = nd.g.ho();
            nd.w = nd.g.wo();
            nd.c = k_alloc;
            nd.c_logical = k_logical;
            nd.conv_index = ++conv_idx;
            nd.need_dgrad = t->nodes.at(nd.in).op != Op::Input;
            const int fan_in = x.c_logical * nd.g.r * nd.g.s;
            // He-uniform bound sqrt(6 / fan_in) times an optional gain (residual branches
            // of the BN-free ResNet use a small gain on their last conv, Fixup-style).
            nd.init_scale = L.value("init_gain", 1.0f) * std::sqrt(6.0f / static_cast<float>(fan_in));
            std::string why;
            if (nd.h < 1 || nd.w < 1 || !geom_valid(nd.g, &why))
                throw std::runtime_error("layer " + nd.name + ": bad geometry " + why);
            if (t->bf16 && !conv_tc_supported(nd.g, ConvMode::Fwd))
                throw std::runtime_error("layer " + nd.name + ": bf16 path needs C % 8 == 0");
            // the planner's per-layer algorithm (Selection.assignment) — obeyed as given
            nd.algo_id = nd.algo == "gemm" ? TCB_ALGO_GEMM
                         : nd.algo == "winograd" ? TCB_ALGO_WINOGRAD
                         : nd.algo == "fft" ? TCB_ALGO_FFT : -1;
            if (nd.algo_id < 0) throw std::runtime_error("layer " + nd.name + ": unknown algo " + nd.algo);
            // tf32 mode: GEMM layers on tensor cores; Winograd / FFT layers run their fp32 kernels
            const int lprec = t->bf16 ? TCB_PREC_BF16
                              : (t->tf32 && nd.algo_id == TCB_ALGO_GEMM) ? TCB_PREC_TF32
                                                                         : TCB_PREC_FFMA_FP32;
            if (!algo_applies(nd.g, nd.algo_id, lprec))
                throw std::runtime_error("layer " + nd.name + ": algorithm " + nd.algo +
                                         " does not apply to this geometry");
            if (nd.residual >= 0) {
                const Node& r = t->nodes.at(nd.residual);
                if (r.h != nd.h || r.w != nd.w || r.c != nd.c)
                    throw std::runtime_error("layer " + nd.name + ": residual shape mismatch");
            }
        } else if (op == "maxpool" || op == "avgpool") {
            nd.op = op == "maxpool" ? Op::MaxPool : Op::AvgPool;
            nd.in = src("in");
            const Node& x = t->nodes.at(nd.in);
            nd.n = x.n;
            nd.c = x.c;
            nd.c_logical = x.c_logical;
            if (nd.op == Op::MaxPool) {
                nd.f = L.at("f").get<int>();
                nd.s = L.value("stride", nd.f);
                nd.p = L.value("pad", 0);
                nd.h = (x.h + 2 * nd.p - nd.f) / nd.s + 1;
                nd.w = (x.w + 2 * nd.p - nd.f) / nd.s + 1;
                if (nd.f > 15 || nd.h < 1 || nd.w < 1)
                    throw std::runtime_error("layer " + nd.name + ": bad pool window");
            } else if (L.contains("f")) {
                // windowed average pool (Inception's 3x3 / s1 / p1 branch pool)
                nd.f = L.at("f").get<int>();
                nd.s = L.value("stride", nd.f);
                nd.p = L.value("pad", 0);
                nd.h = (x.h + 2 * nd.p - nd.f) / nd.s + 1;
                nd.w = (x.w + 2 * nd.p - nd.f) / nd.s + 1;
                if (nd.f < 1 || nd.h < 1 || nd.w < 1 || !avgpool2d_supported(t->dt, nd.c))
                    throw std::runtime_error("layer " + nd.name + ": bad average-pool window / channels");
            } else {
                nd.h = nd.w = 1;
            }
        } else if (op == "concat") {
            // channel concatenation of same-size NHWC tensors (Inception branch outputs)
            nd.op = Op::Concat;
            for (const json& nm : L.at("in")) {
                auto it = by_name.find(nm.get<std::string>());
                if (it == by_name.end()) throw std::runtime_error("unknown tensor " + nm.dump());
                const Node& x = t->nodes.at(it->second);
                if (nd.ins.empty()) {
                    nd.n = x.n;
                    nd.h = x.h;
                    nd.w = x.w;
                } else if (x.n != nd.n || x.h != nd.h || x.w != nd.w) {
                    throw std::runtime_error("layer " + nd.name + ": concat inputs differ in size");
                }
                if (x.c != x.c_logical)
                    throw std::runtime_error("layer " + nd.name + ": concat input " + x.name +
                                             " has padded channels");
                nd.ins.push_back(it->second);
                nd.coff.push_back(nd.c);
                nd.c += x.c;
            }
            if (nd.ins.size() < 2) throw std::runtime_error("layer " + nd.name + ": concat needs 2+ inputs");
            nd.c_logical = nd.c;
            nd.in = nd.ins[0];
        } else if (op == "loss") {
            nd.op = Op::Loss;
            nd.in = src("in");
            const Node& x = t->nodes.at(nd.in);
            if (x.h != 1 || x.w != 1 || x.c_logical != t->classes)
                throw std::runtime_error("loss input must be N x 1 x 1 x classes");
            t->logits = nd.in;
        } else {
            throw std::runtime_error("unknown op " + op);
        }
        by_name[nd.name] = static_cast<int>(t->nodes.size());
        t->nodes.push_back(std::move(nd));
    }
    if (t->logits < 0) throw std::runtime_error("model has no loss layer");

    // Backward plan: who contributes to each tensor's gradient.
    const int count = static_cast<int>(t->nodes.size());
    for (int i = 0; i < count; ++i) {
        const Node& nd = t->nodes[i];
        if (nd.op == Op::Conv) {
            if (nd.need_dgrad) t->nodes[nd.in].compute_from.push_back(i);
            if (nd.residual >= 0 && t->nodes[nd.residual].op != Op::Input)
                t->nodes[nd.residual].alias_from.push_back(i);
        } else if (nd.op == Op::MaxPool || nd.op == Op::AvgPool) {
            if (t->nodes[nd.in].op != Op::Input) t->nodes[nd.in].compute_from.push_back(i);
        } else if (nd.op == Op::Concat) {
            for (int j : nd.ins)
                if (t->nodes[j].op != Op::Input) t->nodes[j].compute_from.push_back(i);
        }
    }
    for (Node& nd : t->nodes) {
        if (!nd.compute_from.empty())
            nd.final_writer = *std::min_element(nd.compute_from.begin(), nd.compute_from.end());
        // A tensor whose gradient arrives only through one residual path and whose
        // producer has no ReLU (a projection shortcut) shares that gradient buffer.
        nd.grad_alias = nd.compute_from.empty() && nd.alias_from.size() == 1 && !nd.relu
                            ? nd.alias_from[0]
                            : -1;
    }
    return TCB_OK;
}

// ---------------------------------------------------------------- arena ---
struct Bump {
    size_t top = 0;
    size_t take(size_t bytes) {
        const size_t off = top;
        top += round_up(std::max<size_t>(bytes, 1), kAlign);
        return off;
    }
};

void plan_params(tcb_trainer* t) {
    size_t off = 0, logical = 0;
    for (Node& nd : t->nodes) {
        if (nd.op != Op::Conv) continue;
        nd.wcount = size_t(nd.g.k) * nd.g.r * nd.g.s * nd.g.c;
        nd.woff = off;
        off = round_up(off + nd.wcount, kParamAlign);
        logical += size_t(nd.c_logical) * nd.g.r * nd.g.s * t->nodes[nd.in].c_logical;
        if (nd.bias) {
            nd.boff = off;
            off = round_up(off + nd.g.k, kParamAlign);
            logical += nd.c_logical;
        }
    }
    t->bias_total = 0;
    for (Node& nd : t->nodes)
        if (nd.op == Op::Conv && nd.bias) {
            nd.bcomp = t->bias_total;
            t->bias_total += nd.g.k;
        }
    t->param_count = logical;
    const size_t unit = size_t(t->world) * kParamAlign;
    t->param_padded = round_up(std::max<size_t>(off, 1), unit);
    t->shard = t->param_padded / t->world;
    // shard s is complete after the backward wgrad of the lowest-index conv
    // touching it (backward runs from the last node down); shards holding only
    // padding go out with the first wgrad
    t->shard_trigger.clear();
    {
        std::vector<int> first_node(t->world, -1);
        int last_conv = -1;
        for (int i = 0; i < static_cast<int>(t->nodes.size()); ++i) {
            const Node& nd = t->nodes[i];
            if (nd.op != Op::Conv) continue;
            last_conv = i;
            const size_t lo = nd.woff, hi = (nd.bias ? nd.boff + nd.g.k : nd.woff + nd.wcount);
            for (size_t sh = lo / t->shard; sh < static_cast<size_t>(t->world) && sh * t->shard < hi; ++sh)
                if (first_node[sh] < 0) first_node[sh] = i;
        }
        for (int sh = t->world - 1; sh >= 0; --sh)
            t->shard_trigger[first_node[sh] >= 0 ? first_node[sh] : last_conv].push_back(sh);
    }
}

// dry: lay the arena out (offsets, arena_bytes, algorithm_ws_bytes) without
// allocating — the exact HBM need of the step for the planner (tcb_trainer_layout)
int allocate(tcb_trainer* t, bool dry = false) {
    const size_t es = dtype_size(t->dt);
    Bump b;
    plan_params(t);
    t->off_param = b.take(t->param_padded * 4);
    t->off_grad = b.take(t->param_padded * 4);
    t->off_mom = b.take(t->param_padded * 4);  // only the owned shard is used
    t->off_wc = t->bf16 ? b.take(t->param_padded * 2) : t->off_param;
    if (t->async_ps) t->off_wc2 = b.take(t->param_padded * 2);
    t->bias_from_wc = t->bf16 && (t->world > 1 || t->async_ps) && t->bias_total > 0;
    if (t->bias_from_wc)
        for (int k = 0; k < (t->async_ps ? 2 : 1); ++k) t->off_biasc[k] = b.take(t->bias_total * 4);
    size_t ws = 0, colsum = 0;
    for (Node& nd : t->nodes) {
        const size_t elems = size_t(nd.n) * nd.h * nd.w * nd.c;
        if (nd.op == Op::Loss) continue;
        nd.act = b.take(elems * es);
        if (nd.op != Op::Input && nd.grad_alias < 0) nd.grad = b.take(elems * es);
        if (nd.op == Op::MaxPool) nd.argmax = b.take(elems);
        if (nd.op == Op::Conv) {
            nd.narrow = t->bf16 && nd.algo_id == TCB_ALGO_GEMM && conv_tc_narrow(nd.g);
            if (nd.narrow && nd.in == 0 && conv_stem_applies(nd.g))
                t->stem_node = static_cast<int>(&nd - t->nodes.data());
            if (nd.algo_id == TCB_ALGO_GEMM) {
                if (nd.narrow) {
                    const size_t nb = std::max(conv_tc_workspace(nd.g, ConvMode::Wgrad),
                                               conv_tc_workspace(nd.g, ConvMode::Fwd));
                    nd.nws = b.take(nb);
                    t->algorithm_ws_bytes += round_up(std::max<size_t>(nb, 1), kAlign);
                }
                else
                    ws = std::max(ws, t->bf16   ? std::max(conv_tc_workspace(nd.g, ConvMode::Wgrad),
                                                           conv_tc_workspace(nd.g, ConvMode::Fwd))
                                      : t->tf32 ? conv_tf32_workspace(nd.g, ConvMode::Wgrad)
                                                : conv_ffma_workspace(nd.g, ConvMode::Wgrad));
                nd.pack_wT = t->bf16 && nd.need_dgrad && conv_tc_dgrad_needs_pack(nd.g);
                if (nd.pack_wT) nd.wT = b.take(nd.wcount * 2);
            } else {
                // Winograd / FFT transformed planes; one shared region, passes run in order
                for (ConvMode m : {ConvMode::Fwd, ConvMode::Dgrad, ConvMode::Wgrad})
                    ws = std::max(ws, nd.algo_id == TCB_ALGO_WINOGRAD ? winograd_workspace(nd.g, m, t->dt)
                                                                      : fft_workspace(nd.g, m));
            }
            if (nd.bias) colsum = std::max(colsum, column_sum_workspace(nd.n * nd.h * nd.w, nd.g.k));
        }
    }
    t->fused_pool = -1;
    if (t->stem_node >= 0 && t->cfg.value("fuse_stem_pool", false)) {
        const Node& sn = t->nodes[t->stem_node];
        int consumers = 0, pool = -1;
        for (size_t j = 0; j < t->nodes.size(); ++j) {
            const Node& c = t->nodes[j];
            bool uses = c.in == t->stem_node || c.residual == t->stem_node;
            for (int k : c.ins) uses = uses || k == t->stem_node;
            if (!uses) continue;
            ++consumers;
            if (c.op == Op::MaxPool && c.in == t->stem_node && c.f == 3 && c.s == 2 && c.p == 1) pool = static_cast<int>(j);
        }
        if (consumers == 1 && pool >= 0 && sn.relu && conv_stem_pool_fusable(sn.g)) t->fused_pool = pool;
    }
    for (Node& nd : t->nodes) {
        nd.chain.clear();
        nd.tmp.clear();
        for (int c : nd.compute_from) {
            if (c == nd.final_writer) continue;
            const Node& con = t->nodes[c];
            if ((con.op == Op::Conv && con.algo_id == TCB_ALGO_GEMM) || (con.op == Op::AvgPool && con.f > 0))
                nd.chain.push_back(c);
            else
                nd.tmp[c] = b.take(size_t(nd.n) * nd.h * nd.w * nd.c * es);
        }
        if (!nd.chain.empty()) nd.acc = b.take(size_t(nd.n) * nd.h * nd.w * nd.c * es);
    }
    for (int i = static_cast<int>(t->nodes.size()) - 1; i >= 0; --i)
        if (t->nodes[i].grad_alias >= 0) t->nodes[i].grad = t->nodes[t->nodes[i].grad_alias].grad;
    t->ws_bytes = ws;
    t->colsum_bytes = colsum;
    t->off_ws = b.take(ws);
    t->off_pack_jobs = b.take((t->async_ps ? 2 : 1) * t->nodes.size() * sizeof(PackDgradJob));
    t->off_counters = b.take(conv_tc_counter_ints() * sizeof(int));
    t->off_colsum = b.take(colsum);
    t->off_labels = b.take(size_t(t->batch) * 4);
    t->off_loss = b.take(size_t(t->batch + 1) * 4);
    const Node& in = t->nodes[0];
    t->off_input_f32 = b.take(size_t(in.n) * in.h * in.w * in.c_logical * 4);
    t->stage_bytes = size_t(in.n) * in.h * in.w * in.c_logical * 4;  // fp32 worst case
    for (int k = 0; k < 2; ++k) {
        t->off_stage[k] = b.take(t->stage_bytes);
        t->off_stage_labels[k] = b.take(size_t(t->batch) * 4);
    }
    t->arena_bytes = b.top;
    t->algorithm_ws_bytes += round_up(std::max<size_t>(ws, 1), kAlign);
    if (dry) return TCB_OK;
    cudaError_t e = cudaMalloc(&t->arena, t->arena_bytes);
    if (e != cudaSuccess)
        return fail(TCB_ERR_OOM, "arena of " + std::to_string(t->arena_bytes) + " bytes: " +
                                     cudaGetErrorString(e));
    // zeroed once: the split-K counters in the workspaces must start at 0 (they reset themselves)
    return check_cuda(cudaMemset(t->arena, 0, t->arena_bytes), "arena memset");
}

int pack_input(tcb_trainer* t, cudaStream_t st) {
    const Node& in = t->nodes[0];
    const size_t px = size_t(in.n) * in.h * in.w;
    const float* src = t->at<float>(t->off_input_f32);
    t->launches++;
    TRY(check_cuda(pack_channels(t->dt, src, t->at(in.act), px, in.c_logical, in.c, st), "pack_input"));
    if (t->stem_node >= 0) {
        const Node& sn = t->nodes[t->stem_node];
        t->launches++;
        TRY(check_cuda(conv_stem_pack_input(sn.g, t->at(in.act), t->at(sn.nws), st), "pack_input stem rows"));
    }
    return TCB_OK;
}

int refresh_biases(tcb_trainer* t, const void* wc, int k, cudaStream_t st);

int initialize(tcb_trainer* t, cudaStream_t st) {
    // parameters: deterministic per-layer streams, tag = 1000 + conv index
    float* param = t->at<float>(t->off_param);
    TRY_CUDA(cudaMemsetAsync(param, 0, t->param_padded * 4, st));
    TRY_CUDA(cudaMemsetAsync(t->at(t->off_mom), 0, t->param_padded * 4, st));
    TRY_CUDA(cudaMemsetAsync(t->grad_ptr(), 0, t->param_padded * 4, st));
    for (const Node& nd : t->nodes) {
        if (nd.op != Op::Conv) continue;
        const int cl = t->nodes[nd.in].c_logical, cp = nd.g.c;
        // logical filters k < c_logical; padded filters (k >= c_logical) stay zero
        const size_t outer = size_t(nd.c_logical) * nd.g.r * nd.g.s;
        if (cl == cp) {
            TRY_CUDA(fill_uniform(DType::F32, param + nd.woff, outer * cl, t->seed,
                                  1000 + nd.conv_index, -nd.init_scale, nd.init_scale, st));
        } else {
            // generate the logical stream in the grad buffer, scatter into padded channels
            float* scratch = t->grad_ptr();
            TRY_CUDA(fill_uniform(DType::F32, scratch, outer * cl, t->seed, 1000 + nd.conv_index,
                                  -nd.init_scale, nd.init_scale, st));
            TRY_CUDA(pack_channels(DType::F32, scratch, param + nd.woff, outer, cl, cp, st));
        }
    }
    if (t->bf16)
        TRY_CUDA(cast(DType::F32, param, DType::BF16, t->wc_ptr(), t->param_padded, st));
    if (t->async_ps)  // W_0 in both buffers
        TRY_CUDA(cudaMemcpyAsync(t->wc_buf(1), t->wc_buf(0), t->param_padded * 2, cudaMemcpyDeviceToDevice, st));
    for (int k = 0; k < (t->async_ps ? 2 : 1); ++k) TRY(refresh_biases(t, t->wc_buf(k), k, st));
    // synthetic mini-batch: worker r uses seed + r (distinct mini-batches);
    // "data_rank" overrides r (tests replay one rank's batch on a single GPU)
    const Node& in = t->nodes[0];
    const uint64_t data_seed = t->seed + static_cast<uint64_t>(t->cfg.value("data_rank", t->rank));
    TRY_CUDA(fill_uniform(DType::F32, t->at(t->off_input_f32), size_t(in.n) * in.h * in.w * in.c_logical,
                          data_seed, 1, -1.f, 1.f, st));
    TRY_CUDA(fill_labels(t->at<int32_t>(t->off_labels), t->batch, t->classes, data_seed, st));
    TRY(pack_input(t, st));
    TRY_CUDA(cudaMemsetAsync(t->grad_ptr(), 0, t->param_padded * 4, st));
    TRY_CUDA(cudaStreamSynchronize(st));
    t->initialized = true;
    return TCB_OK;
}

// ------------------------------------------------------------------ step ---
int refresh_transposes(tcb_trainer* t, cudaStream_t st) {
    if (!t->bf16) return TCB_OK;
    // one job table per bf16 weight buffer: asynchronous PS alternates the
    // buffer the step reads (wc_rd), and the packed w^T must come from the same
    // weights as the forward and the other dgrads of that step
    const int nbuf = t->async_ps ? 2 : 1;
    if (!t->pack_jobs_ready) {
        int blocks = 0, njobs = 0;
        for (int b = 0; b < nbuf; ++b) {
            std::vector<PackDgradJob> jobs;
            blocks = 0;
            for (const Node& nd : t->nodes) {
                if (nd.op != Op::Conv || !nd.pack_wT) continue;
                jobs.push_back({static_cast<__nv_bfloat16*>(t->wc_buf(b)) + nd.woff, t->at(nd.wT), nd.g, blocks});
                blocks += pack_dgrad_blocks(nd.g);
            }
            njobs = static_cast<int>(jobs.size());
            if (!jobs.empty())
                TRY_CUDA(cudaMemcpy(t->at<PackDgradJob>(t->off_pack_jobs) + size_t(b) * t->nodes.size(), jobs.data(),
                                    jobs.size() * sizeof(PackDgradJob), cudaMemcpyHostToDevice));
        }
        t->pack_njobs = njobs;
        t->pack_blocks = blocks;
        t->pack_jobs_ready = true;
    }
    if (t->pack_njobs == 0) return TCB_OK;
    const size_t table = t->async_ps ? static_cast<size_t>(t->wc_rd) : 0;
    TRY_CUDA(pack_dgrad_weights_batched(t->at<PackDgradJob>(t->off_pack_jobs) + table * t->nodes.size(),
                                        t->pack_njobs, t->pack_blocks, st));
    t->launches++;
    return TCB_OK;
}

int forward(tcb_trainer* t, cudaStream_t st) {
    for (const Node& nd : t->nodes) {
        const Node* x = nd.in >= 0 ? &t->nodes[nd.in] : nullptr;
        switch (nd.op) {
            case Op::Input: break;
            case Op::Conv: {
                Epilogue ep;
                ep.bias = !nd.bias ? nullptr
                          : t->bias_from_wc ? t->at<float>(t->off_biasc[t->async_ps ? t->wc_rd : 0]) + nd.bcomp
                                            : t->at<float>(t->off_param) + nd.boff;
                ep.residual = nd.residual >= 0 ? t->at(t->nodes[nd.residual].act) : nullptr;
                ep.relu = nd.relu;
                const size_t idx = static_cast<size_t>(&nd - t->nodes.data());
                t->mark(idx, 0, st);
                const void* wgt = t->bf16 ? static_cast<const void*>(static_cast<__nv_bfloat16*>(t->wc_ptr()) + nd.woff)
                                          : static_cast<const void*>(t->at<float>(t->off_param) + nd.woff);
                if (t->bf16 && static_cast<int>(idx) == t->stem_node && t->fused_pool >= 0) {
                    const Node& pn = t->nodes[t->fused_pool];  // the stem kernel also writes the pool
                    ep.pool_y = t->at(pn.act);
                    ep.pool_arg = t->at<uint8_t>(pn.argmax);
                }
                if (nd.algo_id == TCB_ALGO_WINOGRAD)
                    TRY_CUDA(winograd_fwd(nd.g, t->dt, t->at(x->act), wgt, ep, t->at(nd.act), t->at(t->off_ws), st));
                else if (nd.algo_id == TCB_ALGO_FFT)
                    TRY_CUDA(fft_fwd(nd.g, t->dt, t->at(x->act), wgt, ep, t->at(nd.act), t->at(t->off_ws), st));
                else if (t->bf16)
                    TRY_CUDA(conv_tc_fwd(nd.g, t->at(x->act), static_cast<__nv_bfloat16*>(t->wc_ptr()) + nd.woff,
                                         ep, t->at(nd.act), st,
                                         nd.narrow ? t->at(nd.nws)
                                         : conv_tc_workspace(nd.g, ConvMode::Fwd) ? t->at(t->off_ws)
                                                                                  : nullptr,
                                         static_cast<int>(idx) == t->stem_node));
                else if (t->tf32)
                    TRY_CUDA(conv_tf32_fwd(nd.g, t->at<float>(x->act), t->at<float>(t->off_param) + nd.woff,
                                           ep, t->at<float>(nd.act), st));
                else
                    TRY_CUDA(conv_ffma_fwd(nd.g, t->at<float>(x->act), t->at<float>(t->off_param) + nd.woff,
                                           ep, t->at<float>(nd.act), st));
                t->mark(idx, 1, st);
                t->launches += (t->bf16 && nd.algo_id == TCB_ALGO_GEMM)
                                   ? conv_tc_launches(nd.g, ConvMode::Fwd, static_cast<int>(idx) == t->stem_node)
                                   : 1;
                break;
            }
            case Op::MaxPool:
                if (static_cast<int>(&nd - t->nodes.data()) == t->fused_pool) break;  // done by the stem kernel
                TRY_CUDA(maxpool_fwd(t->dt, t->at(x->act), t->at(nd.act), t->at<uint8_t>(nd.argmax), x->n,
                                     x->h, x->w, x->c, nd.f, nd.s, nd.p, st));
                t->launches++;
                break;
            case Op::AvgPool:
                if (nd.f > 0)
                    TRY_CUDA(avgpool2d_fwd(t->dt, t->at(x->act), t->at(nd.act), x->n, x->h, x->w, x->c, nd.f,
                                           nd.s, nd.p, st));
                else
                    TRY_CUDA(avgpool_global_fwd(t->dt, t->at(x->act), t->at(nd.act), x->n, x->h * x->w, x->c, st));
                t->launches++;
                break;
            case Op::Concat: {
                const size_t rows = size_t(nd.n) * nd.h * nd.w;
                const size_t es = dtype_size(t->dt);
                for (size_t k = 0; k < nd.ins.size(); ++k) {
                    const Node& xi = t->nodes[nd.ins[k]];
                    TRY_CUDA(slice_copy(t->dt, t->at(xi.act), xi.c, t->at<char>(nd.act) + nd.coff[k] * es, nd.c,
                                        xi.c, rows, st));
                    t->launches++;
                }
                break;
            }
            case Op::Loss: {
                const Node& z = t->nodes[t->logits];
                TRY_CUDA(softmax_xent(t->dt, t->at(z.act), t->at<int32_t>(t->off_labels), t->at(z.grad),
                                      t->at<float>(t->off_loss), t->batch, t->classes, z.c, st));
                t->launches += 2;
                break;
            }
        }
    }
    return TCB_OK;
}

// Gradient contribution of consumer `ci` to tensor `ti`: either the final
// G[ti] (with every other contribution fused in) or a temp buffer.
int backward_contribution(tcb_trainer* t, int ci, int ti, cudaStream_t st) {
    Node& tgt = t->nodes[ti];
    const Node& con = t->nodes[ci];
    const bool final = tgt.final_writer == ci;
    const size_t elems = size_t(tgt.n) * tgt.h * tgt.w * tgt.c;
    const bool chained = !final && std::find(tgt.chain.begin(), tgt.chain.end(), ci) != tgt.chain.end();
    void* out = final ? t->at(tgt.grad) : chained ? t->at(tgt.acc) : t->at(tgt.tmp.at(ci));
    const Node* producer = &tgt;
    const bool mask_needed = final && producer->op == Op::Conv && producer->relu;

    // extra contributions to fold in: at the final writer every other one; a
    // chained contribution adds the running sum of the chain (in place)
    // first (and only) chained contribution into a chain buffer nothing else writes
    // before the final writer reads it: pixels this conv's taps never reach keep the
    // zeros of the arena's initial memset across steps (the strided projection's
    // empty dgrad phases need no zero pass)
    const bool sole_chained = chained && tgt.acc_written == 0 && tgt.chain.size() == 1 && tgt.tmp.empty() &&
                              tgt.alias_from.empty();
    std::vector<const void*> extras;
    if (final) {
        if (!tgt.chain.empty()) extras.push_back(t->at(tgt.acc));
        for (const auto& [c, off] : tgt.tmp)
            if (c != ci) extras.push_back(t->at(off));
        for (int a : tgt.alias_from) extras.push_back(t->at(t->nodes[a].grad));
    } else if (chained) {
        if (tgt.acc_written++ > 0) extras.push_back(t->at(tgt.acc));
    }
    if (con.op == Op::Conv) {
        // combine extras into one residual operand for the dgrad epilogue
        const void* residual = nullptr;
        if (extras.size() == 1) {
            residual = extras[0];
        } else if (extras.size() > 1) {
            void* acc = const_cast<void*>(extras[0]);
            for (size_t i = 1; i < extras.size(); ++i) {
                TRY_CUDA(add_inplace(t->dt, acc, extras[i], elems, st));
                t->launches++;
            }
            residual = acc;
        }
        Epilogue ep;
        ep.residual = residual;
        ep.mask = mask_needed ? t->at(tgt.act) : nullptr;
        ep.uncovered_zero = sole_chained && !residual && !ep.mask;
        const void* cw = t->bf16 ? static_cast<const void*>(static_cast<__nv_bfloat16*>(t->wc_ptr()) + con.woff)
                                 : static_cast<const void*>(t->at<float>(t->off_param) + con.woff);
        // a fully connected layer (filter = whole unpadded input map, 1x1 output) runs
        // its dgrad as the equivalent 1x1 conv over a 1x1 image of H*W*C channels:
        // the same memory, dx rows = images and 1/(H*W) of the reduction depth
        // (the other taps only ever meet zero padding)
        const ConvGeom& cg = con.g;
        const bool fc = cg.r == cg.h && cg.s == cg.w && cg.pad_h == 0 && cg.pad_w == 0 && cg.ho() == 1 &&
                        cg.wo() == 1 && (cg.h > 1 || cg.w > 1);
        const ConvGeom dg = fc ? ConvGeom{cg.n, 1, 1, cg.h * cg.w * cg.c, cg.k, 1, 1, 0, 0, 1, 1} : cg;
        if (con.algo_id == TCB_ALGO_WINOGRAD)
            TRY_CUDA(winograd_dgrad(con.g, t->dt, t->at(con.grad), cw, ep, out, t->at(t->off_ws), st));
        else if (con.algo_id == TCB_ALGO_FFT)
            TRY_CUDA(fft_dgrad(con.g, t->dt, t->at(con.grad), cw, ep, out, t->at(t->off_ws), st));
        else if (t->bf16)
            TRY_CUDA(conv_tc_dgrad(dg, t->at(con.grad), cw, (con.pack_wT && !fc) ? t->at(con.wT) : nullptr, ep,
                                   out, st));
        else if (t->tf32)
            TRY_CUDA(conv_tf32_dgrad(dg, t->at<float>(con.grad), t->at<float>(t->off_param) + con.woff,
                                     ep, static_cast<float*>(out), st));
        else
            TRY_CUDA(conv_ffma_dgrad(dg, t->at<float>(con.grad), t->at<float>(t->off_param) + con.woff,
                                     ep, static_cast<float*>(out), st));
        t->launches++;
        return TCB_OK;
    }
    // the ReLU mask fuses into the pool backward when nothing else must be added first
    const bool fuse_mask = mask_needed && extras.empty();
    if (con.op == Op::Concat) {
        // this input's channel range of the concatenated gradient
        size_t k = 0;
        while (con.ins[k] != ti) ++k;
        const void* src = t->at<char>(con.grad) + con.coff[k] * dtype_size(t->dt);
        const size_t rows = size_t(tgt.n) * tgt.h * tgt.w;
        if (fuse_mask && slice_copy_mask_supported(t->dt, src, con.c, out, tgt.c, tgt.c, t->at(tgt.act))) {
            // the producer's ReLU mask in the same pass as the slice copy
            TRY_CUDA(slice_copy_mask(t->dt, src, con.c, out, tgt.c, tgt.c, rows, t->at(tgt.act), st));
            t->launches++;
            return TCB_OK;
        }
        TRY_CUDA(slice_copy(t->dt, src, con.c, out, tgt.c, tgt.c, rows, st));
        t->launches++;
        for (const void* e : extras) {
            TRY_CUDA(add_inplace(t->dt, out, e, elems, st));
            t->launches++;
        }
        if (mask_needed) {
            TRY_CUDA(relu_mask_inplace(t->dt, out, t->at(tgt.act), elems, st));
            t->launches++;
        }
        return TCB_OK;
    }
    if (con.op == Op::AvgPool && con.f > 0 && chained) {  // accumulate into the chain in place
        TRY_CUDA(avgpool2d_bwd(t->dt, t->at(con.grad), out, tgt.n, tgt.h, tgt.w, tgt.c, con.f, con.s, con.p, st,
                               nullptr, extras.empty() ? nullptr : extras[0]));
        t->launches++;
        return TCB_OK;
    }
    if (con.op == Op::MaxPool)
        TRY_CUDA(maxpool_bwd(t->dt, t->at(con.grad), t->at<uint8_t>(con.argmax), out, tgt.n, tgt.h, tgt.w,
                             tgt.c, con.f, con.s, con.p, st, fuse_mask ? t->at(con.act) : nullptr));
    else if (con.f > 0)
        TRY_CUDA(avgpool2d_bwd(t->dt, t->at(con.grad), out, tgt.n, tgt.h, tgt.w, tgt.c, con.f, con.s, con.p, st,
                               fuse_mask ? t->at(tgt.act) : nullptr));
    else
        TRY_CUDA(avgpool_global_bwd(t->dt, t->at(con.grad), out, tgt.n, tgt.h * tgt.w, tgt.c, st,
                                    fuse_mask ? t->at(tgt.act) : nullptr));
    t->launches++;
    for (const void* e : extras) {
        TRY_CUDA(add_inplace(t->dt, out, e, elems, st));
        t->launches++;
    }
    if (mask_needed && !fuse_mask) {
        TRY_CUDA(relu_mask_inplace(t->dt, out, t->at(tgt.act), elems, st));
        t->launches++;
    }
    return TCB_OK;
}

// Overlapped aggregation: reduce each gradient shard that node i completed to
// its owner on the comm stream (same order on every rank).
int issue_ready_shards(tcb_trainer* t, int i, cudaStream_t st) {
    auto it = t->shard_trigger.find(i);
    if (it == t->shard_trigger.end()) return TCB_OK;
    float* grad = t->grad_ptr();
    for (int sh : it->second) {
        TRY_CUDA(cudaEventRecord(t->ev_ready[sh], st));
        TRY_CUDA(cudaStreamWaitEvent(t->comm_stream, t->ev_ready[sh], 0));
        float* g = grad + size_t(sh) * t->shard;
        TRY_NCCL(ncclReduce(g, g, t->shard, ncclFloat32, ncclSum, sh, t->comm_bg, t->comm_stream));
        t->launches++;
    }
    return TCB_OK;
}

int backward(tcb_trainer* t, cudaStream_t st) {
    TRY(refresh_transposes(t, st));
    for (Node& nd : t->nodes) nd.acc_written = 0;
    // overlapped shard reduces run on comm_bg_ctas SMs: keep them free
    conv_tc_set_sm_reserve(t->overlap_active() ? t->comm_bg_ctas : 0);
    struct Reset {
        ~Reset() { conv_tc_set_sm_reserve(0); }
    } reset;
    float* grad = t->grad_ptr();
    for (int i = static_cast<int>(t->nodes.size()) - 1; i >= 0; --i) {
        const Node& nd = t->nodes[i];
        if (nd.op != Op::Input && nd.op != Op::Loss && nd.compute_from.empty() &&
            !nd.alias_from.empty() && nd.grad_alias < 0) {
            // gradient only via residual paths (several, or through a ReLU): combine
            const size_t elems = size_t(nd.n) * nd.h * nd.w * nd.c;
            TRY_CUDA(cudaMemcpyAsync(t->at(nd.grad), t->at(t->nodes[nd.alias_from[0]].grad),
                                     elems * dtype_size(t->dt), cudaMemcpyDeviceToDevice, st));
            for (size_t a = 1; a < nd.alias_from.size(); ++a) {
                TRY_CUDA(add_inplace(t->dt, t->at(nd.grad), t->at(t->nodes[nd.alias_from[a]].grad), elems, st));
                t->launches++;
            }
            if (nd.op == Op::Conv && nd.relu) {
                TRY_CUDA(relu_mask_inplace(t->dt, t->at(nd.grad), t->at(nd.act), elems, st));
                t->launches++;
            }
        }
        if (nd.op == Op::Conv) {
            const Node& x = t->nodes[nd.in];
            // weight (and bias) gradient straight into the flat PS buffer, on a forked
            // stream beside this layer's dgrad (bf16 GEMM layers: their dgrad uses no
            // workspace), joined right after: one pass's tail wave fills with the
            // other's CTAs (ResNet-50 +1.2 %, VGG-16 +1.4 %; $TCB_BWD_CONCURRENT=0 off)
            static const int bwd_conc = [] {
                const char* e = getenv("TCB_BWD_CONCURRENT");
                return e ? atoi(e) : 1;
            }();
            // (per-layer timing runs keep the passes sequential so each one's events
            // bracket that pass alone)
            const bool conc = bwd_conc > 0 && t->bf16 && nd.algo_id == TCB_ALGO_GEMM && nd.need_dgrad &&
                              !t->overlap_active() && !t->layer_timing;
            if (conc && !t->wg_stream) {
                TRY_CUDA(cudaStreamCreateWithFlags(&t->wg_stream, cudaStreamNonBlocking));
                TRY_CUDA(cudaEventCreateWithFlags(&t->wg_fork, cudaEventDisableTiming));
                TRY_CUDA(cudaEventCreateWithFlags(&t->wg_join, cudaEventDisableTiming));
            }
            const cudaStream_t main_st = st;
            if (conc) {
                TRY_CUDA(cudaEventRecord(t->wg_fork, main_st));
                TRY_CUDA(cudaStreamWaitEvent(t->wg_stream, t->wg_fork, 0));
                st = t->wg_stream;
            }
            t->mark(i, 4, st);
            if (nd.algo_id == TCB_ALGO_WINOGRAD)
                TRY_CUDA(winograd_wgrad(nd.g, t->dt, t->at(nd.grad), t->at(x.act), grad + nd.woff,
                                        t->at(t->off_ws), st));
            else if (nd.algo_id == TCB_ALGO_FFT)
                TRY_CUDA(fft_wgrad(nd.g, t->dt, t->at(nd.grad), t->at(x.act), grad + nd.woff,
                                   t->at(t->off_ws), st));
            else if (t->bf16)
                TRY_CUDA(conv_tc_wgrad(nd.g, t->at(nd.grad), t->at(x.act), grad + nd.woff,
                                       t->at(nd.narrow ? nd.nws : t->off_ws), st, nd.narrow,
                                       t->fused_split_reduce ? t->at<int>(t->off_counters) : nullptr));
            else if (t->tf32)
                TRY_CUDA(conv_tf32_wgrad(nd.g, t->at<float>(nd.grad), t->at<float>(x.act), grad + nd.woff,
                                         t->at(t->off_ws), st));
            else
                TRY_CUDA(conv_ffma_wgrad(nd.g, t->at<float>(nd.grad), t->at<float>(x.act), grad + nd.woff,
                                         t->at(t->off_ws), st));
            t->launches += (t->bf16 && nd.algo_id == TCB_ALGO_GEMM) ? conv_tc_launches(nd.g, ConvMode::Wgrad, nd.narrow, t->fused_split_reduce) : 2;
            if (nd.bias) {
                TRY_CUDA(column_sum(t->dt, t->at(nd.grad), grad + nd.boff, nd.n * nd.h * nd.w, nd.g.k,
                                    t->at<float>(t->off_colsum), st));
                t->launches += 2;
            }
            t->mark(i, 5, st);
            if (conc) {
                TRY_CUDA(cudaEventRecord(t->wg_join, st));
                st = main_st;
            }
            if (t->overlap_active()) TRY(issue_ready_shards(t, i, st));
            if (nd.need_dgrad) {
                t->mark(i, 2, st);
                TRY(backward_contribution(t, i, nd.in, st));
                t->mark(i, 3, st);
            }
            if (conc) TRY_CUDA(cudaStreamWaitEvent(st, t->wg_join, 0));
        } else if (nd.op == Op::MaxPool || nd.op == Op::AvgPool) {
            if (t->nodes[nd.in].op != Op::Input) TRY(backward_contribution(t, i, nd.in, st));
        } else if (nd.op == Op::Concat) {
            for (int j : nd.ins)
                if (t->nodes[j].op != Op::Input) TRY(backward_contribution(t, i, j, st));
        }
    }
    return TCB_OK;
}

// fp32 bias copy k <- the bias segments of bf16 weight buffer `wc`
int refresh_biases(tcb_trainer* t, const void* wc, int k, cudaStream_t st) {
    if (!t->bias_from_wc) return TCB_OK;
    for (const Node& nd : t->nodes) {
        if (nd.op != Op::Conv || !nd.bias) continue;
        TRY_CUDA(cast(DType::BF16, static_cast<const __nv_bfloat16*>(wc) + nd.boff, DType::F32,
                      t->at<float>(t->off_biasc[k]) + nd.bcomp, nd.g.k, st));
        t->launches++;
    }
    return TCB_OK;
}

// wc_out: the bf16 weight buffer the update writes (-1: the one the step read)
int aggregate_and_update(tcb_trainer* t, cudaStream_t st, cudaEvent_t after_rs, cudaEvent_t after_sgd,
                         int wc_out = -1) {
    float* grad = t->grad_ptr();
    float* param = t->at<float>(t->off_param);
    float* mom = t->at<float>(t->off_mom);
    const float gscale = 1.0f / static_cast<float>(t->world);
    const ncclDataType_t wdt = t->bf16 ? ncclBfloat16 : ncclFloat32;
    const size_t wes = t->bf16 ? 2 : 4;
    char* wc = static_cast<char*>(wc_out >= 0 ? t->wc_buf(wc_out) : t->wc_ptr());
    void* wc_mc = wc_out >= 0 ? t->wc_mc_buf(wc_out) : t->wc_mc;
    const int owners = (t->n_ps > 0 && t->n_ps < t->world) ? t->n_ps : t->world;

    if (t->overlap_active()) {
        // shard reduces already in flight on the comm stream (issued during
        // backward); own-shard SGD and the all-gather follow there, and the
        // compute stream waits only at the end
        cudaStream_t cs = t->comm_stream;
        if (after_rs) TRY_CUDA(cudaEventRecord(after_rs, cs));
        const size_t o = t->rank * t->shard;
        TRY_CUDA(sgd_momentum(param + o, grad + o, mom + o, t->dt, t->bf16 ? wc + o * 2 : nullptr, t->shard,
                              t->lr, t->momentum, t->weight_decay, gscale, cs));
        t->launches++;
        if (after_sgd) TRY_CUDA(cudaEventRecord(after_sgd, cs));
        TRY_NCCL(ncclAllGather(wc + o * wes, wc, t->shard, wdt, t->comm, cs));
        t->launches++;
        TRY_CUDA(cudaEventRecord(t->ev_comm_done, cs));
        TRY_CUDA(cudaStreamWaitEvent(st, t->ev_comm_done, 0));
    } else if (t->nvls) {
        // PS shards = GPUs over NVSwitch multicast: every GPU's gradients are
        // written (barrier) -> one kernel reduces the own shard in the switch,
        // applies SGD and multicasts the bf16 weights -> all weights delivered
        // (barrier) before the next forward reads them
        TRY_CUDA(nvls_barrier(t->pads_dev, t->nvls_epoch, t->nvls_slot0, t->rank, t->world, st,
                              t->nvls_epoch + 1, t->nvls_timeout_ns));
        if (after_rs) TRY_CUDA(cudaEventRecord(after_rs, st));
        const size_t o = t->rank * t->shard;
        TRY_CUDA(ps_nvls_update(t->grad_mc, grad, param, mom, wc_mc, o, t->shard, t->lr, t->momentum,
                                t->weight_decay, gscale, st));
        if (after_sgd) TRY_CUDA(cudaEventRecord(after_sgd, st));
        TRY_CUDA(nvls_barrier(t->pads_dev, t->nvls_epoch, t->nvls_slot0, t->rank, t->world, st,
                              t->nvls_epoch + 1, t->nvls_timeout_ns));
        t->launches += 3;
    } else if (t->world > 1 && owners == t->world) {
        // PS shards = GPUs: reduce-scatter (in place) -> SGD on own shard -> all-gather
        TRY_NCCL(ncclReduceScatter(grad, grad + t->rank * t->shard, t->shard, ncclFloat32, ncclSum,
                                   t->comm, st));
        t->launches++;
        if (after_rs) TRY_CUDA(cudaEventRecord(after_rs, st));
        const size_t o = t->rank * t->shard;
        TRY_CUDA(sgd_momentum(param + o, grad + o, mom + o, t->dt, t->bf16 ? wc + o * 2 : nullptr, t->shard,
                              t->lr, t->momentum, t->weight_decay, gscale, st));
        t->launches++;
        if (after_sgd) TRY_CUDA(cudaEventRecord(after_sgd, st));
        TRY_NCCL(ncclAllGather(wc + o * wes, wc, t->shard, wdt, t->comm, st));
        t->launches++;
    } else if (t->world > 1) {
        // N_ps < G: shard j (of N_ps) is owned by rank j; every worker pushes its
        // full gradient to the owners (Lemma 2's N_w * S_p / N_ps ingress).
        const size_t per = round_up((t->param_padded + owners - 1) / owners, kParamAlign);
        TRY_NCCL(ncclGroupStart());
        for (int j = 0; j < owners; ++j) {
            const size_t o = j * per;
            if (o >= t->param_padded) break;
            const size_t cnt = std::min(per, t->param_padded - o);
            TRY_NCCL(ncclReduce(grad + o, grad + o, cnt, ncclFloat32, ncclSum, j, t->comm, st));
        }
        TRY_NCCL(ncclGroupEnd());
        t->launches++;
        if (after_rs) TRY_CUDA(cudaEventRecord(after_rs, st));
        if (t->rank < owners) {
            const size_t o = t->rank * per;
            if (o < t->param_padded) {
                const size_t cnt = std::min(per, t->param_padded - o);
                TRY_CUDA(sgd_momentum(param + o, grad + o, mom + o, t->dt, t->bf16 ? wc + o * 2 : nullptr,
                                      cnt, t->lr, t->momentum, t->weight_decay, gscale, st));
                t->launches++;
            }
        }
        if (after_sgd) TRY_CUDA(cudaEventRecord(after_sgd, st));
        TRY_NCCL(ncclGroupStart());
        for (int j = 0; j < owners; ++j) {
            const size_t o = j * per;
            if (o >= t->param_padded) break;
            const size_t cnt = std::min(per, t->param_padded - o);
            TRY_NCCL(ncclBroadcast(wc + o * wes, wc + o * wes, cnt, wdt, j, t->comm, st));
        }
        TRY_NCCL(ncclGroupEnd());
        t->launches++;
    } else {
        if (after_rs) TRY_CUDA(cudaEventRecord(after_rs, st));
        TRY_CUDA(sgd_momentum(param, grad, mom, t->dt, t->bf16 ? wc : nullptr, t->param_padded, t->lr,
                              t->momentum, t->weight_decay, gscale, st));
        t->launches++;
        if (after_sgd) TRY_CUDA(cudaEventRecord(after_sgd, st));
    }
    return refresh_biases(t, wc, wc_out >= 0 ? wc_out : 0, st);
}

}  // namespace
}  // namespace tcb

#define TCB_API extern "C" __attribute__((visibility("default")))

TCB_API int tcb_trainer_create(const char* config_json, tcb_trainer** out) {
    if (!config_json || !out) return fail(TCB_ERR_INVALID, "NULL argument");
    auto t = std::make_unique<tcb_trainer>();
    try {
        t->cfg = json::parse(config_json);
        TRY(build_graph(t.get()));
    } catch (const std::exception& e) {
        return fail(TCB_ERR_INVALID, std::string("model config: ") + e.what());
    }
    *out = t.release();
    return TCB_OK;
}

TCB_API int tcb_trainer_destroy(tcb_trainer* t) {
    if (!t) return TCB_OK;
    if (t->graph_exec) cudaGraphExecDestroy(t->graph_exec);
    if (t->graph_stream) {
        cudaStreamSynchronize(t->graph_stream);
        cudaStreamDestroy(t->graph_stream);
        cudaEventDestroy(t->graph_in);
        cudaEventDestroy(t->graph_out);
    }
    if (t->wg_stream) {
        cudaStreamSynchronize(t->wg_stream);
        cudaStreamDestroy(t->wg_stream);
        cudaEventDestroy(t->wg_fork);
        cudaEventDestroy(t->wg_join);
    }
    if (t->comm_stream) {
        cudaStreamSynchronize(t->comm_stream);
        for (cudaEvent_t e : t->ev_ready) cudaEventDestroy(e);
        if (t->ev_comm_done) cudaEventDestroy(t->ev_comm_done);
        cudaStreamDestroy(t->comm_stream);
    }
    if (t->ps_stream) {
        cudaStreamSynchronize(t->ps_stream);
        cudaStreamDestroy(t->ps_stream);
        cudaEventDestroy(t->ev_bwd_done);
        for (cudaEvent_t e : t->ev_upd) cudaEventDestroy(e);
    }
    if (t->comm_bg) ncclCommDestroy(t->comm_bg);
    if (t->comm) ncclCommDestroy(t->comm);
    if (t->copy_stream) {
        cudaStreamSynchronize(t->copy_stream);
        cudaStreamDestroy(t->copy_stream);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(t->staged[k]);
            cudaEventDestroy(t->consumed[k]);
        }
    }
    for (cudaEvent_t& e : t->ph.e)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (t->ev_h2d[i]) cudaEventDestroy(t->ev_h2d[i]);
        if (t->ev_prep[i]) cudaEventDestroy(t->ev_prep[i]);
    }
    for (auto& a : t->lev)
        for (cudaEvent_t e : a)
            if (e) cudaEventDestroy(e);
    if (t->arena) cudaFree(t->arena);
    if (t->nvls_epoch) cudaFree(t->nvls_epoch);
    delete t;
    return TCB_OK;
}

TCB_API int tcb_nccl_unique_id(uint8_t* id128) {
    if (!id128) return fail(TCB_ERR_INVALID, "NULL argument");
    ncclUniqueId id;
    TRY_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof(id));
    return TCB_OK;
}

TCB_API int tcb_trainer_join(tcb_trainer* t, int rank, int world, const uint8_t* id128) {
    if (!t || world < 1 || rank < 0 || rank >= world) return fail(TCB_ERR_INVALID, "bad rank/world");
    if (t->initialized) return fail(TCB_ERR_INVALID, "join before the first step");
    t->rank = rank;
    t->world = world;
    if (world > 1) {
        if (!id128) return fail(TCB_ERR_INVALID, "NCCL id required for world > 1");
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        TRY_NCCL(ncclCommInitRank(&t->comm, world, id, rank));
        if (t->overlap) {
            ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
            cfg.minCTAs = 1;
            cfg.maxCTAs = std::max(1, t->comm_bg_ctas);
            TRY_NCCL(ncclCommSplit(t->comm, 0, rank, &t->comm_bg, &cfg));
            TRY_CUDA(cudaStreamCreateWithFlags(&t->comm_stream, cudaStreamNonBlocking));
            t->ev_ready.resize(world);
            for (cudaEvent_t& e : t->ev_ready) TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            TRY_CUDA(cudaEventCreateWithFlags(&t->ev_comm_done, cudaEventDisableTiming));
        }
    }
    return TCB_OK;
}

TCB_API int tcb_trainer_layout(const char* config_json, char** json_out) {
    if (!config_json || !json_out) return fail(TCB_ERR_INVALID, "NULL argument");
    auto t = std::make_unique<tcb_trainer>();
    try {
        t->cfg = json::parse(config_json);
        TRY(build_graph(t.get()));
        TRY(allocate(t.get(), /*dry=*/true));
    } catch (const std::exception& e) {
        return fail(TCB_ERR_INVALID, std::string("model config: ") + e.what());
    }
    json d;
    d["arena_bytes"] = t->arena_bytes;
    d["algorithm_workspace_bytes"] = t->algorithm_ws_bytes;
    d["resident_bytes"] = t->arena_bytes - t->algorithm_ws_bytes;
    d["param_padded"] = t->param_padded;
    d["param_count"] = t->param_count;
    d["batch"] = t->batch;
    int convs = 0;
    for (const Node& nd : t->nodes) convs += nd.op == Op::Conv;
    d["conv_layers"] = convs;
    const std::string out = d.dump();
    *json_out = static_cast<char*>(std::malloc(out.size() + 1));
    std::memcpy(*json_out, out.c_str(), out.size() + 1);
    return TCB_OK;
}

TCB_API int tcb_trainer_attach_nvls(tcb_trainer* t, void* grad, const void* grad_mc, void* wcompute,
                                    void* wcompute_mc, void* const* signal_pads_dev, size_t signal_pad_bytes) {
    if (!t || !grad || !grad_mc || !wcompute || !wcompute_mc || !signal_pads_dev)
        return fail(TCB_ERR_INVALID, "NULL argument");
    {
        // the barrier's slots sit at the top of the pad, clear of the low slots the
        // symmetric-memory runtime uses for its own barriers
        const long words = static_cast<long>(signal_pad_bytes / sizeof(uint32_t));
        const long slot0 = std::min<long>(2048, words - t->world);
        if (slot0 < 256)
            return fail(TCB_ERR_INVALID, "signal pad of " + std::to_string(signal_pad_bytes) +
                                             " bytes is too small for the NVLS barrier of " +
                                             std::to_string(t->world) + " ranks");
        t->nvls_slot0 = static_cast<int>(slot0);
        if (const char* e = std::getenv("TCB_NVLS_TIMEOUT_MS"))
            t->nvls_timeout_ns = static_cast<uint64_t>(std::max(1L, std::atol(e))) * 1000000ull;
    }
    if (t->initialized) return fail(TCB_ERR_INVALID, "attach before the first step");
    if (!t->bf16) return fail(TCB_ERR_UNSUPPORTED, "the NVLS parameter-server path is bf16-only");
    if (t->world < 2 || (t->n_ps > 0 && t->n_ps < t->world))
        return fail(TCB_ERR_UNSUPPORTED, "the NVLS path needs world > 1 and PS shards = GPUs");
    if (t->overlap) return fail(TCB_ERR_INVALID, "overlap_comm and the NVLS path are exclusive");
    if (reinterpret_cast<uintptr_t>(grad) % 16 || reinterpret_cast<uintptr_t>(grad_mc) % 16 ||
        reinterpret_cast<uintptr_t>(wcompute) % 16 || reinterpret_cast<uintptr_t>(wcompute_mc) % 16)
        return fail(TCB_ERR_INVALID, "NVLS buffers must be 16-byte aligned");
    t->ext_grad = static_cast<float*>(grad);
    t->grad_mc = static_cast<const float*>(grad_mc);
    t->ext_wc = wcompute;
    t->wc_mc = wcompute_mc;
    t->pads_dev = reinterpret_cast<uint32_t* const*>(signal_pads_dev);
    if (!t->nvls_epoch) {
        TRY_CUDA(cudaMalloc(&t->nvls_epoch, 2 * sizeof(uint32_t)));
        TRY_CUDA(cudaMemset(t->nvls_epoch, 0, 2 * sizeof(uint32_t)));
    }
    t->nvls = true;
    return TCB_OK;
}

// Failure detection: NCCL's asynchronous errors (a peer died, a network /
// NVLink error) are polled on the host without blocking; on one the
// communicators are aborted so no collective hangs, and the trainer is poisoned.
static int poll_comm_errors(tcb_trainer* t) {
    if (!t->failed.empty()) return fail(TCB_ERR_NCCL, t->failed);
    for (ncclComm_t* c : {&t->comm, &t->comm_bg}) {
        if (!*c) continue;
        ncclResult_t async = ncclSuccess;
        const ncclResult_t r = ncclCommGetAsyncError(*c, &async);
        if (r != ncclSuccess || (async != ncclSuccess && async != ncclInProgress)) {
            t->failed = std::string("NCCL communicator failed: ") +
                        ncclGetErrorString(r != ncclSuccess ? r : async) + " (communicators aborted)";
            if (t->comm_bg) ncclCommAbort(t->comm_bg);
            if (t->comm) ncclCommAbort(t->comm);
            t->comm_bg = t->comm = nullptr;
            return fail(TCB_ERR_NCCL, t->failed);
        }
    }
    return TCB_OK;
}

// Full health check (synchronises `st`): NCCL async errors and the NVLS
// barrier's timeout flag.
static int check_health(tcb_trainer* t, cudaStream_t st) {
    TRY(poll_comm_errors(t));
    if (t->nvls_epoch) {
        uint32_t flag = 0;
        TRY_CUDA(cudaMemcpyAsync(&flag, t->nvls_epoch + 1, sizeof(flag), cudaMemcpyDeviceToHost, st));
        TRY_CUDA(cudaStreamSynchronize(st));
        if (flag != 0) {
            t->failed = "NVLS parameter-server barrier timed out: a peer rank did not arrive within " +
                        std::to_string(t->nvls_timeout_ns / 1000000) + " ms";
            return fail(TCB_ERR_NCCL, t->failed);
        }
    }
    return TCB_OK;
}

TCB_API int tcb_trainer_health(tcb_trainer* t, void* stream) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    return check_health(t, static_cast<cudaStream_t>(stream));
}

static int ensure_ready(tcb_trainer* t, cudaStream_t st) {
    if (t->initialized) return TCB_OK;
    if (!t->arena) TRY(allocate(t));
    for (cudaEvent_t& e : t->ph.e)
        if (!e) TRY_CUDA(cudaEventCreate(&e));
    return initialize(t, st);
}

TCB_API int tcb_trainer_set_batch(tcb_trainer* t, const float* host_images, const int32_t* host_labels,
                                  void* stream) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    auto st = static_cast<cudaStream_t>(stream);
    TRY(ensure_ready(t, st));
    const Node& in = t->nodes[0];
    if (host_images) {
        TRY_CUDA(cudaMemcpyAsync(t->at(t->off_input_f32), host_images,
                                 size_t(in.n) * in.h * in.w * in.c_logical * 4, cudaMemcpyHostToDevice, st));
        TRY(pack_input(t, st));
    }
    if (host_labels)
        TRY_CUDA(cudaMemcpyAsync(t->at(t->off_labels), host_labels, size_t(t->batch) * 4,
                                 cudaMemcpyHostToDevice, st));
    return TCB_OK;
}

TCB_API int tcb_trainer_stage_batch(tcb_trainer* t, const void* host_images, int format,
                                    const int32_t* host_labels) {
    if (!t || !host_images || !host_labels) return fail(TCB_ERR_INVALID, "NULL argument");
    if (format != TCB_INPUT_F32 && format != TCB_INPUT_U8)
        return fail(TCB_ERR_INVALID, "format must be TCB_INPUT_F32 or TCB_INPUT_U8");
    if (t->stage_w - t->stage_r >= 2)
        return fail(TCB_ERR_INVALID, "two batches already staged; run a step first");
    TRY(ensure_ready(t, t->stream));
    if (!t->copy_stream) {
        TRY_CUDA(cudaStreamCreateWithFlags(&t->copy_stream, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            TRY_CUDA(cudaEventCreateWithFlags(&t->staged[k], cudaEventDisableTiming));
            TRY_CUDA(cudaEventCreateWithFlags(&t->consumed[k], cudaEventDisableTiming));
        }
    }
    const int k = static_cast<int>(t->stage_w % 2);
    // the slot is rewritten only after the step that consumed it has packed it
    if (t->consumed_recorded[k]) TRY_CUDA(cudaStreamWaitEvent(t->copy_stream, t->consumed[k], 0));
    const Node& in = t->nodes[0];
    const size_t elems = size_t(in.n) * in.h * in.w * in.c_logical;
    if (t->timing) {
        if (!t->ev_h2d[0])
            for (int i = 0; i < 2; ++i) {
                TRY_CUDA(cudaEventCreate(&t->ev_h2d[i]));
                TRY_CUDA(cudaEventCreate(&t->ev_prep[i]));
            }
        TRY_CUDA(cudaEventRecord(t->ev_h2d[0], t->copy_stream));
    }
    TRY_CUDA(cudaMemcpyAsync(t->at(t->off_stage[k]), host_images,
                             elems * (format == TCB_INPUT_U8 ? 1 : 4), cudaMemcpyHostToDevice,
                             t->copy_stream));
    TRY_CUDA(cudaMemcpyAsync(t->at(t->off_stage_labels[k]), host_labels, size_t(t->batch) * 4,
                             cudaMemcpyHostToDevice, t->copy_stream));
    if (t->timing) {
        TRY_CUDA(cudaEventRecord(t->ev_h2d[1], t->copy_stream));
        t->h2d_timed = true;
    }
    TRY_CUDA(cudaEventRecord(t->staged[k], t->copy_stream));
    t->stage_format[k] = format;
    ++t->stage_w;
    return TCB_OK;
}

// The oldest staged batch (if any) becomes this step's input.
static int consume_staged(tcb_trainer* t, cudaStream_t st) {
    if (t->stage_r == t->stage_w) return TCB_OK;
    const int k = static_cast<int>(t->stage_r % 2);
    TRY_CUDA(cudaStreamWaitEvent(st, t->staged[k], 0));
    const Node& in = t->nodes[0];
    const size_t px = size_t(in.n) * in.h * in.w;
    const bool timed = t->timing && t->ev_prep[0];
    if (timed) TRY_CUDA(cudaEventRecord(t->ev_prep[0], st));
    const Node* sn = t->stem_node >= 0 ? &t->nodes[t->stem_node] : nullptr;
    if (t->stage_format[k] == TCB_INPUT_U8 && sn) {
        TRY_CUDA(conv_stem_pack_u8(sn->g, t->at<uint8_t>(t->off_stage[k]), in.c_logical, t->at(in.act),
                                   t->at(sn->nws), st));
    } else {
        if (t->stage_format[k] == TCB_INPUT_U8)
            TRY_CUDA(pack_channels_u8(t->dt, t->at<uint8_t>(t->off_stage[k]), t->at(in.act), px, in.c_logical,
                                      in.c, st));
        else
            TRY_CUDA(pack_channels(t->dt, t->at<float>(t->off_stage[k]), t->at(in.act), px, in.c_logical, in.c,
                                   st));
        if (sn) {
            TRY_CUDA(conv_stem_pack_input(sn->g, t->at(in.act), t->at(sn->nws), st));
            t->launches++;
        }
    }
    TRY_CUDA(cudaMemcpyAsync(t->at(t->off_labels), t->at(t->off_stage_labels[k]), size_t(t->batch) * 4,
                             cudaMemcpyDeviceToDevice, st));
    if (timed) {
        TRY_CUDA(cudaEventRecord(t->ev_prep[1], st));
        t->prep_timed = true;
    }
    TRY_CUDA(cudaEventRecord(t->consumed[k], st));
    t->consumed_recorded[k] = true;
    ++t->stage_r;
    t->launches++;
    return TCB_OK;
}

// The step's launches (everything after the staged-input conversion) are
// recorded once into a CUDA graph and replayed: every kernel argument, tensor
// map and NCCL buffer is fixed for the trainer's lifetime. Timed steps (phase
// or layer events) run eagerly; $TCB_GRAPH=0 / config "cuda_graph": false
// disables the graph.
static int step_body(tcb_trainer* t, cudaStream_t st) {
    TRY(forward(t, st));
    TRY(backward(t, st));
    return aggregate_and_update(t, st, nullptr, nullptr);
}

static int graph_step(tcb_trainer* t, cudaStream_t st) {
    // captured and replayed on the trainer's own stream (the caller's may be the
    // legacy default stream, which cannot be captured), fenced by events
    if (!t->graph_stream) {
        TRY_CUDA(cudaStreamCreateWithFlags(&t->graph_stream, cudaStreamNonBlocking));
        TRY_CUDA(cudaEventCreateWithFlags(&t->graph_in, cudaEventDisableTiming));
        TRY_CUDA(cudaEventCreateWithFlags(&t->graph_out, cudaEventDisableTiming));
    }
    cudaStream_t gs = t->graph_stream;
    if (!t->graph_exec) {
        cudaGraph_t g = nullptr;
        TRY_CUDA(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
        const int rc = step_body(t, gs);
        const cudaError_t ce = cudaStreamEndCapture(gs, &g);
        if (rc != TCB_OK) {
            if (g) cudaGraphDestroy(g);
            return rc;
        }
        TRY_CUDA(ce);
        const cudaError_t ie = cudaGraphInstantiate(&t->graph_exec, g, 0);
        cudaGraphDestroy(g);
        TRY_CUDA(ie);
        t->graph_launches = t->launches;
    }
    t->launches = t->graph_launches;
    TRY_CUDA(cudaEventRecord(t->graph_in, st));
    TRY_CUDA(cudaStreamWaitEvent(gs, t->graph_in, 0));
    TRY_CUDA(cudaGraphLaunch(t->graph_exec, gs));
    TRY_CUDA(cudaEventRecord(t->graph_out, gs));
    return check_cuda(cudaStreamWaitEvent(st, t->graph_out, 0), "graph fence");
}

// Asynchronous PS step s: forward / backward on the caller's stream with
// W_max(s-1,0); the aggregation + update on ps_stream writes W_s+1 into the
// other weight buffer while step s+1 computes. Waits: forward s needs update
// s-2 (it wrote W_s-1); backward s rewrites the gradient update s-1 reads.
static int async_step(tcb_trainer* t, cudaStream_t st) {
    if (!t->ps_stream) {
        if (!t->bf16 || t->overlap || (t->n_ps > 0 && t->n_ps < t->world))
            return fail(TCB_ERR_UNSUPPORTED, "ps_async needs bf16, PS shards = GPUs and no overlap_comm");
        if (t->nvls && !t->wc2_mc)
            return fail(TCB_ERR_INVALID, "ps_async over NVLS needs tcb_trainer_attach_nvls_async");
        int lo = 0, hi = 0;
        TRY_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TRY_CUDA(cudaStreamCreateWithPriority(&t->ps_stream, cudaStreamNonBlocking, hi));
        TRY_CUDA(cudaEventCreateWithFlags(&t->ev_bwd_done, cudaEventDisableTiming));
        for (auto& e : t->ev_upd) TRY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const long long s = t->step_idx;
    t->wc_rd = s >= 1 ? static_cast<int>((s - 1) % 2) : 0;
    if (s >= 2) TRY_CUDA(cudaStreamWaitEvent(st, t->ev_upd[(s - 2) % 2], 0));
    cudaEvent_t* e = t->ph.e;
    if (t->timing) TRY_CUDA(cudaEventRecord(e[0], st));
    TRY(forward(t, st));
    if (t->timing) TRY_CUDA(cudaEventRecord(e[1], st));
    if (s >= 1) TRY_CUDA(cudaStreamWaitEvent(st, t->ev_upd[(s - 1) % 2], 0));
    TRY(backward(t, st));
    if (t->timing) TRY_CUDA(cudaEventRecord(e[2], st));
    TRY_CUDA(cudaEventRecord(t->ev_bwd_done, st));
    TRY_CUDA(cudaStreamWaitEvent(t->ps_stream, t->ev_bwd_done, 0));
    TRY(aggregate_and_update(t, t->ps_stream, t->timing ? e[3] : nullptr, t->timing ? e[4] : nullptr,
                             static_cast<int>((s + 1) % 2)));
    TRY_CUDA(cudaEventRecord(t->ev_upd[s % 2], t->ps_stream));
    if (t->timing) {  // phase timing measures the update itself: join it
        TRY_CUDA(cudaStreamWaitEvent(st, t->ev_upd[s % 2], 0));
        TRY_CUDA(cudaEventRecord(e[5], st));
    }
    ++t->step_idx;
    return check_cuda(cudaGetLastError(), "async step");
}

// The caller's stream waits for every update issued so far (asynchronous PS);
// a no-op otherwise.
TCB_API int tcb_trainer_finish(tcb_trainer* t, void* stream) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    if (t->async_ps && t->step_idx > 0)
        TRY_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), t->ev_upd[(t->step_idx - 1) % 2], 0));
    return TCB_OK;
}

TCB_API int tcb_trainer_attach_nvls_async(tcb_trainer* t, void* wcompute2, void* wcompute2_mc) {
    if (!t || !wcompute2 || !wcompute2_mc) return fail(TCB_ERR_INVALID, "NULL argument");
    if (!t->nvls || !t->async_ps) return fail(TCB_ERR_INVALID, "attach_nvls first, with ps_async");
    if (t->initialized) return fail(TCB_ERR_INVALID, "attach before the first step");
    t->ext_wc2 = wcompute2;
    t->wc2_mc = wcompute2_mc;
    return TCB_OK;
}

TCB_API int tcb_trainer_step(tcb_trainer* t, void* stream) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    TRY(poll_comm_errors(t));
    auto st = static_cast<cudaStream_t>(stream);
    TRY(ensure_ready(t, st));
    t->launches = 0;
    TRY(consume_staged(t, st));
    const int staged_launches = t->launches;
    // eager warm-up steps first (one-time kernel attribute setup stays out of the capture)
    if (t->use_graph && !t->timing && !t->layer_timing && ++t->eager_steps > 2) {
        TRY(graph_step(t, st));
        t->launches += staged_launches;
        return TCB_OK;
    }
    if (t->async_ps) return async_step(t, st);
    cudaEvent_t* e = t->ph.e;
    if (t->timing) TRY_CUDA(cudaEventRecord(e[0], st));
    TRY(forward(t, st));
    if (t->timing) TRY_CUDA(cudaEventRecord(e[1], st));
    TRY(backward(t, st));
    if (t->timing) TRY_CUDA(cudaEventRecord(e[2], st));
    TRY(aggregate_and_update(t, st, t->timing ? e[3] : nullptr, t->timing ? e[4] : nullptr));
    if (t->timing) TRY_CUDA(cudaEventRecord(e[5], st));
    return check_cuda(cudaGetLastError(), "step");
}

TCB_API int tcb_trainer_loss(tcb_trainer* t, float* loss_host, void* stream) {
    if (!t || !loss_host) return fail(TCB_ERR_INVALID, "NULL argument");
    auto st = static_cast<cudaStream_t>(stream);
    TRY_CUDA(cudaMemcpyAsync(loss_host, t->at(t->off_loss), 4, cudaMemcpyDeviceToHost, st));
    TRY_CUDA(cudaStreamSynchronize(st));
    return check_health(t, st);
}

TCB_API int tcb_trainer_enable_timing(tcb_trainer* t, int on) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    t->timing = on != 0;
    return TCB_OK;
}

TCB_API int tcb_trainer_phase_times(tcb_trainer* t, float* ms5) {
    if (!t || !ms5) return fail(TCB_ERR_INVALID, "NULL argument");
    if (!t->timing) return fail(TCB_ERR_INVALID, "timing not enabled");
    cudaEvent_t* e = t->ph.e;
    TRY_CUDA(cudaEventSynchronize(e[5]));
    for (int i = 0; i < 5; ++i) TRY_CUDA(cudaEventElapsedTime(&ms5[i], e[i], e[i + 1]));
    return TCB_OK;
}

// Paper steps 3-4 of the last timed staged batch: {host-to-device copy ms
// (copy stream), on-device preparation ms (uint8 -> compute dtype)}; -1 where
// no staged batch was timed.
TCB_API int tcb_trainer_data_times(tcb_trainer* t, float* ms2) {
    if (!t || !ms2) return fail(TCB_ERR_INVALID, "NULL argument");
    ms2[0] = ms2[1] = -1.f;
    if (t->h2d_timed) {
        TRY_CUDA(cudaEventSynchronize(t->ev_h2d[1]));
        TRY_CUDA(cudaEventElapsedTime(&ms2[0], t->ev_h2d[0], t->ev_h2d[1]));
    }
    if (t->prep_timed) {
        TRY_CUDA(cudaEventSynchronize(t->ev_prep[1]));
        TRY_CUDA(cudaEventElapsedTime(&ms2[1], t->ev_prep[0], t->ev_prep[1]));
    }
    return TCB_OK;
}

TCB_API int tcb_trainer_enable_layer_timing(tcb_trainer* t, int on) {
    if (!t) return fail(TCB_ERR_INVALID, "NULL trainer");
    if (on && t->lev.empty()) {
        t->lev.resize(t->nodes.size());
        for (auto& a : t->lev)
            for (cudaEvent_t& e : a) TRY_CUDA(cudaEventCreate(&e));
    }
    t->layer_timing = on != 0;
    return TCB_OK;
}

// JSON [{name, conv_index, flop, fwd_ms, dgrad_ms|null, wgrad_ms}] of the last step
// (flop = 2*N*Ho*Wo*K*C*R*S with logical channel counts).
TCB_API int tcb_trainer_layer_times(tcb_trainer* t, char** json_out) {
    if (!t || !json_out) return fail(TCB_ERR_INVALID, "NULL argument");
    if (t->lev.empty()) return fail(TCB_ERR_INVALID, "layer timing never enabled");
    json out = json::array();
    for (size_t i = 0; i < t->nodes.size(); ++i) {
        const Node& nd = t->nodes[i];
        if (nd.op != Op::Conv) continue;
        auto& e = t->lev[i];
        TRY_CUDA(cudaEventSynchronize(e[5]));
        float f = 0, w = 0, d = 0;
        TRY_CUDA(cudaEventElapsedTime(&f, e[0], e[1]));
        TRY_CUDA(cudaEventElapsedTime(&w, e[4], e[5]));
        if (nd.need_dgrad) TRY_CUDA(cudaEventElapsedTime(&d, e[2], e[3]));
        json r;
        r["name"] = nd.name;
        r["conv_index"] = nd.conv_index;
        r["flop"] = 2.0 * nd.n * nd.h * nd.w * nd.c_logical * t->nodes[nd.in].c_logical * nd.g.r * nd.g.s;
        r["fwd_ms"] = f;
        r["dgrad_ms"] = nd.need_dgrad ? json(d) : json(nullptr);
        r["wgrad_ms"] = w;
        out.push_back(std::move(r));
    }
    const std::string s = out.dump();
    *json_out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*json_out, s.c_str(), s.size() + 1);
    return TCB_OK;
}

TCB_API int tcb_trainer_launch_count(tcb_trainer* t, int* count) {
    if (!t || !count) return fail(TCB_ERR_INVALID, "NULL argument");
    *count = t->launches;
    return TCB_OK;
}

TCB_API int tcb_trainer_describe(tcb_trainer* t, char** json_out) {
    if (!t || !json_out) return fail(TCB_ERR_INVALID, "NULL argument");
    if (!t->arena) plan_params(t);
    json d;
    d["precision"] = t->bf16 ? "bf16" : t->tf32 ? "tf32" : "ffma";
    d["batch"] = t->batch;
    d["classes"] = t->classes;
    d["world"] = t->world;
    d["rank"] = t->rank;
    d["param_count"] = t->param_count;
    d["param_padded"] = t->param_padded;
    d["shard"] = t->shard;
    d["arena_bytes"] = t->arena_bytes;
    json layers = json::array();
    for (size_t i = 0; i < t->nodes.size(); ++i) {
        const Node& nd = t->nodes[i];
        json L;
        L["index"] = i;
        L["name"] = nd.name;
        static const char* ops[] = {"input", "conv", "maxpool", "avgpool", "loss", "concat"};
        L["op"] = ops[static_cast<int>(nd.op)];
        L["in"] = nd.in;
        L["residual"] = nd.residual;
        L["shape"] = {nd.n, nd.h, nd.w, nd.c};
        L["c_logical"] = nd.c_logical;
        if (nd.op == Op::Conv) {
            L["conv_index"] = nd.conv_index;
            L["geom"] = {nd.g.n, nd.g.h, nd.g.w, nd.g.c, nd.g.k, nd.g.r, nd.g.s, nd.g.pad_h, nd.g.pad_w,
                         nd.g.stride_h, nd.g.stride_w};
            L["relu"] = nd.relu;
            L["bias"] = nd.bias;
            L["woff"] = nd.woff;
            L["wcount"] = nd.wcount;
            L["boff"] = nd.bias ? json(nd.boff) : json(nullptr);
            L["init_scale"] = nd.init_scale;
            L["algo"] = nd.algo;
            L["stem_rows"] = static_cast<int>(i) == t->stem_node;
            L["stem_pool_fused"] = static_cast<int>(i) == t->stem_node && t->fused_pool >= 0;
            L["explicit_im2col"] = nd.narrow && static_cast<int>(i) != t->stem_node;
            L["packed_dgrad_weights"] = nd.pack_wT;
            const size_t first = nd.woff / std::max<size_t>(t->shard, 1);
            const size_t last_el = (nd.bias ? nd.boff + nd.g.k : nd.woff + nd.wcount) - 1;
            L["shards"] = {first, last_el / std::max<size_t>(t->shard, 1)};
        }
        if (nd.op == Op::MaxPool || (nd.op == Op::AvgPool && nd.f > 0)) L["pool"] = {nd.f, nd.s, nd.p};
        if (nd.op == Op::Concat) {
            L["ins"] = nd.ins;
            L["coff"] = nd.coff;
        }
        layers.push_back(std::move(L));
    }
    d["layers"] = std::move(layers);
    const std::string s = d.dump();
    *json_out = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*json_out, s.c_str(), s.size() + 1);
    return TCB_OK;
}

TCB_API int tcb_trainer_tensor(tcb_trainer* t, const char* name, void** ptr, size_t* bytes) {
    if (!t || !name || !ptr) return fail(TCB_ERR_INVALID, "NULL argument");
    if (!t->arena) return fail(TCB_ERR_INVALID, "trainer not initialised (run a step or set_batch)");
    const std::string n(name);
    const size_t es = dtype_size(t->dt);
    size_t b = 0;
    void* p = nullptr;
    auto node_bytes = [&](const Node& nd) { return size_t(nd.n) * nd.h * nd.w * nd.c * es; };
    if (n == "param") { p = t->at(t->off_param); b = t->param_padded * 4; }
    else if (n == "grad") { p = t->grad_ptr(); b = t->param_padded * 4; }
    else if (n == "momentum") { p = t->at(t->off_mom); b = t->param_padded * 4; }
    else if (n == "wcompute") {  // the latest weights (asynchronous PS: W_step_idx)
        p = t->async_ps ? t->wc_buf(static_cast<int>(t->step_idx % 2)) : t->wc_ptr();
        b = t->param_padded * es;
    }
    else if (n == "labels") { p = t->at(t->off_labels); b = size_t(t->batch) * 4; }
    else if (n == "loss") { p = t->at(t->off_loss); b = size_t(t->batch + 1) * 4; }
    else if (n == "input") { p = t->at(t->nodes[0].act); b = node_bytes(t->nodes[0]); }
    else if (n == "input_f32") {
        const Node& in = t->nodes[0];
        p = t->at(t->off_input_f32);
        b = size_t(in.n) * in.h * in.w * in.c_logical * 4;
    } else if (n.rfind("argmax:", 0) == 0) {
        const int i = std::stoi(n.substr(7));
        if (i < 0 || i >= static_cast<int>(t->nodes.size()) || t->nodes[i].op != Op::MaxPool)
            return fail(TCB_ERR_INVALID, "no such argmax tensor");
        const Node& nd = t->nodes[i];
        p = t->at(nd.argmax);
        b = size_t(nd.n) * nd.h * nd.w * nd.c;
    } else if (n.rfind("act:", 0) == 0 || n.rfind("dact:", 0) == 0) {
        const bool grad = n[0] == 'd';
        const int i = std::stoi(n.substr(grad ? 5 : 4));
        if (i < 0 || i >= static_cast<int>(t->nodes.size())) return fail(TCB_ERR_INVALID, "bad node index");
        const Node& nd = t->nodes[i];
        if (nd.op == Op::Loss || (grad && nd.op == Op::Input)) return fail(TCB_ERR_INVALID, "no such tensor");
        p = t->at(grad ? nd.grad : nd.act);
        b = node_bytes(nd);
    } else {
        return fail(TCB_ERR_INVALID, "unknown tensor " + n);
    }
    *ptr = p;
    if (bytes) *bytes = b;
    return TCB_OK;
}
