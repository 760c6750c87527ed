// B200 profiler: measures every (conv layer, algorithm, mini-batch) on the
// device and emits the reference's cost catalog — the boundary through which
// measured GPU costs enter the planner (CostEntry, /root/reference/proj/
// include/traincap/catalog.hpp:19-27; README.md:197-199 "profile on the
// target hardware into catalog rows").
//
//   time_seconds = median over reps of (fwd + dgrad + wgrad) CUDA-event time
//                  (dgrad omitted for layer 1, whose input needs no gradient —
//                  exactly the passes the training step runs)
//   memory_bits  = 8 * the plan's workspace bytes (split-K partials, packed
//                  dgrad weights, Winograd/FFT transformed planes)
//
// Algorithms that do not apply to a layer (TCB_ERR_UNSUPPORTED) or whose
// buffers do not fit in HBM produce no row — absence is a value in the
// reference's catalog. The catalog is assembled and
// serialised by this build's traincap::AlgorithmCatalog / save_catalog, so the
// CSV round-trips doubles exactly.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>
#include <json.hpp>

#include "runtime.h"
#include "tcb.h"
#include "tcb/kernels.h"
#include "traincap/api.hpp"

#define TCB_API extern "C" __attribute__((visibility("default")))

namespace tcb {
namespace {

using json = nlohmann::json;

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (cudaMalloc(&p, std::max<size_t>(bytes, 256)) != cudaSuccess) p = nullptr;
        if (p) cudaMemset(p, 0, std::max<size_t>(bytes, 256));  // workspaces: split-K counters at 0
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct Measured {
    bool ok = false;
    double fwd_ms = 0, dgrad_ms = 0, wgrad_ms = 0, total_ms = 0;
    size_t workspace = 0;
    std::string why;
};

int algo_id(const std::string& a) {
    if (a == "gemm") return TCB_ALGO_GEMM;
    if (a == "winograd") return TCB_ALGO_WINOGRAD;
    if (a == "fft") return TCB_ALGO_FFT;
    return -1;
}

// fused: the in-kernel split-K wgrad reduction, exactly as the executor runs it
// (config "fused_split_reduce" / $TCB_FUSED_SPLIT_REDUCE, default off), so the
// catalog's wgrad cost is the one the step pays.
Measured measure(const ConvGeom& g, int algo, int prec, bool need_dgrad, int reps, cudaStream_t st,
                 bool fused) {
    Measured m;
    if (!algo_applies(g, algo, prec)) {
        m.why = "unsupported";
        return m;
    }
    const ConvPlanLayout L = conv_plan_layout(g, algo, prec);
    const DType dt = prec == TCB_PREC_BF16 ? DType::BF16 : DType::F32;
    const size_t es = dtype_size(dt);
    const size_t nx = size_t(g.n) * g.h * g.w * g.c, nw = size_t(g.k) * g.r * g.s * g.c;
    const size_t ny = size_t(g.n) * g.ho() * g.wo() * g.k;
    DevBuf x(nx * es), w(nw * es), y(ny * es), dy(ny * es), dx(nx * es), dw(nw * 4), db(g.k * 4),
        ws(L.total);
    if (!x.p || !w.p || !y.p || !dy.p || !dx.p || !dw.p || !db.p || !ws.p) {
        cudaGetLastError();
        m.why = "does not fit in HBM";
        return m;
    }
    fill_uniform(dt, x.p, nx, 1, 1, -1.f, 1.f, st);
    fill_uniform(dt, w.p, nw, 1, 2, -0.05f, 0.05f, st);
    fill_uniform(dt, dy.p, ny, 1, 3, -1.f, 1.f, st);
    auto* wTp = static_cast<char*>(ws.p) + L.off_wT;
    Epilogue none;
    auto run_fwd = [&]() -> cudaError_t {
        if (algo == TCB_ALGO_GEMM && prec == TCB_PREC_TF32)
            return conv_tf32_fwd(g, static_cast<float*>(x.p), static_cast<float*>(w.p), none,
                                 static_cast<float*>(y.p), st);
        if (algo == TCB_ALGO_GEMM)
            // split-K forwards (fc layers) run as in the executor, through the workspace
            return dt == DType::BF16 ? conv_tc_fwd(g, x.p, w.p, none, y.p, st,
                                                   !conv_tc_narrow(g) && conv_tc_workspace(g, ConvMode::Fwd) ? ws.p
                                                                                                            : nullptr)
                                     : conv_ffma_fwd(g, static_cast<float*>(x.p), static_cast<float*>(w.p),
                                                     none, static_cast<float*>(y.p), st);
        if (algo == TCB_ALGO_WINOGRAD) return winograd_fwd(g, dt, x.p, w.p, none, y.p, ws.p, st);
        return fft_fwd(g, dt, x.p, w.p, none, y.p, ws.p, st);
    };
    auto run_dgrad = [&]() -> cudaError_t {
        if (algo == TCB_ALGO_GEMM) {
            if (dt == DType::BF16) {
                // the packing pass is part of the measured dgrad where the geometry needs it
                cudaError_t e = conv_tc_dgrad_needs_pack(g) ? pack_dgrad_weights(DType::BF16, w.p, wTp, g, st)
                                                            : cudaSuccess;
                return e != cudaSuccess ? e : conv_tc_dgrad(g, dy.p, w.p, wTp, none, dx.p, st);
            }
            if (prec == TCB_PREC_TF32)
                return conv_tf32_dgrad(g, static_cast<float*>(dy.p), static_cast<float*>(w.p), none,
                                       static_cast<float*>(dx.p), st);
            return conv_ffma_dgrad(g, static_cast<float*>(dy.p), static_cast<float*>(w.p), none,
                                   static_cast<float*>(dx.p), st);
        }
        if (algo == TCB_ALGO_WINOGRAD) return winograd_dgrad(g, dt, dy.p, w.p, none, dx.p, ws.p, st);
        return fft_dgrad(g, dt, dy.p, w.p, none, dx.p, ws.p, st);
    };
    auto run_wgrad = [&]() -> cudaError_t {
        if (algo == TCB_ALGO_GEMM && prec == TCB_PREC_TF32)
            return conv_tf32_wgrad(g, static_cast<float*>(dy.p), static_cast<float*>(x.p),
                                   static_cast<float*>(dw.p), ws.p, st);
        if (algo == TCB_ALGO_GEMM)
            return dt == DType::BF16 ? conv_tc_wgrad(g, dy.p, x.p, static_cast<float*>(dw.p), ws.p, st,
                                                     false,
                                                     fused ? reinterpret_cast<int*>(static_cast<char*>(ws.p) +
                                                                                    L.off_counters)
                                                           : nullptr)
                                     : conv_ffma_wgrad(g, static_cast<float*>(dy.p), static_cast<float*>(x.p),
                                                       static_cast<float*>(dw.p), ws.p, st);
        if (algo == TCB_ALGO_WINOGRAD)
            return winograd_wgrad(g, dt, dy.p, x.p, static_cast<float*>(dw.p), ws.p, st);
        return fft_wgrad(g, dt, dy.p, x.p, static_cast<float*>(dw.p), ws.p, st);
    };
    cudaEvent_t ev[4];
    for (auto& e : ev) cudaEventCreate(&e);
    std::vector<double> f, d, wg, tot;
    cudaError_t err = cudaSuccess;
    for (int it = -1; it < reps && err == cudaSuccess; ++it) {  // it == -1: warm-up
        cudaEventRecord(ev[0], st);
        err = run_fwd();
        cudaEventRecord(ev[1], st);
        if (err == cudaSuccess && need_dgrad) err = run_dgrad();
        cudaEventRecord(ev[2], st);
        if (err == cudaSuccess) err = run_wgrad();
        cudaEventRecord(ev[3], st);
        if (err == cudaSuccess) err = cudaEventSynchronize(ev[3]);
        if (err != cudaSuccess || it < 0) continue;
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, ev[0], ev[1]);
        cudaEventElapsedTime(&b, ev[1], ev[2]);
        cudaEventElapsedTime(&c, ev[2], ev[3]);
        f.push_back(a);
        d.push_back(b);
        wg.push_back(c);
        tot.push_back(double(a) + b + c);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    if (err != cudaSuccess) {
        m.why = cudaGetErrorString(err);
        cudaGetLastError();
        return m;
    }
    auto median = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v[v.size() / 2];
    };
    m.ok = true;
    m.fwd_ms = median(f);
    m.dgrad_ms = need_dgrad ? median(d) : 0.0;
    m.wgrad_ms = median(wg);
    m.total_ms = median(tot);
    m.workspace = L.total;
    return m;
}

}  // namespace
}  // namespace tcb

using namespace tcb;

// Request JSON:
//   {"layers": [{"h","w","c","k","r","s","pad_h","pad_w","stride_h","stride_w"}, ...],
//    "batches": [32, 64, ...], "algorithms": ["gemm", "winograd", "fft"],
//    "precision": "bf16"|"tf32"|"ffma", "reps": 5}
//   (a layer may carry "c_alloc", "k_alloc", "c_valid": the executor's allocation)
// Reply JSON: {"csv": <catalog CSV>, "rows": [per-measurement detail], "skipped": [...]}.
TCB_API int tcb_profile_catalog(const char* request_json, char** reply_out) {
    if (!request_json || !reply_out) return fail(TCB_ERR_INVALID, "NULL argument");
    try {
        const json req = json::parse(request_json);
        const std::string pname = req.value("precision", std::string("bf16"));
        const bool bf16 = pname == "bf16";
        const int prec = bf16 ? TCB_PREC_BF16 : pname == "tf32" ? TCB_PREC_TF32 : TCB_PREC_FFMA_FP32;
        // tensor-core layouts pad channels: 16-byte chunks = 8 bf16 / 4 fp32
        const int cpad = bf16 ? 8 : prec == TCB_PREC_TF32 ? 4 : 1;
        const int reps = std::max(1, req.value("reps", 5));
        const char* fe = std::getenv("TCB_FUSED_SPLIT_REDUCE");
        const bool fused = req.value("fused_split_reduce", fe != nullptr && fe[0] == '1');
        std::vector<traincap::CostEntry> rows;
        json detail = json::array(), skipped = json::array();
        cudaStream_t st = nullptr;
        int layer_id = 0;
        for (const json& L : req.at("layers")) {
            ++layer_id;
            for (const json& bj : req.at("batches")) {
                const int n = bj.get<int>();
                const int c_log = L.at("c").get<int>();
                // "c_alloc" / "k_alloc" / "c_valid": the executor's channel allocation
                // (tcb_trainer_describe), so the catalog times what the step runs
                ConvGeom g{n,
                           L.at("h").get<int>(),
                           L.at("w").get<int>(),
                           L.value("c_alloc", (c_log + cpad - 1) / cpad * cpad),
                           L.value("k_alloc", (L.at("k").get<int>() + cpad - 1) / cpad * cpad),
                           L.at("r").get<int>(),
                           L.value("s", L.at("r").get<int>()),
                           L.value("pad_h", 0),
                           L.value("pad_w", L.value("pad_h", 0)),
                           L.value("stride_h", 1),
                           L.value("stride_w", L.value("stride_h", 1))};
                if (L.contains("c_valid") && L.at("c_valid").get<int>() < g.c) g.c_valid = L.at("c_valid").get<int>();
                for (const json& aj : req.at("algorithms")) {
                    const std::string algo = aj.get<std::string>();
                    const int id = algo_id(algo);
                    if (id < 0) return fail(TCB_ERR_INVALID, "unknown algorithm " + algo);
                    const Measured m = measure(g, id, prec, layer_id > 1, reps, st, fused);
                    if (!m.ok) {
                        skipped.push_back({{"layer_id", layer_id}, {"batch", n}, {"algorithm", algo},
                                           {"why", m.why}});
                        continue;
                    }
                    rows.push_back({layer_id, algo, n, m.total_ms / 1e3,
                                    static_cast<std::int64_t>(m.workspace) * 8});
                    detail.push_back({{"layer_id", layer_id}, {"batch", n}, {"algorithm", algo},
                                      {"fwd_ms", m.fwd_ms}, {"dgrad_ms", m.dgrad_ms},
                                      {"wgrad_ms", m.wgrad_ms}, {"total_ms", m.total_ms},
                                      {"workspace_bytes", m.workspace}});
                }
            }
        }
        json out;
        out["csv"] = traincap::save_catalog(traincap::AlgorithmCatalog(rows), traincap::CatalogFormat::csv);
        out["rows"] = std::move(detail);
        out["skipped"] = std::move(skipped);
        const std::string s = out.dump();
        *reply_out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(*reply_out, s.c_str(), s.size() + 1);
        return TCB_OK;
    } catch (const traincap::Error& e) {
        return fail(TCB_ERR_INVALID, std::string("catalog: ") + e.what());
    } catch (const std::exception& e) {
        return fail(TCB_ERR_INVALID, e.what());
    }
}
