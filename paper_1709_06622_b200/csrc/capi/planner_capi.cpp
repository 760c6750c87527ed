// C-ABI over the traincap C++ planner API: one JSON-in / JSON-out entry point.
//
// This translation unit uses only public traincap:: names, so it compiles
// unchanged against this build's headers (exported as tcb_planner_call) and
// against the reference's headers (oracle/Makefile builds it with
// -DTCB_PLANNER_PREFIX=tcref_ and -Dtraincap=tcref into oracle/_ref/). The
// parity suite sends identical requests to both and compares the replies —
// which also proves the API is a drop-in for the reference's.
//
// Exceptions never cross the boundary: every error becomes
// {"error": {"type": <traincap class>, "message": ..., "line"/"layer_id": ...}}.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include <json.hpp>

#include "traincap/batch_plan.hpp"
#include "traincap/catalog.hpp"
#include "traincap/conv_select.hpp"
#include "traincap/errors.hpp"
#include "traincap/io.hpp"
#include "traincap/mem_model.hpp"
#include "traincap/net_model.hpp"
#include "traincap/report.hpp"
#include "traincap/scale_plan.hpp"
#include "traincap/units.hpp"
#include "traincap/util.hpp"

#ifndef TCB_PLANNER_PREFIX
#define TCB_PLANNER_PREFIX tcb_
#endif
#define TCB_CAT2(a, b) a##b
#define TCB_CAT(a, b) TCB_CAT2(a, b)
#define TCB_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

using J = nlohmann::ordered_json;
namespace tc = traincap;

J num(double v) {
    if (std::isfinite(v)) return J(v);
    if (std::isnan(v)) return J("nan");
    return J(v > 0 ? "inf" : "-inf");
}

tc::NetworkSpec network_of(const J& v) {
    if (v.is_string()) {
        std::istringstream in(v.get<std::string>());
        return tc::load_network(in);
    }
    // Structured form, built directly (lets tests hand in invalid values).
    tc::NetworkSpec net;
    const auto& inp = v.at("input");
    net.input_shape = {inp.at(0).get<std::int64_t>(), inp.at(1).get<std::int64_t>(),
                       inp.at(2).get<std::int64_t>()};
    int id = 0;
    for (const auto& f : v.at("features")) {
        tc::FeatureLayerSpec l;
        l.kind = f.at(0).get<std::string>() == "pool" ? tc::LayerKind::pooling
                                                      : tc::LayerKind::convolution;
        l.filter_size = f.at(1).get<std::int64_t>();
        l.stride = f.at(2).get<std::int64_t>();
        l.padding = f.at(3).get<std::int64_t>();
        l.filter_count = f.at(4).get<std::int64_t>();
        l.layer_id = ++id;
        net.feature_layers.push_back(l);
    }
    int cid = 0;
    for (const auto& c : v.at("classifier"))
        net.classifier_layers.push_back({c.get<std::int64_t>(), ++cid});
    return net;
}

tc::CatalogFormat format_of(const J& req) {
    return req.value("format", std::string("csv")) == "json" ? tc::CatalogFormat::json
                                                             : tc::CatalogFormat::csv;
}

tc::AlgorithmCatalog catalog_of(const J& req) {
    std::istringstream in(req.at("catalog").get<std::string>());
    return tc::load_catalog(in, format_of(req));
}

J entry_json(const tc::CostEntry& e) {
    J o;
    o["layer_id"] = e.layer_id;
    o["algorithm"] = e.algorithm;
    o["batch_size"] = e.batch_size;
    o["time_seconds"] = num(e.time_seconds);
    o["memory_bits"] = e.memory_bits;
    return o;
}

tc::LayerOptions options_of(const J& v) {
    tc::LayerOptions opts;
    for (const auto& layer : v) {
        std::vector<tc::CostEntry> row;
        for (const auto& e : layer) {
            tc::CostEntry c;
            c.layer_id = e.at("layer_id").get<int>();
            c.algorithm = e.at("algorithm").get<std::string>();
            c.batch_size = e.at("batch_size").get<std::int64_t>();
            c.time_seconds = e.at("time_seconds").get<double>();
            c.memory_bits = e.at("memory_bits").get<std::int64_t>();
            row.push_back(c);
        }
        opts.push_back(std::move(row));
    }
    return opts;
}

J breakdown_json(const tc::MemoryBreakdown& b) {
    J o;
    o["feature_maps"] = b.feature_maps;
    o["model_params"] = b.model_params;
    o["classifier"] = b.classifier;
    o["gpu_total"] = b.gpu_total;
    o["bound"] = b.bound;
    o["batch_size"] = b.batch_size;
    return o;
}

J solve_json(const tc::SolveResult& r) {
    J o;
    o["feasible"] = r.feasible();
    o["min_achievable_memory"] = r.min_achievable_memory;
    if (r.feasible()) {
        J a = J::object();
        for (const auto& [layer, algo] : r.selection->assignment) a[std::to_string(layer)] = algo;
        o["assignment"] = std::move(a);
        o["total_time"] = num(r.selection->total_time);
        o["total_memory"] = r.selection->total_memory;
    }
    return o;
}

J plan_json(const tc::BatchPlan& p) {
    J o;
    J cands = J::array();
    for (const auto& c : p.candidates) {
        J x;
        x["batch_size"] = c.batch_size;
        x["breakdown"] = breakdown_json(c.breakdown);
        x["solve"] = solve_json(c.solve);
        x["epoch_time_seconds"] = c.epoch_time_seconds ? num(*c.epoch_time_seconds) : J(nullptr);
        x["throughput"] = c.throughput ? num(*c.throughput) : J(nullptr);
        x["memory_limited_layers"] = c.memory_limited_layers;
        cands.push_back(std::move(x));
    }
    o["candidates"] = std::move(cands);
    o["recommended"] = p.recommended ? J(*p.recommended) : J(nullptr);
    J adv = J::array();
    for (const auto& a : p.advisories) {
        J x;
        x["kind"] = tc::to_string(a.kind);
        x["message"] = a.message;
        x["affected_layers"] = a.affected_layers;
        adv.push_back(std::move(x));
    }
    o["advisories"] = std::move(adv);
    return o;
}

J scaling_json(const std::vector<tc::ScalingEstimate>& t) {
    J rows = J::array();
    for (const auto& s : t) rows.push_back(J::array({s.gpus, num(s.efficiency), num(s.speedup)}));
    return rows;
}

tc::StepTrace trace_of(const J& req) {
    std::istringstream in(req.at("trace").get<std::string>());
    return tc::load_step_trace(in);
}

J dispatch(const J& req) {
    const std::string op = req.at("op").get<std::string>();
    J out;
    if (op == "propagate_shapes") {
        J s = J::array();
        for (const auto& t : tc::propagate_shapes(network_of(req.at("network"))))
            s.push_back(J::array({t.width, t.height, t.depth}));
        out["shapes"] = std::move(s);
    } else if (op == "validate_network") {
        J v = J::array();
        for (const auto& x : tc::validate_network(network_of(req.at("network"))))
            v.push_back(J::array({x.layer_id, x.message}));
        out["violations"] = std::move(v);
    } else if (op == "network_summary") {
        const auto net = network_of(req.at("network"));
        out["conv_layers"] = net.convolution_layer_count();
        out["feature_layers"] = net.feature_layers.size();
        out["classifier_layers"] = net.classifier_layers.size();
    } else if (op == "memory_bound") {
        out = breakdown_json(tc::memory_bound(req.at("gpu_bits").get<std::int64_t>(),
                                              network_of(req.at("network")),
                                              req.at("batch").get<std::int64_t>()));
    } else if (op == "feature_map_memory") {
        const auto net = network_of(req.at("network"));
        out["bits"] = tc::feature_map_memory(net, tc::propagate_shapes(net),
                                             req.at("batch").get<std::int64_t>());
    } else if (op == "model_param_memory") {
        out["bits"] = tc::model_param_memory(network_of(req.at("network")));
    } else if (op == "classifier_memory") {
        std::vector<tc::ClassifierLayerSpec> cl;
        int id = 0;
        for (const auto& n : req.at("layers")) cl.push_back({n.get<std::int64_t>(), ++id});
        out["bits"] = tc::classifier_memory(cl);
    } else if (op == "parameter_bits") {
        out["bits"] = tc::parameter_bits(network_of(req.at("network")));
    } else if (op == "load_catalog") {
        const auto cat = catalog_of(req);
        out["layer_count"] = cat.layer_count();
        out["batch_sizes"] = cat.declared_batch_sizes();
        out["algorithms"] = cat.algorithms();
        J e = J::array();
        for (const auto& x : cat.entries()) e.push_back(entry_json(x));
        out["entries"] = std::move(e);
        out["csv"] = tc::save_catalog(cat, tc::CatalogFormat::csv);
        out["json"] = tc::save_catalog(cat, tc::CatalogFormat::json);
        if (req.contains("batch")) {
            const auto b = req.at("batch").get<std::int64_t>();
            J opts = J::array();
            for (int l = 1; l <= cat.layer_count(); ++l) {
                J row = J::array();
                for (const auto& x : cat.options(l, b)) row.push_back(entry_json(x));
                opts.push_back(std::move(row));
            }
            out["options"] = std::move(opts);
            out["has_batch"] = cat.has_batch_size(b);
        }
    } else if (op == "catalog_options") {
        J opts = J::array();
        for (const auto& row : tc::catalog_options(catalog_of(req), req.at("batch").get<std::int64_t>())) {
            J r = J::array();
            for (const auto& x : row) r.push_back(entry_json(x));
            opts.push_back(std::move(r));
        }
        out["options"] = std::move(opts);
    } else if (op == "solve") {
        const auto opts = options_of(req.at("options"));
        const auto bound = req.at("bound").get<std::int64_t>();
        out = solve_json(req.value("brute", false) ? tc::brute_force_selection(opts, bound)
                                                   : tc::solve_selection(opts, bound));
    } else if (op == "solve_catalog") {
        const auto cat = catalog_of(req);
        const auto b = req.at("batch").get<std::int64_t>();
        const auto bound = req.at("bound").get<std::int64_t>();
        out = solve_json(req.value("brute", false) ? tc::brute_force_selection(cat, b, bound)
                                                   : tc::solve_selection(cat, b, bound));
    } else if (op == "plan_batch_size") {
        const auto cat = catalog_of(req);
        std::vector<std::int64_t> cands;
        if (req.contains("candidates"))
            cands = req.at("candidates").get<std::vector<std::int64_t>>();
        else
            cands = tc::default_batch_candidates(cat);
        out = plan_json(tc::plan_batch_size(network_of(req.at("network")), cat,
                                            req.at("gpu_bits").get<std::int64_t>(),
                                            req.at("dataset").get<std::int64_t>(), cands));
#ifndef TCB_REFERENCE_SHIM  // this build's extension: the reference planner has no branched-graph entry
    } else if (op == "plan_batch_size_graph") {
        // branched networks: resident bits per candidate from the executor layout
        const auto cat = catalog_of(req);
        std::vector<std::pair<std::int64_t, std::int64_t>> res;
        for (const auto& [k, v] : req.at("resident_bits").items())
            res.emplace_back(std::stoll(k), v.get<std::int64_t>());
        std::sort(res.begin(), res.end());
        out = plan_json(tc::plan_batch_size_resident(cat, res, req.at("gpu_bits").get<std::int64_t>(),
                                                     req.at("dataset").get<std::int64_t>()));
#endif
    } else if (op == "default_batch_candidates") {
        out["candidates"] = tc::default_batch_candidates(catalog_of(req));
    } else if (op == "model_caveats") {
        out["caveats"] = tc::model_caveats();
    } else if (op == "efficiency") {
        out["value"] = num(tc::efficiency(req.at("gpus").get<int>(), req.at("r").get<double>()));
    } else if (op == "scaling_table") {
        out["table"] = scaling_json(
            tc::scaling_table(req.at("max_gpus").get<int>(), req.at("r").get<double>()));
    } else if (op == "max_overhead_ratio") {
        out["value"] = num(
            tc::max_overhead_ratio(req.at("gpus").get<int>(), req.at("alpha").get<double>()));
    } else if (op == "recommend_gpus") {
        const auto rec = tc::recommend_gpus(req.at("target").get<double>(),
                                            req.at("r").get<double>(),
                                            req.at("max_gpus").get<int>());
        out["gpus"] = rec.gpus ? J(*rec.gpus) : J(nullptr);
        out["speedup_cap"] = num(rec.speedup_cap);
    } else if (op == "load_step_trace" || op == "estimate_overhead_ratio") {
        const auto tr = trace_of(req);
        J t = J::object();
        for (const auto& [s, v] : tr.times) t[tc::to_string(s)] = num(v);
        out["times"] = std::move(t);
        J h = J::array();
        for (const auto s : tr.hidden) h.push_back(tc::to_string(s));
        out["hidden"] = std::move(h);
        if (op == "estimate_overhead_ratio") {
            const auto p = tc::estimate_overhead_ratio(tr.times, tr.hidden);
            out["compute_time"] = num(p.compute_time);
            out["overhead_time"] = num(p.overhead_time);
            out["ratio"] = num(p.ratio());
        }
    } else if (op == "min_parameter_servers") {
        tc::ClusterSpec spec{req.at("workers").get<int>(), req.at("param_bytes").get<double>(),
                             req.at("bandwidth").get<double>(), req.value("gpus", 1)};
        out["servers"] = tc::min_parameter_servers(spec, req.at("compute_time").get<double>());
    } else if (op == "parse_bytes") {
        out["value"] = num(tc::parse_bytes(req.at("text").get<std::string>()));
    } else if (op == "parse_bandwidth") {
        out["value"] = num(tc::parse_bandwidth(req.at("text").get<std::string>()));
    } else if (op == "human_bytes") {
        out["text"] = tc::human_bytes(req.at("value").get<double>());
    } else if (op == "to_shortest_string") {
        out["text"] = tc::to_shortest_string(req.at("value").get<double>());
    } else if (op == "parse_number") {
        const auto t = req.at("text").get<std::string>();
        const auto d = tc::parse_double(t);
        const auto i = tc::parse_int(t);
        out["double"] = d ? num(*d) : J(nullptr);
        out["int"] = i ? J(*i) : J(nullptr);
    } else if (op == "run_plan") {
        tc::PlanRequest pr;
        pr.network_path = req.at("network_path").get<std::string>();
        pr.catalog_path = req.at("catalog_path").get<std::string>();
        pr.gpu_memory_bits = req.at("gpu_bits").get<std::int64_t>();
        pr.dataset_size = req.at("dataset").get<std::int64_t>();
        if (req.contains("candidates"))
            pr.candidates = req.at("candidates").get<std::vector<std::int64_t>>();
        pr.max_gpus = req.value("max_gpus", 8);
        pr.overhead_ratio = req.value("ro", 0.0);
        pr.workers = req.value("workers", 1);
        pr.bandwidth_bytes_per_sec = req.value("bandwidth", 1.25e9);
        if (req.contains("param_size")) pr.param_size_bytes = req.at("param_size").get<double>();
        pr.verify = req.value("verify", false);
        const auto rep = tc::run_plan(pr);
        out["json"] = tc::render_plan_json(rep, req.value("timestamp", std::string("T")));
        std::ostringstream txt;
        tc::render_plan_text(rep, txt);
        out["text"] = txt.str();
        out["recommended"] = rep.plan.recommended ? J(*rep.plan.recommended) : J(nullptr);
        out["parameter_servers"] = rep.parameter_servers ? J(*rep.parameter_servers) : J(nullptr);
    } else if (op == "render_scale") {
        tc::ScaleReport sr;
        sr.overhead_ratio = req.at("r").get<double>();
        if (req.contains("steps_path")) sr.steps_path = req.at("steps_path").get<std::string>();
        sr.table = tc::scaling_table(req.at("max_gpus").get<int>(), sr.overhead_ratio);
        if (req.contains("target")) {
            sr.target_speedup = req.at("target").get<double>();
            sr.recommendation =
                tc::recommend_gpus(*sr.target_speedup, sr.overhead_ratio, req.at("max_gpus").get<int>());
        }
        out["json"] = tc::render_scale_json(sr, req.value("timestamp", std::string("T")));
        std::ostringstream txt;
        tc::render_scale_text(sr, txt);
        out["text"] = txt.str();
    } else if (op == "render_ps") {
        tc::PsReport pr;
        pr.spec = {req.at("workers").get<int>(), req.at("param_bytes").get<double>(),
                   req.at("bandwidth").get<double>(), 1};
        pr.compute_time_seconds = req.at("compute_time").get<double>();
        pr.servers = tc::min_parameter_servers(pr.spec, pr.compute_time_seconds);
        out["json"] = tc::render_ps_json(pr, req.value("timestamp", std::string("T")));
        std::ostringstream txt;
        tc::render_ps_text(pr, txt);
        out["text"] = txt.str();
    } else {
        throw std::invalid_argument("unknown op `" + op + "`");
    }
    return out;
}

J error_json(const char* type, const std::string& msg) {
    J e;
    e["type"] = type;
    e["message"] = msg;
    J o;
    o["error"] = std::move(e);
    return o;
}

char* to_c_string(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

}  // namespace

TCB_EXPORT char* TCB_CAT(TCB_PLANNER_PREFIX, planner_call)(const char* request_json) {
    J reply;
    try {
        reply = dispatch(J::parse(request_json));
    } catch (const tc::ParseError& e) {
        reply = error_json("ParseError", e.what());
        reply["error"]["line"] = e.line();
    } catch (const tc::NonPositiveShapeError& e) {
        reply = error_json("NonPositiveShapeError", e.what());
        reply["error"]["layer_id"] = e.layer_id();
    } catch (const tc::DuplicateKeyError& e) {
        reply = error_json("DuplicateKeyError", e.what());
    } catch (const tc::IncompleteCatalogError& e) {
        reply = error_json("IncompleteCatalogError", e.what());
    } catch (const tc::OverflowError& e) {
        reply = error_json("OverflowError", e.what());
    } catch (const tc::DomainError& e) {
        reply = error_json("DomainError", e.what());
    } catch (const tc::UnitError& e) {
        reply = error_json("UnitError", e.what());
    } catch (const tc::MissingComputeStepError& e) {
        reply = error_json("MissingComputeStepError", e.what());
    } catch (const tc::InstanceTooLargeError& e) {
        reply = error_json("InstanceTooLargeError", e.what());
    } catch (const tc::CandidateNotInCatalogError& e) {
        reply = error_json("CandidateNotInCatalogError", e.what());
    } catch (const tc::ValidationError& e) {
        reply = error_json("ValidationError", e.what());
    } catch (const tc::Error& e) {
        reply = error_json("Error", e.what());
    } catch (const std::exception& e) {
        reply = error_json("BadRequest", e.what());
    }
    return to_c_string(reply.dump());
}

TCB_EXPORT void TCB_CAT(TCB_PLANNER_PREFIX, planner_free)(char* p) { std::free(p); }
