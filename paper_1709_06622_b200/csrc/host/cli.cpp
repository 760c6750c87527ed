// `traincap` command line: plan / scale / ps / catalog-validate, same options
// and exit codes as the reference (/root/reference/proj/src/cli.cpp:19-210):
// 0 success, 2 no feasible mini-batch, 1 malformed input. CLI11 is not
// available in this image, so arguments are parsed by hand here.
#include <cmath>
#include <cstring>
#include <functional>
#include <iostream>
#include <map>

#include "traincap/api.hpp"

namespace traincap {

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::int64_t bytes_to_bits(double bytes) {
    const double bits = bytes * 8.0;
    if (!(bits >= 1) || bits > 9.0e18) throw UnitError("memory size out of range");
    return static_cast<std::int64_t>(std::llround(bits));
}

// Minimal option scanner: `--name value`, `--name=value`, `--flag`, positionals.
struct Args {
    std::map<std::string, std::string> opts;
    std::vector<std::string> flags;
    std::vector<std::string> pos;

    Args(int argc, const char* const* argv, int first, const std::vector<std::string>& flag_names) {
        for (int i = first; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) {
                pos.push_back(a);
                continue;
            }
            const auto eq = a.find('=');
            std::string name = a.substr(2, eq == std::string::npos ? std::string::npos : eq - 2);
            if (std::find(flag_names.begin(), flag_names.end(), name) != flag_names.end()) {
                flags.push_back(name);
                continue;
            }
            if (eq != std::string::npos) {
                opts[name] = a.substr(eq + 1);
            } else {
                if (i + 1 >= argc) throw Usage("option --" + name + " needs a value");
                opts[name] = argv[++i];
            }
        }
    }
    bool has(const std::string& k) const { return opts.count(k) > 0; }
    bool flag(const std::string& k) const {
        return std::find(flags.begin(), flags.end(), k) != flags.end();
    }
    std::string need(const std::string& k) const {
        auto it = opts.find(k);
        if (it == opts.end()) throw Usage("--" + k + " is required");
        return it->second;
    }
    std::string get(const std::string& k, const std::string& dflt) const {
        auto it = opts.find(k);
        return it == opts.end() ? dflt : it->second;
    }
    void only(const std::vector<std::string>& allowed) const {
        for (const auto& kv : opts)
            if (std::find(allowed.begin(), allowed.end(), kv.first) == allowed.end())
                throw Usage("unknown option --" + kv.first);
    }
};

std::int64_t as_int(const std::string& s, const char* what) {
    if (auto v = parse_int(s)) return *v;
    throw Usage(std::string(what) + ": not an integer: " + s);
}
double as_double(const std::string& s, const char* what) {
    if (auto v = parse_double(s)) return *v;
    throw Usage(std::string(what) + ": not a number: " + s);
}
std::string as_format(const std::string& s) {
    if (s != "text" && s != "json") throw Usage("--format must be text or json");
    return s;
}

int cmd_plan(const Args& a) {
    a.only({"network", "catalog", "gpu-memory", "dataset-size", "candidates", "gmax", "ro",
            "workers", "bandwidth", "param-size", "format"});
    PlanRequest req;
    req.network_path = a.need("network");
    req.catalog_path = a.need("catalog");
    const std::string mem = a.need("gpu-memory");
    req.dataset_size = as_int(a.need("dataset-size"), "--dataset-size");
    if (a.has("candidates")) {
        std::string list = a.get("candidates", "");
        std::size_t start = 0;
        while (start <= list.size()) {
            const std::size_t c = list.find(',', start);
            req.candidates.push_back(as_int(list.substr(start, c - start), "--candidates"));
            if (c == std::string::npos) break;
            start = c + 1;
        }
    }
    req.max_gpus = static_cast<int>(as_int(a.get("gmax", "8"), "--gmax"));
    req.overhead_ratio = as_double(a.get("ro", "0"), "--ro");
    req.workers = static_cast<int>(as_int(a.get("workers", "1"), "--workers"));
    const std::string format = as_format(a.get("format", "text"));
    req.gpu_memory_bits = bytes_to_bits(parse_bytes(mem));
    req.bandwidth_bytes_per_sec = parse_bandwidth(a.get("bandwidth", "10Gbps"));
    if (a.has("param-size")) req.param_size_bytes = parse_bytes(a.get("param-size", ""));
    req.verify = a.flag("verify");

    const PlanReport rep = run_plan(req);
    if (format == "json")
        std::cout << render_plan_json(rep, current_timestamp());
    else
        render_plan_text(rep, std::cout);
    return rep.plan.recommended ? 0 : 2;
}

int cmd_scale(const Args& a) {
    a.only({"ro", "steps", "target", "gmax", "format"});
    if (a.has("ro") == a.has("steps")) throw DomainError("pass exactly one of --ro or --steps");
    ScaleReport rep;
    const int gmax = static_cast<int>(as_int(a.get("gmax", "8"), "--gmax"));
    const std::string format = as_format(a.get("format", "text"));
    if (a.has("ro")) {
        rep.overhead_ratio = as_double(a.get("ro", ""), "--ro");
        if (rep.overhead_ratio < 0) throw DomainError("overhead ratio must be >= 0");
    } else {
        const StepTrace tr = load_step_trace_file(a.get("steps", ""));
        rep.overhead_ratio = estimate_overhead_ratio(tr.times, tr.hidden).ratio();
        rep.steps_path = a.get("steps", "");
    }
    rep.table = scaling_table(gmax, rep.overhead_ratio);
    if (a.has("target")) {
        rep.target_speedup = as_double(a.get("target", ""), "--target");
        rep.recommendation = recommend_gpus(*rep.target_speedup, rep.overhead_ratio, gmax);
    }
    if (format == "json")
        std::cout << render_scale_json(rep, current_timestamp());
    else
        render_scale_text(rep, std::cout);
    return 0;
}

int cmd_ps(const Args& a) {
    a.only({"format"});
    if (a.pos.size() != 4) throw Usage("ps takes: param-size workers bandwidth compute-time");
    PsReport rep;
    rep.spec.param_size_bytes = parse_bytes(a.pos[0]);
    rep.spec.worker_count = static_cast<int>(as_int(a.pos[1], "workers"));
    rep.spec.bandwidth_bytes_per_sec = parse_bandwidth(a.pos[2]);
    rep.spec.gpu_count = 1;
    rep.compute_time_seconds = as_double(a.pos[3], "compute-time");
    const std::string format = as_format(a.get("format", "text"));
    rep.servers = min_parameter_servers(rep.spec, rep.compute_time_seconds);
    if (format == "json")
        std::cout << render_ps_json(rep, current_timestamp());
    else
        render_ps_text(rep, std::cout);
    return 0;
}

int cmd_catalog_validate(const Args& a) {
    a.only({"catalog-format"});
    if (a.pos.size() != 1) throw Usage("catalog-validate takes one catalog file");
    const std::string fmt = a.get("catalog-format", "");
    if (!fmt.empty() && fmt != "csv" && fmt != "json")
        throw Usage("--catalog-format must be csv or json");
    const AlgorithmCatalog cat =
        fmt.empty() ? load_catalog_file(a.pos[0])
                    : load_catalog_file(a.pos[0], fmt == "json" ? CatalogFormat::json
                                                                : CatalogFormat::csv);
    std::cout << "catalog ok: " << cat.entries().size() << " entries, " << cat.layer_count()
              << " layers, " << cat.algorithms().size() << " algorithms, "
              << cat.declared_batch_sizes().size() << " batch sizes\n";
    return 0;
}

const char* kUsage =
    "usage: traincap <plan|scale|ps|catalog-validate> [options]\n"
    "  plan --network F --catalog F --gpu-memory 12GiB --dataset-size N [--candidates a,b]\n"
    "       [--gmax 8] [--ro R] [--workers W] [--bandwidth 10Gbps] [--param-size 180MB]\n"
    "       [--format text|json] [--verify]\n"
    "  scale (--ro R | --steps F) [--target S] [--gmax 8] [--format text|json]\n"
    "  ps <param-size> <workers> <bandwidth> <compute-seconds> [--format text|json]\n"
    "  catalog-validate <file> [--catalog-format csv|json]\n";

}  // namespace

int run_cli(int argc, const char* const* argv) {
    if (argc < 2) {
        std::cerr << kUsage;
        return 1;
    }
    const std::string sub = argv[1];
    if (sub == "-h" || sub == "--help") {
        std::cout << kUsage;
        return 0;
    }
    try {
        if (sub == "plan") return cmd_plan(Args(argc, argv, 2, {"verify"}));
        if (sub == "scale") return cmd_scale(Args(argc, argv, 2, {}));
        if (sub == "ps") return cmd_ps(Args(argc, argv, 2, {}));
        if (sub == "catalog-validate") return cmd_catalog_validate(Args(argc, argv, 2, {}));
        std::cerr << "unknown subcommand `" << sub << "`\n" << kUsage;
        return 1;
    } catch (const Usage& u) {
        std::cerr << u.what() << "\n" << kUsage;
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}

}  // namespace traincap
