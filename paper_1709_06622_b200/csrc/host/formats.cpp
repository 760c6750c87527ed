// Cost catalog (validated table of measured T_{k,l}, M_{k,l}) and the two
// text formats that feed the planner: `.net` networks and step traces.
//
// Behaviour follows the reference boundary:
//   catalog invariants + queries   /root/reference/proj/src/catalog.cpp:48-121
//   CSV / JSON readers, writer     /root/reference/proj/src/catalog.cpp:125-244
//   `.net` + step-trace parsers    /root/reference/proj/src/io.cpp:32-138
// The B200 profiler (csrc/host/profiler.cpp) writes catalogs through
// save_catalog, so doubles must survive a write/read round trip bit-exactly.
#include <algorithm>
#include <fstream>
#include <sstream>
#include <tuple>

#include <json.hpp>

#include "traincap/api.hpp"

namespace traincap {

namespace {

constexpr std::string_view kCatalogHeader =
    "layer_id,algorithm,batch_size,time_seconds,memory_bits";

void require_valid_row(const CostEntry& e, std::size_t line) {
    if (e.layer_id < 1) throw ParseError("layer_id must be >= 1", line);
    if (e.algorithm.empty()) throw ParseError("algorithm name must be non-empty", line);
    if (e.batch_size < 1) throw ParseError("batch_size must be >= 1", line);
    if (!(e.time_seconds > 0.0)) throw ParseError("time_seconds must be > 0", line);
    if (e.memory_bits < 0) throw ParseError("memory_bits must be >= 0", line);
}

bool row_order(const CostEntry& a, const CostEntry& b) {
    return std::tie(a.layer_id, a.batch_size, a.algorithm) <
           std::tie(b.layer_id, b.batch_size, b.algorithm);
}

bool option_order(const CostEntry& a, const CostEntry& b) {
    return std::tie(a.time_seconds, a.memory_bits, a.algorithm) <
           std::tie(b.time_seconds, b.memory_bits, b.algorithm);
}

}  // namespace

// ------------------------------------------------------------- catalog ----

AlgorithmCatalog::AlgorithmCatalog(std::vector<CostEntry> rows,
                                   const std::vector<std::size_t>* source_lines) {
    const auto origin = [&](std::size_t i) { return source_lines ? (*source_lines)[i] : i + 1; };

    // Field checks and duplicate keys, in input order.
    std::map<std::tuple<int, std::string, std::int64_t>, std::size_t> first_seen;
    for (std::size_t i = 0; i < rows.size(); ++i) {
        const CostEntry& r = rows[i];
        require_valid_row(r, origin(i));
        auto key = std::make_tuple(r.layer_id, r.algorithm, r.batch_size);
        auto hit = first_seen.find(key);
        if (hit != first_seen.end())
            throw DuplicateKeyError("duplicate catalog key (layer " + std::to_string(r.layer_id) +
                                    ", " + r.algorithm + ", batch " +
                                    std::to_string(r.batch_size) + ") on lines " +
                                    std::to_string(origin(hit->second)) + " and " +
                                    std::to_string(origin(i)));
        first_seen.emplace(std::move(key), i);
    }
    if (rows.empty()) throw IncompleteCatalogError("catalog has no entries");

    std::set<std::int64_t> batches;
    std::set<std::string> algos;
    std::set<std::pair<int, std::int64_t>> covered;
    for (const CostEntry& r : rows) {
        layers_ = std::max(layers_, r.layer_id);
        batches.insert(r.batch_size);
        algos.insert(r.algorithm);
        covered.emplace(r.layer_id, r.batch_size);
    }
    batches_.assign(batches.begin(), batches.end());
    algos_.assign(algos.begin(), algos.end());

    // Every (layer 1..q, declared batch) must be plannable; this also forces
    // the layer ids to be contiguous.
    for (int layer = 1; layer <= layers_; ++layer)
        for (std::int64_t b : batches_)
            if (!covered.count({layer, b}))
                throw IncompleteCatalogError("no algorithm profiled for layer " +
                                             std::to_string(layer) + " at batch size " +
                                             std::to_string(b));

    std::sort(rows.begin(), rows.end(), row_order);
    rows_ = std::move(rows);
}

bool AlgorithmCatalog::has_batch_size(std::int64_t b) const {
    return std::binary_search(batches_.begin(), batches_.end(), b);
}

std::optional<CostEntry> AlgorithmCatalog::query(int layer_id, const AlgorithmId& algorithm,
                                                 std::int64_t batch_size) const {
    auto it = std::find_if(rows_.begin(), rows_.end(), [&](const CostEntry& r) {
        return r.layer_id == layer_id && r.batch_size == batch_size && r.algorithm == algorithm;
    });
    if (it == rows_.end()) return std::nullopt;
    return *it;
}

std::vector<CostEntry> AlgorithmCatalog::options(int layer_id, std::int64_t batch_size) const {
    std::vector<CostEntry> picked;
    std::copy_if(rows_.begin(), rows_.end(), std::back_inserter(picked), [&](const CostEntry& r) {
        return r.layer_id == layer_id && r.batch_size == batch_size;
    });
    std::sort(picked.begin(), picked.end(), option_order);
    return picked;
}

// ------------------------------------------------------ catalog readers ----

namespace {

std::vector<std::string> csv_fields(std::string_view row) {
    std::vector<std::string> out;
    for (;;) {
        std::size_t comma = row.find(',');
        out.emplace_back(trim(row.substr(0, comma)));
        if (comma == std::string_view::npos) return out;
        row.remove_prefix(comma + 1);
    }
}

AlgorithmCatalog read_csv(std::istream& in) {
    std::string text;
    if (!std::getline(in, text)) throw ParseError("empty catalog file");
    std::size_t line = 1;
    if (trim(text) != kCatalogHeader)
        throw ParseError("expected header `" + std::string(kCatalogHeader) + "`", line);

    std::vector<CostEntry> rows;
    std::vector<std::size_t> where;
    while (std::getline(in, text)) {
        ++line;
        if (trim(text).empty()) continue;
        std::vector<std::string> f = csv_fields(text);
        if (f.size() != 5)
            throw ParseError("expected 5 comma-separated fields, got " + std::to_string(f.size()),
                             line);
        const auto layer = parse_int(f[0]);
        const auto batch = parse_int(f[2]);
        const auto secs = parse_double(f[3]);
        const auto bits = parse_int(f[4]);
        if (!layer) throw ParseError("layer_id is not an integer: `" + f[0] + "`", line);
        if (!batch) throw ParseError("batch_size is not an integer: `" + f[2] + "`", line);
        if (!secs) throw ParseError("time_seconds is not a number: `" + f[3] + "`", line);
        if (!bits) throw ParseError("memory_bits is not an integer: `" + f[4] + "`", line);
        CostEntry r;
        r.layer_id = static_cast<int>(*layer);
        r.algorithm = f[1];
        r.batch_size = *batch;
        r.time_seconds = *secs;
        r.memory_bits = *bits;
        require_valid_row(r, line);
        rows.push_back(std::move(r));
        where.push_back(line);
    }
    return AlgorithmCatalog(std::move(rows), &where);
}

AlgorithmCatalog read_json(std::istream& in) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(in);
    } catch (const nlohmann::json::parse_error& e) {
        throw ParseError(std::string("invalid JSON: ") + e.what());
    }
    if (!doc.is_array()) throw ParseError("catalog JSON must be an array of entry objects");

    static const char* const kKeys[] = {"layer_id", "algorithm", "batch_size", "time_seconds",
                                        "memory_bits"};
    std::vector<CostEntry> rows;
    std::vector<std::size_t> where;
    std::size_t pos = 0;
    for (const auto& item : doc) {
        ++pos;  // JSON "lines" are 1-based array positions
        if (!item.is_object()) throw ParseError("catalog entry is not an object", pos);
        for (const char* k : kKeys)
            if (!item.contains(k)) throw ParseError(std::string("missing key `") + k + "`", pos);
        CostEntry r;
        try {
            r.layer_id = item.at("layer_id").get<int>();
            r.algorithm = item.at("algorithm").get<std::string>();
            r.batch_size = item.at("batch_size").get<std::int64_t>();
            r.time_seconds = item.at("time_seconds").get<double>();
            r.memory_bits = item.at("memory_bits").get<std::int64_t>();
        } catch (const nlohmann::json::exception& ex) {
            throw ParseError(std::string("bad entry field: ") + ex.what(), pos);
        }
        require_valid_row(r, pos);
        rows.push_back(std::move(r));
        where.push_back(pos);
    }
    return AlgorithmCatalog(std::move(rows), &where);
}

}  // namespace

AlgorithmCatalog load_catalog(std::istream& source, CatalogFormat format) {
    if (format == CatalogFormat::json) return read_json(source);
    return read_csv(source);
}

AlgorithmCatalog load_catalog_file(const std::string& path, CatalogFormat format) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open catalog file: " + path);
    return load_catalog(in, format);
}

AlgorithmCatalog load_catalog_file(const std::string& path) {
    const bool json = path.size() >= 5 && path.compare(path.size() - 5, 5, ".json") == 0;
    return load_catalog_file(path, json ? CatalogFormat::json : CatalogFormat::csv);
}

std::string save_catalog(const AlgorithmCatalog& catalog, CatalogFormat format) {
    if (format == CatalogFormat::json) {
        auto arr = nlohmann::ordered_json::array();
        for (const CostEntry& r : catalog.entries()) {
            nlohmann::ordered_json o;
            o["layer_id"] = r.layer_id;
            o["algorithm"] = r.algorithm;
            o["batch_size"] = r.batch_size;
            o["time_seconds"] = r.time_seconds;
            o["memory_bits"] = r.memory_bits;
            arr.push_back(std::move(o));
        }
        return arr.dump(2) + "\n";
    }
    std::string out(kCatalogHeader);
    out += '\n';
    for (const CostEntry& r : catalog.entries()) {
        out += std::to_string(r.layer_id) + ',' + r.algorithm + ',' +
               std::to_string(r.batch_size) + ',' + to_shortest_string(r.time_seconds) + ',' +
               std::to_string(r.memory_bits) + '\n';
    }
    return out;
}

// ---------------------------------------------------------- text files ----

namespace {

// Whitespace-separated words up to a word that starts with '#'.
std::vector<std::string> words(const std::string& line) {
    std::vector<std::string> out;
    std::istringstream ss(line);
    for (std::string w; ss >> w;) {
        if (w[0] == '#') break;
        out.push_back(std::move(w));
    }
    return out;
}

std::int64_t integer(const std::string& tok, const char* label, std::size_t line) {
    if (auto v = parse_int(tok)) return *v;
    throw ParseError(std::string(label) + " is not an integer: `" + tok + "`", line);
}

}  // namespace

NetworkSpec load_network(std::istream& source) {
    NetworkSpec net;
    bool seen_input = false, classifier_started = false;
    int next_feature = 0, next_fc = 0;
    std::size_t line = 0;

    for (std::string text; std::getline(source, text);) {
        ++line;
        const std::vector<std::string> w = words(text);
        if (w.empty()) continue;
        const std::string& op = w[0];
        const auto arity = [&](std::size_t want) {
            if (w.size() - 1 != want)
                throw ParseError("`" + op + "` takes " + std::to_string(want) +
                                     " arguments, got " + std::to_string(w.size() - 1),
                                 line);
        };

        if (op == "input") {
            arity(3);
            if (seen_input) throw ParseError("duplicate `input` line", line);
            const std::int64_t wd = integer(w[1], "input width", line);
            const std::int64_t ht = integer(w[2], "input height", line);
            const std::int64_t dp = integer(w[3], "input depth", line);
            net.input_shape = {wd, ht, dp};
            seen_input = true;
            continue;
        }
        if (!seen_input)
            throw ParseError("network file must start with an `input B H D` line", line);

        if (op == "fc") {
            arity(1);
            classifier_started = true;
            const std::int64_t n = integer(w[1], "neuron count", line);
            net.classifier_layers.push_back({n, ++next_fc});
            continue;
        }
        if (op != "conv" && op != "pool")
            throw ParseError("unknown directive `" + op + "` (expected input, conv, pool, or fc)",
                             line);
        if (classifier_started) throw ParseError("feature layer after the first `fc` layer", line);

        FeatureLayerSpec layer;
        layer.layer_id = ++next_feature;
        if (op == "conv") {
            arity(4);
            layer.kind = LayerKind::convolution;
            layer.filter_count = integer(w[4], "filter count", line);
        } else {
            arity(3);
            layer.kind = LayerKind::pooling;
        }
        layer.filter_size = integer(w[1], "filter size", line);
        layer.stride = integer(w[2], "stride", line);
        layer.padding = integer(w[3], "padding", line);
        net.feature_layers.push_back(layer);
    }
    if (!seen_input) throw ParseError("network file has no `input` line");
    return net;
}

NetworkSpec load_network_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open network file: " + path);
    return load_network(in);
}

StepTrace load_step_trace(std::istream& source) {
    StepTrace trace;
    std::size_t line = 0;
    for (std::string text; std::getline(source, text);) {
        ++line;
        const std::vector<std::string> w = words(text);
        if (w.empty()) continue;
        if (w.size() < 2 || w.size() > 3)
            throw ParseError("expected `<step> <seconds> [hidden]`", line);
        const auto step = pipeline_step_from_string(w[0]);
        if (!step) throw ParseError("unknown pipeline step `" + w[0] + "`", line);
        if (trace.times.count(*step)) throw ParseError("duplicate step `" + w[0] + "`", line);
        const auto secs = parse_double(w[1]);
        if (!secs) throw ParseError("step time is not a number: `" + w[1] + "`", line);
        trace.times[*step] = *secs;
        if (w.size() == 3) {
            if (w[2] != "hidden")
                throw ParseError("trailing token must be `hidden`, got `" + w[2] + "`", line);
            trace.hidden.insert(*step);
        }
    }
    return trace;
}

StepTrace load_step_trace_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open step-times file: " + path);
    return load_step_trace(in);
}

}  // namespace traincap
