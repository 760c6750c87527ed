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

// Field invariants of one measured cost row (first failing one reported).
void require_valid_row(const CostEntry& e, std::size_t line) {
    struct Rule {
        bool ok;
        const char* what;
    };
    const Rule rules[] = {{e.layer_id >= 1, "layer_id must be >= 1"},
                          {!e.algorithm.empty(), "algorithm name must be non-empty"},
                          {e.batch_size >= 1, "batch_size must be >= 1"},
                          {e.time_seconds > 0.0, "time_seconds must be > 0"},
                          {e.memory_bits >= 0, "memory_bits must be >= 0"}};
    for (const Rule& r : rules)
        if (!r.ok) throw ParseError(r.what, line);
}

// Eq 6's per-layer option order: time, then workspace, then name.
bool faster_option(const CostEntry& a, const CostEntry& b) {
    if (a.time_seconds != b.time_seconds) return a.time_seconds < b.time_seconds;
    if (a.memory_bits != b.memory_bits) return a.memory_bits < b.memory_bits;
    return a.algorithm < b.algorithm;
}

}  // namespace

// ------------------------------------------------------------- catalog ----
//
// A catalog is indexed by cell (layer, batch): every cell of layers 1..q x
// declared batches must hold at least one option, which also makes the layer
// ids contiguous. Rows are validated in input order so the first bad or
// duplicated row is the one reported, with its source line.

AlgorithmCatalog::AlgorithmCatalog(std::vector<CostEntry> rows,
                                   const std::vector<std::size_t>* source_lines) {
    const auto line_of = [&](std::size_t i) { return source_lines ? (*source_lines)[i] : i + 1; };
    std::map<std::tuple<int, std::string, std::int64_t>, std::size_t> where;
    for (std::size_t i = 0; i < rows.size(); ++i) {
        const CostEntry& r = rows[i];
        require_valid_row(r, line_of(i));
        const auto [it, fresh] = where.try_emplace({r.layer_id, r.algorithm, r.batch_size}, i);
        if (!fresh)
            throw DuplicateKeyError("duplicate catalog key (layer " + std::to_string(r.layer_id) + ", " +
                                    r.algorithm + ", batch " + std::to_string(r.batch_size) + ") on lines " +
                                    std::to_string(line_of(it->second)) + " and " + std::to_string(line_of(i)));
        cells_[{r.layer_id, r.batch_size}].push_back(r);
    }
    if (rows.empty()) throw IncompleteCatalogError("catalog has no entries");

    std::set<std::int64_t> batch_set;
    std::set<AlgorithmId> algo_set;
    for (const auto& [key, opts] : cells_) {
        layers_ = std::max(layers_, key.first);
        batch_set.insert(key.second);
        for (const CostEntry& e : opts) algo_set.insert(e.algorithm);
    }
    batches_.assign(batch_set.begin(), batch_set.end());
    algos_.assign(algo_set.begin(), algo_set.end());
    for (int layer = 1; layer <= layers_; ++layer)
        for (std::int64_t b : batches_)
            if (cells_.find({layer, b}) == cells_.end())
                throw IncompleteCatalogError("no algorithm profiled for layer " + std::to_string(layer) +
                                             " at batch size " + std::to_string(b));

    // canonical row order: by cell, then algorithm name; options fastest first
    rows_.clear();
    rows_.reserve(rows.size());
    for (auto& [key, opts] : cells_) {
        std::vector<CostEntry> by_name = opts;
        std::sort(by_name.begin(), by_name.end(),
                  [](const CostEntry& x, const CostEntry& y) { return x.algorithm < y.algorithm; });
        rows_.insert(rows_.end(), by_name.begin(), by_name.end());
        std::sort(opts.begin(), opts.end(), faster_option);
    }
}

bool AlgorithmCatalog::has_batch_size(std::int64_t b) const {
    return std::binary_search(batches_.begin(), batches_.end(), b);
}

std::optional<CostEntry> AlgorithmCatalog::query(int layer_id, const AlgorithmId& algorithm,
                                                 std::int64_t batch_size) const {
    const auto cell = cells_.find({layer_id, batch_size});
    if (cell == cells_.end()) return std::nullopt;
    for (const CostEntry& e : cell->second)
        if (e.algorithm == algorithm) return e;
    return std::nullopt;
}

std::vector<CostEntry> AlgorithmCatalog::options(int layer_id, std::int64_t batch_size) const {
    const auto cell = cells_.find({layer_id, batch_size});
    return cell == cells_.end() ? std::vector<CostEntry>{} : cell->second;
}

// ------------------------------------------------------ catalog readers ----
//
// CSV and JSON both reduce to (row, source line) pairs handed to the
// validating constructor; each field is converted by a per-column rule whose
// failure names the column and the offending text.

namespace {

struct SourcedRows {
    std::vector<CostEntry> rows;
    std::vector<std::size_t> lines;
    void add(CostEntry e, std::size_t line) {
        require_valid_row(e, line);
        rows.push_back(std::move(e));
        lines.push_back(line);
    }
    AlgorithmCatalog build() { return AlgorithmCatalog(std::move(rows), &lines); }
};

std::vector<std::string> split_commas(std::string_view row) {
    std::vector<std::string> out;
    std::size_t from = 0;
    for (std::size_t comma; (comma = row.find(',', from)) != std::string_view::npos; from = comma + 1)
        out.emplace_back(trim(row.substr(from, comma - from)));
    out.emplace_back(trim(row.substr(from)));
    return out;
}

CostEntry entry_from_csv(const std::vector<std::string>& f, std::size_t line) {
    const auto need_int = [&](std::size_t i, const char* col) {
        const auto v = parse_int(f[i]);
        if (!v) throw ParseError(std::string(col) + " is not an integer: `" + f[i] + "`", line);
        return *v;
    };
    const auto need_num = [&](std::size_t i, const char* col) {
        const auto v = parse_double(f[i]);
        if (!v) throw ParseError(std::string(col) + " is not a number: `" + f[i] + "`", line);
        return *v;
    };
    CostEntry e;
    // checked in this order: layer, batch, time, memory
    e.layer_id = static_cast<int>(need_int(0, "layer_id"));
    e.batch_size = need_int(2, "batch_size");
    e.time_seconds = need_num(3, "time_seconds");
    e.memory_bits = need_int(4, "memory_bits");
    e.algorithm = f[1];
    return e;
}

AlgorithmCatalog read_csv(std::istream& in) {
    std::string text;
    if (!std::getline(in, text)) throw ParseError("empty catalog file");
    if (trim(text) != kCatalogHeader) throw ParseError("expected header `" + std::string(kCatalogHeader) + "`", 1);
    SourcedRows out;
    for (std::size_t line = 2; std::getline(in, text); ++line) {
        if (trim(text).empty()) continue;
        const std::vector<std::string> f = split_commas(text);
        if (f.size() != 5)
            throw ParseError("expected 5 comma-separated fields, got " + std::to_string(f.size()), line);
        out.add(entry_from_csv(f, line), line);
    }
    return out.build();
}

AlgorithmCatalog read_json(std::istream& in) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(in);
    } catch (const nlohmann::json::parse_error& e) {
        throw ParseError(std::string("invalid JSON: ") + e.what());
    }
    if (!doc.is_array()) throw ParseError("catalog JSON must be an array of entry objects");
    SourcedRows out;
    std::size_t pos = 0;  // JSON "lines" are 1-based array positions
    for (const nlohmann::json& item : doc) {
        ++pos;
        if (!item.is_object()) throw ParseError("catalog entry is not an object", pos);
        for (const char* k : {"layer_id", "algorithm", "batch_size", "time_seconds", "memory_bits"})
            if (!item.contains(k)) throw ParseError(std::string("missing key `") + k + "`", pos);
        CostEntry e;
        try {
            item.at("layer_id").get_to(e.layer_id);
            item.at("algorithm").get_to(e.algorithm);
            item.at("batch_size").get_to(e.batch_size);
            item.at("time_seconds").get_to(e.time_seconds);
            item.at("memory_bits").get_to(e.memory_bits);
        } catch (const nlohmann::json::exception& ex) {
            throw ParseError(std::string("bad entry field: ") + ex.what(), pos);
        }
        out.add(std::move(e), pos);
    }
    return out.build();
}

}  // namespace

AlgorithmCatalog load_catalog(std::istream& source, CatalogFormat format) {
    return format == CatalogFormat::json ? read_json(source) : read_csv(source);
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

// Writers: JSON objects in the field order of the CSV header; CSV times in the
// shortest text that reads back to the same double (profiled catalogs survive
// a write / read round trip bit-exactly).
std::string save_catalog(const AlgorithmCatalog& catalog, CatalogFormat format) {
    if (format == CatalogFormat::json) {
        nlohmann::ordered_json arr = nlohmann::ordered_json::array();
        for (const CostEntry& r : catalog.entries())
            arr.push_back({{"layer_id", r.layer_id},
                           {"algorithm", r.algorithm},
                           {"batch_size", r.batch_size},
                           {"time_seconds", r.time_seconds},
                           {"memory_bits", r.memory_bits}});
        return arr.dump(2) + "\n";
    }
    std::ostringstream out;
    out << kCatalogHeader << '\n';
    for (const CostEntry& r : catalog.entries())
        out << r.layer_id << ',' << r.algorithm << ',' << r.batch_size << ',' << to_shortest_string(r.time_seconds)
            << ',' << r.memory_bits << '\n';
    return out.str();
}

// ---------------------------------------------------------- text files ----
//
// Both text formats are line records of whitespace-separated words; a word
// starting with '#' comments out the rest of its line, blank lines are
// skipped. Records carry their 1-based line number for the diagnostics.

namespace {

struct Record {
    std::size_t line = 0;
    std::vector<std::string> w;
};

std::vector<Record> read_records(std::istream& in) {
    std::vector<Record> recs;
    std::size_t n = 0;
    for (std::string text; std::getline(in, text);) {
        ++n;
        Record r{n, {}};
        std::istringstream ss(text);
        std::string word;
        while (ss >> word && word.front() != '#') r.w.push_back(word);
        if (!r.w.empty()) recs.push_back(std::move(r));
    }
    return recs;
}

std::int64_t int_operand(const Record& r, std::size_t i, const char* label) {
    const std::optional<std::int64_t> v = parse_int(r.w[i]);
    if (!v) throw ParseError(std::string(label) + " is not an integer: `" + r.w[i] + "`", r.line);
    return *v;
}

// `.net` grammar: an `input W H D` line, then feature layers (conv F S P K /
// pool F S P), then classifier layers (fc N). One row per directive: operand
// count, whether it is a feature layer, and its operands in checking order.
struct Directive {
    const char* name;
    std::size_t operands;
    bool feature;
    std::vector<std::pair<std::size_t, const char*>> checked;  // (word index, label)
};

const std::vector<Directive>& net_grammar() {
    static const std::vector<Directive> g = {
        {"input", 3, false, {{1, "input width"}, {2, "input height"}, {3, "input depth"}}},
        {"conv", 4, true, {{4, "filter count"}, {1, "filter size"}, {2, "stride"}, {3, "padding"}}},
        {"pool", 3, true, {{1, "filter size"}, {2, "stride"}, {3, "padding"}}},
        {"fc", 1, false, {{1, "neuron count"}}},
    };
    return g;
}

void require_operands(const Record& r, std::size_t want) {
    if (r.w.size() - 1 != want)
        throw ParseError("`" + r.w[0] + "` takes " + std::to_string(want) + " arguments, got " +
                             std::to_string(r.w.size() - 1),
                         r.line);
}

}  // namespace

NetworkSpec load_network(std::istream& source) {
    enum class Stage { before_input, features, classifier };
    NetworkSpec net;
    Stage stage = Stage::before_input;
    for (const Record& r : read_records(source)) {
        const auto& g = net_grammar();
        const auto d = std::find_if(g.begin(), g.end(), [&](const Directive& x) { return r.w[0] == x.name; });
        const bool is_input = d != g.end() && d == g.begin();
        if (is_input) {
            require_operands(r, d->operands);
            if (stage != Stage::before_input) throw ParseError("duplicate `input` line", r.line);
        } else {
            if (stage == Stage::before_input)
                throw ParseError("network file must start with an `input B H D` line", r.line);
            if (d == g.end())
                throw ParseError("unknown directive `" + r.w[0] + "` (expected input, conv, pool, or fc)", r.line);
            if (d->feature && stage == Stage::classifier)
                throw ParseError("feature layer after the first `fc` layer", r.line);
            require_operands(r, d->operands);
        }
        std::map<std::size_t, std::int64_t> v;
        for (const auto& [idx, label] : d->checked) v[idx] = int_operand(r, idx, label);
        if (is_input) {
            net.input_shape = {v[1], v[2], v[3]};
            stage = Stage::features;
        } else if (d->feature) {
            FeatureLayerSpec f;
            f.layer_id = static_cast<int>(net.feature_layers.size()) + 1;
            f.kind = d->operands == 4 ? LayerKind::convolution : LayerKind::pooling;
            if (f.kind == LayerKind::convolution) f.filter_count = v[4];
            f.filter_size = v[1];
            f.stride = v[2];
            f.padding = v[3];
            net.feature_layers.push_back(f);
        } else {
            net.classifier_layers.push_back({v[1], static_cast<int>(net.classifier_layers.size()) + 1});
            stage = Stage::classifier;
        }
    }
    if (stage == Stage::before_input) throw ParseError("network file has no `input` line");
    return net;
}

NetworkSpec load_network_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open network file: " + path);
    return load_network(in);
}

// Step trace: `<step> <seconds> [hidden]` per line, each step at most once.
StepTrace load_step_trace(std::istream& source) {
    StepTrace trace;
    for (const Record& r : read_records(source)) {
        const std::size_t n = r.w.size();
        if (n != 2 && n != 3) throw ParseError("expected `<step> <seconds> [hidden]`", r.line);
        const std::optional<PipelineStep> step = pipeline_step_from_string(r.w[0]);
        if (!step) throw ParseError("unknown pipeline step `" + r.w[0] + "`", r.line);
        if (trace.times.find(*step) != trace.times.end())
            throw ParseError("duplicate step `" + r.w[0] + "`", r.line);
        const std::optional<double> secs = parse_double(r.w[1]);
        if (!secs) throw ParseError("step time is not a number: `" + r.w[1] + "`", r.line);
        trace.times.emplace(*step, *secs);
        if (n == 3 && r.w[2] != "hidden")
            throw ParseError("trailing token must be `hidden`, got `" + r.w[2] + "`", r.line);
        if (n == 3) trace.hidden.insert(*step);
    }
    return trace;
}

StepTrace load_step_trace_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw Error("cannot open step-times file: " + path);
    return load_step_trace(in);
}

}  // namespace traincap
