// Geometry (Eq 1), exact memory accounting (Eq 2-5), number/unit parsing.
//
// Semantics follow the reference planner:
//   text helpers   /root/reference/proj/src/util.cpp:8-44
//   units          /root/reference/proj/src/units.cpp:28-80
//   Eq 1 shapes    /root/reference/proj/src/net_model.cpp:36-99
//   Eq 2-5 memory  /root/reference/proj/src/mem_model.cpp:30-109
// All integer arithmetic is overflow-checked; overflow raises OverflowError.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "traincap/api.hpp"

namespace traincap {

namespace {

struct Checked {
    const char* what;
    std::int64_t mul(std::int64_t a, std::int64_t b) const {
        std::int64_t r;
        if (__builtin_mul_overflow(a, b, &r)) throw OverflowError(what);
        return r;
    }
    std::int64_t add(std::int64_t a, std::int64_t b) const {
        std::int64_t r;
        if (__builtin_add_overflow(a, b, &r)) throw OverflowError(what);
        return r;
    }
    std::int64_t sub(std::int64_t a, std::int64_t b) const {
        std::int64_t r;
        if (__builtin_sub_overflow(a, b, &r)) throw OverflowError(what);
        return r;
    }
};

constexpr Checked kShapeMath{"integer overflow in shape arithmetic"};
constexpr Checked kMemMath{"integer overflow in memory arithmetic"};

bool is_blank(char c) { return c == ' ' || c == '\t' || c == '\r'; }

// Rounds toward negative infinity (a filter wider than the padded input
// yields a negative numerator; C++ division would round it toward zero).
std::int64_t div_floor(std::int64_t n, std::int64_t d) {
    std::int64_t q = n / d;
    std::int64_t r = n % d;
    return (r != 0 && ((r < 0) != (d < 0))) ? q - 1 : q;
}

std::int64_t out_extent(std::int64_t in, const FeatureLayerSpec& l) {
    return div_floor(in + 2 * l.padding - l.filter_size, l.stride) + 1;
}

}  // namespace

// ----------------------------------------------------------------- text ----

std::string_view trim(std::string_view s) {
    std::size_t b = 0, e = s.size();
    while (b < e && is_blank(s[b])) ++b;
    while (e > b && is_blank(s[e - 1])) --e;
    return s.substr(b, e - b);
}

std::string to_shortest_string(double value) {
    // Smallest %g precision that survives a from_chars round trip.
    char text[64] = {0};
    int digits = 0;
    while (++digits <= 17) {
        std::snprintf(text, sizeof text, "%.*g", digits, value);
        double parsed = 0.0;
        auto res = std::from_chars(text, text + std::strlen(text), parsed);
        if (res.ec == std::errc() && parsed == value) break;
    }
    return std::string(text);
}

template <typename T>
static std::optional<T> parse_whole(std::string_view token) {
    std::string_view t = trim(token);
    if (t.empty()) return std::nullopt;
    T out{};
    const char* end = t.data() + t.size();
    auto res = std::from_chars(t.data(), end, out);
    if (res.ec != std::errc() || res.ptr != end) return std::nullopt;
    return out;
}

std::optional<double> parse_double(std::string_view token) { return parse_whole<double>(token); }
std::optional<std::int64_t> parse_int(std::string_view token) {
    return parse_whole<std::int64_t>(token);
}

// ---------------------------------------------------------------- units ----

namespace {

struct Quantity {
    double number;
    std::string_view unit;
};

Quantity split_quantity(std::string_view text) {
    std::string_view t = trim(text);
    double v = 0.0;
    auto res = std::from_chars(t.data(), t.data() + t.size(), v);
    if (res.ec != std::errc() || res.ptr == t.data())
        throw UnitError("expected a number with a unit suffix, got `" + std::string(t) + "`");
    return {v, trim(t.substr(static_cast<std::size_t>(res.ptr - t.data())))};
}

double bytes_per_unit(std::string_view unit) {
    struct U {
        const char* name;
        double scale;
    };
    static const U table[] = {
        {"B", 1.0},
        {"KB", 1e3},
        {"MB", 1e6},
        {"GB", 1e9},
        {"TB", 1e12},
        {"KiB", 1024.0},
        {"MiB", 1024.0 * 1024},
        {"GiB", 1024.0 * 1024 * 1024},
        {"TiB", 1024.0 * 1024 * 1024 * 1024},
    };
    for (const U& u : table)
        if (unit == u.name) return u.scale;
    throw UnitError("unknown byte unit `" + std::string(unit) +
                    "` (use B, KB, MB, GB, TB or KiB, MiB, GiB, TiB)");
}

}  // namespace

double parse_bytes(std::string_view text) {
    Quantity q = split_quantity(text);
    if (q.unit.empty())
        throw UnitError("byte quantity `" + std::string(text) + "` needs an explicit unit suffix");
    return q.number * bytes_per_unit(q.unit);
}

double parse_bandwidth(std::string_view text) {
    Quantity q = split_quantity(text);
    if (q.unit.empty())
        throw UnitError("bandwidth `" + std::string(text) + "` needs an explicit unit suffix");
    static const std::pair<const char*, double> bit_rates[] = {
        {"bps", 1.0}, {"Kbps", 1e3}, {"Mbps", 1e6}, {"Gbps", 1e9}, {"Tbps", 1e12}};
    for (const auto& [name, scale] : bit_rates)
        if (q.unit == name) return scale == 1.0 ? q.number / 8.0 : q.number * scale / 8.0;
    if (q.unit.size() > 2 && q.unit.substr(q.unit.size() - 2) == "/s")
        return q.number * bytes_per_unit(q.unit.substr(0, q.unit.size() - 2));
    throw UnitError("unknown bandwidth unit `" + std::string(q.unit) +
                    "` (use bps/Kbps/Mbps/Gbps/Tbps or a byte unit plus /s, e.g. GB/s)");
}

std::string human_bytes(double bytes) {
    static const char* names[] = {"B", "KiB", "MiB", "GiB", "TiB"};
    int k = 0;
    double v = bytes;
    for (; k < 4 && std::fabs(v) >= 1024.0; ++k) v /= 1024.0;
    char buf[48];
    if (k == 0)
        std::snprintf(buf, sizeof buf, "%.0f %s", v, names[k]);
    else
        std::snprintf(buf, sizeof buf, "%.2f %s", v, names[k]);
    return buf;
}

// -------------------------------------------------------------- network ----

std::int64_t TensorShape::elements() const {
    return kShapeMath.mul(kShapeMath.mul(width, height), depth);
}

int NetworkSpec::convolution_layer_count() const {
    int n = 0;
    for (const FeatureLayerSpec& l : feature_layers) n += l.kind == LayerKind::convolution;
    return n;
}

std::vector<TensorShape> propagate_shapes(const NetworkSpec& network) {
    std::vector<TensorShape> chain(1, network.input_shape);
    chain.reserve(network.feature_layers.size() + 1);
    for (const FeatureLayerSpec& l : network.feature_layers) {
        const TensorShape prev = chain.back();
        TensorShape next{out_extent(prev.width, l), out_extent(prev.height, l),
                         l.kind == LayerKind::convolution ? l.filter_count : prev.depth};
        if (next.width < 1 || next.height < 1)
            throw NonPositiveShapeError("layer " + std::to_string(l.layer_id) +
                                            ": filter exceeds padded input, output shape "
                                            "collapses",
                                        l.layer_id);
        chain.push_back(next);
    }
    return chain;
}

std::vector<Violation> validate_network(const NetworkSpec& network) {
    std::vector<Violation> found;
    const TensorShape& in = network.input_shape;
    if (std::min({in.width, in.height, in.depth}) < 1)
        found.push_back({0, "input shape components must all be >= 1"});
    if (network.feature_layers.empty())
        found.push_back({0, "network needs at least one feature-extraction layer"});
    if (network.classifier_layers.empty())
        found.push_back({0, "network needs at least one classifier layer"});

    for (const FeatureLayerSpec& l : network.feature_layers) {
        const bool conv = l.kind == LayerKind::convolution;
        if (l.filter_size < 1) found.push_back({l.layer_id, "filter size must be >= 1"});
        if (l.stride < 1) found.push_back({l.layer_id, "stride must be >= 1"});
        if (l.padding < 0) found.push_back({l.layer_id, "padding must be >= 0"});
        if (!conv && l.filter_count != 0)
            found.push_back({l.layer_id, "pooling layer must have filter count 0"});
        if (conv && l.filter_count < 1)
            found.push_back({l.layer_id, "convolution layer must have filter count >= 1"});
    }
    for (const ClassifierLayerSpec& c : network.classifier_layers)
        if (c.neuron_count < 1)
            found.push_back({c.layer_id, "classifier layer must have neuron count >= 1"});

    // Collapse detection only runs on an otherwise well-formed chain.
    if (found.empty()) {
        try {
            (void)propagate_shapes(network);
        } catch (const NonPositiveShapeError& e) {
            found.push_back({e.layer_id(), e.what()});
        } catch (const OverflowError& e) {
            found.push_back({0, e.what()});
        }
    }
    return found;
}

// --------------------------------------------------------------- memory ----

std::int64_t feature_map_memory(const NetworkSpec& network,
                                const std::vector<TensorShape>& shapes,
                                std::int64_t batch_size) {
    if (shapes.size() != network.feature_layers.size() + 1)
        throw DomainError("shapes must come from propagate_shapes on the same network");
    if (batch_size < 1) throw DomainError("batch size must be >= 1");
    std::int64_t per_sample = 0;
    for (const TensorShape& s : shapes) per_sample = kMemMath.add(per_sample, s.elements());
    return kMemMath.mul(kMemMath.mul(per_sample, batch_size), kValueBits);
}

std::int64_t model_param_memory(const NetworkSpec& network) {
    constexpr std::int64_t kCharge = kGradientReplication * kValueBits;
    std::int64_t bits = 0;
    std::int64_t depth_in = network.input_shape.depth;
    for (const FeatureLayerSpec& l : network.feature_layers) {
        if (l.kind != LayerKind::convolution) continue;  // pooling: no parameters
        const std::int64_t w = kMemMath.mul(kMemMath.mul(l.filter_size, l.filter_size),
                                            kMemMath.mul(depth_in, l.filter_count));
        bits = kMemMath.add(bits, kMemMath.mul(w, kCharge));
        bits = kMemMath.add(bits, kMemMath.mul(l.filter_count, kCharge));
        depth_in = l.filter_count;
    }
    return bits;
}

std::int64_t classifier_memory(const std::vector<ClassifierLayerSpec>& layers) {
    constexpr std::int64_t kCharge = kGradientReplication * kValueBits;
    std::int64_t neurons = 0;
    for (const ClassifierLayerSpec& c : layers) neurons = kMemMath.add(neurons, c.neuron_count);
    std::int64_t bits = kMemMath.mul(neurons, kValueBits);
    for (std::size_t j = 1; j < layers.size(); ++j) {
        const std::int64_t junction =
            kMemMath.mul(layers[j - 1].neuron_count, layers[j].neuron_count);
        bits = kMemMath.add(bits, kMemMath.mul(junction, kCharge));
    }
    // One scalar bias charge per junction, independent of widths (paper's Eq 4 as stated).
    if (!layers.empty())
        bits = kMemMath.add(bits, static_cast<std::int64_t>(layers.size() - 1) * kCharge);
    return bits;
}

MemoryBreakdown memory_bound(std::int64_t gpu_total_bits, const NetworkSpec& network,
                             std::int64_t batch_size) {
    MemoryBreakdown m;
    m.batch_size = batch_size;
    m.gpu_total = gpu_total_bits;
    m.feature_maps = feature_map_memory(network, propagate_shapes(network), batch_size);
    m.model_params = model_param_memory(network);
    m.classifier = classifier_memory(network.classifier_layers);
    std::int64_t left = kMemMath.sub(gpu_total_bits, m.feature_maps);
    left = kMemMath.sub(left, m.model_params);
    m.bound = kMemMath.sub(left, m.classifier);
    return m;
}

std::int64_t parameter_bits(const NetworkSpec& network) {
    const std::int64_t conv_bits = model_param_memory(network) / kGradientReplication;
    const auto& fc = network.classifier_layers;
    std::int64_t fc_bits = 0;
    for (std::size_t j = 1; j < fc.size(); ++j)
        fc_bits = kMemMath.add(
            fc_bits,
            kMemMath.mul(kMemMath.mul(fc[j - 1].neuron_count, fc[j].neuron_count), kValueBits));
    if (!fc.empty())
        fc_bits = kMemMath.add(fc_bits, static_cast<std::int64_t>(fc.size() - 1) * kValueBits);
    return kMemMath.add(conv_bits, fc_bits);
}

}  // namespace traincap
