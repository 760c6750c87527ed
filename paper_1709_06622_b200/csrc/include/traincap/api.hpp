// traincap host API — B200 build.
//
// One header carries the whole planner surface so that the per-module
// forwarding headers (net_model.hpp, catalog.hpp, ...) stay drop-in
// compatible with code written against the reference's include layout
// (/root/reference/proj/include/traincap/*.hpp). Names, types, units and
// exception classes follow the reference contract; the implementation under
// csrc/host/ is independent.
//
// Units everywhere: memory in bits (int64), time in seconds (double),
// bandwidth in bytes/second (double).
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <map>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace traincap __attribute__((visibility("default"))) {

// ---------------------------------------------------------------------------
// Errors (reference: include/traincap/errors.hpp:10-89)
// ---------------------------------------------------------------------------
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class ParseError : public Error {
public:
    ParseError(const std::string& what_msg, std::size_t line = 0)
        : Error(line == 0 ? what_msg : "line " + std::to_string(line) + ": " + what_msg),
          line_(line) {}
    std::size_t line() const noexcept { return line_; }

private:
    std::size_t line_;
};

#define TRAINCAP_SIMPLE_ERROR(Name)      \
    class Name : public Error {          \
    public:                              \
        using Error::Error;              \
    };
TRAINCAP_SIMPLE_ERROR(DuplicateKeyError)
TRAINCAP_SIMPLE_ERROR(IncompleteCatalogError)
TRAINCAP_SIMPLE_ERROR(OverflowError)
TRAINCAP_SIMPLE_ERROR(DomainError)
TRAINCAP_SIMPLE_ERROR(UnitError)
TRAINCAP_SIMPLE_ERROR(MissingComputeStepError)
TRAINCAP_SIMPLE_ERROR(InstanceTooLargeError)
TRAINCAP_SIMPLE_ERROR(CandidateNotInCatalogError)
TRAINCAP_SIMPLE_ERROR(ValidationError)
#undef TRAINCAP_SIMPLE_ERROR

class NonPositiveShapeError : public Error {
public:
    NonPositiveShapeError(const std::string& what_msg, int layer)
        : Error(what_msg), layer_(layer) {}
    int layer_id() const noexcept { return layer_; }

private:
    int layer_;
};

// ---------------------------------------------------------------------------
// Text helpers (reference: include/traincap/util.hpp:11-18)
// ---------------------------------------------------------------------------
std::string to_shortest_string(double value);
std::optional<double> parse_double(std::string_view token);
std::optional<std::int64_t> parse_int(std::string_view token);
std::string_view trim(std::string_view s);

// Unit parsing at the CLI boundary (reference: include/traincap/units.hpp:12-20)
double parse_bytes(std::string_view text);
double parse_bandwidth(std::string_view text);
std::string human_bytes(double bytes);

// ---------------------------------------------------------------------------
// Network model, Eq 1 (reference: include/traincap/net_model.hpp:12-68)
// ---------------------------------------------------------------------------
struct TensorShape {
    std::int64_t width = 0;
    std::int64_t height = 0;
    std::int64_t depth = 0;

    std::int64_t elements() const;
    friend bool operator==(const TensorShape&, const TensorShape&) = default;
};

enum class LayerKind { convolution, pooling };

struct FeatureLayerSpec {
    LayerKind kind = LayerKind::convolution;
    std::int64_t filter_size = 0;
    std::int64_t stride = 0;
    std::int64_t padding = 0;
    std::int64_t filter_count = 0;  // 0 for pooling
    int layer_id = 0;
};

struct ClassifierLayerSpec {
    std::int64_t neuron_count = 0;
    int layer_id = 0;
};

struct NetworkSpec {
    TensorShape input_shape;
    std::vector<FeatureLayerSpec> feature_layers;
    std::vector<ClassifierLayerSpec> classifier_layers;

    int convolution_layer_count() const;
};

struct Violation {
    int layer_id = 0;
    std::string message;
};

std::vector<Violation> validate_network(const NetworkSpec& network);
std::vector<TensorShape> propagate_shapes(const NetworkSpec& network);

// ---------------------------------------------------------------------------
// Memory model, Eq 2-5 (reference: include/traincap/mem_model.hpp:11-52)
// ---------------------------------------------------------------------------
inline constexpr std::int64_t kValueBits = 32;
inline constexpr std::int64_t kGradientReplication = 3;

struct MemoryBreakdown {
    std::int64_t feature_maps = 0;
    std::int64_t model_params = 0;
    std::int64_t classifier = 0;
    std::int64_t gpu_total = 0;
    std::int64_t bound = 0;
    std::int64_t batch_size = 0;
};

std::int64_t feature_map_memory(const NetworkSpec& network,
                                const std::vector<TensorShape>& shapes,
                                std::int64_t batch_size);
std::int64_t model_param_memory(const NetworkSpec& network);
std::int64_t classifier_memory(const std::vector<ClassifierLayerSpec>& classifier_layers);
MemoryBreakdown memory_bound(std::int64_t gpu_total_bits, const NetworkSpec& network,
                             std::int64_t batch_size);
std::int64_t parameter_bits(const NetworkSpec& network);

// ---------------------------------------------------------------------------
// Measured cost catalog (reference: include/traincap/catalog.hpp:14-85)
// ---------------------------------------------------------------------------
using AlgorithmId = std::string;

struct CostEntry {
    int layer_id = 0;
    AlgorithmId algorithm;
    std::int64_t batch_size = 0;
    double time_seconds = 0.0;
    std::int64_t memory_bits = 0;

    friend bool operator==(const CostEntry&, const CostEntry&) = default;
};

enum class CatalogFormat { csv, json };

class AlgorithmCatalog {
public:
    explicit AlgorithmCatalog(std::vector<CostEntry> entries,
                              const std::vector<std::size_t>* source_lines = nullptr);

    int layer_count() const noexcept { return layers_; }
    const std::vector<std::int64_t>& declared_batch_sizes() const noexcept { return batches_; }
    const std::vector<AlgorithmId>& algorithms() const noexcept { return algos_; }
    const std::vector<CostEntry>& entries() const noexcept { return rows_; }

    bool has_batch_size(std::int64_t batch_size) const;
    std::optional<CostEntry> query(int layer_id, const AlgorithmId& algorithm,
                                   std::int64_t batch_size) const;
    std::vector<CostEntry> options(int layer_id, std::int64_t batch_size) const;

    friend bool operator==(const AlgorithmCatalog& a, const AlgorithmCatalog& b) {
        return a.rows_ == b.rows_;
    }

private:
    std::vector<CostEntry> rows_;
    std::vector<std::int64_t> batches_;
    std::vector<AlgorithmId> algos_;
    int layers_ = 0;
    // (layer, batch) -> its profiled options, fastest first (options() / query())
    std::map<std::pair<int, std::int64_t>, std::vector<CostEntry>> cells_;
};

AlgorithmCatalog load_catalog(std::istream& source, CatalogFormat format);
AlgorithmCatalog load_catalog_file(const std::string& path);
AlgorithmCatalog load_catalog_file(const std::string& path, CatalogFormat format);
std::string save_catalog(const AlgorithmCatalog& catalog, CatalogFormat format);

// ---------------------------------------------------------------------------
// Algorithm selection, Eq 6 (reference: include/traincap/conv_select.hpp:14-52)
// ---------------------------------------------------------------------------
struct Selection {
    std::map<int, AlgorithmId> assignment;
    double total_time = 0.0;
    std::int64_t total_memory = 0;
};

struct SolveResult {
    std::optional<Selection> selection;
    std::int64_t min_achievable_memory = 0;

    bool feasible() const noexcept { return selection.has_value(); }
};

using LayerOptions = std::vector<std::vector<CostEntry>>;

LayerOptions catalog_options(const AlgorithmCatalog& catalog, std::int64_t batch_size);
SolveResult solve_selection(const AlgorithmCatalog& catalog, std::int64_t batch_size,
                            std::int64_t memory_bound);
SolveResult solve_selection(const LayerOptions& options, std::int64_t memory_bound);
SolveResult brute_force_selection(const AlgorithmCatalog& catalog, std::int64_t batch_size,
                                  std::int64_t memory_bound);
SolveResult brute_force_selection(const LayerOptions& options, std::int64_t memory_bound);

// ---------------------------------------------------------------------------
// Lemma 1 / Lemma 2 (reference: include/traincap/scale_plan.hpp:17-84)
// ---------------------------------------------------------------------------
enum class PipelineStep {
    parameter_refresh,
    data_loading,
    data_preparation,
    host_to_gpu_transfer,
    gpu_processing,
    parameter_update,
    distributed_update,
};

const char* to_string(PipelineStep step);
std::optional<PipelineStep> pipeline_step_from_string(std::string_view name);

struct OverheadProfile {
    double compute_time = 0.0;
    double overhead_time = 0.0;
    double ratio() const { return overhead_time / compute_time; }
};

struct ClusterSpec {
    int worker_count = 0;
    double param_size_bytes = 0.0;
    double bandwidth_bytes_per_sec = 0.0;
    int gpu_count = 0;
};

struct ScalingEstimate {
    int gpus = 0;
    double efficiency = 0.0;
    double speedup = 0.0;
};

double efficiency(int gpus, double overhead_ratio);
ScalingEstimate estimate_scaling(int gpus, double overhead_ratio);
std::vector<ScalingEstimate> scaling_table(int max_gpus, double overhead_ratio);
double max_overhead_ratio(int gpus, double alpha);

struct GpuRecommendation {
    std::optional<int> gpus;
    double speedup_cap = 0.0;
};

GpuRecommendation recommend_gpus(double target_speedup, double overhead_ratio, int max_gpus);
OverheadProfile estimate_overhead_ratio(const std::map<PipelineStep, double>& step_times,
                                        const std::set<PipelineStep>& hidden_steps);
int min_parameter_servers(const ClusterSpec& spec, double compute_time);

// ---------------------------------------------------------------------------
// Mini-batch sweep, §3.1.3-4 (reference: include/traincap/batch_plan.hpp:14-63)
// ---------------------------------------------------------------------------
enum class AdvisoryKind { reduce_batch, adjust_model, caveat };
const char* to_string(AdvisoryKind kind);

struct Advisory {
    AdvisoryKind kind = AdvisoryKind::caveat;
    std::string message;
    std::vector<int> affected_layers;
};

struct BatchCandidateResult {
    std::int64_t batch_size = 0;
    MemoryBreakdown breakdown;
    SolveResult solve;
    std::optional<double> epoch_time_seconds;
    std::optional<double> throughput;
    std::vector<int> memory_limited_layers;
};

struct BatchPlan {
    std::vector<BatchCandidateResult> candidates;
    std::optional<std::int64_t> recommended;
    std::vector<Advisory> advisories;
};

std::vector<std::int64_t> default_batch_candidates(const AlgorithmCatalog& catalog);
BatchPlan plan_batch_size(const NetworkSpec& network, const AlgorithmCatalog& catalog,
                          std::int64_t gpu_total_bits, std::int64_t dataset_size,
                          const std::vector<std::int64_t>& candidates);
std::vector<Advisory> advise_refinement(const BatchPlan& plan, const NetworkSpec& network);
// Branched networks (ResNet / Inception): no chain memory model
// (Eq 2-5) applies, so the caller supplies each candidate's resident bits —
// the executor's exact HBM layout without the conv workspaces
// (tcb_trainer_layout) — and the workspace bound is gpu_total_bits minus
// them. Selection, epoch time, the recommendation rule and the advisories
// are those of plan_batch_size. Breakdown: feature_maps = resident bits.
BatchPlan plan_batch_size_resident(const AlgorithmCatalog& catalog,
                                   const std::vector<std::pair<std::int64_t, std::int64_t>>& resident_bits,
                                   std::int64_t gpu_total_bits, std::int64_t dataset_size);
std::vector<std::string> model_caveats();

// ---------------------------------------------------------------------------
// File formats (reference: include/traincap/io.hpp:18-31)
// ---------------------------------------------------------------------------
NetworkSpec load_network(std::istream& source);
NetworkSpec load_network_file(const std::string& path);

struct StepTrace {
    std::map<PipelineStep, double> times;
    std::set<PipelineStep> hidden;
};

StepTrace load_step_trace(std::istream& source);
StepTrace load_step_trace_file(const std::string& path);

// ---------------------------------------------------------------------------
// Orchestration + reports (reference: include/traincap/report.hpp:17-82)
// ---------------------------------------------------------------------------
struct PlanRequest {
    std::string network_path;
    std::string catalog_path;
    std::int64_t gpu_memory_bits = 0;
    std::int64_t dataset_size = 0;
    std::vector<std::int64_t> candidates;
    int max_gpus = 8;
    double overhead_ratio = 0.0;
    int workers = 1;
    double bandwidth_bytes_per_sec = 1.25e9;
    std::optional<double> param_size_bytes;
    bool verify = false;
};

struct PlanReport {
    PlanRequest request;
    std::vector<std::int64_t> candidates_used;
    NetworkSpec network;
    std::vector<TensorShape> shapes;
    BatchPlan plan;
    double param_size_bytes = 0.0;
    bool param_size_derived = false;
    std::vector<ScalingEstimate> scaling;
    std::optional<double> compute_time_seconds;
    std::optional<int> parameter_servers;
    std::vector<std::string> caveats;
    bool verified = false;
};

PlanReport run_plan(const PlanRequest& request);
void render_plan_text(const PlanReport& report, std::ostream& out);
std::string render_plan_json(const PlanReport& report, const std::string& timestamp);

struct ScaleReport {
    double overhead_ratio = 0.0;
    std::optional<std::string> steps_path;
    std::vector<ScalingEstimate> table;
    std::optional<double> target_speedup;
    std::optional<GpuRecommendation> recommendation;
};

void render_scale_text(const ScaleReport& report, std::ostream& out);
std::string render_scale_json(const ScaleReport& report, const std::string& timestamp);

struct PsReport {
    ClusterSpec spec;
    double compute_time_seconds = 0.0;
    int servers = 0;
};

void render_ps_text(const PsReport& report, std::ostream& out);
std::string render_ps_json(const PsReport& report, const std::string& timestamp);

std::string current_timestamp();

// CLI entry (reference: include/traincap/cli.hpp:8): exit 0 / 1 input error / 2 infeasible.
int run_cli(int argc, const char* const* argv);

}  // namespace traincap
