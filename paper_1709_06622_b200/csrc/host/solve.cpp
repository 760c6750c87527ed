// Decision layer: Eq 6 algorithm selection, the §3.1.3 mini-batch sweep,
// Lemma 1 (GPU count) and Lemma 2 (parameter-server count).
//
// Contract (what must match the reference bit-for-bit):
//   * solve_selection returns the canonical optimum of
//       min  sum_k T_k   s.t.  sum_k M_k <= bound,  one option per layer,
//     ordered by (total time as a left-to-right double sum in layer order,
//     total memory, algorithm-name sequence) —
//     /root/reference/proj/src/conv_select.cpp:19-29,64-76,182-197.
//   * brute_force_selection enumerates with the same order and refuses
//     instances above 1e7 assignments — conv_select.cpp:199-219.
//   * plan_batch_size / advise_refinement — batch_plan.cpp:17-157.
//   * Lemma 1 / Lemma 2 arithmetic — scale_plan.cpp:8-112.
//
// The search itself is this build's own: a depth-first branch-and-bound
// whose pruning bound is the LP relaxation of the remaining multiple-choice
// knapsack (lower convex hull of each layer's (memory, time) points, greedy
// by slope). It is far tighter than a per-layer minimum when the memory
// bound binds, which is what makes the 53-layer (ResNet-50) and 94-layer
// (Inception-v3) catalogs solvable under reduced-memory sweeps.
#include <algorithm>
#include <cmath>
#include <future>
#include <limits>
#include <numeric>

#include "traincap/api.hpp"

namespace traincap {

namespace {

// Total order used by both solvers on complete assignments.
struct Leaf {
    double time = 0.0;
    std::int64_t memory = 0;
    std::vector<const CostEntry*> pick;
};

bool better_than(double t, std::int64_t m, const std::vector<const CostEntry*>& pick,
                 const std::optional<Leaf>& incumbent) {
    if (!incumbent) return true;
    if (t < incumbent->time) return true;
    if (incumbent->time < t) return false;
    if (m != incumbent->memory) return m < incumbent->memory;
    for (std::size_t i = 0; i < pick.size(); ++i) {
        const int c = pick[i]->algorithm.compare(incumbent->pick[i]->algorithm);
        if (c != 0) return c < 0;
    }
    return false;
}

void require_nonempty(const LayerOptions& options) {
    for (std::size_t i = 0; i < options.size(); ++i)
        if (options[i].empty())
            throw IncompleteCatalogError("layer " + std::to_string(i + 1) +
                                         " has no algorithm options");
}

LayerOptions sorted_copy(const LayerOptions& options) {
    LayerOptions s = options;
    for (auto& layer : s)
        std::sort(layer.begin(), layer.end(), [](const CostEntry& a, const CostEntry& b) {
            if (a.time_seconds != b.time_seconds) return a.time_seconds < b.time_seconds;
            if (a.memory_bits != b.memory_bits) return a.memory_bits < b.memory_bits;
            return a.algorithm < b.algorithm;
        });
    return s;
}

std::int64_t cheapest_memory(const LayerOptions& options) {
    std::int64_t total = 0;
    for (const auto& layer : options) {
        std::int64_t m = layer[0].memory_bits;
        for (const CostEntry& e : layer) m = std::min(m, e.memory_bits);
        total += m;
    }
    return total;
}

Selection make_selection(const Leaf& leaf) {
    Selection s;
    s.total_time = leaf.time;
    s.total_memory = leaf.memory;
    for (std::size_t i = 0; i < leaf.pick.size(); ++i)
        s.assignment[static_cast<int>(i + 1)] = leaf.pick[i]->algorithm;
    return s;
}

// One upgrade step along a layer's lower hull: spend `dm` more bits to save `dt` seconds.
struct HullStep {
    double dm;
    double dt;
    double rate() const { return dt / dm; }
};

class Search {
public:
    Search(const LayerOptions& sorted, std::int64_t bound) : bound_(bound) {
        const std::size_t q = sorted.size();
        kept_.resize(q);
        for (std::size_t i = 0; i < q; ++i) {
            // Options arrive in (time, memory, name) order: keep an option only if
            // it needs strictly less memory than every faster one before it.
            std::int64_t lightest = std::numeric_limits<std::int64_t>::max();
            for (const CostEntry& e : sorted[i])
                if (e.memory_bits < lightest) {
                    kept_[i].push_back(&e);
                    lightest = e.memory_bits;
                }
        }
        // Suffix data for bounds.
        fast_time_.assign(q + 1, 0.0);
        light_mem_.assign(q + 1, 0);
        light_time_.assign(q + 1, 0.0);
        steps_.assign(q + 1, {});
        for (std::size_t i = q; i-- > 0;) {
            const auto& k = kept_[i];  // time ascending, memory strictly descending
            const CostEntry* fastest = k.front();
            const CostEntry* lightest = k.back();
            fast_time_[i] = fast_time_[i + 1] + fastest->time_seconds;
            light_mem_[i] = light_mem_[i + 1] + lightest->memory_bits;
            light_time_[i] = light_time_[i + 1] + lightest->time_seconds;
            steps_[i] = steps_[i + 1];
            for (const HullStep& s : hull_steps(k)) steps_[i].push_back(s);
            std::sort(steps_[i].begin(), steps_[i].end(),
                      [](const HullStep& a, const HullStep& b) { return a.rate() > b.rate(); });
        }
    }

    std::optional<Leaf> run() {
        pick_.reserve(kept_.size());
        dive(0, 0.0, 0);
        return best_;
    }

private:
    // Lower convex hull from the lightest option toward the fastest one.
    static std::vector<HullStep> hull_steps(const std::vector<const CostEntry*>& k) {
        std::vector<const CostEntry*> pts(k.rbegin(), k.rend());  // memory ascending
        std::vector<const CostEntry*> hull;
        for (const CostEntry* p : pts) {
            while (hull.size() >= 2) {
                const CostEntry* a = hull[hull.size() - 2];
                const CostEntry* b = hull.back();
                // Drop b if it lies on or above segment a->p.
                const long double cross =
                    (static_cast<long double>(b->memory_bits) - a->memory_bits) *
                        (static_cast<long double>(p->time_seconds) - a->time_seconds) -
                    (static_cast<long double>(b->time_seconds) - a->time_seconds) *
                        (static_cast<long double>(p->memory_bits) - a->memory_bits);
                if (cross <= 0)
                    hull.pop_back();
                else
                    break;
            }
            hull.push_back(p);
        }
        std::vector<HullStep> out;
        for (std::size_t j = 1; j < hull.size(); ++j) {
            const double dm = static_cast<double>(hull[j]->memory_bits - hull[j - 1]->memory_bits);
            const double dt = hull[j - 1]->time_seconds - hull[j]->time_seconds;
            if (dm > 0 && dt > 0) out.push_back({dm, dt});
        }
        return out;
    }

    // LP-relaxation lower bound on the time of layers [i, q) given `budget` bits.
    double relaxed_time(std::size_t i, double budget) const {
        double t = light_time_[i];
        double room = budget - static_cast<double>(light_mem_[i]);
        for (const HullStep& s : steps_[i]) {
            if (room <= 0) break;
            if (s.dm <= room) {
                t -= s.dt;
                room -= s.dm;
            } else {
                t -= s.dt * (room / s.dm);
                room = 0;
            }
        }
        return std::max(t, fast_time_[i]);
    }

    bool hopeless(std::size_t i, double t, std::int64_t m) const {
        if (m + light_mem_[i] > bound_) return true;
        if (!best_) return false;
        const double slack = 1e-9 * (1.0 + std::fabs(best_->time));
        if (t + fast_time_[i] > best_->time + slack) return true;
        const double lb = relaxed_time(i, static_cast<double>(bound_ - m));
        return t + lb > best_->time + slack;
    }

    void dive(std::size_t i, double t, std::int64_t m) {
        if (hopeless(i, t, m)) return;
        if (i == kept_.size()) {
            if (better_than(t, m, pick_, best_)) best_ = Leaf{t, m, pick_};
            return;
        }
        for (const CostEntry* e : kept_[i]) {
            pick_.push_back(e);
            dive(i + 1, t + e->time_seconds, m + e->memory_bits);
            pick_.pop_back();
        }
    }

    std::int64_t bound_;
    std::vector<std::vector<const CostEntry*>> kept_;
    std::vector<double> fast_time_, light_time_;
    std::vector<std::int64_t> light_mem_;
    std::vector<std::vector<HullStep>> steps_;
    std::vector<const CostEntry*> pick_;
    std::optional<Leaf> best_;
};

void enumerate_all(const LayerOptions& s, std::size_t i, double t, std::int64_t m,
                   std::int64_t bound, std::vector<const CostEntry*>& pick,
                   std::optional<Leaf>& best) {
    if (i == s.size()) {
        if (m <= bound && better_than(t, m, pick, best)) best = Leaf{t, m, pick};
        return;
    }
    for (const CostEntry& e : s[i]) {
        pick.push_back(&e);
        enumerate_all(s, i + 1, t + e.time_seconds, m + e.memory_bits, bound, pick, best);
        pick.pop_back();
    }
}

}  // namespace

LayerOptions catalog_options(const AlgorithmCatalog& catalog, std::int64_t batch_size) {
    LayerOptions out(static_cast<std::size_t>(catalog.layer_count()));
    for (int l = 1; l <= catalog.layer_count(); ++l)
        out[static_cast<std::size_t>(l - 1)] = catalog.options(l, batch_size);
    require_nonempty(out);
    return out;
}

SolveResult solve_selection(const LayerOptions& options, std::int64_t memory_bound) {
    require_nonempty(options);
    const LayerOptions s = sorted_copy(options);
    SolveResult r;
    r.min_achievable_memory = cheapest_memory(s);
    if (r.min_achievable_memory <= memory_bound) {
        if (auto leaf = Search(s, memory_bound).run()) r.selection = make_selection(*leaf);
    }
    return r;
}

SolveResult solve_selection(const AlgorithmCatalog& catalog, std::int64_t batch_size,
                            std::int64_t memory_bound) {
    return solve_selection(catalog_options(catalog, batch_size), memory_bound);
}

SolveResult brute_force_selection(const LayerOptions& options, std::int64_t memory_bound) {
    require_nonempty(options);
    double count = 1.0;
    for (const auto& layer : options) count *= static_cast<double>(layer.size());
    if (count > 1e7)
        throw InstanceTooLargeError("exhaustive enumeration over " + std::to_string(count) +
                                    " assignments exceeds 1e7");
    const LayerOptions s = sorted_copy(options);
    SolveResult r;
    r.min_achievable_memory = cheapest_memory(s);
    std::vector<const CostEntry*> pick;
    std::optional<Leaf> best;
    enumerate_all(s, 0, 0.0, 0, memory_bound, pick, best);
    if (best) r.selection = make_selection(*best);
    return r;
}

SolveResult brute_force_selection(const AlgorithmCatalog& catalog, std::int64_t batch_size,
                                  std::int64_t memory_bound) {
    return brute_force_selection(catalog_options(catalog, batch_size), memory_bound);
}

// --------------------------------------------------------- batch sweep ----

const char* to_string(AdvisoryKind kind) {
    switch (kind) {
        case AdvisoryKind::reduce_batch: return "reduce_batch";
        case AdvisoryKind::adjust_model: return "adjust_model";
        case AdvisoryKind::caveat: return "caveat";
    }
    return "?";
}

std::vector<std::int64_t> default_batch_candidates(const AlgorithmCatalog& catalog) {
    std::vector<std::int64_t> out;
    for (std::int64_t b = 32; b <= 512; b *= 2)
        if (catalog.has_batch_size(b)) out.push_back(b);
    return out;
}

namespace {

constexpr const char* kClassifierCaveat =
    "classifier memory uses a fixed per-junction bias charge and batch-independent "
    "activations; treat classifier totals as approximate";

BatchCandidateResult assess_bound(const AlgorithmCatalog& cat, std::int64_t dataset, std::int64_t b,
                                  const MemoryBreakdown& breakdown) {
    BatchCandidateResult c;
    c.batch_size = b;
    c.breakdown = breakdown;
    const LayerOptions opts = catalog_options(cat, b);
    c.solve = solve_selection(opts, c.breakdown.bound);
    if (!c.solve.feasible()) return c;

    const Selection& sel = *c.solve.selection;
    const std::int64_t rounds = (dataset + b - 1) / b;
    c.epoch_time_seconds = static_cast<double>(rounds) * sel.total_time;
    c.throughput = static_cast<double>(b) / sel.total_time;
    for (std::size_t i = 0; i < opts.size(); ++i) {
        const int layer = static_cast<int>(i + 1);
        const double quickest = opts[i].front().time_seconds;
        const double chosen = cat.query(layer, sel.assignment.at(layer), b)->time_seconds;
        if (chosen > quickest) c.memory_limited_layers.push_back(layer);
    }
    return c;
}

BatchCandidateResult assess(const NetworkSpec& net, const AlgorithmCatalog& cat,
                            std::int64_t gpu_bits, std::int64_t dataset, std::int64_t b) {
    return assess_bound(cat, dataset, b, memory_bound(gpu_bits, net, b));
}

void recommend(BatchPlan& plan) {
    for (const BatchCandidateResult& c : plan.candidates) {
        if (!c.epoch_time_seconds) continue;
        if (!plan.recommended) {
            plan.recommended = c.batch_size;
            continue;
        }
        const auto holder =
            std::find_if(plan.candidates.begin(), plan.candidates.end(),
                         [&](const BatchCandidateResult& x) { return x.batch_size == *plan.recommended; });
        const double incumbent = *holder->epoch_time_seconds;
        const double mine = *c.epoch_time_seconds;
        if (mine < incumbent || (mine == incumbent && c.batch_size > *plan.recommended))
            plan.recommended = c.batch_size;
    }
}

}  // namespace

BatchPlan plan_batch_size_resident(const AlgorithmCatalog& catalog,
                                   const std::vector<std::pair<std::int64_t, std::int64_t>>& resident_bits,
                                   std::int64_t gpu_total_bits, std::int64_t dataset_size) {
    if (resident_bits.empty()) throw DomainError("candidate batch-size list must not be empty");
    if (dataset_size < 1) throw DomainError("dataset size must be >= 1");
    std::vector<std::future<BatchCandidateResult>> work;
    for (const auto& [b, bits] : resident_bits) {
        if (!catalog.has_batch_size(b))
            throw CandidateNotInCatalogError("batch size " + std::to_string(b) +
                                             " is not declared in the catalog");
        if (bits < 0) throw DomainError("resident bits must be >= 0");
        MemoryBreakdown m;
        m.batch_size = b;
        m.gpu_total = gpu_total_bits;
        m.feature_maps = bits;
        if (__builtin_sub_overflow(gpu_total_bits, bits, &m.bound))
            throw OverflowError("integer overflow in memory arithmetic");
        work.push_back(std::async(std::launch::async, assess_bound, std::cref(catalog), dataset_size, b, m));
    }
    BatchPlan plan;
    for (auto& w : work) plan.candidates.push_back(w.get());
    recommend(plan);
    plan.advisories = advise_refinement(plan, NetworkSpec{});
    return plan;
}

BatchPlan plan_batch_size(const NetworkSpec& network, const AlgorithmCatalog& catalog,
                          std::int64_t gpu_total_bits, std::int64_t dataset_size,
                          const std::vector<std::int64_t>& candidates) {
    if (candidates.empty()) throw DomainError("candidate batch-size list must not be empty");
    if (dataset_size < 1) throw DomainError("dataset size must be >= 1");
    for (std::int64_t b : candidates)
        if (!catalog.has_batch_size(b))
            throw CandidateNotInCatalogError("batch size " + std::to_string(b) +
                                             " is not declared in the catalog");
    if (catalog.layer_count() != network.convolution_layer_count())
        throw IncompleteCatalogError("catalog profiles " + std::to_string(catalog.layer_count()) +
                                     " convolution layers but the network has " +
                                     std::to_string(network.convolution_layer_count()));

    // Candidates are independent: evaluate concurrently, collect in input order
    // (the first failing candidate in input order is the one whose error surfaces).
    std::vector<std::future<BatchCandidateResult>> work;
    work.reserve(candidates.size());
    for (std::int64_t b : candidates)
        work.push_back(std::async(std::launch::async, assess, std::cref(network),
                                  std::cref(catalog), gpu_total_bits, dataset_size, b));
    BatchPlan plan;
    for (auto& w : work) plan.candidates.push_back(w.get());
    recommend(plan);
    plan.advisories = advise_refinement(plan, network);
    return plan;
}

std::vector<Advisory> advise_refinement(const BatchPlan& plan, const NetworkSpec&) {
    std::vector<Advisory> out;
    if (!plan.recommended) {
        std::int64_t smallest = 0;
        for (const auto& c : plan.candidates)
            smallest = smallest == 0 ? c.batch_size : std::min(smallest, c.batch_size);
        out.push_back({AdvisoryKind::reduce_batch,
                       "no candidate mini-batch fits in GPU memory; profile and sweep batch "
                       "sizes below " +
                           std::to_string(smallest),
                       {}});
    } else {
        const BatchCandidateResult* chosen = nullptr;
        for (const auto& c : plan.candidates)
            if (c.batch_size == *plan.recommended) chosen = &c;
        for (const auto& c : plan.candidates) {
            const bool faster_smaller = c.batch_size < chosen->batch_size && c.throughput &&
                                        chosen->throughput && *c.throughput > *chosen->throughput;
            if (!faster_smaller) continue;
            out.push_back({AdvisoryKind::reduce_batch,
                           "batch " + std::to_string(c.batch_size) +
                               " sustains higher throughput than the recommended " +
                               std::to_string(chosen->batch_size) +
                               "; consider reducing the mini-batch size",
                           {}});
            break;
        }
        if (!chosen->memory_limited_layers.empty())
            out.push_back({AdvisoryKind::adjust_model,
                           "memory budget forced slower algorithms at batch " +
                               std::to_string(chosen->batch_size) +
                               "; freeing memory (larger strides, leaner filters) on the listed "
                               "layers would unlock the faster ones",
                           chosen->memory_limited_layers});
    }
    out.push_back({AdvisoryKind::caveat, kClassifierCaveat, {}});
    return out;
}

std::vector<std::string> model_caveats() {
    return {
        kClassifierCaveat,
        "candidates are ranked by estimated epoch time only; convergence quality is assumed "
        "equivalent across the swept mini-batch sizes",
        "parameter-server sizing ignores server-side update compute; network transfer is "
        "assumed to dominate",
        "the overhead ratio is treated as a constant; real overheads fluctuate run to run",
    };
}

// ------------------------------------------------------------- lemmas ----

namespace {
constexpr PipelineStep kAllSteps[] = {
    PipelineStep::parameter_refresh,    PipelineStep::data_loading,
    PipelineStep::data_preparation,     PipelineStep::host_to_gpu_transfer,
    PipelineStep::gpu_processing,       PipelineStep::parameter_update,
    PipelineStep::distributed_update,
};
}  // namespace

const char* to_string(PipelineStep step) {
    switch (step) {
        case PipelineStep::parameter_refresh: return "parameter_refresh";
        case PipelineStep::data_loading: return "data_loading";
        case PipelineStep::data_preparation: return "data_preparation";
        case PipelineStep::host_to_gpu_transfer: return "host_to_gpu_transfer";
        case PipelineStep::gpu_processing: return "gpu_processing";
        case PipelineStep::parameter_update: return "parameter_update";
        case PipelineStep::distributed_update: return "distributed_update";
    }
    return "?";
}

std::optional<PipelineStep> pipeline_step_from_string(std::string_view name) {
    for (PipelineStep s : kAllSteps)
        if (name == to_string(s)) return s;
    return std::nullopt;
}

// Lemma 1: alpha = (1 + R_O) / (1 + G R_O).
double efficiency(int gpus, double r) {
    if (gpus < 1) throw DomainError("GPU count must be >= 1");
    if (r < 0) throw DomainError("overhead ratio must be >= 0");
    return (1.0 + r) / (1.0 + gpus * r);
}

ScalingEstimate estimate_scaling(int gpus, double r) {
    const double a = efficiency(gpus, r);
    return ScalingEstimate{gpus, a, a * gpus};
}

std::vector<ScalingEstimate> scaling_table(int max_gpus, double r) {
    if (max_gpus < 1) throw DomainError("GPU count must be >= 1");
    std::vector<ScalingEstimate> rows;
    for (int g = 1; g <= max_gpus; ++g) rows.push_back(estimate_scaling(g, r));
    return rows;
}

double max_overhead_ratio(int gpus, double alpha) {
    if (gpus < 2) throw DomainError("overhead bound needs at least 2 GPUs");
    const bool inside = alpha > 1.0 / gpus && alpha < 1.0;
    if (!inside) throw DomainError("efficiency must lie strictly between 1/G and 1");
    return (1.0 - alpha) / (alpha * gpus - 1.0);
}

GpuRecommendation recommend_gpus(double target, double r, int max_gpus) {
    if (target < 1.0) throw DomainError("target speedup must be >= 1");
    if (max_gpus < 1) throw DomainError("GPU count must be >= 1");
    GpuRecommendation rec;
    rec.speedup_cap = r > 0 ? 1.0 + 1.0 / r : std::numeric_limits<double>::infinity();
    for (int g = 1; g <= max_gpus && !rec.gpus; ++g)
        if (estimate_scaling(g, r).speedup >= target) rec.gpus = g;
    return rec;
}

OverheadProfile estimate_overhead_ratio(const std::map<PipelineStep, double>& times,
                                        const std::set<PipelineStep>& hidden) {
    for (const auto& kv : times)
        if (kv.second < 0)
            throw DomainError(std::string("negative time for step ") + to_string(kv.first));
    const auto gpu = times.find(PipelineStep::gpu_processing);
    if (gpu == times.end() || !(gpu->second > 0))
        throw MissingComputeStepError("step trace needs a positive gpu_processing time");
    OverheadProfile p;
    p.compute_time = gpu->second;
    for (const auto& kv : times)
        if (kv.first != PipelineStep::gpu_processing && !hidden.count(kv.first))
            p.overhead_time += kv.second;
    return p;
}

// Lemma 2: least n >= 1 with T_C >= 2 S_p N_w / (n B_ps).
int min_parameter_servers(const ClusterSpec& spec, double compute_time) {
    if (spec.worker_count < 1) throw DomainError("worker count must be >= 1");
    if (!(spec.param_size_bytes > 0)) throw DomainError("parameter size must be > 0");
    if (!(spec.bandwidth_bytes_per_sec > 0)) throw DomainError("bandwidth must be > 0");
    if (!(compute_time > 0)) throw DomainError("compute time must be > 0");
    const double traffic = 2.0 * spec.param_size_bytes * spec.worker_count;
    const auto hides = [&](std::int64_t n) {
        return compute_time >= traffic / (static_cast<double>(n) * spec.bandwidth_bytes_per_sec);
    };
    // The closed form is exact in real arithmetic; the inequality itself decides
    // the boundary cases rounding can shift.
    std::int64_t n = static_cast<std::int64_t>(
        std::ceil(traffic / (spec.bandwidth_bytes_per_sec * compute_time)));
    n = std::max<std::int64_t>(n, 1);
    while (!hides(n)) ++n;
    while (n > 1 && hides(n - 1)) --n;
    return static_cast<int>(n);
}

}  // namespace traincap
