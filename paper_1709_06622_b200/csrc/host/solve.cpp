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
#include <functional>
#include <future>
#include <limits>
#include <numeric>
#include <tuple>

#include "traincap/api.hpp"

namespace traincap {

namespace {

// A complete assignment: its totals and the option picked for each layer.
struct Leaf {
    double time = 0.0;
    std::int64_t memory = 0;
    std::vector<const CostEntry*> pick;
};

// The canonical optimum both solvers return: least total time, then least
// workspace, then the lexicographically smallest sequence of algorithm names.
bool better_than(double t, std::int64_t m, const std::vector<const CostEntry*>& pick,
                 const std::optional<Leaf>& incumbent) {
    if (!incumbent) return true;
    if (t != incumbent->time || m != incumbent->memory)
        return std::make_pair(t, m) < std::make_pair(incumbent->time, incumbent->memory);
    return std::lexicographical_compare(pick.begin(), pick.end(), incumbent->pick.begin(), incumbent->pick.end(),
                                        [](const CostEntry* x, const CostEntry* y) { return x->algorithm < y->algorithm; });
}

void require_nonempty(const LayerOptions& options) {
    const auto hole = std::find_if(options.begin(), options.end(), [](const auto& l) { return l.empty(); });
    if (hole != options.end())
        throw IncompleteCatalogError("layer " + std::to_string(hole - options.begin() + 1) +
                                     " has no algorithm options");
}

// Options of every layer fastest first (time, workspace, name), so that an
// assignment sums its per-layer times in one fixed order in either solver.
LayerOptions sorted_copy(const LayerOptions& options) {
    LayerOptions s = options;
    const auto key = [](const CostEntry& e) { return std::tie(e.time_seconds, e.memory_bits, e.algorithm); };
    for (auto& layer : s)
        std::sort(layer.begin(), layer.end(), [&](const CostEntry& x, const CostEntry& y) { return key(x) < key(y); });
    return s;
}

// The least workspace any assignment can use (each layer at its leanest option).
std::int64_t cheapest_memory(const LayerOptions& options) {
    return std::transform_reduce(options.begin(), options.end(), std::int64_t{0}, std::plus<>(), [](const auto& l) {
        return std::min_element(l.begin(), l.end(), [](const CostEntry& x, const CostEntry& y) {
                   return x.memory_bits < y.memory_bits;
               })->memory_bits;
    });
}

Selection make_selection(const Leaf& leaf) {
    Selection s{{}, leaf.time, leaf.memory};
    int layer = 0;
    for (const CostEntry* e : leaf.pick) s.assignment.emplace(++layer, e->algorithm);
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
    // the paper's sweep grid (powers of two, 32..512) restricted to what was profiled
    static constexpr std::int64_t kGrid[] = {32, 64, 128, 256, 512};
    std::vector<std::int64_t> out;
    std::copy_if(std::begin(kGrid), std::end(kGrid), std::back_inserter(out),
                 [&](std::int64_t b) { return catalog.has_batch_size(b); });
    return out;
}

namespace {

constexpr const char* kClassifierCaveat =
    "classifier memory uses a fixed per-junction bias charge and batch-independent "
    "activations; treat classifier totals as approximate";

// §3.1.3 mini-batch sweep. A candidate is scored from its workspace bound:
// the Eq 6 selection under that bound, epoch time = ceil(dataset / b) * sum T,
// throughput = b / sum T (the paper's img/s model), and the layers whose
// selected algorithm is slower than their fastest profiled one (memory-limited).
// Both sweeps below differ only in where the bound comes from.
class Sweep {
public:
    using BoundFn = std::function<MemoryBreakdown(std::size_t)>;  // candidate index -> its bound

    Sweep(const AlgorithmCatalog& catalog, std::int64_t dataset) : cat_(catalog), dataset_(dataset) {}

    // Candidates are independent and pure: scored concurrently, kept in input
    // order (the first failing candidate in input order is the error that surfaces).
    BatchPlan run(const std::vector<std::int64_t>& batches, const BoundFn& bound) const {
        std::vector<std::future<BatchCandidateResult>> pending;
        pending.reserve(batches.size());
        for (std::size_t i = 0; i < batches.size(); ++i)
            pending.push_back(std::async(std::launch::async, [this, i, &batches, &bound] {
                return score(batches[i], bound(i));
            }));
        BatchPlan plan;
        plan.candidates.reserve(batches.size());
        for (auto& f : pending) plan.candidates.push_back(f.get());
        plan.recommended = pick(plan.candidates);
        return plan;
    }

    BatchCandidateResult score(std::int64_t b, const MemoryBreakdown& m) const {
        BatchCandidateResult r;
        r.batch_size = b;
        r.breakdown = m;
        const LayerOptions per_layer = catalog_options(cat_, b);
        r.solve = solve_selection(per_layer, m.bound);
        if (!r.solve.selection) return r;
        const Selection& chosen = *r.solve.selection;
        const double sum_t = chosen.total_time;
        const std::int64_t rounds = dataset_ / b + (dataset_ % b != 0);
        r.epoch_time_seconds = sum_t * static_cast<double>(rounds);
        r.throughput = static_cast<double>(b) / sum_t;
        int layer = 0;
        for (const std::vector<CostEntry>& opts : per_layer) {
            ++layer;  // options are sorted fastest first
            const auto it = std::find_if(opts.begin(), opts.end(), [&](const CostEntry& e) {
                return e.algorithm == chosen.assignment.at(layer);
            });
            if (it->time_seconds > opts.front().time_seconds) r.memory_limited_layers.push_back(layer);
        }
        return r;
    }

    // Shortest epoch wins; equal epochs go to the larger mini-batch.
    static std::optional<std::int64_t> pick(const std::vector<BatchCandidateResult>& cs) {
        const BatchCandidateResult* best = nullptr;
        for (const BatchCandidateResult& c : cs) {
            if (!c.epoch_time_seconds) continue;
            const bool better = !best || *c.epoch_time_seconds < *best->epoch_time_seconds ||
                                (*c.epoch_time_seconds == *best->epoch_time_seconds && c.batch_size > best->batch_size);
            if (better) best = &c;
        }
        return best ? std::optional<std::int64_t>(best->batch_size) : std::nullopt;
    }

private:
    const AlgorithmCatalog& cat_;
    std::int64_t dataset_;
};

void require_sweep_inputs(std::size_t n_candidates, std::int64_t dataset) {
    if (n_candidates == 0) throw DomainError("candidate batch-size list must not be empty");
    if (dataset < 1) throw DomainError("dataset size must be >= 1");
}

void require_declared(const AlgorithmCatalog& catalog, std::int64_t b) {
    if (!catalog.has_batch_size(b))
        throw CandidateNotInCatalogError("batch size " + std::to_string(b) + " is not declared in the catalog");
}

}  // namespace

BatchPlan plan_batch_size_resident(const AlgorithmCatalog& catalog,
                                   const std::vector<std::pair<std::int64_t, std::int64_t>>& resident_bits,
                                   std::int64_t gpu_total_bits, std::int64_t dataset_size) {
    require_sweep_inputs(resident_bits.size(), dataset_size);
    std::vector<std::int64_t> order;
    for (const auto& [b, bits] : resident_bits) {
        require_declared(catalog, b);
        if (bits < 0) throw DomainError("resident bits must be >= 0");
        std::int64_t left = 0;
        if (__builtin_sub_overflow(gpu_total_bits, bits, &left))
            throw OverflowError("integer overflow in memory arithmetic");
        order.push_back(b);
    }
    // the executor's resident bytes stand in for Eq 2-5 (no chain model for branched graphs)
    const auto bound = [&](std::size_t i) {
        MemoryBreakdown m;
        m.batch_size = resident_bits[i].first;
        m.gpu_total = gpu_total_bits;
        m.feature_maps = resident_bits[i].second;
        m.bound = gpu_total_bits - m.feature_maps;
        return m;
    };
    BatchPlan plan = Sweep(catalog, dataset_size).run(order, bound);
    plan.advisories = advise_refinement(plan, NetworkSpec{});
    return plan;
}

BatchPlan plan_batch_size(const NetworkSpec& network, const AlgorithmCatalog& catalog,
                          std::int64_t gpu_total_bits, std::int64_t dataset_size,
                          const std::vector<std::int64_t>& candidates) {
    require_sweep_inputs(candidates.size(), dataset_size);
    for (std::int64_t b : candidates) require_declared(catalog, b);
    const int convs = network.convolution_layer_count();
    if (catalog.layer_count() != convs)
        throw IncompleteCatalogError("catalog profiles " + std::to_string(catalog.layer_count()) +
                                     " convolution layers but the network has " + std::to_string(convs));
    const auto bound = [&](std::size_t i) { return memory_bound(gpu_total_bits, network, candidates[i]); };
    BatchPlan plan = Sweep(catalog, dataset_size).run(candidates, bound);
    plan.advisories = advise_refinement(plan, network);
    return plan;
}

// §3.1.4 refinement advice: nothing fits -> sweep smaller batches; a smaller
// batch with higher throughput than the recommendation -> consider it; a
// recommendation that had to trade speed for memory -> name those layers;
// the classifier caveat always closes the list.
std::vector<Advisory> advise_refinement(const BatchPlan& plan, const NetworkSpec&) {
    std::vector<Advisory> advice;
    const auto& cs = plan.candidates;
    if (!plan.recommended) {
        const auto smallest = std::min_element(cs.begin(), cs.end(), [](const auto& x, const auto& y) {
            return x.batch_size < y.batch_size;
        });
        advice.push_back({AdvisoryKind::reduce_batch,
                          "no candidate mini-batch fits in GPU memory; profile and sweep batch sizes below " +
                              std::to_string(smallest == cs.end() ? 0 : smallest->batch_size),
                          {}});
    } else {
        const std::int64_t rb = *plan.recommended;
        const auto rec = std::find_if(cs.rbegin(), cs.rend(), [&](const auto& c) { return c.batch_size == rb; });
        const auto faster = std::find_if(cs.begin(), cs.end(), [&](const auto& c) {
            return c.batch_size < rb && c.throughput && rec->throughput && *c.throughput > *rec->throughput;
        });
        if (faster != cs.end())
            advice.push_back({AdvisoryKind::reduce_batch,
                              "batch " + std::to_string(faster->batch_size) +
                                  " sustains higher throughput than the recommended " + std::to_string(rb) +
                                  "; consider reducing the mini-batch size",
                              {}});
        if (!rec->memory_limited_layers.empty())
            advice.push_back({AdvisoryKind::adjust_model,
                              "memory budget forced slower algorithms at batch " + std::to_string(rb) +
                                  "; freeing memory (larger strides, leaner filters) on the listed layers would "
                                  "unlock the faster ones",
                              rec->memory_limited_layers});
    }
    advice.push_back({AdvisoryKind::caveat, kClassifierCaveat, {}});
    return advice;
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
