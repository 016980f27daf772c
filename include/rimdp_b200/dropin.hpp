// rimdp_b200/dropin.hpp — the reference's solve entry points, on the B200.
//
// Header-only C++20 host layer above the C ABI (include/rimdp_b200.h).  It
// takes the reference's own model and problem types unchanged — IntervalMDP,
// IntervalProbabilities, Specification, Problem, Policy (imdp.hpp,
// interval.hpp, property.hpp under proj/include/rimdp/) — and offers the same
// signatures as the reference's hot-path entry points:
//
//   value_iteration(problem, options)            solver.hpp:149-155
//   control_synthesis(problem, options)          solver.hpp:163-198
//   verify_policy(mdp, policy, spec, options)    solver.hpp:204-251
//   bellman_step(mdp, v_prev, mode, frozen, w)   bellman.hpp:127-133
//   robust_expectation(column, values, mode)     omax.hpp:182-199
//   io::read_native_model<Value>(path)           io/native.hpp:457-561
//
// with the same results (bit-identical on the exact-order kernels, see
// DESIGN.md "Parity") and the same exception types and messages
// (errors.hpp: ModelError{InfeasibleColumn}, NonConvergence,
// PropertyStateOutOfRange, InvalidProperty, InvalidPolicyAction).  Only the
// iteration runs elsewhere: every Bellman step executes in sm_100a kernels
// on the device; there is no CPU fallback — without a device the calls throw
// rimdp::Error.
//
// `Engine<Value>` keeps one IMDP resident in HBM across solves; the free
// functions upload the model per call, like the reference's by-value
// Problem.  See INTEGRATION.md for the two-line dispatch a maintainer adds to
// solver.hpp / bellman.hpp so that existing callers reach this layer.
#pragma once

#include "rimdp_b200.h"

#include "rimdp/bellman.hpp"
#include "rimdp/errors.hpp"
#include "rimdp/imdp.hpp"
#include "rimdp/numeric.hpp"
#include "rimdp/omax.hpp"
#include "rimdp/property.hpp"
#include "rimdp/solver.hpp"

#include <charconv>
#include <cstdint>
#include <span>
#include <string>
#include <type_traits>
#include <utility>
#include <variant>
#include <vector>

namespace rimdp_b200 {

using rimdp::index_t;

/// rimdp::SolverOptions (solver.hpp:19-23) plus the engine's placement fields
/// ("a GPU-count option is added as a new field").  Any options
/// type works with the entry points below; these fields are read when present.
struct SolverOptions : rimdp::SolverOptions {
    int device = 0;            ///< single-GPU solves
    int gpus = 1;              ///< > 1: state-sharded over devices 0 .. gpus-1, V exchanged over NVLink
    std::vector<int> devices;  ///< explicit shard devices (may repeat); overrides gpus when non-empty
};

/// Where an Engine puts the model: one device, or one shard per entry of `devices`.
struct Placement {
    int device = 0;
    std::vector<int> devices;  ///< empty or one entry: single device
};

template <typename Options>
Placement placement_of(const Options& o) {
    Placement p;
    if constexpr (requires { o.device; }) p.device = o.device;
    if constexpr (requires { o.devices; }) p.devices.assign(o.devices.begin(), o.devices.end());
    if constexpr (requires { o.gpus; })
        if (p.devices.empty() && o.gpus > 1)
            for (int g = 0; g < o.gpus; ++g) p.devices.push_back(g);
    return p;
}

template <typename Value>
inline constexpr bool has_device_path = std::is_same_v<Value, double> || std::is_same_v<Value, float>;

template <typename Value>
constexpr rimdp_dtype dtype_of() {
    static_assert(has_device_path<Value>,
                  "the B200 engine computes in float64/float32; Rational has no device path");
    return std::is_same_v<Value, double> ? RIMDP_F64 : RIMDP_F32;
}

namespace detail {

template <typename Value>
std::string shortest(double v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, static_cast<Value>(v));
    return std::string(buf, r.ptr);
}

/// Rethrows a failed C-ABI call as the reference's exception type.
template <typename Value>
[[noreturn]] inline void raise(int status) {
    rimdp_error_info info{};
    rimdp_last_error_info(&info);
    const std::string msg = rimdp_last_error();
    switch (status) {
    case RIMDP_ERR_INFEASIBLE_COLUMN: {
        // omax.hpp:72-80: the message quotes the offending sum in shortest form
        const bool low = info.infeasible_kind == 1;
        throw rimdp::ModelError(
            {rimdp::ViolationKind::InfeasibleColumn,
             std::string(low ? "lower" : "upper") + " bounds sum to " + shortest<Value>(info.infeasible_sum) +
                 (low ? " > 1" : " < 1")});
    }
    case RIMDP_ERR_NON_CONVERGENCE:
        throw rimdp::NonConvergence(info.iterations, info.residual);
    case RIMDP_ERR_INVALID_MODEL: {
        // the upload checks (interval.hpp:132-179): the message is Violation::to_string, "<Kind> ...: <text>"
        const auto colon = msg.find(": ");
        rimdp::Violation v{static_cast<rimdp::ViolationKind>(info.violation_kind),
                           colon == std::string::npos ? msg : msg.substr(colon + 2), info.column, info.row};
        throw rimdp::ModelError(std::move(v));
    }
    default:
        throw rimdp::Error("rimdp_b200: " + msg);
    }
}

inline void check(int status, rimdp_dtype dt) {
    if (status == RIMDP_OK) return;
    if (dt == RIMDP_F64) raise<double>(status);
    raise<float>(status);
}

/// The marshalled form of detail::IterationPlan (solver.hpp:27-80).
template <typename Value>
struct Plan {
    std::vector<Value> initial;
    std::vector<std::uint8_t> frozen;
    bool finite = false;
    std::int64_t horizon = 0;
    double eps = 0;
    const std::vector<Value>* rewards = nullptr;
    Value discount{};
};

template <typename Value>
Plan<Value> make_plan(const rimdp::Specification<Value>& spec, index_t n) {
    rimdp::check_property(spec.property, n); // same validation, same exceptions
    Plan<Value> p;
    p.initial.assign(static_cast<std::size_t>(n), Value(0));
    p.frozen.assign(static_cast<std::size_t>(n), 0);
    std::visit(
        [&](const auto& prop) {
            using P = std::decay_t<decltype(prop)>;
            if constexpr (std::is_same_v<P, rimdp::FiniteTimeReachability> ||
                          std::is_same_v<P, rimdp::InfiniteTimeReachability>) {
                for (index_t g : prop.goal) p.initial[g] = Value(1), p.frozen[g] = 1;
            } else if constexpr (std::is_same_v<P, rimdp::FiniteTimeReachAvoid> ||
                                 std::is_same_v<P, rimdp::InfiniteTimeReachAvoid>) {
                for (index_t g : prop.reach) p.initial[g] = Value(1), p.frozen[g] = 1;
                for (index_t a : prop.avoid) p.frozen[a] = 1;
            } else {
                p.initial = prop.rewards;
                p.rewards = &prop.rewards;
                p.discount = prop.discount;
            }
            if constexpr (requires { prop.horizon; }) {
                p.finite = true;
                p.horizon = prop.horizon;
            } else {
                // eps is compared in Value (NumericTraits::from_double, solver.hpp:75)
                p.eps = static_cast<double>(rimdp::NumericTraits<Value>::from_double(prop.eps));
            }
        },
        spec.property);
    return p;
}

} // namespace detail

namespace io {

/// io::read_native_model (io/native.hpp:457-561) through the engine's native
/// reader (rimdp_native_read, csrc/native_io.cpp): the same container checks
/// and the same MissingFile / SchemaViolation messages, and the same model —
/// the arrays it returns are exactly the validated, aligned CSC pattern the
/// reference builds, so they are assembled without re-validation.  The binary
/// container only (the JSON debug variant is refused with a SchemaViolation).
template <typename Value>
rimdp::IntervalMDP<Value> read_native_model(const std::string& path) {
    static_assert(has_device_path<Value>, "rimdp_b200: only double and float models have a device path");
    const rimdp_dtype dt = dtype_of<Value>();
    rimdp_native_sizes sz{};
    void* h = nullptr;
    const int st = rimdp_native_read(path.c_str(), dt, &sz, &h);
    if (st == RIMDP_ERR_MISSING_FILE) throw rimdp::MissingFile(path);
    if (st == RIMDP_ERR_SCHEMA) {
        const std::string msg = rimdp_last_error();
        const std::string prefix = "schema violation: ";
        throw rimdp::SchemaViolation(msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
    }
    detail::check(st, dt);
    struct Free {
        void* h;
        ~Free() { rimdp_native_free(h); }
    } guard{h};
    std::vector<index_t> stateptr(static_cast<std::size_t>(sz.num_states) + 1), rowval(sz.nnz);
    std::vector<std::int64_t> colptr(static_cast<std::size_t>(sz.num_cols) + 1);
    std::vector<Value> lower(sz.nnz), upper(sz.nnz);
    std::vector<char> labels(static_cast<std::size_t>(sz.label_bytes) + 1);
    detail::check(rimdp_native_take(h, stateptr.data(), colptr.data(), rowval.data(), lower.data(), upper.data(),
                                    labels.data()),
                  dt);
    std::vector<index_t> cp(colptr.begin(), colptr.end()); // the container's int32 colptr, widened and back
    std::vector<std::string> actions;
    actions.reserve(sz.num_cols);
    for (std::size_t i = 0; i < static_cast<std::size_t>(sz.label_bytes);) {
        actions.emplace_back(labels.data() + i);
        i += actions.back().size() + 1;
    }
    auto t = rimdp::IntervalProbabilities<Value>::from_aligned_unchecked(sz.num_states, sz.num_cols, std::move(cp),
                                                                         std::move(rowval), std::move(lower),
                                                                         std::move(upper));
    return rimdp::IntervalMDP<Value>::from_parts_unchecked(std::move(t), std::move(stateptr), std::move(actions));
}

} // namespace io

/// One IMDP resident in HBM (rimdp_model): the device CSC store plus the
/// per-column remainders and the column schedule, built once.
template <typename Value>
class Engine {
public:
    explicit Engine(const rimdp::IntervalMDP<Value>& mdp, int device = 0) : Engine(mdp, Placement{device, {}}) {}

    /// Placement with several devices: the model cut into transition-balanced state shards, one per
    /// device, solved together (rimdp_multi_*); results are bit-identical to one device.
    Engine(const rimdp::IntervalMDP<Value>& mdp, const Placement& where) : mdp_(&mdp) {
        const auto& tp = mdp.transition();
        const auto cp32 = tp.colptr();
        std::vector<std::int64_t> colptr(cp32.begin(), cp32.end()); // int64 on the device
        if (colptr.empty()) colptr.push_back(0);
        rimdp_model_desc d{};
        d.dtype = dtype_of<Value>();
        d.device = where.device;
        d.num_states = mdp.num_states();
        d.num_cols = mdp.num_cols();
        d.nnz = tp.nnz();
        d.stateptr = mdp.stateptr().data();
        d.colptr = colptr.data();
        d.rowval = tp.rowval().data();
        d.lower = tp.lower_values().data();
        d.upper = tp.upper_values().data();
        d.device = where.device;
        if (where.devices.size() > 1) {
            detail::check(rimdp_multi_create(&d, static_cast<int32_t>(where.devices.size()), where.devices.data(),
                                             &multi_),
                          d.dtype);
        } else {
            if (where.devices.size() == 1) d.device = where.devices[0];
            detail::check(rimdp_model_create(&d, &model_), d.dtype);
        }
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() {
        rimdp_model_destroy(model_);
        rimdp_multi_destroy(multi_);
    }

    rimdp_model* handle() const { return model_; }
    bool sharded() const { return multi_ != nullptr; }
    const rimdp::IntervalMDP<Value>& mdp() const { return *mdp_; }

    template <typename Options>
    rimdp::ValueFunction<Value> value_iteration(const rimdp::Specification<Value>& spec,
                                                const Options& options) {
        auto plan = detail::make_plan(spec, mdp_->num_states());
        return run(plan, spec.optimization_mode(), options, nullptr, nullptr, false);
    }

    template <typename Options>
    std::pair<rimdp::Policy, rimdp::ValueFunction<Value>> control_synthesis(
        const rimdp::Specification<Value>& spec, const Options& options) {
        auto plan = detail::make_plan(spec, mdp_->num_states());
        const index_t n = mdp_->num_states();
        auto label = [&](index_t s, index_t c) -> const std::string& {
            return mdp_->action(c >= 0 ? c : mdp_->columns_begin(s));
        };
        if (plan.finite) {
            // row t of the recording = the columns of iteration k = horizon - t (solver.hpp:174-186)
            std::vector<index_t> chosen(static_cast<std::size_t>(n) * static_cast<std::size_t>(plan.horizon));
            auto vf = run(plan, spec.optimization_mode(), options, nullptr, chosen.data(), true);
            rimdp::TimeDependentPolicy pol;
            pol.num_states = n;
            pol.horizon = plan.horizon;
            pol.actions.resize(chosen.size());
            for (std::int64_t t = 0; t < plan.horizon; ++t)
                for (index_t s = 0; s < n; ++s) pol.at(s, t) = label(s, chosen[t * n + s]);
            return {rimdp::Policy(std::move(pol)), std::move(vf)};
        }
        std::vector<index_t> chosen(static_cast<std::size_t>(n), -1);
        auto vf = run(plan, spec.optimization_mode(), options, nullptr, chosen.data(), false);
        rimdp::StationaryPolicy pol;
        pol.actions.reserve(n);
        for (index_t s = 0; s < n; ++s) pol.actions.push_back(label(s, chosen[s]));
        return {rimdp::Policy(std::move(pol)), std::move(vf)};
    }

    template <typename Options>
    rimdp::ValueFunction<Value> verify_policy(const rimdp::Policy& policy, const rimdp::Specification<Value>& spec,
                                              const Options& options) {
        const index_t n = mdp_->num_states();
        auto plan = detail::make_plan(spec, n);
        auto resolve = [&](index_t s, const std::string& lab) {
            const index_t c = mdp_->find_action(s, lab);
            if (c < 0)
                throw rimdp::InvalidPolicyAction("state " + std::to_string(s) + " has no action \"" + lab + "\"");
            return c;
        };
        std::vector<index_t> forced;
        bool td = false;
        if (const auto* st = std::get_if<rimdp::StationaryPolicy>(&policy)) {
            if (static_cast<index_t>(st->actions.size()) != n)
                throw rimdp::InvalidPolicyAction("stationary policy has " + std::to_string(st->actions.size()) +
                                                 " entries for " + std::to_string(n) + " states");
            forced.resize(n);
            for (index_t s = 0; s < n; ++s) forced[s] = resolve(s, st->actions[s]);
        } else {
            const auto& tdp = std::get<rimdp::TimeDependentPolicy>(policy);
            if (!plan.finite)
                throw rimdp::InvalidPolicyAction(
                    "a time-dependent policy cannot be evaluated against an infinite-time property");
            if (tdp.num_states != n || tdp.horizon != plan.horizon)
                throw rimdp::InvalidPolicyAction("policy shape " + std::to_string(tdp.num_states) + "x" +
                                                 std::to_string(tdp.horizon) + " does not match " +
                                                 std::to_string(n) + " states, horizon " +
                                                 std::to_string(plan.horizon));
            td = true;
            forced.resize(static_cast<std::size_t>(n) * static_cast<std::size_t>(plan.horizon));
            // the reference resolves iteration k = 1 (t = horizon - 1) first
            for (std::int64_t t = plan.horizon - 1; t >= 0; --t)
                for (index_t s = 0; s < n; ++s) forced[t * n + s] = resolve(s, tdp.at(s, t));
        }
        return run(plan, spec.optimization_mode(), options, &forced, nullptr, false, td);
    }

    rimdp::BellmanResult<Value> bellman_step(std::span<const Value> v_prev, rimdp::OptimizationMode mode,
                                             std::span<const std::uint8_t> frozen = {}) {
        if (multi_) throw rimdp::Error("rimdp_b200: bellman_step runs on a single-device Engine");
        const index_t n = mdp_->num_states();
        if (static_cast<index_t>(v_prev.size()) != n)
            throw rimdp::Error("rimdp_b200: value vector has " + std::to_string(v_prev.size()) + " entries for " +
                               std::to_string(n) + " states");
        rimdp::BellmanResult<Value> out;
        out.values.resize(n);
        out.chosen_column.resize(n);
        detail::check(rimdp_bellman_step(model_, v_prev.data(),
                                         mode.satisfaction == rimdp::SatisfactionMode::Pessimistic,
                                         mode.strategy == rimdp::StrategyMode::Maximize,
                                         frozen.empty() ? nullptr : frozen.data(), nullptr, out.values.data(),
                                         out.chosen_column.data()),
                      dtype_of<Value>());
        return out;
    }

    /// Robust expectation of every column (bellman.hpp:60-70 for all columns at once).
    std::vector<Value> column_values(std::span<const Value> values, rimdp::SatisfactionMode mode) {
        if (multi_) throw rimdp::Error("rimdp_b200: column_values runs on a single-device Engine");
        std::vector<Value> q(static_cast<std::size_t>(mdp_->num_cols()));
        detail::check(rimdp_column_values(model_, values.data(), mode == rimdp::SatisfactionMode::Pessimistic,
                                          q.data()),
                      dtype_of<Value>());
        return q;
    }

private:
    template <typename Options>
    rimdp::ValueFunction<Value> run(const detail::Plan<Value>& plan, rimdp::OptimizationMode mode,
                                    const Options& options, const std::vector<index_t>* forced, index_t* chosen,
                                    bool record_all, bool forced_td = false) {
        const std::size_t n = plan.initial.size();
        rimdp::ValueFunction<Value> vf;
        vf.values.resize(n);
        vf.residual.resize(n);
        rimdp_plan p{};
        p.pessimistic = mode.satisfaction == rimdp::SatisfactionMode::Pessimistic;
        p.maximize = mode.strategy == rimdp::StrategyMode::Maximize;
        p.finite = plan.finite;
        p.horizon = plan.horizon;
        p.eps = plan.eps;
        p.max_iterations = options.max_iterations;
        p.initial = plan.initial.data();
        p.frozen = plan.frozen.data();
        p.rewards = plan.rewards ? plan.rewards->data() : nullptr;
        p.discount = static_cast<double>(plan.discount);
        p.forced = forced ? forced->data() : nullptr;
        p.forced_time_dependent = forced_td;
        rimdp_outputs o{};
        o.values = vf.values.data();
        o.residual = vf.residual.data();
        std::int64_t iters = 0;
        o.iterations = &iters;
        o.chosen = chosen;
        o.record_all_steps = record_all;
        // on_iteration_f64 (solver.hpp:119-125): one device->host copy per iteration, only when set
        struct Cb {
            const Options* opt;
            std::size_t n;
            std::vector<double> buf;
        } cb{&options, n, {}};
        if (options.on_iteration_f64) {
            o.on_iteration = [](std::int64_t k, const void* v, void* user) {
                auto* c = static_cast<Cb*>(user);
                const Value* vv = static_cast<const Value*>(v);
                c->buf.assign(vv, vv + c->n);
                c->opt->on_iteration_f64(k, std::span<const double>(c->buf));
            };
            o.user = &cb;
        }
        detail::check(multi_ ? rimdp_multi_solve(multi_, &p, &o) : rimdp_solve(model_, &p, &o), dtype_of<Value>());
        vf.iterations = iters;
        return vf;
    }

    const rimdp::IntervalMDP<Value>* mdp_;
    rimdp_model* model_ = nullptr;
    rimdp_multi* multi_ = nullptr;
};

// ---- free functions with the reference's signatures ------------------------

// Options defaults to rimdp_b200::SolverOptions (a rimdp::SolverOptions), so
// `value_iteration(problem)` works as in the reference (solver.hpp:149-155).

template <typename Value, typename Options = SolverOptions>
rimdp::ValueFunction<Value> value_iteration(const rimdp::Problem<Value>& problem, const Options& options = {}) {
    Engine<Value> e(problem.imdp, placement_of(options));
    return e.value_iteration(problem.spec, options);
}

template <typename Value, typename Options = SolverOptions>
std::pair<rimdp::Policy, rimdp::ValueFunction<Value>> control_synthesis(const rimdp::Problem<Value>& problem,
                                                                        const Options& options = {}) {
    Engine<Value> e(problem.imdp, placement_of(options));
    return e.control_synthesis(problem.spec, options);
}

template <typename Value, typename Options = SolverOptions>
rimdp::ValueFunction<Value> verify_policy(const rimdp::IntervalMDP<Value>& mdp, const rimdp::Policy& policy,
                                          const rimdp::Specification<Value>& spec, const Options& options = {}) {
    // the reference validates the property before touching the model (solver.hpp:208)
    (void)detail::make_plan(spec, mdp.num_states());
    Engine<Value> e(mdp, placement_of(options));
    return e.verify_policy(policy, spec, options);
}

template <typename Value>
rimdp::BellmanResult<Value> bellman_step(const rimdp::IntervalMDP<Value>& mdp, std::span<const Value> v_prev,
                                         rimdp::OptimizationMode mode, std::span<const std::uint8_t> frozen = {},
                                         unsigned workers = 0) {
    (void)workers; // host threads: the device grid replaces parallel_for_index
    Engine<Value> e(mdp);
    return e.bellman_step(v_prev, mode, frozen);
}

/// One column as a one-column model over `values` (omax.hpp:182-189).
template <typename Value>
Value robust_expectation(const rimdp::ColumnView<Value>& column, std::span<const Value> values,
                         rimdp::SatisfactionMode mode) {
    const index_t n = static_cast<index_t>(values.size());
    const std::int64_t L = static_cast<std::int64_t>(column.size());
    std::vector<index_t> stateptr(static_cast<std::size_t>(n) + 1, 1);
    stateptr[0] = 0;
    std::int64_t colptr[2] = {0, L};
    rimdp_model_desc d{};
    d.dtype = dtype_of<Value>();
    d.num_states = n;
    d.num_cols = 1;
    d.nnz = L;
    d.stateptr = stateptr.data();
    d.colptr = colptr;
    d.rowval = column.rows.data();
    d.lower = column.lower.data();
    d.upper = column.upper.data();
    rimdp_model* m = nullptr;
    detail::check(rimdp_model_create(&d, &m), d.dtype);
    Value q{};
    const int st = rimdp_column_values(m, values.data(), mode == rimdp::SatisfactionMode::Pessimistic, &q);
    rimdp_model_destroy(m);
    detail::check(st, d.dtype);
    return q;
}

} // namespace rimdp_b200
