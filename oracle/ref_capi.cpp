// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include (header-only C++20, see proj/CMakeLists.txt:12-17)
// and the reference's own test oracle (proj/tests/oracle.hpp).  Compiled by
// oracle/Makefile into oracle/_ref/librimdp_ref.so with -Drimdp=rimdp_ref so it
// can share a process with the B200 engine.  Nothing here re-implements the
// algorithm: every result comes from the reference's own functions:
//   random_imdp / random_point_imdp      random_model.hpp:42-161
//   IntervalProbabilities::from_aligned  interval.hpp:67-77
//   IntervalMDP::from_parts              imdp.hpp:78-84
//   value_iteration / control_synthesis  solver.hpp:149-198
//   verify_policy                        solver.hpp:204-251
//   bellman_step                         bellman.hpp:127-133
//   robust_expectation                   omax.hpp:182-189
//   omaximize_sequential                 omax.hpp:98-112
//   oracle::robust_expectation (LP)      tests/oracle.hpp:28-80
//   oracle::random_feasible_column       tests/oracle.hpp:193-217
//   io::write_native_model / read_native_model  io/native.hpp:424-561
// The one non-reference input is the counter-based workload generator of
// BASELINE configs 4-5 (paper_2401_04068_b200/csrc/generator.cuh, host-side
// and header-only: a workload, not the algorithm), so bench.py's reference
// arm can build those models without loading the engine library.

#include "rimdp/io/native.hpp"
#include "rimdp/random_model.hpp"
#include "rimdp/solver.hpp"
#include "oracle.hpp" // proj/tests/oracle.hpp

#include "generator.cuh" // workload generator of configs 4-5 (host build)

#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <string>
#include <vector>

using rimdp::index_t;

namespace {

enum RefStatus {
    REF_OK = 0,
    REF_MODEL_ERROR = 1,
    REF_NON_CONVERGENCE = 2,
    REF_STATE_OUT_OF_RANGE = 3,
    REF_INVALID_PROPERTY = 4,
    REF_INVALID_POLICY = 5,
    REF_OTHER = 9,
};

struct ErrOut {
    char* buf;
    int len;
    std::int64_t* iters;   // NonConvergence payload
    double* residual;
    int* violation_kind;   // ModelError payload
    std::int64_t* violation_column;
};

void put(const ErrOut& e, const std::string& s) {
    if (e.buf && e.len > 0) {
        std::strncpy(e.buf, s.c_str(), static_cast<std::size_t>(e.len - 1));
        e.buf[e.len - 1] = '\0';
    }
}

template <class F>
int guarded(const ErrOut& e, F&& f) {
    try {
        f();
        return REF_OK;
    } catch (const rimdp::ModelError& ex) {
        put(e, ex.what());
        if (e.violation_kind) *e.violation_kind = static_cast<int>(ex.kind());
        if (e.violation_column) *e.violation_column = ex.violation().column;
        return REF_MODEL_ERROR;
    } catch (const rimdp::NonConvergence& ex) {
        put(e, ex.what());
        if (e.iters) *e.iters = ex.iterations();
        if (e.residual) *e.residual = ex.residual();
        return REF_NON_CONVERGENCE;
    } catch (const rimdp::PropertyStateOutOfRange& ex) {
        put(e, ex.what());
        return REF_STATE_OUT_OF_RANGE;
    } catch (const rimdp::InvalidProperty& ex) {
        put(e, ex.what());
        return REF_INVALID_PROPERTY;
    } catch (const rimdp::InvalidPolicyAction& ex) {
        put(e, ex.what());
        return REF_INVALID_POLICY;
    } catch (const std::exception& ex) {
        put(e, ex.what());
        return REF_OTHER;
    }
}

struct ModelBase {
    virtual ~ModelBase() = default;
};
template <class V>
struct Model : ModelBase {
    rimdp::IntervalMDP<V> mdp;
};

std::vector<std::string> positional_labels(const std::vector<index_t>& stateptr) {
    std::vector<std::string> labels;
    for (std::size_t s = 0; s + 1 < stateptr.size(); ++s)
        for (index_t c = stateptr[s]; c < stateptr[s + 1]; ++c)
            labels.push_back(std::to_string(c - stateptr[s]));
    return labels;
}

} // namespace

extern "C" {

// Spec passed across the shim.  kind: 0 FiniteTimeReachability,
// 1 InfiniteTimeReachability, 2 FiniteTimeReachAvoid, 3 InfiniteTimeReachAvoid,
// 4 FiniteTimeReward, 5 InfiniteTimeReward (property.hpp:14-59).
struct ref_spec {
    int kind;
    const int* reach;
    int nreach;
    const int* avoid;
    int navoid;
    const void* rewards; // Value[n]
    double discount;     // converted with static_cast<Value>
    long long horizon;
    double eps;
    int pessimistic;
    int maximize;
    unsigned workers;
    long long max_iterations;
};

struct ref_err {
    char msg[512];
    long long iterations;
    double residual;
    int violation_kind;
    long long violation_column;
};

} // extern "C"

namespace {

template <class V>
rimdp::Specification<V> make_spec(const ref_spec& sp, index_t n) {
    std::vector<index_t> reach(sp.reach, sp.reach + sp.nreach);
    std::vector<index_t> avoid(sp.avoid, sp.avoid + sp.navoid);
    rimdp::Property<V> prop;
    const V* r = static_cast<const V*>(sp.rewards);
    switch (sp.kind) {
    case 0: prop = rimdp::FiniteTimeReachability{reach, sp.horizon}; break;
    case 1: prop = rimdp::InfiniteTimeReachability{reach, sp.eps}; break;
    case 2: prop = rimdp::FiniteTimeReachAvoid{reach, avoid, sp.horizon}; break;
    case 3: prop = rimdp::InfiniteTimeReachAvoid{reach, avoid, sp.eps}; break;
    case 4:
        prop = rimdp::FiniteTimeReward<V>{std::vector<V>(r, r + (r ? n : 0)),
                                          static_cast<V>(sp.discount), sp.horizon};
        break;
    default:
        prop = rimdp::InfiniteTimeReward<V>{std::vector<V>(r, r + (r ? n : 0)),
                                            static_cast<V>(sp.discount), sp.eps};
        break;
    }
    return {prop, sp.pessimistic ? rimdp::SatisfactionMode::Pessimistic
                                 : rimdp::SatisfactionMode::Optimistic,
            sp.maximize ? rimdp::StrategyMode::Maximize : rimdp::StrategyMode::Minimize};
}

template <class V>
int from_arrays(int n, int ncols, const int* stateptr, const int* colptr, const int* rowval,
                const V* lower, const V* upper, int checked, void** out, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr,
             err ? &err->violation_kind : nullptr, nullptr};
    return guarded(e, [&] {
        const std::int64_t nnz = colptr[ncols];
        std::vector<index_t> sp(stateptr, stateptr + n + 1);
        std::vector<index_t> cp(colptr, colptr + ncols + 1);
        std::vector<index_t> rv(rowval, rowval + nnz);
        std::vector<V> lo(lower, lower + nnz), up(upper, upper + nnz);
        auto labels = positional_labels(sp);
        auto m = new Model<V>;
        if (checked) {
            auto t = rimdp::IntervalProbabilities<V>::from_aligned(n, ncols, cp, rv, lo, up);
            m->mdp = rimdp::IntervalMDP<V>::from_parts(std::move(t), sp, labels);
        } else {
            auto t = rimdp::IntervalProbabilities<V>::from_aligned_unchecked(n, ncols, cp, rv, lo, up);
            m->mdp = rimdp::IntervalMDP<V>::from_parts_unchecked(std::move(t), sp, labels);
        }
        *out = static_cast<ModelBase*>(m);
    });
}

// A counter-generator workload (configs 4-5 law, rimdp_gen::write_column)
// built through the reference's own checked constructors.
template <class V>
int generate_model(int states, int actions, int law, int support, double alpha, int kmax, double lower_scale,
                   double upper_scale, unsigned long long seed, void** out, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr, nullptr, nullptr};
    return guarded(e, [&] {
        rimdp_gen::Params p{states, actions, law, support, kmax, lower_scale, upper_scale, seed};
        std::vector<uint64_t> cdf;
        if (law == 1) cdf = rimdp_gen::power_law_cdf(kmax, alpha);
        const index_t ncols = static_cast<index_t>(states) * actions;
        std::vector<index_t> cp(ncols + 1, 0), sp(states + 1);
        for (index_t c = 0; c < ncols; ++c) cp[c + 1] = cp[c] + rimdp_gen::column_length(p, cdf.data(), c);
        for (int s = 0; s <= states; ++s) sp[s] = s * actions;
        std::vector<index_t> rv(cp[ncols]);
        std::vector<V> lo(cp[ncols]), up(cp[ncols]);
        std::vector<std::int32_t> r32(4096 * 2);
        for (index_t c = 0; c < ncols; ++c) {
            const int k = cp[c + 1] - cp[c];
            if ((int)r32.size() < k) r32.resize(k);
            rimdp_gen::write_column<V>(p, c, k, r32.data(), lo.data() + cp[c], up.data() + cp[c]);
            for (int i = 0; i < k; ++i) rv[cp[c] + i] = r32[i];
        }
        auto labels = positional_labels(sp);
        auto m = new Model<V>;
        auto t = rimdp::IntervalProbabilities<V>::from_aligned(states, ncols, cp, rv, lo, up);
        m->mdp = rimdp::IntervalMDP<V>::from_parts(std::move(t), sp, labels);
        *out = static_cast<ModelBase*>(m);
    });
}

template <class V>
int random_model(int states, int actions, double density, double scale, unsigned long long seed,
                 int point, void** out, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr, nullptr, nullptr};
    return guarded(e, [&] {
        rimdp::RandomModelConfig cfg{states, actions, density, scale, seed};
        auto m = new Model<V>;
        m->mdp = point ? rimdp::random_point_imdp<V>(cfg) : rimdp::random_imdp<V>(cfg);
        *out = static_cast<ModelBase*>(m);
    });
}

template <class V>
void model_export(void* h, int* stateptr, int* colptr, int* rowval, V* lower, V* upper) {
    const auto& mdp = static_cast<Model<V>*>(static_cast<ModelBase*>(h))->mdp;
    const auto& t = mdp.transition();
    auto sp = mdp.stateptr();
    std::copy(sp.begin(), sp.end(), stateptr);
    std::copy(t.colptr().begin(), t.colptr().end(), colptr);
    std::copy(t.rowval().begin(), t.rowval().end(), rowval);
    std::copy(t.lower_values().begin(), t.lower_values().end(), lower);
    std::copy(t.upper_values().begin(), t.upper_values().end(), upper);
}

template <class V>
int write_native(void* h, const char* path, int json_debug, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr, nullptr, nullptr};
    return guarded(e, [&] {
        rimdp::io::write_native_model(path, static_cast<Model<V>*>(static_cast<ModelBase*>(h))->mdp, json_debug != 0);
    });
}

template <class V>
int read_native(const char* path, void** out, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr, nullptr, nullptr};
    return guarded(e, [&] {
        auto m = new Model<V>;
        try {
            m->mdp = rimdp::io::read_native_model<V>(path);
        } catch (...) {
            delete m;
            throw;
        }
        *out = static_cast<ModelBase*>(m);
    });
}

// action labels, each NUL-terminated, concatenated; returns the byte count
template <class V>
long long model_labels(void* h, char* out) {
    const auto& mdp = static_cast<Model<V>*>(static_cast<ModelBase*>(h))->mdp;
    long long n = 0;
    for (const auto& a : mdp.actions()) {
        if (out) std::memcpy(out + n, a.c_str(), a.size() + 1);
        n += static_cast<long long>(a.size()) + 1;
    }
    return n;
}

template <class V>
int solve(void* h, const ref_spec* sp, int synthesize, V* values, V* residual,
          long long* iterations, int* policy_cols, V* trace, long long trace_cap, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, err ? reinterpret_cast<std::int64_t*>(&err->iterations) : nullptr,
             err ? &err->residual : nullptr, err ? &err->violation_kind : nullptr,
             err ? reinterpret_cast<std::int64_t*>(&err->violation_column) : nullptr};
    auto* model = static_cast<Model<V>*>(static_cast<ModelBase*>(h));
    // Problem holds the IMDP by value (property.hpp:73-77): move it in and back
    // out so a timed solve does not pay for a model copy.
    rimdp::Problem<V> problem{std::move(model->mdp), {}};
    struct Restore {
        Model<V>* m;
        rimdp::Problem<V>* p;
        ~Restore() { m->mdp = std::move(p->imdp); }
    } restore{model, &problem};
    return guarded(e, [&] {
        const auto& mdp = problem.imdp;
        const index_t n = mdp.num_states();
        problem.spec = make_spec<V>(*sp, n);
        rimdp::SolverOptions opt;
        opt.workers = sp->workers;
        opt.max_iterations = sp->max_iterations;
        if (trace) {
            opt.on_iteration_f64 = [&](std::int64_t k, std::span<const double> v) {
                if (k > trace_cap) return;
                for (index_t s = 0; s < n; ++s) trace[(k - 1) * n + s] = static_cast<V>(v[s]);
            };
        }
        rimdp::ValueFunction<V> vf;
        if (synthesize) {
            auto [policy, out] = rimdp::control_synthesis(problem, opt);
            vf = std::move(out);
            if (policy_cols) {
                if (auto* st = std::get_if<rimdp::StationaryPolicy>(&policy)) {
                    for (index_t s = 0; s < n; ++s) policy_cols[s] = mdp.find_action(s, st->actions[s]);
                } else {
                    const auto& td = std::get<rimdp::TimeDependentPolicy>(policy);
                    for (index_t s = 0; s < n; ++s)
                        for (std::int64_t t = 0; t < td.horizon; ++t)
                            policy_cols[s * td.horizon + t] = mdp.find_action(s, td.at(s, t));
                }
            }
        } else {
            vf = rimdp::value_iteration(problem, opt);
        }
        std::copy(vf.values.begin(), vf.values.end(), values);
        std::copy(vf.residual.begin(), vf.residual.end(), residual);
        *iterations = vf.iterations;
    });
}

template <class V>
int verify(void* h, const ref_spec* sp, const int* policy_cols, int time_dependent, long long horizon,
           V* values, V* residual, long long* iterations, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, err ? reinterpret_cast<std::int64_t*>(&err->iterations) : nullptr,
             err ? &err->residual : nullptr, nullptr, nullptr};
    return guarded(e, [&] {
        const auto& mdp = static_cast<Model<V>*>(static_cast<ModelBase*>(h))->mdp;
        const index_t n = mdp.num_states();
        auto label = [&](int col) { return col >= 0 && col < mdp.num_cols() ? mdp.action(col) : std::string("<none>"); };
        rimdp::Policy policy;
        if (time_dependent) {
            rimdp::TimeDependentPolicy td;
            td.num_states = n;
            td.horizon = horizon;
            for (std::int64_t i = 0; i < n * horizon; ++i) td.actions.push_back(label(policy_cols[i]));
            policy = td;
        } else {
            rimdp::StationaryPolicy st;
            for (index_t s = 0; s < n; ++s) st.actions.push_back(label(policy_cols[s]));
            policy = st;
        }
        rimdp::SolverOptions opt;
        opt.workers = sp->workers;
        opt.max_iterations = sp->max_iterations;
        auto vf = rimdp::verify_policy(mdp, policy, make_spec<V>(*sp, n), opt);
        std::copy(vf.values.begin(), vf.values.end(), values);
        std::copy(vf.residual.begin(), vf.residual.end(), residual);
        *iterations = vf.iterations;
    });
}

template <class V>
int step(void* h, const V* v, int pessimistic, int maximize, const unsigned char* frozen,
         unsigned workers, V* out_v, int* out_chosen, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr,
             err ? &err->violation_kind : nullptr, nullptr};
    return guarded(e, [&] {
        const auto& mdp = static_cast<Model<V>*>(static_cast<ModelBase*>(h))->mdp;
        const index_t n = mdp.num_states();
        std::span<const std::uint8_t> fz;
        if (frozen) fz = std::span<const std::uint8_t>(frozen, n);
        auto r = rimdp::bellman_step<V>(
            mdp, std::span<const V>(v, n),
            {maximize ? rimdp::StrategyMode::Maximize : rimdp::StrategyMode::Minimize,
             pessimistic ? rimdp::SatisfactionMode::Pessimistic : rimdp::SatisfactionMode::Optimistic},
            fz, workers);
        std::copy(r.values.begin(), r.values.end(), out_v);
        std::copy(r.chosen_column.begin(), r.chosen_column.end(), out_chosen);
    });
}

template <class V>
int column_expectation(int len, const int* rows, const V* lower, const V* upper, const V* values,
                       int pessimistic, V* out, V* p_out, ref_err* err) {
    ErrOut e{err ? err->msg : nullptr, err ? 512 : 0, nullptr, nullptr,
             err ? &err->violation_kind : nullptr, nullptr};
    return guarded(e, [&] {
        rimdp::ColumnView<V> col{std::span<const index_t>(rows, len), std::span<const V>(lower, len),
                                 std::span<const V>(upper, len)};
        const std::size_t nv = len == 0 ? 0 : static_cast<std::size_t>(*std::max_element(rows, rows + len)) + 1;
        auto mode = pessimistic ? rimdp::SatisfactionMode::Pessimistic : rimdp::SatisfactionMode::Optimistic;
        *out = rimdp::robust_expectation<V>(col, std::span<const V>(values, nv), mode);
        if (p_out) {
            auto ord = rimdp::value_ordering<V>(col.rows, std::span<const V>(values, nv), mode);
            auto p = rimdp::omaximize_sequential<V>(ord, col.lower, col.upper);
            std::copy(p.begin(), p.end(), p_out);
        }
    });
}

} // namespace

extern "C" {

int ref_model_from_arrays_f64(int n, int ncols, const int* sp, const int* cp, const int* rv,
                              const double* lo, const double* up, int checked, void** out, ref_err* err) {
    return from_arrays<double>(n, ncols, sp, cp, rv, lo, up, checked, out, err);
}
int ref_model_from_arrays_f32(int n, int ncols, const int* sp, const int* cp, const int* rv,
                              const float* lo, const float* up, int checked, void** out, ref_err* err) {
    return from_arrays<float>(n, ncols, sp, cp, rv, lo, up, checked, out, err);
}
int ref_model_random_f64(int states, int actions, double density, double scale,
                         unsigned long long seed, int point, void** out, ref_err* err) {
    return random_model<double>(states, actions, density, scale, seed, point, out, err);
}
int ref_model_random_f32(int states, int actions, double density, double scale,
                         unsigned long long seed, int point, void** out, ref_err* err) {
    return random_model<float>(states, actions, density, scale, seed, point, out, err);
}
int ref_model_generate_f64(int states, int actions, int law, int support, double alpha, int kmax, double lscale,
                           double uscale, unsigned long long seed, void** out, ref_err* err) {
    return generate_model<double>(states, actions, law, support, alpha, kmax, lscale, uscale, seed, out, err);
}
int ref_model_generate_f32(int states, int actions, int law, int support, double alpha, int kmax, double lscale,
                           double uscale, unsigned long long seed, void** out, ref_err* err) {
    return generate_model<float>(states, actions, law, support, alpha, kmax, lscale, uscale, seed, out, err);
}
// Transitions of a generator workload at any size (column lengths only).
long long ref_generate_nnz(int states, int actions, int law, int support, double alpha, int kmax,
                           unsigned long long seed) {
    rimdp_gen::Params p{states, actions, law, support, kmax, 0.0, 0.0, seed};
    std::vector<uint64_t> cdf;
    if (law == 1) cdf = rimdp_gen::power_law_cdf(kmax, alpha);
    long long z = 0;
    const long long ncols = static_cast<long long>(states) * actions;
    for (long long c = 0; c < ncols; ++c) z += rimdp_gen::column_length(p, cdf.data(), c);
    return z;
}
void ref_model_free(void* h) { delete static_cast<ModelBase*>(h); }

void ref_model_sizes_f64(void* h, int* n, int* ncols, long long* nnz) {
    const auto& m = static_cast<Model<double>*>(static_cast<ModelBase*>(h))->mdp;
    *n = m.num_states();
    *ncols = m.num_cols();
    *nnz = m.num_transitions();
}
void ref_model_sizes_f32(void* h, int* n, int* ncols, long long* nnz) {
    const auto& m = static_cast<Model<float>*>(static_cast<ModelBase*>(h))->mdp;
    *n = m.num_states();
    *ncols = m.num_cols();
    *nnz = m.num_transitions();
}
void ref_model_export_f64(void* h, int* sp, int* cp, int* rv, double* lo, double* up) {
    model_export<double>(h, sp, cp, rv, lo, up);
}
void ref_model_export_f32(void* h, int* sp, int* cp, int* rv, float* lo, float* up) {
    model_export<float>(h, sp, cp, rv, lo, up);
}

int ref_write_native_f64(void* h, const char* path, int json, ref_err* err) { return write_native<double>(h, path, json, err); }
int ref_write_native_f32(void* h, const char* path, int json, ref_err* err) { return write_native<float>(h, path, json, err); }
int ref_read_native_f64(const char* path, void** out, ref_err* err) { return read_native<double>(path, out, err); }
int ref_read_native_f32(const char* path, void** out, ref_err* err) { return read_native<float>(path, out, err); }
long long ref_model_labels_f64(void* h, char* out) { return model_labels<double>(h, out); }
long long ref_model_labels_f32(void* h, char* out) { return model_labels<float>(h, out); }

int ref_solve_f64(void* h, const ref_spec* sp, int synth, double* v, double* res, long long* it,
                  int* pol, double* trace, long long cap, ref_err* err) {
    return solve<double>(h, sp, synth, v, res, it, pol, trace, cap, err);
}
int ref_solve_f32(void* h, const ref_spec* sp, int synth, float* v, float* res, long long* it,
                  int* pol, float* trace, long long cap, ref_err* err) {
    return solve<float>(h, sp, synth, v, res, it, pol, trace, cap, err);
}
int ref_verify_policy_f64(void* h, const ref_spec* sp, const int* pol, int td, long long horizon,
                          double* v, double* res, long long* it, ref_err* err) {
    return verify<double>(h, sp, pol, td, horizon, v, res, it, err);
}
int ref_verify_policy_f32(void* h, const ref_spec* sp, const int* pol, int td, long long horizon,
                          float* v, float* res, long long* it, ref_err* err) {
    return verify<float>(h, sp, pol, td, horizon, v, res, it, err);
}
int ref_bellman_step_f64(void* h, const double* v, int pess, int maxi, const unsigned char* frozen,
                         unsigned workers, double* ov, int* oc, ref_err* err) {
    return step<double>(h, v, pess, maxi, frozen, workers, ov, oc, err);
}
int ref_bellman_step_f32(void* h, const float* v, int pess, int maxi, const unsigned char* frozen,
                         unsigned workers, float* ov, int* oc, ref_err* err) {
    return step<float>(h, v, pess, maxi, frozen, workers, ov, oc, err);
}
int ref_robust_expectation_f64(int len, const int* rows, const double* lo, const double* up,
                               const double* values, int pess, double* out, double* p, ref_err* err) {
    return column_expectation<double>(len, rows, lo, up, values, pess, out, p, err);
}
int ref_robust_expectation_f32(int len, const int* rows, const float* lo, const float* up,
                               const float* values, int pess, float* out, float* p, ref_err* err) {
    return column_expectation<float>(len, rows, lo, up, values, pess, out, p, err);
}

// The reference test-suite's independent break-point LP (tests/oracle.hpp:28-80).
double ref_lp_expectation_f64(int len, const double* lo, const double* up, const double* values,
                              int minimize) {
    return oracle::robust_expectation<double>(std::vector<double>(lo, lo + len),
                                              std::vector<double>(up, up + len),
                                              std::vector<double>(values, values + len), minimize != 0);
}

// Reproduces the reference tests' random columns (tests/oracle.hpp:187-217,
// test_omax.cpp:73-208 pattern): `count` columns of size nmin + rng() % nmod,
// each followed by `len` uniform01 values.  Returns total entries written.
long long ref_test_columns_f64(unsigned long long seed, int count, int nmin, int nmod, double scale,
                               int with_values, int* lens, double* lo, double* up, double* values,
                               long long cap) {
    std::mt19937_64 rng(seed);
    std::vector<double> l, u;
    long long off = 0;
    for (int rep = 0; rep < count; ++rep) {
        const std::size_t n = static_cast<std::size_t>(nmin) + rng() % static_cast<std::uint64_t>(nmod);
        oracle::random_feasible_column<double>(rng, n, l, u, scale);
        if (off + static_cast<long long>(n) > cap) return -1;
        lens[rep] = static_cast<int>(n);
        for (std::size_t i = 0; i < n; ++i) {
            lo[off + i] = l[i];
            up[off + i] = u[i];
        }
        if (with_values)
            for (std::size_t i = 0; i < n; ++i) values[off + i] = oracle::uniform01(rng);
        off += static_cast<long long>(n);
    }
    return off;
}

} // extern "C"
