// Drop-in parity: the reference's C++ entry points (rimdp::, the unmodified
// header-only CPU library under /root/reference/proj/include, compiled in as
// the checker) against the same entry points on the B200 engine
// (rimdp_b200::, include/rimdp_b200/dropin.hpp over the C ABI), on the same
// Problem objects in one process.
//
// TEST INFRASTRUCTURE: the reference code here is the oracle, never the thing
// measured.  Built by paper_2401_04068_b200/build.py (build_cpp_tests) into
// tests/cpp/_build/dropin_parity; run by tests/test_dropin_cpp.py.
//
//   dropin_parity              all parity cases (needs a CUDA device)
//   dropin_parity --no-device  checks that every entry point fails loudly
//                              (rimdp::Error) when no device is visible
//
// Cases mirror the reference's own hot-path tests (test_solver.cpp,
// test_omax.cpp): the paper model in all four modes, random models in every
// property kind, reach-avoid, rewards, policy synthesis and re-verification,
// single Bellman steps, single columns, the error paths, and native IMDPCSC1
// containers read by both readers (test_io.cpp).
#include "rimdp/io/native.hpp"
#include "rimdp/random_model.hpp"
#include "rimdp/solver.hpp"
#include "rimdp_b200/dropin.hpp"

#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <cstring>
#include <functional>
#include <random>
#include <string>

using namespace rimdp;

namespace {

int g_checks = 0, g_fail = 0;

#define EXPECT(cond, ...)                                                                    \
    do {                                                                                     \
        ++g_checks;                                                                          \
        if (!(cond)) {                                                                       \
            ++g_fail;                                                                        \
            std::fprintf(stderr, "FAIL %s:%d: %s  ", __FILE__, __LINE__, #cond);             \
            std::fprintf(stderr, __VA_ARGS__);                                               \
            std::fprintf(stderr, "\n");                                                      \
        }                                                                                    \
    } while (0)

// Parity bar per model: bit-exact where every evaluated column runs an
// exact-order kernel, else |diff| <= tol (north_star: 1e-12 per iteration,
// 1e-9 at convergence) with identical iteration counts.
template <typename Value>
bool same(const std::vector<Value>& a, const std::vector<Value>& b, double tol, double* worst = nullptr) {
    if (a.size() != b.size()) return false;
    double w = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        if (tol == 0) {
            if (std::memcmp(&a[i], &b[i], sizeof(Value)) != 0) return false;
        } else {
            w = std::max(w, std::fabs(static_cast<double>(a[i]) - static_cast<double>(b[i])));
        }
    }
    if (worst) *worst = w;
    return tol == 0 || w <= tol;
}

SolverOptions opts(std::int64_t max_iter = 1'000'000) {
    SolverOptions o;
    o.max_iterations = max_iter;
    return o;
}

Problem<double> paper_problem(Specification<double> spec) {
    // the running example of PAPER.md:116-133 (three states, sink = state 2)
    using IP = IntervalProbabilities<double>;
    auto s0 = IP::from_dense({{0.0, 0.5}, {0.1, 0.3}, {0.2, 0.1}}, {{0.5, 0.7}, {0.6, 0.5}, {0.7, 0.3}});
    auto s1 = IP::from_dense({{0.1, 0.2}, {0.2, 0.3}, {0.3, 0.4}}, {{0.6, 0.6}, {0.5, 0.5}, {0.4, 0.4}});
    auto s2 = IP::from_dense({{0.0}, {0.0}, {1.0}}, {{0.0}, {0.0}, {1.0}});
    std::vector<StateBlock<double>> blocks{{{"a1", "a2"}, s0}, {{"a1", "a2"}, s1}, {{"sink"}, s2}};
    return {build_imdp<double>(blocks), std::move(spec)};
}

const SatisfactionMode kSat[2] = {SatisfactionMode::Pessimistic, SatisfactionMode::Optimistic};
const StrategyMode kStr[2] = {StrategyMode::Maximize, StrategyMode::Minimize};

bool same_policy(const Policy& a, const Policy& b) {
    if (a.index() != b.index()) return false;
    if (const auto* s = std::get_if<StationaryPolicy>(&a)) return s->actions == std::get<StationaryPolicy>(b).actions;
    const auto& x = std::get<TimeDependentPolicy>(a);
    const auto& y = std::get<TimeDependentPolicy>(b);
    return x.num_states == y.num_states && x.horizon == y.horizon && x.actions == y.actions;
}

template <typename Value>
void compare_solve(const std::string& name, const Problem<Value>& pr, double tol, std::int64_t max_iter = 1'000'000) {
    const auto o = opts(max_iter);
    auto [rp, rv] = rimdp::control_synthesis(pr, o);
    auto [gp, gv] = rimdp_b200::control_synthesis(pr, o);
    double w = 0;
    EXPECT(rv.iterations == gv.iterations, "%s iterations ref %lld dev %lld", name.c_str(), (long long)rv.iterations,
           (long long)gv.iterations);
    EXPECT(same(rv.values, gv.values, tol, &w), "%s values (worst %.3g)", name.c_str(), w);
    EXPECT(same(rv.residual, gv.residual, tol, &w), "%s residual (worst %.3g)", name.c_str(), w);
    if (tol == 0) EXPECT(same_policy(rp, gp), "%s policy", name.c_str());
    auto vi = rimdp_b200::value_iteration(pr, o);
    EXPECT(same(vi.values, gv.values, 0), "%s value_iteration == control_synthesis", name.c_str());
    EXPECT(vi.iterations == gv.iterations, "%s iterations vi/cs", name.c_str());
    if (max_iter == 1'000'000) { // the reference's default options (solver.hpp:149-155)
        auto vd = rimdp_b200::value_iteration(pr);
        EXPECT(same(vd.values, gv.values, 0) && vd.iterations == gv.iterations, "%s default options", name.c_str());
    }
    // the sharded multi-GPU solve (SolverOptions::devices; two and three shards on device 0 here): the
    // same bits as one device, strategies included
    for (int world : {2, 3}) {
        rimdp_b200::SolverOptions mo;
        mo.max_iterations = max_iter;
        mo.devices.assign(world, 0);
        auto [mp, mv] = rimdp_b200::control_synthesis(pr, mo);
        EXPECT(mv.iterations == gv.iterations && same(mv.values, gv.values, 0) && same(mv.residual, gv.residual, 0) &&
                   same_policy(mp, gp),
               "%s sharded x%d == single device", name.c_str(), world);
    }
    // re-verify the synthesized policy (solver.hpp:204-251)
    auto rver = rimdp::verify_policy(pr.imdp, rp, pr.spec, o);
    auto gver = rimdp_b200::verify_policy(pr.imdp, rp, pr.spec, o);
    EXPECT(rver.iterations == gver.iterations, "%s verify iterations %lld %lld", name.c_str(),
           (long long)rver.iterations, (long long)gver.iterations);
    EXPECT(same(rver.values, gver.values, tol, &w), "%s verify values (worst %.3g)", name.c_str(), w);
}

template <typename E, typename F>
std::string thrown(F&& f) {
    try {
        f();
    } catch (const E& e) {
        return std::string("ok:") + e.what();
    } catch (const std::exception& e) {
        return std::string("other:") + e.what();
    }
    return "none";
}

void paper_cases() {
    for (auto sat : kSat)
        for (auto str : kStr) {
            const std::string tag = std::string("paper/") + to_string(str) + "/" + to_string(sat);
            compare_solve(tag + "/F10", paper_problem({FiniteTimeReachability{{2}, 10}, sat, str}), 0);
            compare_solve(tag + "/Finf", paper_problem({InfiniteTimeReachability{{2}, 1e-6}, sat, str}), 0);
            compare_solve(tag + "/RA", paper_problem({FiniteTimeReachAvoid{{2}, {1}, 7}, sat, str}), 0);
            compare_solve(tag + "/Rw", paper_problem({InfiniteTimeReward<double>{{1.0, 0.5, 0.0}, 0.9, 1e-8}, sat, str}),
                          0);
            // one Bellman step from [0, 0, 1] with state 2 frozen (test_omax.cpp:210-251)
            auto pr = paper_problem({FiniteTimeReachability{{2}, 1}, sat, str});
            std::vector<double> v{0.0, 0.0, 1.0};
            std::vector<std::uint8_t> fz{0, 0, 1};
            auto r = rimdp::bellman_step<double>(pr.imdp, v, {str, sat}, fz);
            auto g = rimdp_b200::bellman_step<double>(pr.imdp, v, {str, sat}, fz);
            EXPECT(same(r.values, g.values, 0), "%s step values", tag.c_str());
            EXPECT(r.chosen_column == g.chosen_column, "%s step columns", tag.c_str());
        }
}

template <typename Value>
void random_cases(const char* label, RandomModelConfig cfg, double tol) {
    auto mdp = random_imdp<Value>(cfg);
    const index_t n = mdp.num_states();
    std::vector<index_t> goal{n - 1}, avoid{0};
    std::vector<Value> rew(n);
    std::mt19937_64 rng(cfg.seed + 99);
    for (auto& x : rew) x = static_cast<Value>((rng() >> 11) * 0x1.0p-53);
    for (auto sat : kSat)
        for (auto str : kStr) {
            const std::string tag = std::string(label) + "/" + to_string(str) + "/" + to_string(sat);
            compare_solve<Value>(tag + "/F25", {mdp, {FiniteTimeReachability{goal, 25}, sat, str}}, tol);
            compare_solve<Value>(tag + "/Finf", {mdp, {InfiniteTimeReachability{goal, 1e-6}, sat, str}}, tol);
            compare_solve<Value>(tag + "/RAinf", {mdp, {InfiniteTimeReachAvoid{goal, avoid, 1e-6}, sat, str}}, tol);
            compare_solve<Value>(tag + "/RwF", {mdp, {FiniteTimeReward<Value>{rew, Value(0.9), 12}, sat, str}}, tol);
            compare_solve<Value>(tag + "/RwInf",
                                 {mdp, {InfiniteTimeReward<Value>{rew, Value(0.8), 1e-5}, sat, str}}, tol);
            // single columns through robust_expectation (omax.hpp:182-189)
            std::vector<Value> v(n);
            for (auto& x : v) x = static_cast<Value>((rng() >> 11) * 0x1.0p-53);
            for (index_t c = 0; c < std::min<index_t>(mdp.num_cols(), 3); ++c) {
                const auto col = mdp.transition().column(c);
                const Value a = rimdp::robust_expectation<Value>(col, v, sat);
                const Value b = rimdp_b200::robust_expectation<Value>(col, v, sat);
                EXPECT(tol == 0 ? std::memcmp(&a, &b, sizeof a) == 0 : std::fabs(double(a) - double(b)) <= tol,
                       "%s column %d: %.17g vs %.17g", tag.c_str(), c, double(a), double(b));
            }
        }
}

void error_cases() {
    // infeasible column: lower bounds sum to 1.2 (test_omax.cpp:54-62)
    auto tp = IntervalProbabilities<double>::from_aligned_unchecked(2, 2, {0, 2, 3}, {0, 1, 1}, {0.6, 0.6, 1.0},
                                                                    {0.7, 0.7, 1.0});
    auto bad = IntervalMDP<double>::from_parts_unchecked(tp, {0, 1, 2}, {"a", "b"});
    Problem<double> pr{bad, {FiniteTimeReachability{{1}, 3}, SatisfactionMode::Pessimistic, StrategyMode::Maximize}};
    const auto r = thrown<ModelError>([&] { rimdp::value_iteration(pr, opts()); });
    const auto g = thrown<ModelError>([&] { rimdp_b200::value_iteration(pr, opts()); });
    EXPECT(r == g && r.rfind("ok:", 0) == 0, "infeasible: ref '%s' dev '%s'", r.c_str(), g.c_str());
    // upper bounds below 1
    auto tp2 = IntervalProbabilities<double>::from_aligned_unchecked(2, 2, {0, 2, 3}, {0, 1, 1}, {0.1, 0.1, 1.0},
                                                                     {0.3, 0.25, 1.0});
    auto bad2 = IntervalMDP<double>::from_parts_unchecked(tp2, {0, 1, 2}, {"a", "b"});
    Problem<double> pr2{bad2, {FiniteTimeReachability{{1}, 3}, SatisfactionMode::Optimistic, StrategyMode::Minimize}};
    const auto r2 = thrown<ModelError>([&] { rimdp::value_iteration(pr2, opts()); });
    const auto g2 = thrown<ModelError>([&] { rimdp_b200::value_iteration(pr2, opts()); });
    EXPECT(r2 == g2 && r2.rfind("ok:", 0) == 0, "infeasible upper: ref '%s' dev '%s'", r2.c_str(), g2.c_str());
    // NonConvergence at the cap (solver.hpp:131-133)
    auto slow = paper_problem({InfiniteTimeReachability{{2}, 1e-14}, SatisfactionMode::Pessimistic,
                               StrategyMode::Maximize});
    std::int64_t ri = -1, gi = -2;
    std::string rm, gm;
    try {
        rimdp::value_iteration(slow, opts(7));
    } catch (const NonConvergence& e) {
        ri = e.iterations();
        rm = e.what();
    }
    try {
        rimdp_b200::value_iteration(slow, opts(7));
    } catch (const NonConvergence& e) {
        gi = e.iterations();
        gm = e.what();
    }
    EXPECT(ri == gi && rm == gm, "non-convergence: ref %lld '%s' dev %lld '%s'", (long long)ri, rm.c_str(),
           (long long)gi, gm.c_str());
    // property validation (property.hpp:132-180)
    auto oob = paper_problem({FiniteTimeReachability{{7}, 3}, SatisfactionMode::Pessimistic, StrategyMode::Maximize});
    EXPECT(thrown<PropertyStateOutOfRange>([&] { rimdp::value_iteration(oob, opts()); }) ==
               thrown<PropertyStateOutOfRange>([&] { rimdp_b200::value_iteration(oob, opts()); }),
           "state out of range");
    auto ov = paper_problem({FiniteTimeReachAvoid{{2}, {2}, 3}, SatisfactionMode::Pessimistic, StrategyMode::Maximize});
    EXPECT(thrown<InvalidProperty>([&] { rimdp::value_iteration(ov, opts()); }) ==
               thrown<InvalidProperty>([&] { rimdp_b200::value_iteration(ov, opts()); }),
           "overlapping reach/avoid");
    // policy resolution (solver.hpp:211-248)
    auto pp = paper_problem({FiniteTimeReachability{{2}, 3}, SatisfactionMode::Pessimistic, StrategyMode::Maximize});
    Policy badpol = StationaryPolicy{{"a1", "zz", "sink"}};
    EXPECT(thrown<InvalidPolicyAction>([&] { rimdp::verify_policy(pp.imdp, badpol, pp.spec, opts()); }) ==
               thrown<InvalidPolicyAction>([&] { rimdp_b200::verify_policy(pp.imdp, badpol, pp.spec, opts()); }),
           "invalid policy label");
    auto inf = paper_problem({InfiniteTimeReachability{{2}, 1e-6}, SatisfactionMode::Pessimistic,
                              StrategyMode::Maximize});
    TimeDependentPolicy td;
    td.num_states = 3;
    td.horizon = 2;
    td.actions = {"a1", "a1", "a2", "a2", "sink", "sink"};
    EXPECT(thrown<InvalidPolicyAction>([&] { rimdp::verify_policy(inf.imdp, Policy(td), inf.spec, opts()); }) ==
               thrown<InvalidPolicyAction>([&] { rimdp_b200::verify_policy(inf.imdp, Policy(td), inf.spec, opts()); }),
           "time-dependent policy vs infinite property");
    // per-iteration callback (solver.hpp:119-125)
    std::vector<std::vector<double>> rt, gt;
    auto o1 = opts(), o2 = opts();
    o1.on_iteration_f64 = [&](std::int64_t, std::span<const double> v) { rt.emplace_back(v.begin(), v.end()); };
    o2.on_iteration_f64 = [&](std::int64_t, std::span<const double> v) { gt.emplace_back(v.begin(), v.end()); };
    auto trp = paper_problem({FiniteTimeReachability{{2}, 12}, SatisfactionMode::Optimistic, StrategyMode::Maximize});
    rimdp::value_iteration(trp, o1);
    rimdp_b200::value_iteration(trp, o2);
    EXPECT(rt == gt && rt.size() == 12, "on_iteration_f64 trajectory");
}

int no_device() {
    auto pr = paper_problem({FiniteTimeReachability{{2}, 3}, SatisfactionMode::Pessimistic, StrategyMode::Maximize});
    const std::string g = thrown<rimdp::Error>([&] { rimdp_b200::value_iteration(pr, opts()); });
    std::printf("no-device: %s\n", g.c_str());
    return g.find("no CUDA device") != std::string::npos ? 0 : 1;
}

// io::read_native_model against rimdp_b200::io::read_native_model on the same
// container files: identical models (IntervalMDP::operator==), identical
// exception types and messages.  Host-only: runs with or without a device.
template <typename Value>
void native_case(const char* label, const IntervalMDP<Value>& mdp) {
    const std::string path = std::string("/tmp/dropin_native_") + label + ".imdpcsc";
    io::write_native_model(path, mdp);
    const auto a = io::read_native_model<Value>(path);
    const auto b = rimdp_b200::io::read_native_model<Value>(path);
    EXPECT(a == b, "%s: models differ", label);
    EXPECT(b == mdp, "%s: round trip differs", label);
    // truncated container: the same SchemaViolation text
    {
        std::ifstream in(path, std::ios::binary);
        std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        out.write(bytes.data(), static_cast<std::streamsize>(bytes.size() / 2));
    }
    std::string ea, eb;
    try { io::read_native_model<Value>(path); } catch (const SchemaViolation& e) { ea = e.what(); }
    try { rimdp_b200::io::read_native_model<Value>(path); } catch (const SchemaViolation& e) { eb = e.what(); }
    EXPECT(!ea.empty() && ea == eb, "%s: truncated: '%s' vs '%s'", label, ea.c_str(), eb.c_str());
    std::remove(path.c_str());
    ea.clear();
    eb.clear();
    try { io::read_native_model<Value>(path); } catch (const MissingFile& e) { ea = e.what(); }
    try { rimdp_b200::io::read_native_model<Value>(path); } catch (const MissingFile& e) { eb = e.what(); }
    EXPECT(!ea.empty() && ea == eb, "%s: missing: '%s' vs '%s'", label, ea.c_str(), eb.c_str());
}

void native_cases() {
    native_case<double>("r200x4", random_imdp<double>({200, 4, 24.0 / 200, 1.0 / 24, 8}));
    native_case<float>("f32r60", random_imdp<float>({60, 3, 0.2, 1.0 / 12, 9}));
}

} // namespace

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--no-device") == 0) {
        native_cases(); // host-only reader
        if (g_fail) return 1;
        return no_device();
    }
    native_cases();
    paper_cases();
    error_cases();
    // short columns only (warp kernel, exact order): bit-exact
    random_cases<double>("r40x3", {40, 3, 0.2, 0.2, 3}, 0);
    random_cases<double>("r200x4k24", {200, 4, 24.0 / 200, 1.0 / 24, 8}, 0);
    random_cases<float>("f32r60", {60, 3, 0.2, 1.0 / 12, 9}, 0);
    // long columns (> 32 entries): tolerance bar
    random_cases<double>("r150dense", {150, 2, 1.0, 1.0 / 150, 6}, 1e-12);
    random_cases<double>("r300k90", {300, 3, 0.3, 1.0 / 90, 5}, 1e-12);
    std::printf("dropin_parity: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
