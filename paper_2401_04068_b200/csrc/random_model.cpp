// Seeded workload generator with the reference's exact law, so the engine and
// the CPU reference ingest byte-identical models for BASELINE configs 2-3.
//
// Restates random_imdp / random_point_imdp (random_model.hpp:42-161): per
// column a partial Fisher-Yates draw of ceil(density * n) destinations from a
// pool that persists across columns, sorted; lower = u * scale,
// upper = min(lower + v * (1 - scale), 1) with u, v = (rng() >> 11) * 2^-53,
// redrawn until sum(lower) <= 1 <= sum(upper) in the value type; then the
// checked from_aligned path drops [0, 0] entries (interval.hpp:261-279).
// std::mt19937_64 is fully specified by the standard, so the streams match.
#include "rimdp_b200_workloads.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

namespace {

double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

template <class V>
struct Gen {
    std::vector<int32_t> stateptr;
    std::vector<int64_t> colptr;
    std::vector<int32_t> rows;
    std::vector<V> lower, upper;
};

template <class V>
void interval_model(Gen<V>& g, int32_t n, int32_t actions, double density, double scale, uint64_t seed) {
    const int32_t support = std::clamp<int32_t>(static_cast<int32_t>(std::ceil(density * n)), 1, n);
    std::mt19937_64 rng(seed);
    std::vector<int32_t> pool(n), pick(support);
    for (int32_t i = 0; i < n; ++i) pool[i] = i;
    std::vector<V> lo(support), up(support);
    g.stateptr.assign(1, 0);
    g.colptr.assign(1, 0);
    g.rows.reserve(static_cast<size_t>(n) * actions * support);
    g.lower.reserve(g.rows.capacity());
    g.upper.reserve(g.rows.capacity());
    for (int32_t s = 0; s < n; ++s) {
        for (int32_t a = 0; a < actions; ++a) {
            for (;;) {
                for (int32_t i = 0; i < support; ++i) {
                    const int32_t j = i + static_cast<int32_t>(rng() % static_cast<uint64_t>(n - i));
                    std::swap(pool[i], pool[j]);
                    pick[i] = pool[i];
                }
                std::sort(pick.begin(), pick.end());
                V ls(0), us(0);
                for (int32_t i = 0; i < support; ++i) {
                    const double u = uniform01(rng), v = uniform01(rng);
                    const double l = u * scale;
                    double h = std::min(l + v * (1.0 - scale), 1.0);
                    if (support == 1) h = 1.0;
                    lo[i] = static_cast<V>(l);
                    up[i] = static_cast<V>(h);
                    ls += lo[i];
                    us += up[i];
                }
                if (ls <= V(1) && us >= V(1)) break;
            }
            for (int32_t i = 0; i < support; ++i) {
                if (lo[i] == V(0) && up[i] == V(0)) continue; // drop_empty_intervals
                g.rows.push_back(pick[i]);
                g.lower.push_back(lo[i]);
                g.upper.push_back(up[i]);
            }
            g.colptr.push_back(static_cast<int64_t>(g.rows.size()));
        }
        g.stateptr.push_back(static_cast<int32_t>(g.colptr.size() - 1));
    }
}

template <class V>
void point_model(Gen<V>& g, int32_t n, int32_t actions, double density, uint64_t seed) {
    const int32_t support = std::clamp<int32_t>(static_cast<int32_t>(std::ceil(density * n)), 1, n);
    std::mt19937_64 rng(seed);
    std::vector<int32_t> pool(n), pick(support);
    for (int32_t i = 0; i < n; ++i) pool[i] = i;
    g.stateptr.assign(1, 0);
    g.colptr.assign(1, 0);
    std::vector<V> w(support);
    for (int32_t s = 0; s < n; ++s) {
        for (int32_t a = 0; a < actions; ++a) {
            for (int32_t i = 0; i < support; ++i) {
                const int32_t j = i + static_cast<int32_t>(rng() % static_cast<uint64_t>(n - i));
                std::swap(pool[i], pool[j]);
                pick[i] = pool[i];
            }
            std::sort(pick.begin(), pick.end());
            V total(0);
            for (int32_t i = 0; i < support; ++i) {
                w[i] = static_cast<V>(uniform01(rng) + 1e-3);
                total += w[i];
            }
            V acc(0);
            for (int32_t i = 0; i < support; ++i) {
                V p = (i + 1 == support) ? V(V(1) - acc) : V(w[i] / total);
                if (p < V(0)) p = V(0);
                acc += p;
                if (p == V(0)) continue; // [0, 0] entries are dropped by from_aligned
                g.rows.push_back(pick[i]);
                g.lower.push_back(p);
                g.upper.push_back(p);
            }
            g.colptr.push_back(static_cast<int64_t>(g.rows.size()));
        }
        g.stateptr.push_back(static_cast<int32_t>(g.colptr.size() - 1));
    }
}

struct Holder {
    int dtype;
    Gen<double> d;
    Gen<float> f;
};

} // namespace

extern "C" {

int rimdp_random_imdp(int32_t num_states, int32_t actions, double density, double scale, uint64_t seed,
                      int32_t point, int32_t dtype, rimdp_random_sizes* sizes, void** handle) {
    if (num_states <= 0 || actions <= 0 || !sizes || !handle || !(density > 0)) return 1;
    auto* h = new Holder;
    h->dtype = dtype;
    if (dtype == 0) {
        point ? point_model(h->d, num_states, actions, density, seed)
              : interval_model(h->d, num_states, actions, density, scale, seed);
        sizes->nnz = static_cast<int64_t>(h->d.rows.size());
    } else {
        point ? point_model(h->f, num_states, actions, density, seed)
              : interval_model(h->f, num_states, actions, density, scale, seed);
        sizes->nnz = static_cast<int64_t>(h->f.rows.size());
    }
    sizes->num_states = num_states;
    sizes->num_cols = num_states * actions;
    *handle = h;
    return 0;
}

int rimdp_random_imdp_take(void* handle, int32_t* stateptr, int64_t* colptr, int32_t* rowval, void* lower,
                           void* upper) {
    auto* h = static_cast<Holder*>(handle);
    if (!h) return 1;
    auto copy = [&](auto& g, size_t es) {
        std::memcpy(stateptr, g.stateptr.data(), sizeof(int32_t) * g.stateptr.size());
        std::memcpy(colptr, g.colptr.data(), sizeof(int64_t) * g.colptr.size());
        std::memcpy(rowval, g.rows.data(), sizeof(int32_t) * g.rows.size());
        std::memcpy(lower, g.lower.data(), es * g.lower.size());
        std::memcpy(upper, g.upper.data(), es * g.upper.size());
    };
    if (h->dtype == 0)
        copy(h->d, 8);
    else
        copy(h->f, 4);
    delete h;
    return 0;
}

} // extern "C"
