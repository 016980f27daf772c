// sm_100a kernels of the robust Bellman operator.
//
// Reference semantics (proj/include/rimdp/, all f64/f32 paths):
//   per column   omax_remainder (omax.hpp:64-85)  — precomputed once per model
//                value_ordering (omax.hpp:41-58) / column_value (bellman.hpp:60-70)
//                omaximize_sequential (omax.hpp:98-112)
//                row-order dot (omax.hpp:169-173)
//   per state    bellman_step_impl (bellman.hpp:75-118)
//   per iterate  reward update, residual, stop test (solver.hpp:107-134)
//
// Arithmetic order:
//   * every kernel makes the reference's greedy decisions exactly: the
//     adversary ordering is found by exact integer argmin over
//     (order-preserving key of V[row], position) — position order is row
//     order because rows are strictly increasing (csc.hpp:98-101) — and
//     `consumed` is accumulated sequentially along that ordering up to the
//     cut;
//   * the row-order kernels (omax_tiny, omax_short, omax_medium, omax_long,
//     action_reduce, bellman_short) also sum the expectation sequentially in
//     row order with separate round-to-nearest mul/add, so their results
//     are bit-identical to the reference;
//   * the single-pass / selection kernels (omax_long_tree, omax_wbucket,
//     omax_bucket, omax_select, omax_sorted) sum the expectation — and the
//     last four the gaps below the cut — in tree order (the paper's parallel
//     form): within a few ulps (north_star: 1e-12 per iteration).  The
//     scheduler routes float32 models to the row-order kernels only (see
//     engine.cu column_class), where a few ulps exceed the stop tolerance.
#pragma once

#include "numeric.cuh"

#include <climits>
#include <cstdint>
#include <cstring>
#include <type_traits>

namespace rimdp_dev {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kShortLen = 32;        // columns with <= 32 entries: one lane per entry
constexpr int kShortBatch = 16;      // columns per warp batch in the short kernel
constexpr int kWarpsPerBlock = 8;
constexpr int kMaxPartial = 4;       // partially-filled positions tracked per long column
#ifndef RIMDP_SHORT_BLOCKS_PER_SM
#define RIMDP_SHORT_BLOCKS_PER_SM 4
#endif
constexpr int kShortBlocksPerSm = RIMDP_SHORT_BLOCKS_PER_SM; // resident blocks of bellman_short

// Device loop state of one solve.
struct Ctl {
    unsigned long long res_bits[2]; // max residual of iteration k, slot k & 1
    unsigned int arrive;            // blocks of the action kernel that finished
    int done;                       // stop condition reached; later launches are no-ops
    int status;                     // 0 ok, 1 non-convergence, 2 internal
    unsigned int arrive_stop;       // blocks of the sharded stop test that finished
    long long k;                    // iterations completed
    double res_last;                // max residual of the last iteration, as double
    int class_early;                // many-kernel iterations: class kernels start before their predecessor ends
};

// Start of a column-class kernel.  Normally (pdl_enter) it waits for its
// predecessor grid, then lets its successor launch.  In iterations of many
// class kernels (C5: a dozen) the classes are independent of each other — they
// read V_{k-1} and write disjoint q entries — so with ctl->class_early the
// kernel lets its successor launch at once and only thread 0 of block 0 waits
// for the predecessor: the next class's blocks take over SMs as this one's
// blocks retire (no drain bubble between class kernels), and a grid still
// cannot complete before its predecessor, so the action kernel (full wait)
// sees every class finished.  The iteration's first class kernel follows a
// plain-launched gate (value_range or pdl_gate), which orders it after the
// previous iteration.  Kernels that read a predecessor's output (selection /
// exact_dot / fallback passes, action_reduce) keep the full wait.
__device__ __forceinline__ void pdl_enter_class(const Ctl* ctl) {
    if (ctl && ctl->class_early) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    } else {
        pdl_enter();
    }
}

__global__ void pdl_gate() {}

// ---------------------------------------------------------------------------
// Model preparation: per-column remainder and feasibility (omax.hpp:64-85),
// and gap = upper - lower in place of upper.  Sequential in row order, so the
// sums carry the reference's rounding.
// One warp per column: coalesced 32-entry chunks; gap = upper - lower and
// the largest gap are elementwise / order-free, while the two running sums
// are kept sequential in row order by lanes 0 (lower) and 1 (gap) reading the
// chunk back from shared memory.
template <class T>
__global__ void __launch_bounds__(256)
prepare_columns(int ncols, const long long* __restrict__ colptr, const T* __restrict__ lower,
                T* __restrict__ upper_to_gap, T* __restrict__ rem, unsigned char* __restrict__ infeasible,
                T* __restrict__ quoted_sum, T* __restrict__ maxgap, int* __restrict__ n_infeasible) {
    using N = Num<T>;
    __shared__ T st[8][2][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = blockIdx.x * 8 + w; c < ncols; c += gridDim.x * 8) {
        const long long b = colptr[c], e = colptr[c + 1];
        T run = T(0), mg = T(0); // lane 0: sum of lower, lane 1: sum of gaps
        for (long long j0 = b; j0 < e; j0 += 32) {
            const long long j = j0 + lane;
            T l = T(0), g = T(0);
            if (j < e) {
                l = lower[j];
                g = N::sub(upper_to_gap[j], l);
                upper_to_gap[j] = g;
                mg = g > mg ? g : mg;
            }
            st[w][0][lane] = l;
            st[w][1][lane] = g;
            __syncwarp();
            if (lane < 2) {
                const int m = static_cast<int>(e - j0 < 32 ? e - j0 : 32);
                for (int i = 0; i < m; ++i) run = N::add(run, st[w][lane][i]);
            }
            __syncwarp();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T x = __shfl_xor_sync(0xffffffffu, mg, o);
            mg = x > mg ? x : mg;
        }
        const T ls = __shfl_sync(0xffffffffu, run, 0), gs = __shfl_sync(0xffffffffu, run, 1);
        if (lane == 0) {
            maxgap[c] = mg;
            unsigned char bad = 0;
            T qs = T(0);
            if (ls > N::add(T(1), N::tol())) {
                bad = 1;
                qs = ls;
            } else if (N::add(ls, gs) < N::sub(T(1), N::tol())) {
                bad = 2;
                qs = N::add(ls, gs);
            }
            T r = N::sub(T(1), ls);
            if (r < T(0)) r = T(0);
            if (r > gs) r = gs;
            rem[c] = r;
            infeasible[c] = bad;
            quoted_sum[c] = qs;
            if (bad) atomicAdd(n_infeasible, 1);
        }
    }
}

// Device-side model validation at upload, in the
// reference's report order: CscMatrix::structural_violation (csc.hpp:89-104:
// per column, per entry: row in range, then strictly increasing rows) over
// every column first, then IntervalProbabilities::validate's entry checks
// (interval.hpp:148-164: per entry lower in [0,1] and finite, upper likewise,
// lower <= upper).  One warp per column; the first violation of the model is
// the minimum of (column, entry, check) keys, folded with atomicMin:
//   first[0] structural: column << 32 | entry << 1 | (0 range, 1 order)
//   first[1] entries:    column << 32 | entry << 2 | (0 lower, 1 upper, 2 order)
// Runs before prepare_columns turns `upper` into gaps.
template <class T>
__global__ void __launch_bounds__(256)
validate_entries(int ncols, const long long* __restrict__ colptr, const int* __restrict__ rows,
                 const T* __restrict__ lower, const T* __restrict__ upper, int n, unsigned long long* __restrict__ first) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = blockIdx.x * 8 + w; c < ncols; c += gridDim.x * 8) {
        const long long b = colptr[c], e = colptr[c + 1];
        unsigned long long sk = ~0ull, ek = ~0ull;
        int prev = 0;
        for (long long j0 = b; j0 < e; j0 += 32) {
            const long long j = j0 + lane;
            const bool in = j < e;
            const int r = in ? rows[j] : 0;
            int before = __shfl_up_sync(kFull, r, 1);
            if (lane == 0) before = prev;
            prev = __shfl_sync(kFull, r, 31);
            if (in) {
                const unsigned long long pos = static_cast<unsigned long long>(j - b);
                if (r < 0 || r >= n) sk = min(sk, (pos << 1) | 0ull);
                else if (j > b && r <= before) sk = min(sk, (pos << 1) | 1ull);
                const T l = lower[j], u = upper[j];
                // !(0 <= x <= 1) is true for NaN; +-inf fail the range test too (Traits::is_finite)
                if (!(l >= T(0) && l <= T(1))) ek = min(ek, (pos << 2) | 0ull);
                else if (!(u >= T(0) && u <= T(1))) ek = min(ek, (pos << 2) | 1ull);
                else if (l > u) ek = min(ek, (pos << 2) | 2ull); // the first check the reference pushes
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            sk = min(sk, __shfl_xor_sync(kFull, sk, o));
            ek = min(ek, __shfl_xor_sync(kFull, ek, o));
        }
        if (lane == 0) {
            if (sk != ~0ull) atomicMin(first, (static_cast<unsigned long long>(c) << 32) | sk);
            if (ek != ~0ull) atomicMin(first + 1, (static_cast<unsigned long long>(c) << 32) | ek);
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-wide exact argmin helpers.

// Lane holding the smallest (key, lane) among lanes with `active`, or -1.
template <class Bits>
__device__ __forceinline__ int warp_argmin_lane(Bits key, bool active) {
    if (__ballot_sync(kFull, active) == 0u) return -1;
    bool cand = active;
    if constexpr (sizeof(Bits) == 8) {
        const unsigned hi = static_cast<unsigned>(key >> 32);
        const unsigned mhi = __reduce_min_sync(kFull, active ? hi : 0xffffffffu);
        cand = cand && hi == mhi;
        const unsigned lo = static_cast<unsigned>(key);
        const unsigned mlo = __reduce_min_sync(kFull, cand ? lo : 0xffffffffu);
        cand = cand && lo == mlo;
    } else {
        const unsigned mk = __reduce_min_sync(kFull, active ? static_cast<unsigned>(key) : 0xffffffffu);
        cand = cand && static_cast<unsigned>(key) == mk;
    }
    return __ffs(__ballot_sync(kFull, cand)) - 1;
}

// Smallest (key, pos) over lanes with `active`; returns false when none.
template <class Bits>
__device__ __forceinline__ bool warp_argmin_pos(Bits key, int pos, bool active, Bits& kout, int& pout) {
    if (__ballot_sync(kFull, active) == 0u) return false;
    bool cand = active;
    Bits k;
    if constexpr (sizeof(Bits) == 8) {
        const unsigned hi = static_cast<unsigned>(key >> 32);
        const unsigned mhi = __reduce_min_sync(kFull, active ? hi : 0xffffffffu);
        cand = cand && hi == mhi;
        const unsigned lo = static_cast<unsigned>(key);
        const unsigned mlo = __reduce_min_sync(kFull, cand ? lo : 0xffffffffu);
        cand = cand && lo == mlo;
        k = (static_cast<Bits>(mhi) << 32) | mlo;
    } else {
        const unsigned mk = __reduce_min_sync(kFull, active ? static_cast<unsigned>(key) : 0xffffffffu);
        cand = cand && static_cast<unsigned>(key) == mk;
        k = mk;
    }
    pout = static_cast<int>(__reduce_min_sync(kFull, cand ? static_cast<unsigned>(pos) : 0xffffffffu));
    kout = k;
    return true;
}

// ---------------------------------------------------------------------------
// Short columns (<= 32 entries).
//
// A warp walks a stream of columns in batches of 16 (the first batch per
// warp static, the rest handed out by an atomic work counter).  For each column, lane i owns entry i: coalesced loads of
// (row, lower, gap), one V gather, and the greedy assignment driven by exact
// warp argmins — one per position that receives extra mass (1-3 on typical
// models).  Products V[row_i] * p_i are staged in shared memory; at the end
// of a batch lane t sums column t's products sequentially in row order.
//
// Latency: the row -> V gather is a dependent pair of memory round trips, so
// the kernel is software-pipelined three deep — while column i is reduced,
// (lower, gap, V[row]) of column i+1 and the rows of column i+2 are in
// flight.  Column metadata (start, length, rem) lives in a 32-lane window:
// lanes 0-15 hold the current batch, lanes 16-31 the next one, prefetched a
// whole batch ahead.
template <class T>
__device__ __forceinline__ typename Num<T>::Bits order_key(T v, bool pess) {
    using Bits = typename Num<T>::Bits;
    using SBits = typename std::conditional<sizeof(T) == 8, long long, int>::type;
    constexpr Bits kMsb = Bits(1) << (8 * sizeof(Bits) - 1);
    Bits b;
    const T z = Num<T>::add(v, T(0)); // -0 -> +0: the reference orders with != (ties by row)
    memcpy(&b, &z, sizeof b);
    const Bits s = static_cast<Bits>(static_cast<SBits>(b) >> (8 * sizeof(Bits) - 1));
    return pess ? (b ^ (s | kMsb)) : (b ^ (~s & ~kMsb));
}

// Lane with the smallest (key, lane); inactive lanes carry the all-ones key.
// The high word usually decides alone (one lane holds the minimum high
// word): then the second redux is skipped (warp-uniform branch).
template <class Bits>
__device__ __forceinline__ int warp_argmin_sentinel(Bits key) {
    if constexpr (sizeof(Bits) == 8) {
        const unsigned hi = static_cast<unsigned>(key >> 32), lo = static_cast<unsigned>(key);
        const unsigned mhi = __reduce_min_sync(kFull, hi);
        const unsigned wh = __ballot_sync(kFull, hi == mhi);
        if ((wh & (wh - 1u)) == 0u) return __ffs(wh) - 1;
        const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
        return __ffs(__ballot_sync(kFull, hi == mhi && lo == mlo)) - 1;
    } else {
        const unsigned mk = __reduce_min_sync(kFull, static_cast<unsigned>(key));
        return __ffs(__ballot_sync(kFull, static_cast<unsigned>(key) == mk)) - 1;
    }
}

template <class T, bool kPess>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 5)
omax_short(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
           const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
           const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl,
           unsigned* __restrict__ work) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    // +2: 16-byte aligned rows for the paired loads of the row-order sums, still spread over the banks
    __shared__ __align__(16) T xs[kWarpsPerBlock][kShortBatch][kShortLen + 2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerBlock + w, nw = gridDim.x * kWarpsPerBlock;
    // batches: the first one static, the rest handed out by a work counter
    auto next_batch = [&]() -> int {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(work, 1u);
        return nw + static_cast<int>(__shfl_sync(kFull, t, 0));
    };
    int base = gw * kShortBatch;
    if (base >= nlist) return;
    int nbase = next_batch() * kShortBatch;

    // metadata window: lane j describes column j of [current batch | next batch]
    int mc = -1, mlen = 0;
    long long mbeg = 0;
    T mrem = T(0);
    auto load_meta = [&](int batch_base) {
        const int idx = batch_base + (lane & (kShortBatch - 1));
        mc = -1;
        mlen = 0;
        mbeg = 0;
        mrem = T(0);
        if (batch_base < nlist && idx < nlist) {
            mc = __ldg(list + idx);
            mbeg = __ldg(colptr + mc);
            mlen = static_cast<int>(__ldg(colptr + mc + 1) - mbeg);
            mrem = __ldg(rem + mc);
        }
    };
    load_meta(lane < kShortBatch ? base : nbase);

    // pipeline prologue: data of column 0, rows of column 1
    long long bn = __shfl_sync(kFull, mbeg, 0), bnn = __shfl_sync(kFull, mbeg, 1);
    int Ln = __shfl_sync(kFull, mlen, 0), Lnn = __shfl_sync(kFull, mlen, 1);
    int rowA = lane < Ln ? __ldg(rows + bn + lane) : 0;
    T lc = T(0), gc = T(0), vc = T(0);
    int Lc = Ln;
    if (lane < Ln) {
        lc = __ldg(lower + bn + lane);
        gc = __ldg(gap + bn + lane);
        vc = __ldg(V + rowA);
    }
    bn = bnn;
    Ln = Lnn;
    rowA = lane < Ln ? __ldg(rows + bn + lane) : 0;
    bnn = __shfl_sync(kFull, mbeg, 2);
    Lnn = __shfl_sync(kFull, mlen, 2);

    for (;;) {
        for (int s = 0; s < kShortBatch; ++s) {
            // stage D: (lower, gap, V[row]) of column i+1
            T ln = T(0), gn = T(0), vn = T(0);
            if (lane < Ln) {
                ln = __ldg(lower + bn + lane);
                gn = __ldg(gap + bn + lane);
                vn = __ldg(V + rowA);
            }
            // stage R: rows of column i+2
            const int rowB = lane < Lnn ? __ldg(rows + bnn + lane) : 0;
            // stage C: the greedy O-max of column i (omax.hpp:98-112)
            const T r = __shfl_sync(kFull, mrem, s);
            const bool valid = lane < Lc;
            Bits key = valid ? order_key<T>(vc, kPess) : ~Bits(0);
            T consumed = T(0);
            T avail = r;
            T mine = T(-1); // the avail at this lane's pick (picks only happen with avail > 0)
            for (int nsel = 0; avail > T(0) && nsel < Lc; ++nsel) {
                const int sel = warp_argmin_sentinel(key);
                const T gs = __shfl_sync(kFull, gc, sel);
                {   // branch-free winner update; the winner's share is formed once, after the loop
                    const bool me = lane == sel;
                    mine = me ? avail : mine;
                    key = me ? ~Bits(0) : key;
                }
                consumed = N::add(consumed, gs);
                avail = N::sub(r, consumed);
            }
            // omax.hpp:107: p = lower + (gap < avail ? gap : avail) for a picked position, lower otherwise
            const T p = mine > T(0) ? N::add(lc, gc < mine ? gc : mine) : lc;
            if (valid) xs[w][s][lane] = N::mul(vc, p);
            // rotate the pipeline; metadata of column i+3 = window lane s+3
            lc = ln;
            gc = gn;
            vc = vn;
            Lc = Ln;
            rowA = rowB;
            bn = bnn;
            Ln = Lnn;
            bnn = __shfl_sync(kFull, mbeg, s + 3);
            Lnn = __shfl_sync(kFull, mlen, s + 3);
        }
        // row-order expectation of the batch's columns (omax.hpp:169-173)
        __syncwarp();
        if (lane < kShortBatch && mc >= 0) {
            T acc = T(0);
            int i = 0;
            if constexpr (sizeof(T) == 8) {
                const double2* x2 = reinterpret_cast<const double2*>(xs[w][lane]);
                for (; i + 2 <= mlen; i += 2) {
                    const double2 y = x2[i >> 1];
                    acc = N::add(acc, y.x);
                    acc = N::add(acc, y.y);
                }
            }
            for (; i < mlen; ++i) acc = N::add(acc, xs[w][lane][i]);
            q[mc] = acc;
        }
        __syncwarp();
        base = nbase;
        if (base >= nlist) break;
        nbase = next_batch() * kShortBatch;
        // shift the window and prefetch the batch after next
        const int c2 = __shfl_down_sync(kFull, mc, kShortBatch);
        const long long b2 = __shfl_down_sync(kFull, mbeg, kShortBatch);
        const int l2 = __shfl_down_sync(kFull, mlen, kShortBatch);
        const T r2 = __shfl_down_sync(kFull, mrem, kShortBatch);
        if (lane < kShortBatch) {
            mc = c2;
            mbeg = b2;
            mlen = l2;
            mrem = r2;
        } else {
            load_meta(nbase);
        }
    }
}

// ---------------------------------------------------------------------------
// Short columns (17 .. 32 entries), two per warp step (omax_pair): lanes
// 0-15 take column A, lanes 16-31 column B, lane l of a half owning the two
// consecutive entries 2l, 2l+1 — one 128-bit load per array (`double2`
// lower / gap, `int2` rows) when the column starts on an even entry.  The two
// greedy loops (omax.hpp:98-112) run side by side: each pick step is one
// half-masked exact argmin per column over (order key, position) and one
// shuffle of the winners' gaps, so the per-pick and per-column instructions
// (reductions, metadata shuffles, loop control) serve two columns.  Products
// are staged in shared memory and lane t sums column t in row order
// (omax.hpp:169-173), as in omax_short: bit-exact.  Same three-deep
// pipeline as omax_short, one pair per stage.
template <class T, bool kPess>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 4)
omax_pair(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
          const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
          const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl,
          unsigned* __restrict__ work) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    constexpr int P = kShortBatch / 2; // pairs per batch
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    __shared__ __align__(16) T xs[kWarpsPerBlock][kShortBatch][kShortLen + 2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int h = lane >> 4, j0 = 2 * (lane & 15);
    const unsigned half = h ? 0xffff0000u : 0x0000ffffu;
    const unsigned long long pstream = l2_evict_first_policy();
    const int gw = blockIdx.x * kWarpsPerBlock + w, nw = gridDim.x * kWarpsPerBlock;
    auto next_batch = [&]() -> int {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(work, 1u);
        return nw + static_cast<int>(__shfl_sync(kFull, t, 0));
    };
    int base = gw * kShortBatch;
    if (base >= nlist) return;
    int nbase = next_batch() * kShortBatch;

    // metadata window: lane j describes column j of [current batch | next batch]
    int mc = -1, mlen = 0;
    long long mbeg = 0;
    T mrem = T(0);
    auto load_meta = [&](int batch_base) {
        const int idx = batch_base + (lane & (kShortBatch - 1));
        mc = -1;
        mlen = 0;
        mbeg = 0;
        mrem = T(0);
        if (batch_base < nlist && idx < nlist) {
            mc = __ldg(list + idx);
            mbeg = __ldg(colptr + mc);
            mlen = static_cast<int>(__ldg(colptr + mc + 1) - mbeg);
            mrem = __ldg(rem + mc);
        }
    };
    load_meta(lane < kShortBatch ? base : nbase);
    auto gather = [&](const int (&rw)[2], int L, T (&v)[2]) {
#pragma unroll
        for (int e = 0; e < 2; ++e) v[e] = j0 + e < L ? __ldg(V + rw[e]) : T(0);
    };

    // pipeline prologue: data of pair 0, rows of pair 1 (this lane's column of each)
    long long bn = __shfl_sync(kFull, mbeg, h), bnn = __shfl_sync(kFull, mbeg, 2 + h);
    int Ln = __shfl_sync(kFull, mlen, h), Lnn = __shfl_sync(kFull, mlen, 2 + h);
    int rowA[2], rowB[2];
    T lc[2], gc[2], vc[2], ln[2], gn[2], vn[2];
    ld_run<2>(rows + bn, j0, Ln, (bn & 1) == 0, pstream, rowA);
    ld_run<2>(lower + bn, j0, Ln, (bn & 1) == 0, pstream, lc);
    ld_run<2>(gap + bn, j0, Ln, (bn & 1) == 0, pstream, gc);
    gather(rowA, Ln, vc);
    int Lc = Ln;
    bn = bnn;
    Ln = Lnn;
    ld_run<2>(rows + bn, j0, Ln, (bn & 1) == 0, pstream, rowA);
    bnn = __shfl_sync(kFull, mbeg, 4 + h);
    Lnn = __shfl_sync(kFull, mlen, 4 + h);

    for (;;) {
        for (int s = 0; s < P; ++s) {
            // stage D: (lower, gap, V[row]) of pair i+1; stage R: rows of pair i+2
            ld_run<2>(lower + bn, j0, Ln, (bn & 1) == 0, pstream, ln);
            ld_run<2>(gap + bn, j0, Ln, (bn & 1) == 0, pstream, gn);
            gather(rowA, Ln, vn);
            ld_run<2>(rows + bnn, j0, Lnn, (bnn & 1) == 0, pstream, rowB);
            // stage C: the two greedy O-maxes of pair i
            const T r = __shfl_sync(kFull, mrem, 2 * s + h);
            Bits key[2];
            T pa[2]; // avail at this entry's pick, -1 if not picked (picks only happen with avail > 0)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                key[e] = j0 + e < Lc ? order_key<T>(vc[e], kPess) : ~Bits(0);
                pa[e] = T(-1);
            }
            T consumed = T(0), avail = r;
            for (int nsel = 0;; ++nsel) {
                const bool act = avail > T(0) && nsel < Lc;
                if (!__any_sync(kFull, act)) break;
                const bool second = key[1] < key[0]; // ties keep the lower position
                const Bits bk = second ? key[1] : key[0];
                bool cand;
                unsigned wb;
                if constexpr (sizeof(Bits) == 8) {
                    const unsigned hi = act ? static_cast<unsigned>(bk >> 32) : 0xffffffffu;
                    const unsigned m0 = __reduce_min_sync(kFull, h == 0 ? hi : 0xffffffffu);
                    const unsigned m1 = __reduce_min_sync(kFull, h == 1 ? hi : 0xffffffffu);
                    cand = act && hi == (h ? m1 : m0);
                    wb = __ballot_sync(kFull, cand);
                    const unsigned a = wb & 0xffffu, b = wb >> 16;
                    if ((a & (a - 1u)) | (b & (b - 1u))) { // a half with several equal high words
                        const unsigned lo = cand ? static_cast<unsigned>(bk) : 0xffffffffu;
                        const unsigned l0 = __reduce_min_sync(kFull, h == 0 ? lo : 0xffffffffu);
                        const unsigned l1 = __reduce_min_sync(kFull, h == 1 ? lo : 0xffffffffu);
                        cand = cand && lo == (h ? l1 : l0);
                        wb = __ballot_sync(kFull, cand);
                    }
                } else {
                    const unsigned k = act ? static_cast<unsigned>(bk) : 0xffffffffu;
                    const unsigned m0 = __reduce_min_sync(kFull, h == 0 ? k : 0xffffffffu);
                    const unsigned m1 = __reduce_min_sync(kFull, h == 1 ? k : 0xffffffffu);
                    cand = act && k == (h ? m1 : m0);
                    wb = __ballot_sync(kFull, cand);
                }
                // lowest lane of the half among equal keys = lowest position (rows ascending, csc.hpp:98-101)
                const unsigned mine = wb & half;
                const int sel = mine ? __ffs(mine) - 1 : lane;
                const T gs = __shfl_sync(kFull, second ? gc[1] : gc[0], sel);
                if (act) {
                    if (lane == sel) {
                        if (second) {
                            pa[1] = avail;
                            key[1] = ~Bits(0);
                        } else {
                            pa[0] = avail;
                            key[0] = ~Bits(0);
                        }
                    }
                    consumed = N::add(consumed, gs);
                    avail = N::sub(r, consumed);
                }
            }
            {   // omax.hpp:107: p = lower + (gap < avail ? gap : avail) for a picked position, lower otherwise
                T x[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const T p = pa[e] > T(0) ? N::add(lc[e], gc[e] < pa[e] ? gc[e] : pa[e]) : lc[e];
                    x[e] = N::mul(vc[e], p);
                }
                if constexpr (sizeof(T) == 8) {
                    *reinterpret_cast<double2*>(&xs[w][2 * s + h][j0]) = make_double2(x[0], x[1]);
                } else {
                    xs[w][2 * s + h][j0] = x[0];
                    xs[w][2 * s + h][j0 + 1] = x[1];
                }
            }
            // rotate the pipeline; metadata of pair i+3 = window lanes 2(s+3), 2(s+3)+1
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                lc[e] = ln[e];
                gc[e] = gn[e];
                vc[e] = vn[e];
                rowA[e] = rowB[e];
            }
            Lc = Ln;
            bn = bnn;
            Ln = Lnn;
            bnn = __shfl_sync(kFull, mbeg, (2 * (s + 3) + h) & 31);
            Lnn = __shfl_sync(kFull, mlen, (2 * (s + 3) + h) & 31);
        }
        // row-order expectation of the batch's columns (omax.hpp:169-173)
        __syncwarp();
        if (lane < kShortBatch && mc >= 0) {
            T acc = T(0);
            int i = 0;
            if constexpr (sizeof(T) == 8) {
                const double2* x2 = reinterpret_cast<const double2*>(xs[w][lane]);
                for (; i + 2 <= mlen; i += 2) {
                    const double2 y = x2[i >> 1];
                    acc = N::add(acc, y.x);
                    acc = N::add(acc, y.y);
                }
            }
            for (; i < mlen; ++i) acc = N::add(acc, xs[w][lane][i]);
            q[mc] = acc;
        }
        __syncwarp();
        base = nbase;
        if (base >= nlist) break;
        nbase = next_batch() * kShortBatch;
        // shift the window and prefetch the batch after next
        const int c2 = __shfl_down_sync(kFull, mc, kShortBatch);
        const long long b2 = __shfl_down_sync(kFull, mbeg, kShortBatch);
        const int l2 = __shfl_down_sync(kFull, mlen, kShortBatch);
        const T r2 = __shfl_down_sync(kFull, mrem, kShortBatch);
        if (lane < kShortBatch) {
            mc = c2;
            mbeg = b2;
            mlen = l2;
            mrem = r2;
        } else {
            load_meta(nbase);
        }
    }
}

// ---------------------------------------------------------------------------
// Tiny columns (<= SEG entries, SEG = 4, 8 or 16): 32 / SEG columns per warp
// step, one SEG-lane segment per column (power-law models are dominated by
// columns of 1-4 entries, which would leave most of omax_short's lanes
// idle).  Segment reductions use redux/shfl/ballot with the segment's lane
// mask, so the segments' greedy loops (omax.hpp:98-112) run independently;
// the expectation is summed sequentially in row order by shuffling the
// segment's products to its first lane (omax.hpp:169-173): bit-exact.
// Two-stage pipeline: the next step's metadata and rows are in flight while
// the current step is reduced.
// kPacked: the class's columns were copied into item-ordered packed arrays at
// upload (pack_columns): `colptr` / `rem` / the entry arrays are indexed by
// list position, `list` only maps a position to its column for the q write.
// Power-law models have millions of 1-16-entry columns scattered through the
// store; packed, a warp step reads one contiguous run instead of a few
// partially used sectors per column.
template <class T, bool kPess, int SEG, bool kPacked = false>
__global__ void __launch_bounds__(256)
omax_tiny(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
          const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
          const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    constexpr int CPW = 32 / SEG;
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    const int lane = threadIdx.x & 31, sg = lane / SEG, sl = lane % SEG;
    const unsigned segmask = (SEG == 32 ? kFull : ((1u << SEG) - 1u)) << (sg * SEG);
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int nsteps = (nlist + CPW - 1) / CPW;
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    int step = gw;
    if (step >= nsteps) return;
    auto meta = [&](int st, int& c, long long& b, int& L, T& r) {
        const int idx = st * CPW + sg;
        c = -1;
        b = 0;
        L = 0;
        r = T(0);
        if (st < nsteps && idx < nlist) {
            c = __ldg(list + idx);
            const int ci = kPacked ? idx : c;
            b = __ldg(colptr + ci);
            L = static_cast<int>(__ldg(colptr + ci + 1) - b);
            r = __ldg(rem + ci);
        }
    };
    int c, L;
    long long b;
    T r;
    meta(step, c, b, L, r);
    int row = sl < L ? ld_hint(rows + b + sl, pstream) : 0;
    for (;;) {
        T l = T(0), g = T(0), v = T(0);
        if (sl < L) {
            l = ld_hint(lower + b + sl, pstream);
            g = ld_hint(gap + b + sl, pstream);
            v = ld_hint(V + row, pval);
        }
        const int nstep = step + nw;
        int c2, L2;
        long long b2;
        T r2;
        meta(nstep, c2, b2, L2, r2);
        const int row2 = sl < L2 ? ld_hint(rows + b2 + sl, pstream) : 0;
        // greedy of this segment's column.  The loop is warp-uniform (segments
        // that are done idle through it) and every collective uses the full
        // mask: per-segment masks in divergent code serialise per segment.
        Bits key = sl < L ? order_key<T>(v, kPess) : ~Bits(0);
        T p = l, consumed = T(0), avail = r;
        int nsel = 0;
        for (;;) {
            const bool active = avail > T(0) && nsel < L;
            if (!__any_sync(kFull, active)) break;
            // segment minimum of the key: xor butterfly inside the segment
            Bits mk = key;
#pragma unroll
            for (int o = SEG / 2; o > 0; o >>= 1) {
                const Bits y = __shfl_xor_sync(kFull, mk, o);
                mk = y < mk ? y : mk;
            }
            const int sel = __ffs(__ballot_sync(kFull, key == mk) & segmask) - 1; // lowest lane = lowest position
            const T gs = __shfl_sync(kFull, g, sel < 0 ? lane : sel);
            if (active) {
                if (lane == sel) {
                    p = N::add(l, g < avail ? g : avail);
                    key = ~Bits(0);
                }
                consumed = N::add(consumed, gs);
                avail = N::sub(r, consumed);
                ++nsel;
            }
        }
        const T x = sl < L ? N::mul(v, p) : T(0);
        const int maxL = __reduce_max_sync(kFull, static_cast<unsigned>(L));
        T acc = T(0);
        for (int i = 0; i < maxL; ++i) {
            const T y = __shfl_sync(kFull, x, sg * SEG + (i < SEG ? i : 0));
            if (i < L) acc = N::add(acc, y);
        }
        if (sl == 0 && c >= 0) q[c] = acc;
        step = nstep;
        if (step >= nsteps) break;
        c = c2;
        b = b2;
        L = L2;
        r = r2;
        row = row2;
    }
}

// omax_tiny by ranks instead of repeated argmins.  Each lane counts its
// entry's rank in its segment's (key, position) order (SEG independent
// shuffles, no dependent chain), scatters its gap to that slot of the warp's
// shared-memory row, and then every lane replays the reference's `consumed`
// chain (omax.hpp:102-110) over the sorted gaps up to the end of the column,
// taking avail at its own rank:
//   avail_k = r - (g_(0) + ... + g_(k-1))   (sequential, as the reference)
//   p       = avail_k > 0 ? l + min(g, avail_k) : l
// avail is non-increasing along the chain (g >= 0), so "avail_k > 0" is the
// reference's loop condition at step k.  The row-order dot is the segment
// leader's sequential sum over the products staged in the same row.  Same
// arithmetic as omax_tiny, so the same bits; about a third of its
// instructions for columns with several picks.
template <class T, bool kPess, int SEG, bool kPacked = false>
__global__ void __launch_bounds__(256)
omax_tiny_rank(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
               const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
               const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    constexpr int CPW = 32 / SEG;
    __shared__ __align__(16) T rowbuf[8][32];
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    const int lane = threadIdx.x & 31, sg = lane / SEG, sl = lane % SEG;
    T* sb = rowbuf[threadIdx.x >> 5] + sg * SEG;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const int nsteps = (nlist + CPW - 1) / CPW;
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    int step = gw;
    if (step >= nsteps) return;
    auto meta = [&](int st, int& c, long long& b, int& L, T& r) {
        const int idx = st * CPW + sg;
        c = -1;
        b = 0;
        L = 0;
        r = T(0);
        if (st < nsteps && idx < nlist) {
            c = __ldg(list + idx);
            const int ci = kPacked ? idx : c;
            b = __ldg(colptr + ci);
            L = static_cast<int>(__ldg(colptr + ci + 1) - b);
            r = __ldg(rem + ci);
        }
    };
    int c, L;
    long long b;
    T r;
    meta(step, c, b, L, r);
    int row = sl < L ? ld_hint(rows + b + sl, pstream) : 0;
    for (;;) {
        T l = T(0), g = T(0), v = T(0);
        if (sl < L) {
            l = ld_hint(lower + b + sl, pstream);
            g = ld_hint(gap + b + sl, pstream);
            v = ld_hint(V + row, pval);
        }
        const int nstep = step + nw;
        int c2, L2;
        long long b2;
        T r2;
        meta(nstep, c2, b2, L2, r2);
        const int row2 = sl < L2 ? ld_hint(rows + b2 + sl, pstream) : 0;
        // rank of the entry in the segment's (key, position) order
        const Bits key = sl < L ? order_key<T>(v, kPess) : ~Bits(0);
        int rank = 0;
#pragma unroll
        for (int j = 0; j < SEG; ++j) {
            const Bits kj = __shfl_sync(kFull, key, sg * SEG + j);
            rank += (kj < key) | ((kj == key) & (j < sl));
        }
        if (sl < L) sb[rank] = g;
        __syncwarp();
        // the greedy's `consumed` chain over the sorted gaps; p at this lane's rank
        T consumed = T(0), p = l;
#pragma unroll
        for (int k = 0; k < SEG; ++k) {
            if (k < L) {
                const T a = N::sub(r, consumed);
                if (k == rank && a > T(0)) p = N::add(l, g < a ? g : a);
                consumed = N::add(consumed, sb[k]);
            }
        }
        __syncwarp();
        sb[sl] = sl < L ? N::mul(v, p) : T(0);
        __syncwarp();
        if (sl == 0 && c >= 0) {
            T acc = T(0);
#pragma unroll
            for (int i = 0; i < SEG; ++i)
                if (i < L) acc = N::add(acc, sb[i]);
            q[c] = acc;
        }
        __syncwarp();
        step = nstep;
        if (step >= nsteps) break;
        c = c2;
        b = b2;
        L = L2;
        r = r2;
        row = row2;
    }
}

// Copies the columns of a class list into item-ordered packed arrays (see
// omax_tiny's kPacked).  One thread per column (tiny columns: <= 16 entries).
template <class T>
__global__ void __launch_bounds__(256)
pack_columns(int n, const int* __restrict__ list, const long long* __restrict__ colptr, const long long* __restrict__ pk_beg,
             const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
             const T* __restrict__ rem, int* __restrict__ pk_rows, T* __restrict__ pk_lower, T* __restrict__ pk_gap,
             T* __restrict__ pk_rem) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int c = list[i];
        const long long b = colptr[c], e = colptr[c + 1], o = pk_beg[i];
        for (long long k = b; k < e; ++k) {
            pk_rows[o + (k - b)] = rows[k];
            pk_lower[o + (k - b)] = lower[k];
            pk_gap[o + (k - b)] = gap[k];
        }
        pk_rem[i] = rem[c];
    }
}

// ---------------------------------------------------------------------------
// Medium columns (33 .. 32*E entries, few greedy picks): omax_short widened
// to E entries per lane.  Lane i owns positions i, 32 + i, ..., 32(E-1) + i,
// so every load is still one coalesced 128/256-byte segment per e.  A warp
// walks batches of B columns (metadata window: lanes [0, B) the current
// batch, [B, 2B) the next), with the same three-deep pipeline: the rows of
// column i+2 and (lower, gap, V[row]) of column i+1 are in flight while
// column i is reduced.  Each greedy pick is an exact warp argmin of
// (key, position): every lane first takes the minimum of its own E entries
// (its positions increase with e, so the first minimum wins ties), then the
// warp reduces the key words and the position.  Products are staged in
// shared memory and lane t < B sums column t in row order, so the result is
// bit-identical to the reference (omax.hpp:98-112, 169-173).
template <int E>
struct MediumShape {
    static constexpr int B = E == 2 ? 8 : 4;       // columns per batch
    static constexpr int W = 8;                    // warps per block
    static constexpr int Len = 32 * E;
};

template <class T, bool kPess, int E, int kMinBlocks = 1>
__global__ void __launch_bounds__(MediumShape<E>::W * 32, kMinBlocks)
omax_medium(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
            const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
            const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl,
            unsigned* __restrict__ work) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    using Sh = MediumShape<E>;
    constexpr int B = Sh::B, W = Sh::W, LEN = Sh::Len;
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    // +2: rows stay 16-byte aligned for the vector product stores and lane t's sequential reads of row t
    // still spread over the banks
    __shared__ __align__(16) T xs[W][B][LEN + 2];
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gw = blockIdx.x * W + w, nw = gridDim.x * W;
    auto next_batch = [&]() -> int {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(work, 1u);
        return nw + static_cast<int>(__shfl_sync(kFull, t, 0));
    };
    int base = gw * B;
    if (base >= nlist) return;
    int nbase = next_batch() * B;

    int mc = -1, mlen = 0;
    long long mbeg = 0;
    T mrem = T(0);
    auto load_meta = [&](int batch_base) {
        const int idx = batch_base + (lane & (B - 1));
        mc = -1;
        mlen = 0;
        mbeg = 0;
        mrem = T(0);
        if (lane < 2 * B && idx < nlist) {
            mc = __ldg(list + idx);
            mbeg = __ldg(colptr + mc);
            mlen = static_cast<int>(__ldg(colptr + mc + 1) - mbeg);
            mrem = __ldg(rem + mc);
        }
    };
    load_meta(lane < B ? base : nbase);

    long long bn = __shfl_sync(kFull, mbeg, 0), bnn = __shfl_sync(kFull, mbeg, 1);
    int Ln = __shfl_sync(kFull, mlen, 0), Lnn = __shfl_sync(kFull, mlen, 1);
    // lane l owns the E consecutive entries [l E, l E + E) of a column: one 64/128-bit load per array when
    // the column starts on an E-entry boundary (config 4: always)
    const int j0 = lane * E;
    int rowA[E], rowB[E];
    T lc[E], gc[E], vc[E], ln[E], gn[E], vn[E];
    ld_run<E>(rows + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, rowA);
    ld_run<E>(lower + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, lc);
    ld_run<E>(gap + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, gc);
#pragma unroll
    for (int e = 0; e < E; ++e) vc[e] = j0 + e < Ln ? ld_hint(V + rowA[e], pval) : T(0);
    int Lc = Ln;
    bn = bnn;
    Ln = Lnn;
    ld_run<E>(rows + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, rowA);
    bnn = __shfl_sync(kFull, mbeg, 2);
    Lnn = __shfl_sync(kFull, mlen, 2);

    for (;;) {
        for (int s = 0; s < B; ++s) {
            ld_run<E>(lower + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, ln);
            ld_run<E>(gap + bn, j0, Ln, (bn & (E - 1)) == 0, pstream, gn);
#pragma unroll
            for (int e = 0; e < E; ++e) vn[e] = j0 + e < Ln ? ld_hint(V + rowA[e], pval) : T(0);
            ld_run<E>(rows + bnn, j0, Lnn, (bnn & (E - 1)) == 0, pstream, rowB);
            // greedy O-max of column s (omax.hpp:98-112)
            const T r = __shfl_sync(kFull, mrem, s);
            Bits key[E];
            T pick_avail[E]; // avail at this entry's pick, -1 if not picked (picks only happen with avail > 0)
#pragma unroll
            for (int e = 0; e < E; ++e) {
                key[e] = j0 + e < Lc ? order_key<T>(vc[e], kPess) : ~Bits(0);
                pick_avail[e] = T(-1);
            }
            T consumed = T(0), avail = r;
            for (int nsel = 0; avail > T(0) && nsel < Lc; ++nsel) {
                // lane-local (key, e) minimum, then the warp-wide one
                Bits bk = key[0];
                int be = 0;
#pragma unroll
                for (int e = 1; e < E; ++e)
                    if (key[e] < bk) {
                        bk = key[e];
                        be = e;
                    }
                bool cand = true;
                unsigned single = 0u; // a lane whose high key word is the unique minimum decides alone
                if constexpr (sizeof(Bits) == 8) {
                    const unsigned hi = static_cast<unsigned>(bk >> 32), lo = static_cast<unsigned>(bk);
                    const unsigned mhi = __reduce_min_sync(kFull, hi);
                    cand = hi == mhi;
                    const unsigned wh = __ballot_sync(kFull, cand);
                    if ((wh & (wh - 1u)) == 0u) {
                        single = wh;
                    } else {
                        const unsigned mlo = __reduce_min_sync(kFull, cand ? lo : 0xffffffffu);
                        cand = cand && lo == mlo;
                    }
                } else {
                    const unsigned mk = __reduce_min_sync(kFull, static_cast<unsigned>(bk));
                    cand = static_cast<unsigned>(bk) == mk;
                }
                // ties of the key go to the lowest position = row (csc.hpp:98-101); a lane's own entries are
                // in position order, so its (key, e) minimum already prefers the lower e on ties
                int sel_lane, sel_e;
                if (single) {
                    sel_lane = __ffs(single) - 1;
                    sel_e = __shfl_sync(kFull, be, sel_lane);
                } else {
                    const unsigned pos = __reduce_min_sync(kFull, cand ? static_cast<unsigned>(j0 + be) : 0xffffffffu);
                    sel_lane = static_cast<int>(pos / E);
                    sel_e = static_cast<int>(pos % E);
                }
                T mine = gc[0];
#pragma unroll
                for (int e = 1; e < E; ++e)
                    if (e == sel_e) mine = gc[e];
                const T gs = __shfl_sync(kFull, mine, sel_lane);
                if (lane == sel_lane) {
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        if (e == sel_e) {
                            pick_avail[e] = avail;
                            key[e] = ~Bits(0);
                        }
                }
                consumed = N::add(consumed, gs);
                avail = N::sub(r, consumed);
            }
            {
                T x[E];
#pragma unroll
                for (int e = 0; e < E; ++e) { // omax.hpp:107; entries past the column are never read
                    const T a = pick_avail[e];
                    const T p = a > T(0) ? N::add(lc[e], gc[e] < a ? gc[e] : a) : lc[e];
                    x[e] = N::mul(vc[e], p);
                }
                if constexpr (E == 2 && sizeof(T) == 8) {
                    *reinterpret_cast<double2*>(&xs[w][s][j0]) = make_double2(x[0], x[1]);
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) xs[w][s][j0 + e] = x[e];
                }
            }
            // rotate the pipeline
#pragma unroll
            for (int e = 0; e < E; ++e) {
                lc[e] = ln[e];
                gc[e] = gn[e];
                vc[e] = vn[e];
                rowA[e] = rowB[e];
            }
            Lc = Ln;
            bn = bnn;
            Ln = Lnn;
            bnn = __shfl_sync(kFull, mbeg, s + 3);
            Lnn = __shfl_sync(kFull, mlen, s + 3);
        }
        __syncwarp();
        if (lane < B && mc >= 0) {
            T acc = T(0);
            int i = 0;
            if constexpr (sizeof(T) == 8) {
                const double2* x2 = reinterpret_cast<const double2*>(xs[w][lane]);
                for (; i + 2 <= mlen; i += 2) {
                    const double2 y = x2[i >> 1];
                    acc = N::add(acc, y.x);
                    acc = N::add(acc, y.y);
                }
            }
            for (; i < mlen; ++i) acc = N::add(acc, xs[w][lane][i]);
            q[mc] = acc;
        }
        __syncwarp();
        base = nbase;
        if (base >= nlist) break;
        nbase = next_batch() * B;
        const int c2 = __shfl_down_sync(kFull, mc, B);
        const long long b2 = __shfl_down_sync(kFull, mbeg, B);
        const int l2 = __shfl_down_sync(kFull, mlen, B);
        const T r2 = __shfl_down_sync(kFull, mrem, B);
        if (lane < B) {
            mc = c2;
            mbeg = b2;
            mlen = l2;
            mrem = r2;
        } else {
            load_meta(nbase);
        }
    }
}

// ---------------------------------------------------------------------------
// Long columns (> 32 entries) with few greedy picks.  One warp per group of
// kLongGroup columns.
//
// Phase A, one column at a time — scan: one coalesced pass over the column
// (rows, V[row]; four 32-entry chunks in flight per lane) in which every
// lane keeps its kLongTopK smallest (order key, position, gap) in a register
// list.  Greedy: each pick is an exact warp argmin over the lanes' list
// heads; the winner pops its head.  The lists hold every position the greedy
// can reach before some lane runs dry — if one does while it still owns
// unseen positions, the greedy continues with full rescans: a warp argmin
// over the entries strictly after the previous pick.  Only positions whose
// assignment is clipped by the remaining mass (g >= avail) need their value
// remembered; every other picked position receives lower + gap.  The result
// (last pick, clipped positions) goes to shared memory.
//
// Phase B, the group's columns interleaved: chunk by chunk (32 entries of
// each column), the warp forms the products V[row] * p in shared memory and
// lane j adds column j's 32 products to its running sum — sequentially in
// row order, so bit-exact (omax.hpp:169-173), with the group's sums advancing
// in parallel instead of one lane summing one column.
constexpr int kLongTopK = 2;
constexpr int kLongGroup = 4;

template <class T>
struct LongCut {
    typename Num<T>::Bits lastk;
    int lastp;   // -1: nothing picked
    int npart;
    int ppos[kMaxPartial];
    T pval[kMaxPartial];
};

// kVs: the whole value vector (nv entries) is staged in shared memory once
// per block and gathered from there (small models, e.g. config 3's 2000
// states), instead of from L1/L2 where the column stream keeps evicting it.
constexpr int kLongVsMaxBytes = 64 * 1024;

template <class T, bool kPess, bool kVs>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
omax_long(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
          const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
          const T* __restrict__ rem, const T* __restrict__ Vg, int nv, T* __restrict__ q, Ctl* __restrict__ ctl) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    constexpr int K = kLongTopK, U = 4, G = kLongGroup;
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    constexpr int UB = 2; // phase B: chunks per round
    __shared__ T xs[kWarpsPerBlock][G][32 * UB + 1];
    __shared__ LongCut<T> cuts[kWarpsPerBlock][G];
    extern __shared__ __align__(16) unsigned char vs_raw[];
    const T* __restrict__ V = Vg;
    if constexpr (kVs) {
        T* vs = reinterpret_cast<T*>(vs_raw);
        for (int i = threadIdx.x; i < nv; i += blockDim.x) vs[i] = __ldg(Vg + i);
        __syncthreads();
        V = vs;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerBlock + w, nw = gridDim.x * kWarpsPerBlock;
    for (int base = gw * G; base < nlist; base += nw * G) {
        // lane j < G describes column j of the group
        int mc = -1, mlen = 0;
        long long mbeg = 0;
        T mrem = T(0);
        if (lane < G && base + lane < nlist) {
            mc = __ldg(list + base + lane);
            mbeg = __ldg(colptr + mc);
            mlen = static_cast<int>(__ldg(colptr + mc + 1) - mbeg);
            mrem = __ldg(rem + mc);
        }
        const int ng = min(G, nlist - base);
        // ---- phase A: greedy of each column ----
        for (int jc = 0; jc < ng; ++jc) {
            const long long b = __shfl_sync(kFull, mbeg, jc);
            const int L = __shfl_sync(kFull, mlen, jc);
            const T r = __shfl_sync(kFull, mrem, jc);
            Bits hk[K];
            int hp[K];
            T hg[K];
#pragma unroll
            for (int t = 0; t < K; ++t) {
                hk[t] = ~Bits(0);
                hp[t] = INT_MAX;
                hg[t] = T(0);
            }
            int seen = 0;
            for (int j0 = 0; j0 < L; j0 += 32 * U) {
                int rw[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + u * 32 + lane;
                    rw[u] = j < L ? __ldg(rows + b + j) : 0;
                }
                T vv[U], gg[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + u * 32 + lane;
                    vv[u] = j < L ? V[rw[u]] : T(0);
                    gg[u] = j < L ? __ldg(gap + b + j) : T(0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int j = j0 + u * 32 + lane;
                    if (j < L) {
                        ++seen;
                        const Bits k = N::key(vv[u], kPess);
                        // positions of a lane increase, so an equal key ranks after: strict <
                        if (k < hk[K - 1]) {
                            Bits ck = k;
                            int cp = j;
                            T cg = gg[u];
#pragma unroll
                            for (int t = 0; t < K; ++t) {
                                // a displaced entry can tie the next one: order by (key, pos)
                                if (ck < hk[t] || (ck == hk[t] && cp < hp[t])) {
                                    const Bits tk = hk[t];
                                    const int tp = hp[t];
                                    const T tg = hg[t];
                                    hk[t] = ck;
                                    hp[t] = cp;
                                    hg[t] = cg;
                                    ck = tk;
                                    cp = tp;
                                    cg = tg;
                                }
                            }
                        }
                    }
                }
            }
            // greedy along the adversary ordering (omax.hpp:98-112)
            bool any = false;
            Bits lastk = 0;
            int lastp = -1;
            int npart = 0;
            int ppos[kMaxPartial];
            T pval[kMaxPartial];
            T consumed = T(0);
            int popped = 0;
            bool dry = false; // some lane emptied its list while owning unseen positions
            for (;;) {
                const T avail = N::sub(r, consumed);
                if (!(avail > T(0))) break;
                if (__any_sync(kFull, dry)) break;
                Bits mk;
                int mp;
                if (!warp_argmin_pos(hk[0], hp[0], hp[0] != INT_MAX, mk, mp)) break; // every position picked
                const bool mine = hp[0] == mp;
                const T g = __shfl_sync(kFull, hg[0], __ffs(__ballot_sync(kFull, mine)) - 1);
                if (mine) {
#pragma unroll
                    for (int t = 0; t < K - 1; ++t) {
                        hk[t] = hk[t + 1];
                        hp[t] = hp[t + 1];
                        hg[t] = hg[t + 1];
                    }
                    hk[K - 1] = ~Bits(0);
                    hp[K - 1] = INT_MAX;
                    ++popped;
                    dry = hp[0] == INT_MAX && seen > popped;
                }
                if (!(g < avail)) {
                    if (npart < kMaxPartial) {
                        ppos[npart] = mp;
                        pval[npart] = N::add(__ldg(lower + b + mp), avail);
                    }
                    ++npart;
                }
                consumed = N::add(consumed, g);
                any = true;
                lastk = mk;
                lastp = mp;
            }
            // continuation with full rescans once a lane's list ran dry
            if (__any_sync(kFull, dry)) {
                for (;;) {
                    const T avail = N::sub(r, consumed);
                    if (!(avail > T(0))) break;
                    Bits bk = ~Bits(0);
                    int bp = INT_MAX;
                    bool have = false;
                    for (int j = lane; j < L; j += 32) {
                        const Bits k = N::key(V[__ldg(rows + b + j)], kPess);
                        const bool after = !any || k > lastk || (k == lastk && j > lastp);
                        if (after && (!have || k < bk || (k == bk && j < bp))) {
                            bk = k;
                            bp = j;
                            have = true;
                        }
                    }
                    Bits mk;
                    int mp;
                    if (!warp_argmin_pos(bk, bp, have, mk, mp)) break;
                    const T g = __ldg(gap + b + mp);
                    if (!(g < avail)) {
                        if (npart < kMaxPartial) {
                            ppos[npart] = mp;
                            pval[npart] = N::add(__ldg(lower + b + mp), avail);
                        }
                        ++npart;
                    }
                    consumed = N::add(consumed, g);
                    any = true;
                    lastk = mk;
                    lastp = mp;
                }
            }
            if (npart > kMaxPartial && lane == 0 && ctl) atomicExch(&ctl->status, 2);
            if (lane == 0) {
                LongCut<T>& cu = cuts[w][jc];
                cu.lastk = lastk;
                cu.lastp = any ? lastp : -1;
                cu.npart = npart < kMaxPartial ? npart : kMaxPartial;
                for (int t = 0; t < kMaxPartial; ++t) {
                    cu.ppos[t] = t < npart ? ppos[t] : -1;
                    cu.pval[t] = t < npart ? pval[t] : T(0);
                }
            }
        }
        __syncwarp();
        // ---- phase B: row-order expectations of the group, chunk by chunk ----
        const int maxL = __reduce_max_sync(kFull, static_cast<unsigned>(mlen));
        T acc = T(0);
        for (int j0 = 0; j0 < maxL; j0 += 32 * UB) {
            // loads of G x UB chunks in flight: rows first, then (V, lower) of each
            int rw[G][UB];
            T lw[G][UB];
#pragma unroll
            for (int jc = 0; jc < G; ++jc) {
                const long long b = __shfl_sync(kFull, mbeg, jc);
                const int L = __shfl_sync(kFull, mlen, jc);
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int j = j0 + u * 32 + lane;
                    const bool ok = jc < ng && j < L;
                    rw[jc][u] = ok ? __ldg(rows + b + j) : 0;
                    lw[jc][u] = ok ? __ldg(lower + b + j) : T(0);
                }
            }
#pragma unroll
            for (int jc = 0; jc < G; ++jc) {
                const long long b = __shfl_sync(kFull, mbeg, jc);
                const int L = __shfl_sync(kFull, mlen, jc);
                const LongCut<T>& cu = cuts[w][jc];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int j = j0 + u * 32 + lane;
                    if (jc < ng && j < L) {
                        const T v = V[rw[jc][u]];
                        const T l = lw[jc][u];
                        T p = l;
                        if (cu.lastp >= 0) {
                            const Bits k = N::key(v, kPess);
                            if (k < cu.lastk || (k == cu.lastk && j <= cu.lastp)) {
                                p = N::add(l, __ldg(gap + b + j));
                                for (int t = 0; t < cu.npart; ++t)
                                    if (cu.ppos[t] == j) p = cu.pval[t];
                            }
                        }
                        xs[w][jc][u * 32 + lane] = N::mul(v, p);
                    }
                }
            }
            __syncwarp();
            if (lane < ng) {
                const int m = min(32 * UB, mlen - j0);
                for (int t = 0; t < m; ++t) acc = N::add(acc, xs[w][lane][t]);
            }
            __syncwarp();
        }
        if (lane < ng) q[mc] = acc;
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// Long columns with few greedy picks, single pass (the default for class-1
// columns; RIMDP_LONG=exact keeps the bit-exact omax_long above).
//
// One warp per column, one coalesced pass over (row, lower, gap) with U
// chunks of 32 entries in flight per lane.  During the pass every lane keeps
// its running sum of V[row] * lower (its own positions, in row order) and its
// kLongTopK smallest (order key, position, gap); the greedy then pops the
// lanes' list heads with exact warp argmins (omax.hpp:98-112), as omax_long's
// phase A, and adds V_j * min(g_j, avail) for each pick — V_j is recovered
// exactly from the order key.  A lane that runs dry while owning unseen
// positions switches the warp to full rescans (rows and gaps only).
//   q = sum_lanes(sum V l) + sum_picks V_j min(g_j, avail_j)
// So the column data crosses HBM exactly once (omax_long reads rows and
// lower twice to sum the products in row order).  The sum is in lane/tree
// order instead of the reference's row order: within a few ulps (north_star:
// 1e-12 per iteration), deterministic.  The picks, hence the cut, are exact.
template <class T, bool kPess, bool kVs>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
omax_long_tree(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
               const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
               const T* __restrict__ rem, const T* __restrict__ Vg, int nv, T* __restrict__ q,
               const Ctl* __restrict__ ctl) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    constexpr int K = kLongTopK, U = 4;
    pdl_enter_class(ctl);
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    extern __shared__ __align__(16) unsigned char vs_raw[];
    const T* __restrict__ V = Vg;
    if constexpr (kVs) {
        T* vs = reinterpret_cast<T*>(vs_raw);
        for (int i = threadIdx.x; i < nv; i += blockDim.x) vs[i] = __ldg(Vg + i);
        __syncthreads();
        V = vs;
    }
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerBlock + w, nw = gridDim.x * kWarpsPerBlock;
    for (int item = gw; item < nlist; item += nw) {
        const int c = __ldg(list + item);
        const long long b = __ldg(colptr + c);
        const int L = static_cast<int>(__ldg(colptr + c + 1) - b);
        const T r = __ldg(rem + c);
        Bits hk[K];
        int hp[K];
        T hg[K];
#pragma unroll
        for (int t = 0; t < K; ++t) {
            hk[t] = ~Bits(0);
            hp[t] = INT_MAX;
            hg[t] = T(0);
        }
        int seen = 0;
        T acc = T(0);
        for (int j0 = 0; j0 < L; j0 += 32 * U) {
            int rw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * 32 + lane;
                rw[u] = j < L ? ld_hint(rows + b + j, pstream) : 0;
            }
            T ll[U], gg[U], vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * 32 + lane;
                ll[u] = j < L ? ld_hint(lower + b + j, pstream) : T(0);
                gg[u] = j < L ? ld_hint(gap + b + j, pstream) : T(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * 32 + lane;
                if constexpr (kVs) vv[u] = j < L ? V[rw[u]] : T(0);
                else vv[u] = j < L ? ld_hint(V + rw[u], pval) : T(0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + u * 32 + lane;
                if (j < L) {
                    ++seen;
                    acc = N::add(acc, N::mul(vv[u], ll[u]));
                    const Bits k = N::key(vv[u], kPess);
                    if (k < hk[K - 1]) {
                        Bits ck = k;
                        int cp = j;
                        T cg = gg[u];
#pragma unroll
                        for (int t = 0; t < K; ++t) {
                            if (ck < hk[t] || (ck == hk[t] && cp < hp[t])) {
                                const Bits tk = hk[t];
                                const int tp = hp[t];
                                const T tg = hg[t];
                                hk[t] = ck;
                                hp[t] = cp;
                                hg[t] = cg;
                                ck = tk;
                                cp = tp;
                                cg = tg;
                            }
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = N::add(acc, __shfl_xor_sync(kFull, acc, o));
        // greedy along the adversary ordering (omax.hpp:98-112)
        T extra = T(0), consumed = T(0);
        bool any = false;
        Bits lastk = 0;
        int lastp = -1, popped = 0;
        bool dry = false;
        for (;;) {
            const T avail = N::sub(r, consumed);
            if (!(avail > T(0))) break;
            if (__any_sync(kFull, dry)) break;
            Bits mk;
            int mp;
            if (!warp_argmin_pos(hk[0], hp[0], hp[0] != INT_MAX, mk, mp)) break;
            const bool mine = hp[0] == mp;
            const T g = __shfl_sync(kFull, hg[0], __ffs(__ballot_sync(kFull, mine)) - 1);
            if (mine) {
#pragma unroll
                for (int t = 0; t < K - 1; ++t) {
                    hk[t] = hk[t + 1];
                    hp[t] = hp[t + 1];
                    hg[t] = hg[t + 1];
                }
                hk[K - 1] = ~Bits(0);
                hp[K - 1] = INT_MAX;
                ++popped;
                dry = hp[0] == INT_MAX && seen > popped;
            }
            extra = N::add(extra, N::mul(N::value(mk, kPess), g < avail ? g : avail));
            consumed = N::add(consumed, g);
            any = true;
            lastk = mk;
            lastp = mp;
        }
        if (__any_sync(kFull, dry)) {
            for (;;) {
                const T avail = N::sub(r, consumed);
                if (!(avail > T(0))) break;
                Bits bk = ~Bits(0);
                int bp = INT_MAX;
                bool have = false;
                for (int j = lane; j < L; j += 32) {
                    const Bits k = N::key(V[__ldg(rows + b + j)], kPess);
                    const bool after = !any || k > lastk || (k == lastk && j > lastp);
                    if (after && (!have || k < bk || (k == bk && j < bp))) {
                        bk = k;
                        bp = j;
                        have = true;
                    }
                }
                Bits mk;
                int mp;
                if (!warp_argmin_pos(bk, bp, have, mk, mp)) break;
                const T g = __ldg(gap + b + mp);
                extra = N::add(extra, N::mul(N::value(mk, kPess), g < avail ? g : avail));
                consumed = N::add(consumed, g);
                any = true;
                lastk = mk;
                lastp = mp;
            }
        }
        if (lane == 0) q[c] = N::add(acc, extra);
    }
}

// ---------------------------------------------------------------------------
// Sorted long columns (33 .. 8192 entries, many picks): one CTA per column.
//
// The column's support is sorted by the adversary ordering with a bitonic
// network in shared memory, then the greedy assignment is evaluated in the
// paper's cumsum form (omaximize_prefix, omax.hpp:118-138):
// with E_j the sum of the gaps before sorted position j, position j receives
// lower + min(gap, rem - E_j) when rem - E_j > 0 and lower otherwise.  E_j
// comes from a block-wide prefix scan and the expectation from a block-wide
// reduction, so every position is independent — the north_star's warp-shuffle
// scan design.  Sums are in tree order rather than the reference's
// sequential order: results agree within a few ulps (tests bound them by
// 1e-12), deterministically.
//
// Sort key: (order key of V[row] with its low log2(N) bits dropped) | pos, a
// unique u64 whose order is the reference's (V, row) order except among
// entries whose keys differ only in the dropped bits; those runs are detected
// after the sort and re-sorted exactly by the full (key, pos) (rare: values
// within 2^-40 relative of each other).
template <int kLogN>
struct SortedShape {
    static constexpr int N = 1 << kLogN;
    static constexpr int threads = N / 4 < 32 ? 32 : (N / 4 > 512 ? 512 : N / 4);
    static constexpr int E = N / threads; // sorted elements per thread in the scan
    template <class T>
    static constexpr size_t smem() { return N * (8 + sizeof(T)) + 32 * sizeof(T) + 16; }
};

//
// kExact (the float32 default for many-pick long columns, engine.cu
// launch_sorted): after the sort, one thread walks the sorted gaps with the
// reference's sequential `consumed` (omax.hpp:102-110) and one thread sums
// V[row] * p in row order (omax.hpp:169-173), so the result is bit-identical
// to robust_expectation; the parallel scan / tree sums below are skipped.
template <class T, bool kPess, int kLogN, bool kExact = false>
__global__ void __launch_bounds__(SortedShape<kLogN>::threads)
omax_sorted(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
            const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
            const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl,
            const int* __restrict__ count_dev = nullptr) {
    using N_ = Num<T>;
    using Bits = typename N_::Bits;
    using Sh = SortedShape<kLogN>;
    constexpr int N = Sh::N, NT = Sh::threads, E = Sh::E;
    constexpr unsigned long long kPosMask = (1ull << kLogN) - 1;
    pdl_enter();
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    // dynamic shared memory (SortedShape::smem bytes): sort keys (later the
    // available mass by position), gaps by position, warp partials, fix flag
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem_raw);
    T* sgap = reinterpret_cast<T*>(skey + N);
    T* wsum = sgap + N;
    int& fix = *reinterpret_cast<int*>(wsum + 32);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (count_dev) nlist = *count_dev; // fallback list of exact_sort (omax_exact.cuh)
    for (int item = blockIdx.x; item < nlist; item += gridDim.x) {
        const int c = list[item];
        const long long b = colptr[c];
        const int L = static_cast<int>(colptr[c + 1] - b);
        const T r = rem[c];
        // load: keys and gaps by position; padding sorts last
        for (int j = tid; j < N; j += NT) {
            unsigned long long k = ~0ull;
            if (j < L) {
                const Bits full = N_::key(__ldg(V + __ldg(rows + b + j)), kPess);
                if constexpr (sizeof(Bits) == 8)
                    k = ((static_cast<unsigned long long>(full) >> kLogN) << kLogN) | static_cast<unsigned long long>(j);
                else
                    k = (static_cast<unsigned long long>(full) << kLogN) | static_cast<unsigned long long>(j);
                sgap[j] = __ldg(gap + b + j);
            }
            skey[j] = k;
        }
        if (tid == 0) fix = 0;
        __syncthreads();
        // bitonic sort, ascending
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < N / 2; i += NT) {
                    const int lo = 2 * j * (i / j) + (i % j), hi = lo + j;
                    const unsigned long long x = skey[lo], y = skey[hi];
                    const bool up = (lo & k) == 0;
                    if ((x > y) == up) {
                        skey[lo] = y;
                        skey[hi] = x;
                    }
                }
                __syncthreads();
            }
        }
        if constexpr (sizeof(Bits) == 8) {
            // exact order among entries whose truncated keys collide
            for (int j = tid; j + 1 < L; j += NT) {
                const unsigned long long x = skey[j], y = skey[j + 1];
                if ((x >> kLogN) == (y >> kLogN)) {
                    const Bits fx = N_::key(__ldg(V + __ldg(rows + b + (x & kPosMask))), kPess);
                    const Bits fy = N_::key(__ldg(V + __ldg(rows + b + (y & kPosMask))), kPess);
                    if (fx > fy) fix = 1;
                }
            }
            __syncthreads();
            if (fix) {
                if (tid == 0) {
                    // insertion sort by (full key, pos): the input is nearly sorted
                    for (int j = 1; j < L; ++j) {
                        const unsigned long long x = skey[j];
                        const Bits fx = N_::key(__ldg(V + __ldg(rows + b + (x & kPosMask))), kPess);
                        int t = j - 1;
                        while (t >= 0) {
                            const unsigned long long y = skey[t];
                            const Bits fy = N_::key(__ldg(V + __ldg(rows + b + (y & kPosMask))), kPess);
                            if (fy < fx || (fy == fx && (y & kPosMask) < (x & kPosMask))) break;
                            skey[t + 1] = y;
                            --t;
                        }
                        skey[t + 1] = x;
                    }
                }
                __syncthreads();
            }
        }
        if constexpr (kExact) {
            // greedy along the sorted order, sequential as omaximize_sequential (omax.hpp:102-110):
            // sgap[pos] becomes the extra share min(gap, avail) of every picked position
            __shared__ int picks;
            if (tid == 0) {
                T consumed = T(0);
                int j = 0;
                for (; j < L; ++j) {
                    const T avail = N_::sub(r, consumed);
                    if (!(avail > T(0))) break;
                    const int o = static_cast<int>(skey[j] & kPosMask);
                    const T g = sgap[o];
                    sgap[o] = g < avail ? g : avail;
                    consumed = N_::add(consumed, g);
                }
                picks = j;
            }
            __syncthreads();
            for (int j = picks + tid; j < L; j += NT) sgap[skey[j] & kPosMask] = T(-1); // not picked: p = lower
            __syncthreads();
            // products by position, then the row-order dot (omax.hpp:169-173) by one thread
            T* prod = reinterpret_cast<T*>(skey);
            for (int j = tid; j < L; j += NT) {
                const T l = __ldg(lower + b + j), x = sgap[j];
                prod[j] = N_::mul(__ldg(V + __ldg(rows + b + j)), x >= T(0) ? N_::add(l, x) : l);
            }
            __syncthreads();
            if (tid == 0) {
                T dot = T(0);
                for (int j = 0; j < L; ++j) dot = N_::add(dot, prod[j]);
                q[c] = dot;
            }
            __syncthreads();
            continue;
        }
        // prefix scan of the gaps in sorted order: thread tid owns sorted [tid*E, tid*E+E)
        int pos[E];
        T g[E];
        T run = T(0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = tid * E + e;
            pos[e] = j < L ? static_cast<int>(skey[j] & kPosMask) : -1;
            g[e] = pos[e] >= 0 ? sgap[pos[e]] : T(0);
            run = N_::add(run, g[e]);
        }
        // block exclusive scan of the per-thread totals
        T incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T y = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl = N_::add(incl, y);
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads(); // also: every thread has read its keys before they are overwritten
        if (wid == 0) {
            T w = lane < NT / 32 ? wsum[lane] : T(0);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const T y = __shfl_up_sync(kFull, w, o);
                if (lane >= o) w = N_::add(w, y);
            }
            if (lane < NT / 32) wsum[lane] = w; // inclusive warp prefix
        }
        __syncthreads();
        T excl = __shfl_up_sync(kFull, incl, 1);
        if (lane == 0) excl = T(0);
        if (wid > 0) excl = N_::add(excl, wsum[wid - 1]);
        // available mass at each sorted position, stored by position
        T* avail_by_pos = reinterpret_cast<T*>(skey);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (pos[e] >= 0) avail_by_pos[pos[e]] = N_::sub(r, excl);
            excl = N_::add(excl, g[e]);
        }
        __syncthreads();
        // expectation (tree order)
        T acc = T(0);
        for (int j = tid; j < L; j += NT) {
            const T a = avail_by_pos[j];
            const T l = __ldg(lower + b + j);
            const T gg = sgap[j];
            const T p = a > T(0) ? N_::add(l, gg < a ? gg : a) : l;
            acc = N_::add(acc, N_::mul(__ldg(V + __ldg(rows + b + j)), p));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = N_::add(acc, __shfl_xor_sync(kFull, acc, o));
        __syncthreads();
        if (lane == 0) wsum[wid] = acc;
        __syncthreads();
        if (tid == 0) {
            T t = T(0);
            for (int w = 0; w < NT / 32; ++w) t = N_::add(t, wsum[w]);
            q[c] = t;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Long columns with many greedy picks (33 .. 8192 entries): selection of the
// greedy's cut over per-thread sorted runs, instead of a full sort.
//
// The greedy (omax.hpp:98-112) gives every position before the cut c its
// full gap, c the rest of the remainder and every later position nothing,
// where c is the last position (in the adversary order of (V[row], row)) whose
// prefix gap sum F(c) < rem.  So the expectation is
//     q = sum_i V_i l_i + sum_{i before c} V_i g_i + V_c min(g_c, rem - F(c))
// and only c and F(c) are needed, not the order itself.
//
// Work unit: a group of NT threads per column, E = 2..8 entries per thread
// (thread t owns positions e * NT + t: coalesced loads).  Each thread sorts
// its E entries by (order key, position) in registers (bitonic network) and
// publishes the sorted run to shared memory with exclusive prefix sums of g
// and of V g.  Selection passes: every thread keeps a candidate index range
// [lo, hi) of its run; a pivot P splits each range by one binary search, a
// group reduction adds the gap mass below P (differences of the run
// prefixes) and decides the side holding c (base + mass < rem: c >= P); the
// next pivot is the median of the largest remaining range, so each pass
// roughly halves the candidates: about log2(L) passes of O(log E) work per
// thread, against a full sort's log2(L)^2 / 2 barrier stages.
//
// Groups of NT = 32 (up to 256 entries) are warps: reductions by shuffles
// only.  Larger columns take one CTA (NT = 64 .. 1024): one barrier per pass,
// warp partials double-buffered.  The sums run in a different order than
// the reference's sequential loops, so results are within a few ulps of it
// (tests bound them by 1e-12 per step); deterministic.
template <int LG>
struct SelectShape {
    static constexpr int Len = 1 << LG;
    static constexpr int E = 8;                        // entries per thread
    static constexpr int LogE = 3;
    static constexpr int NT = Len / E;                 // threads per column: 8 .. 1024
    static constexpr int Block = NT < 32 ? 256 : NT;
    static constexpr int Groups = Block / NT;          // columns per block
    static constexpr int NW = NT > 32 ? NT / 32 : 1;   // warps per column
    template <class T>
    static constexpr size_t group_bytes() {
        // keys, (E+1) x NT prefix sums of g and of V g, u16 positions
        return ((size_t)Len * sizeof(typename Num<T>::Bits) + 2 * sizeof(T) * (size_t)(Len + NT) +
                2 * (size_t)Len + 15) / 16 * 16;
    }
    template <class T>
    static constexpr size_t smem() {
        // CTA columns: per-warp partials (sum, count, two pivot proposals) + the decision
        return Groups * group_bytes<T>() + (NW > 1 ? NW * (sizeof(T) + 16) + 32 : 0);
    }
};

template <class T>
__device__ __forceinline__ T value_of_key(typename Num<T>::Bits k, bool pess) {
    using Bits = typename Num<T>::Bits;
    constexpr Bits kMsb = Bits(1) << (8 * sizeof(Bits) - 1);
    const Bits b = pess ? k : ~k;
    const Bits raw = (b & kMsb) ? (b & ~kMsb) : ~b;
    T v;
    memcpy(&v, &raw, sizeof v);
    return v;
}

// Pivot proposal: (range length, permuted thread, index of the range
// median), compared as one integer so that a max-reduction picks the largest
// range; ties between equal lengths (late passes: ranges of one entry) go to
// a pass-dependent pseudo-random thread, so the pivot stays a random
// candidate instead of degenerating to an extreme one.
__device__ __forceinline__ unsigned sel_perm(int t, int pass) {
    return ((static_cast<unsigned>(t) + static_cast<unsigned>(pass) * 158u) * 757u) & 1023u;
}
__device__ __forceinline__ int sel_unperm(unsigned x, int pass) {
    return static_cast<int>((x * 349u - static_cast<unsigned>(pass) * 158u) & 1023u); // 757 * 349 = 1 mod 1024
}
__device__ __forceinline__ unsigned sel_pack(int n, int t, int mid, int pass) {
    return n > 0 ? (static_cast<unsigned>(n) << 14) | (sel_perm(t, pass) << 4) | static_cast<unsigned>(mid) : 0u;
}

// Reductions over the lanes of a segment of S <= 32 lanes: xor butterflies
// with offsets < S stay inside the segment, so they run with the full mask
// (per-segment masks would serialise per segment); sums in a fixed tree
// order, so deterministic.
template <int S, class T>
__device__ __forceinline__ T seg_sum(T x) {
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) x = Num<T>::add(x, __shfl_xor_sync(kFull, x, o));
    return x;
}
template <int S>
__device__ __forceinline__ unsigned seg_addu(unsigned x) {
    if constexpr (S == 32) {
        return __reduce_add_sync(kFull, x);
    } else {
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
        return x;
    }
}
template <int S>
__device__ __forceinline__ unsigned seg_maxu(unsigned x) {
    if constexpr (S == 32) {
        return __reduce_max_sync(kFull, x);
    } else {
#pragma unroll
        for (int o = S / 2; o > 0; o >>= 1) {
            const unsigned y = __shfl_xor_sync(kFull, x, o);
            x = y > x ? y : x;
        }
        return x;
    }
}

template <class T, bool kPess, int LG>
__global__ void __launch_bounds__(SelectShape<LG>::Block)
omax_select(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
            const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
            const T* __restrict__ rem, const T* __restrict__ V, T* __restrict__ q, const Ctl* __restrict__ ctl,
            const int* __restrict__ nlist_dev) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    using Sh = SelectShape<LG>;
    pdl_enter();
    if (nlist_dev) nlist = *nlist_dev; // fallback list of omax_bucket
    constexpr int E = Sh::E, NT = Sh::NT, NW = Sh::NW, LOGE = Sh::LogE;
    constexpr int S = NT < 32 ? NT : 32; // lanes of one column inside a warp
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int grp = threadIdx.x / NT, t = threadIdx.x % NT, wig = t >> 5;
    unsigned char* gb = smem_raw + grp * Sh::template group_bytes<T>();
    Bits* rk = reinterpret_cast<Bits*>(gb);                       // [E][NT] sorted keys
    T* rpre = reinterpret_cast<T*>(gb + Sh::Len * sizeof(Bits)); // [E+1][NT] exclusive prefix of g
    T* rvg = rpre + (Sh::Len + NT);                               // [E+1][NT] exclusive prefix of V g
    unsigned short* rp = reinterpret_cast<unsigned short*>(rvg + (Sh::Len + NT)); // [E][NT] positions
    // CTA columns: warp partials and the decision of warp 0
    T* psl = reinterpret_cast<T*>(smem_raw + Sh::Groups * Sh::template group_bytes<T>());
    unsigned* pu = reinterpret_cast<unsigned*>(psl + NW);           // [NW][3]: count, packL, packR
    T* dbase = reinterpret_cast<T*>(pu + ((3 * NW + 1) & ~1));      // decision: base (8-byte aligned)
    unsigned* dword = reinterpret_cast<unsigned*>(dbase + 1);      // decision: side, ncand, pack
    const int ngroups = gridDim.x * Sh::Groups;
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();

    for (int item0 = blockIdx.x * Sh::Groups; item0 < nlist; item0 += ngroups) {
        const int item = item0 + grp;
        const bool live = item < nlist;
        int L = 0;
        long long b = 0;
        T r = T(0);
        int c = -1;
        if (live) {
            c = __ldg(list + item);
            b = __ldg(colptr + c);
            L = static_cast<int>(__ldg(colptr + c + 1) - b);
            r = __ldg(rem + c);
        }
        // ---- load this thread's entries; sum of V l ----
        int rw[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = e * NT + t;
            rw[e] = pos < L ? ld_hint(rows + b + pos, pstream) : 0;
        }
        Bits k[E];
        int p[E];
        T g[E];
        T acc = T(0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = e * NT + t;
            k[e] = ~Bits(0);
            p[e] = 0xffff;
            g[e] = T(0);
            if (pos < L) {
                const T v = ld_hint(V + rw[e], pval);
                k[e] = order_key<T>(v, kPess);
                p[e] = pos;
                g[e] = ld_hint(gap + b + pos, pstream);
                acc = N::add(acc, N::mul(v, ld_hint(lower + b + pos, pstream)));
            }
        }
        const int cnt = min(E, max(0, (L - t + NT - 1) / NT));
        // ---- sort the run by (key, position): bitonic network in registers ----
#pragma unroll
        for (int size = 2; size <= E; size <<= 1) {
#pragma unroll
            for (int stride = size / 2; stride > 0; stride >>= 1) {
#pragma unroll
                for (int i = 0; i < E; ++i) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const bool up = (i & size) == 0;
                        const bool gt = k[i] > k[j] || (k[i] == k[j] && p[i] > p[j]);
                        if (gt == up) {
                            const Bits tk = k[i];
                            k[i] = k[j];
                            k[j] = tk;
                            const int tp = p[i];
                            p[i] = p[j];
                            p[j] = tp;
                            const T tg = g[i];
                            g[i] = g[j];
                            g[j] = tg;
                        }
                    }
                }
            }
        }
        {
            T sg = T(0), svg = T(0);
            rpre[t] = sg;
            rvg[t] = svg;
#pragma unroll
            for (int i = 0; i < E; ++i) {
                rk[i * NT + t] = k[i];
                rp[i * NT + t] = static_cast<unsigned short>(p[i]);
                if (i < cnt) {
                    sg = N::add(sg, g[i]);
                    svg = N::add(svg, N::mul(value_of_key<T>(k[i], kPess), g[i]));
                }
                rpre[(i + 1) * NT + t] = sg;
                rvg[(i + 1) * NT + t] = svg;
            }
        }
        // ---- selection of the cut ----
        int lo = 0, hi = cnt;
        unsigned pack = seg_maxu<S>(sel_pack(cnt, t, cnt / 2, 0));
        if constexpr (NW > 1) {
            if (lane == 0) pu[wig] = pack;
            __syncthreads();
            pack = pu[0];
#pragma unroll
            for (int i = 1; i < NW; ++i) pack = pu[i] > pack ? pu[i] : pack;
            __syncthreads();
        } else {
            __syncwarp();
        }
        T base = T(0);
        const bool picks = live && r > T(0);
        // segment columns: the pass loop is warp-uniform (done segments idle
        // through it), so every collective runs convergent with the full mask
        bool act = picks;
        int ncand = L;
        if (NW > 1 ? picks : __any_sync(kFull, act)) {
            for (int pass = 0;; ++pass) {
                // (a segment that is done idles on its own first entry)
                const int ts = act ? sel_unperm((pack >> 4) & 1023u, pass) : t;
                const int ms = act ? static_cast<int>(pack & 15u) : 0;
                const Bits pk = rk[ms * NT + ts];
                const int pp = rp[ms * NT + ts];
                // first index of [lo, hi) with (key, pos) >= (pk, pp)
                int i0 = lo, i1 = hi;
#pragma unroll
                for (int st = 0; st <= LOGE; ++st) {
                    if (i0 < i1) {
                        const int m = (i0 + i1) >> 1;
                        const Bits km = rk[m * NT + t];
                        const int pm = rp[m * NT + t];
                        if (km < pk || (km == pk && pm < pp)) i0 = m + 1;
                        else i1 = m;
                    }
                }
                const int split = i0;
                T sl = lo < split ? N::sub(rpre[split * NT + t], rpre[lo * NT + t]) : T(0);
                int nl = split - lo;
                const bool ownsP = t == ts && split < hi && split == ms;
                const int rs = split + (ownsP ? 1 : 0);
                unsigned packL = sel_pack(nl, t, lo + nl / 2, pass + 1);
                unsigned packR = sel_pack(hi - rs, t, rs + (hi - rs) / 2, pass + 1);
                sl = seg_sum<S>(sl);
                nl = static_cast<int>(seg_addu<S>(static_cast<unsigned>(nl)));
                packL = seg_maxu<S>(packL);
                packR = seg_maxu<S>(packR);
                bool right;
                if constexpr (NW > 1) {
                    if (lane == 0) {
                        psl[wig] = sl;
                        pu[3 * wig + 0] = static_cast<unsigned>(nl);
                        pu[3 * wig + 1] = packL;
                        pu[3 * wig + 2] = packR;
                    }
                    __syncthreads();
                    if (wig == 0) {
                        // warp 0 combines the warp partials and decides
                        T ws = lane < NW ? psl[lane] : T(0);
                        ws = seg_sum<32>(ws);
                        const unsigned wn = __reduce_add_sync(kFull, lane < NW ? pu[3 * lane] : 0u);
                        const unsigned wl = __reduce_max_sync(kFull, lane < NW ? pu[3 * lane + 1] : 0u);
                        const unsigned wr = __reduce_max_sync(kFull, lane < NW ? pu[3 * lane + 2] : 0u);
                        if (lane == 0) {
                            const bool rt = N::add(base, ws) < r;
                            dbase[0] = rt ? N::add(base, ws) : base;
                            dword[0] = rt;
                            dword[1] = static_cast<unsigned>(rt ? ncand - static_cast<int>(wn) : static_cast<int>(wn));
                            dword[2] = rt ? wr : wl;
                        }
                    }
                    __syncthreads();
                    right = dword[0] != 0;
                    base = dbase[0];
                    ncand = static_cast<int>(dword[1]);
                    pack = dword[2];
                    if (right) lo = split;
                    else hi = split;
                    if (ncand <= 1) break;
                } else {
                    right = N::add(base, sl) < r; // the cut is at or after the pivot
                    if (act) {
                        if (right) {
                            base = N::add(base, sl);
                            ncand -= nl;
                            pack = packR;
                            lo = split;
                        } else {
                            ncand = nl;
                            pack = packL;
                            hi = split;
                        }
                        act = ncand > 1;
                    }
                    if (!__any_sync(kFull, act)) break;
                }
            }
        }
        // ---- expectation: sum V l + sum_{before c} V g + V_c min(g_c, rem - F(c)) ----
        if (picks) {
            acc = N::add(acc, rvg[lo * NT + t]);
            if (hi - lo == 1) { // this thread owns the cut
                const T vc = value_of_key<T>(rk[lo * NT + t], kPess);
                const T gc = __ldg(gap + b + rp[lo * NT + t]);
                const T avail = N::sub(r, base);
                acc = N::add(acc, N::mul(vc, gc < avail ? gc : avail));
            }
        }
        acc = seg_sum<S>(acc);
        if constexpr (NW > 1) {
            if (lane == 0) psl[wig] = acc;
            __syncthreads();
            if (t == 0) {
                T s2 = psl[0];
                for (int i = 1; i < NW; ++i) s2 = N::add(s2, psl[i]);
                q[c] = s2;
            }
            __syncthreads();
        } else {
            if (t == 0 && live) q[c] = acc;
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// Long many-pick columns (257 .. 8192 entries), O(L) path: value buckets.
//
// One CTA per column, thread t owning positions e * NT + t (E = 8).  With w
// the value in adversary order (V pessimistic, -V optimistic), the column's
// entries are cut into B equal-width buckets of [w_min, w_max]: the bucket
// index is a monotone function of w, so buckets are contiguous in the
// adversary order and ties share a bucket.  Gap mass per bucket is
// accumulated in shared memory as fixed-point integers (g * Sc truncated,
// Sc = 2^31 / (L * max gap): no overflow; integer atomics, deterministic).
// Since truncation loses < 1 unit per entry, the exact mass before bucket b
// lies in [F_b, F_b + L) (F_b the fixed mass before b, L the column length),
// which brackets the bucket of the cut c (the last entry whose prefix gap
// mass is < rem) in [b_lo, b_hi]:  b_lo = last bucket with F_b + L <= rem * Sc
// (certainly reached), b_hi = last bucket with F_b < rem * Sc.  (Empty
// buckets in the bracket hold no entries; no count histogram is needed.)
// Entries below b_lo are before c: their exact gap sum (double, tree order)
// is the base, and their V g is added to the expectation.  The <= kBucketCap
// entries of [b_lo, b_hi] are resolved exactly by warp 0: bitonic sort by
// (order key, position), exclusive prefix of the gaps from the base, the cut
// is the last entry whose prefix is < rem.
//   q = sum V l + sum_{before c} V g + V_c min(g_c, rem - F(c))
// A column whose bracket holds more than kBucketCap entries (heavy ties,
// clustered values) is appended to a fallback list for omax_select.  Sums are
// in tree order: within a few ulps of the reference (1e-12 tests).
constexpr int kBucketCap = 64;

// f32 entries take half the registers: 16 entries per thread, half the
// threads per column, twice the columns in flight per SM (C5 f32 1.98 ->
// 1.91 ms per iteration).  RIMDP_BUCKET_F32_E16=0: 8 entries as for f64.
#ifndef RIMDP_BUCKET_F32_E16
#define RIMDP_BUCKET_F32_E16 1
#endif
template <int LG, class TV = double>
struct BucketShape {
    static constexpr int Len = 1 << LG;
    static constexpr int E = (sizeof(TV) == 4 && RIMDP_BUCKET_F32_E16) ? 16 : 8;
    static constexpr int NT = Len / E;    // 64 .. 1024
    static constexpr int NW = NT / 32;
    static constexpr int B = Len / 4 < 1024 ? Len / 4 : 1024; // ~4 entries per bucket
    static constexpr int MinBlocks = NT >= 1024 ? 1 : 1024 / NT;
    template <class T>
    static constexpr size_t smem() {
        // hist (u32 x B) x 2 (alternate columns); candidates (key, pos, g, V) x kBucketCap; partials
        // (sum g below the bracket, sum V l + V g below) x NW; warp scan totals; decision words x 2
        return 2 * 4 * B + kBucketCap * (8 + 4 + 2 * sizeof(T)) + NW * (2 * sizeof(T) + 16) + 64;
    }
};

// Range of the value vector as order keys of the ascending order (slot
// [0] = min, [1] = max), for omax_bucket's value buckets.  Launches
// alternate between two slots; each launch resets the other one.
template <class T>
__global__ void __launch_bounds__(256)
value_range(int n, const T* __restrict__ V, unsigned long long* __restrict__ slot,
            unsigned long long* __restrict__ other) {
    using Bits = typename Num<T>::Bits;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        other[0] = ~0ull;
        other[1] = 0ull;
    }
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const unsigned long long k = static_cast<unsigned long long>(static_cast<Bits>(order_key<T>(__ldg(V + i), true)));
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a = __shfl_xor_sync(kFull, lo, o), z = __shfl_xor_sync(kFull, hi, o);
        lo = a < lo ? a : lo;
        hi = z > hi ? z : hi;
    }
    // one pair of global atomics per block (per warp they serialise on the two words: 12 -> 4 us at C5)
    __shared__ unsigned long long wl[8], wh[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        wl[w] = lo;
        wh[w] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) {
            lo = wl[i] < lo ? wl[i] : lo;
            hi = wh[i] > hi ? wh[i] : hi;
        }
        if (lo != ~0ull) atomicMin(slot, lo);
        atomicMax(slot + 1, hi);
    }
}

// Many-pick columns of 257 .. 8192 entries: one CTA per column, E = 8
// entries per thread, kept in registers (no shared-memory staging).
//
// Equal-width value buckets of w = +-V (along the adversary order) over the
// range of the whole value vector (value_range, one launch per iteration:
// no per-column min/max pass) are monotone in the order (omax.hpp:41-58), so
// buckets are contiguous and ties share a bucket.  Values outside the range
// cannot occur; the index is clamped anyway.  A fixed-point gap histogram
// uses u32 shared atomics at a scale chosen per column so it cannot
// overflow; it is deterministic.  Since truncation loses < 1 unit per entry,
// the exact mass before bucket b lies in [F_b, F_b + L) (F_b the fixed mass
// before b), which brackets the bucket of the cut c (the last entry whose
// prefix gap mass is < rem) in [b_lo, b_hi]:  b_lo = last bucket with
// F_b + L <= rem * Sc (certainly reached), b_hi = last bucket with
// F_b < rem * Sc; the fixed-point total is <= 2^31, so the scan is 32-bit.
// Entries below b_lo are before c: their exact gap sum (double, tree order)
// is the base, and their V g is added to the expectation.  The <= kBucketCap
// entries of [b_lo, b_hi] are resolved exactly by the greedy itself, run by
// the last warp to finish the column: exact warp argmins over (order key,
// position), `consumed` continued sequentially from the base.
//   q = sum V l + sum_{before c} V g + V_c min(g_c, rem - F(c))
// A column whose bracket holds more than kBucketCap entries (heavy ties,
// clustered values) is appended to a fallback list for omax_select.  Sums are
// in tree order: within a few ulps of the reference (1e-12 tests).
// Three barriers per column (histogram, scan, bracket); the last warp to
// deposit its partials completes the column (arrival counter), the others
// go on; the histogram and the decision words alternate between two buffers
// so the next column needs no trailing barrier.
template <class T, bool kPess, int LG>
__global__ void __launch_bounds__(BucketShape<LG, T>::NT, BucketShape<LG, T>::MinBlocks)
omax_bucket(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
            const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
            const T* __restrict__ rem, const T* __restrict__ maxgap, const T* __restrict__ V, T* __restrict__ q,
            const Ctl* __restrict__ ctl, int* __restrict__ fallback, int* __restrict__ nfallback,
            int* __restrict__ other_nfallback, const unsigned long long* __restrict__ vrange,
            unsigned* __restrict__ work) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    using Sh = BucketShape<LG, T>;
    constexpr int E = Sh::E, NT = Sh::NT, NW = Sh::NW, B = Sh::B, CAP = kBucketCap;
    pdl_enter_class(ctl);
    // fallback counters alternate between launches: this launch counts into
    // nfallback and clears the other one for the next launch (every earlier
    // launch, and the selection pass that read it, has completed)
    if (blockIdx.x == 0 && threadIdx.x == 0) *other_nfallback = 0;
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned* hbuf = reinterpret_cast<unsigned*>(smem_raw);           // [2][hist B]
    unsigned long long* ckey = reinterpret_cast<unsigned long long*>(hbuf + 2 * B);
    T* cg = reinterpret_cast<T*>(ckey + CAP);
    T* cv = cg + CAP;
    int* cpos = reinterpret_cast<int*>(cv + CAP);
    T* pa = reinterpret_cast<T*>(cpos + CAP);   // [NW] sum g below the bracket
    T* pb = pa + NW;                            // [NW] sum V l + sum V g below the bracket
    unsigned long long* wtot = reinterpret_cast<unsigned long long*>(pb + NW); // [2][NW] warp scan totals
    int* dwb = reinterpret_cast<int*>(wtot + 2 * NW); // [2][b_lo + 1, b_hi + 1, -, candidate counter]
    const int t = threadIdx.x, lane = t & 31, wig = t >> 5;
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    // value range: buckets over [wlo, whi] of w = +-V
    const T vmin = value_of_key<T>(static_cast<Bits>(__ldg(vrange)), true);
    const T vmax = value_of_key<T>(static_cast<Bits>(__ldg(vrange + 1)), true);
    const T wlo = kPess ? vmin : -vmax, whi = kPess ? vmax : -vmin;
    const T span = N::sub(whi, wlo);
    const T bscale = span > T(0) ? T(B) / span : T(0);
    auto bucket_of = [&](T val) -> int {
        const T w = kPess ? val : -val;
        int x = static_cast<int>(N::mul(N::sub(w, wlo), bscale));
        x = x > 0 ? x : 0;
        return x < B - 1 ? x : B - 1;
    };
    for (int i = t; i < 2 * B; i += NT) hbuf[i] = 0u;
    if (t < 8) dwb[t] = 0;
    __syncthreads();
    unsigned par = 0;
    // columns are taken dynamically (work counter; the first one per CTA is blockIdx.x): thread 0 claims
    // the CTA's next column while this one loads, every thread reads it behind B1 (alternating slots)
    __shared__ int next_slot[2];
    int next_item = nlist;

    for (int item = blockIdx.x; item < nlist; item = next_item) {
        if (t == 0) next_slot[par] = work ? static_cast<int>(gridDim.x + atomicAdd(work, 1u)) : item + static_cast<int>(gridDim.x);
        const int c = __ldg(list + item);
        const long long b = __ldg(colptr + c);
        const int L = static_cast<int>(__ldg(colptr + c + 1) - b);
        const T r = __ldg(rem + c);
        const bool picks = r > T(0);
        unsigned* hist = hbuf + par * B;
        int* dw = dwb + par * 4;
        // ---- load (registers); sum V l; fixed-point gap histogram ----
        int rw[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = e * NT + t;
            rw[e] = pos < L ? ld_hint(rows + b + pos, pstream) : 0;
        }
        T v[E], g[E];
        T acc = T(0);
#pragma unroll
        for (int h = 0; h < E; h += E / 2) { // two halves: 3 x E/2 loads in flight, fewer registers
            T l[E / 2];
#pragma unroll
            for (int i = 0; i < E / 2; ++i) {
                const int e = h + i, pos = e * NT + t;
                v[e] = T(0);
                g[e] = T(0);
                l[i] = T(0);
                if (pos < L) {
                    v[e] = ld_hint(V + rw[e], pval);
                    g[e] = ld_hint(gap + b + pos, pstream);
                    l[i] = ld_hint(lower + b + pos, pstream);
                }
            }
#pragma unroll
            for (int i = 0; i < E / 2; ++i) {
                const int e = h + i, pos = e * NT + t;
                if (pos < L) acc = N::add(acc, N::mul(v[e], l[i]));
            }
        }
        const T gm = __ldg(maxgap + c);
        const double sc = gm > T(0) ? 2147483648.0 / ((double)L * (double)gm) : 0.0;
        if (picks) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e * NT + t < L) atomicAdd(hist + bucket_of(v[e]), static_cast<unsigned>((double)g[e] * sc));
            }
        }
        __syncthreads(); // B1: histogram complete
        next_item = next_slot[par];
        {   // the next column's buffers: their last readers (the previous column) are past B1
            unsigned* oh = hbuf + (par ^ 1u) * B;
            for (int i = t; i < B; i += NT) oh[i] = 0u;
            if (t < 4) dwb[(par ^ 1u) * 4 + t] = 0;
        }
        T bs = T(0);
        if (picks) {
            // ---- bracket of the cut's bucket: block-wide exclusive scan of the buckets ----
            // (the fixed-point total is <= 2^31: 32-bit prefixes)
            constexpr int PB = B / NT > 0 ? B / NT : 1; // buckets per thread
            unsigned fm = 0;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
                const int bb = t * PB + i;
                if (bb < B) fm += hist[bb];
            }
            unsigned em = fm;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned a = __shfl_up_sync(kFull, em, o);
                if (lane >= o) em += a;
            }
            if (lane == 31) wtot[wig] = em;
            __syncthreads(); // B2
            em -= fm;
            // totals of the warps before this one: one load per lane and a warp reduction
            em += __reduce_add_sync(kFull, lane < wig ? static_cast<unsigned>(wtot[lane]) : 0u);
            {
                // truncation lost < 1 unit per entry, < L before any bucket
                const double R = (double)r * sc, RL = R - (double)L;
                int blo = -1, bhi = -1;
#pragma unroll
                for (int i = 0; i < PB; ++i) {
                    const int bb = t * PB + i;
                    if (bb < B) {
                        if ((double)em <= RL) blo = bb;
                        if ((double)em < R) bhi = bb;
                        em += hist[bb];
                    }
                }
                // one shared atomic per warp (the whole block would otherwise hit the same two words)
                const unsigned wlo = __reduce_max_sync(kFull, static_cast<unsigned>(blo + 1));
                const unsigned whi = __reduce_max_sync(kFull, static_cast<unsigned>(bhi + 1));
                if (lane == 0) {
                    if (wlo > 0) atomicMax(dw + 0, static_cast<int>(wlo));
                    if (whi > 0) atomicMax(dw + 1, static_cast<int>(whi));
                }
            }
            __syncthreads(); // B3
            const int blo = dw[0] > 0 ? dw[0] - 1 : 0; // the first entry is always reached (rem > 0)
            const int bhi = dw[1] - 1;
            // ---- entries before the bracket; candidates to shared memory ----
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = e * NT + t;
                if (pos < L) {
                    const int bb = bucket_of(v[e]);
                    if (bb < blo) {
                        bs = N::add(bs, g[e]);
                        acc = N::add(acc, N::mul(v[e], g[e]));
                    } else if (bb <= bhi) {
                        const int slot = atomicAdd(dw + 3, 1);
                        if (slot < CAP) {
                            ckey[slot] = static_cast<unsigned long long>(order_key<T>(v[e], kPess));
                            cg[slot] = g[e];
                            cv[slot] = v[e];
                            cpos[slot] = pos;
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            bs = N::add(bs, __shfl_xor_sync(kFull, bs, o));
            acc = N::add(acc, __shfl_xor_sync(kFull, acc, o));
        }
        if (lane == 0) {
            pa[wig] = bs;
            pb[wig] = acc;
        }
        // The last warp to get here completes the column; the others go on to
        // the next one at once (no block barrier: an arrival counter, dw[2],
        // with CTA-scope fences on both sides).  The shared state it reads —
        // partials, candidates, dw — is rewritten only after the next
        // column's B1, which this warp reaches after finishing.
        __threadfence_block();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(reinterpret_cast<unsigned*>(dw + 2), 1u) == static_cast<unsigned>(NW - 1);
        last = __shfl_sync(kFull, last, 0);
        par ^= 1u;
        if (!last) continue;
        __threadfence_block();
        const int K = picks ? *reinterpret_cast<volatile int*>(dw + 3) : 0;
        if (K > CAP) {
            // too many entries in the bracket (ties, clustered values): selection kernel
            if (lane == 0) fallback[atomicAdd(nfallback, 1)] = c;
            continue;
        }
        // ---- the last warp: the greedy (omax.hpp:98-112) inside the bracket, q ----
        // Two candidates per lane (slots lane, 32 + lane).  `consumed` starts
        // at the exact base below the bracket and grows along the adversary
        // order: each pick is the exact warp argmin over (order key, position),
        // so only the picks up to the cut are walked (typically a handful).
        // The picks' shares are summed in pick order, so q does not depend on
        // which slot a candidate landed in.
        T add = T(0);
        if (picks && K > 0) {
            T base = pa[0];
#pragma unroll
            for (int i = 1; i < NW; ++i) base = N::add(base, pa[i]);
            unsigned long long k0 = lane < K ? ckey[lane] : ~0ull;
            unsigned long long k1 = 32 + lane < K ? ckey[32 + lane] : ~0ull;
            const int p0 = lane < K ? cpos[lane] : INT_MAX, p1 = 32 + lane < K ? cpos[32 + lane] : INT_MAX;
            const T g0 = lane < K ? cg[lane] : T(0), g1 = 32 + lane < K ? cg[32 + lane] : T(0);
            const T v0 = lane < K ? cv[lane] : T(0), v1 = 32 + lane < K ? cv[32 + lane] : T(0);
            T consumed = base;
            T avail = N::sub(r, consumed);
            for (int nsel = 0; avail > T(0) && nsel < K; ++nsel) {
                const bool first = k0 < k1 || (k0 == k1 && p0 < p1);
                const unsigned long long lk = first ? k0 : k1;
                const int lp = first ? p0 : p1;
                const unsigned hi = static_cast<unsigned>(lk >> 32), lo = static_cast<unsigned>(lk);
                const unsigned mhi = __reduce_min_sync(kFull, hi);
                bool cand = hi == mhi;
                const unsigned mlo = __reduce_min_sync(kFull, cand ? lo : 0xffffffffu);
                cand = cand && lo == mlo;
                const unsigned mp = __reduce_min_sync(kFull, cand ? static_cast<unsigned>(lp) : 0xffffffffu);
                cand = cand && static_cast<unsigned>(lp) == mp;
                const int sel = __ffs(__ballot_sync(kFull, cand)) - 1;
                const T gl = first ? g0 : g1, vl = first ? v0 : v1;
                const T gs = __shfl_sync(kFull, gl, sel);
                // the share of the pick, summed in pick order (candidate slots are not deterministic)
                add = N::add(add, __shfl_sync(kFull, N::mul(vl, gl < avail ? gl : avail), sel));
                if (lane == sel) {
                    if (first) k0 = ~0ull;
                    else k1 = ~0ull;
                }
                consumed = N::add(consumed, gs);
                avail = N::sub(r, consumed);
            }
        }
        // ---- q = sum of the warps' partials + the bracket's share (warp-uniform) ----
        if (lane == 0) {
            T s2 = pb[0];
            for (int i = 1; i < NW; ++i) s2 = N::add(s2, pb[i]);
            q[c] = N::add(s2, add);
        }
    }
}

// Many-pick columns of 33 .. 256 entries: omax_bucket's method at warp
// scale.  One warp per column, E = Len / 32 entries per lane in registers,
// B = Len / 4 value buckets over the value vector's range (value_range), a
// fixed-point gap histogram in the warp's shared memory, a warp scan for the
// bracket [b_lo, b_hi], no block barriers.  The bracket's entries (<= 32)
// are compacted one per lane in position order (ballot ranks) and resolved by
// the greedy itself (omax.hpp:98-112): exact warp argmins over their order
// keys, `consumed` continued sequentially from the exact base (the gaps
// below the bracket, tree order), so only the few picks inside the bracket
// are walked.  A bracket of more than 32 entries goes to the fallback list
// (omax_select).  Tree-order sums: within a few ulps of the reference.
template <int LG>
struct WBucketShape {
    static constexpr int Len = 1 << LG;
    static constexpr int E = Len / 32;          // 2, 4, 8
    static constexpr int B = Len / 4;           // 16, 32, 64
    static constexpr int PB = B >= 32 ? B / 32 : 1;
    static constexpr int W = 8;                 // warps per block
    static constexpr int WarpBytes = 4 * B + 32 * (8 + 2 * 8);
};

template <class T, bool kPess, int LG>
__global__ void __launch_bounds__(WBucketShape<LG>::W * 32)
omax_wbucket(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
             const int* __restrict__ rows, const T* __restrict__ lower, const T* __restrict__ gap,
             const T* __restrict__ rem, const T* __restrict__ maxgap, const T* __restrict__ V, T* __restrict__ q,
             const Ctl* __restrict__ ctl, int* __restrict__ fallback, int* __restrict__ nfallback,
             int* __restrict__ other_nfallback, const unsigned long long* __restrict__ vrange) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    using Sh = WBucketShape<LG>;
    constexpr int E = Sh::E, B = Sh::B, PB = Sh::PB, W = Sh::W;
    pdl_enter_class(ctl);
    if (blockIdx.x == 0 && threadIdx.x == 0) *other_nfallback = 0;
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    __shared__ __align__(16) unsigned char smem[W * Sh::WarpBytes];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned* hist = reinterpret_cast<unsigned*>(smem + w * Sh::WarpBytes);
    unsigned long long* ckey = reinterpret_cast<unsigned long long*>(hist + B);
    T* cg = reinterpret_cast<T*>(ckey + 32);
    T* cv = cg + 32;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned long long pstream = l2_evict_first_policy(), pval = l2_evict_last_policy();
    const T vmin = value_of_key<T>(static_cast<Bits>(__ldg(vrange)), true);
    const T vmax = value_of_key<T>(static_cast<Bits>(__ldg(vrange + 1)), true);
    const T wlo = kPess ? vmin : -vmax, whi = kPess ? vmax : -vmin;
    const T span = N::sub(whi, wlo);
    const T bscale = span > T(0) ? T(B) / span : T(0);
    auto bucket_of = [&](T val) -> int {
        const T wv = kPess ? val : -val;
        int x = static_cast<int>(N::mul(N::sub(wv, wlo), bscale));
        x = x > 0 ? x : 0;
        return x < B - 1 ? x : B - 1;
    };
    // static assignment: a dynamic claim per column (work counter, as omax_bucket) measured 1.6% slower
    // here (one atomic and its round trip per warp per column of 33-256 entries)
    const int gw = blockIdx.x * W + w, nw = gridDim.x * W;
    for (int item = gw; item < nlist; item += nw) {
        const int c = __ldg(list + item);
        const long long b = __ldg(colptr + c);
        const int L = static_cast<int>(__ldg(colptr + c + 1) - b);
        const T r = __ldg(rem + c);
        const T gm = __ldg(maxgap + c); // issued with the other metadata, not behind the column's loads
        const bool picks = r > T(0);
        int rw[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = e * 32 + lane;
            rw[e] = pos < L ? ld_hint(rows + b + pos, pstream) : 0;
        }
        T v[E], g[E];
        T acc = T(0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int pos = e * 32 + lane;
            v[e] = T(0);
            g[e] = T(0);
            if (pos < L) {
                v[e] = ld_hint(V + rw[e], pval);
                g[e] = ld_hint(gap + b + pos, pstream);
                acc = N::add(acc, N::mul(v[e], ld_hint(lower + b + pos, pstream)));
            }
        }
        T add = T(0);
        if (picks) {
            // ---- fixed-point gap histogram (warp-private) ----
#pragma unroll
            for (int i = lane; i < B; i += 32) hist[i] = 0u;
            __syncwarp();
            const double sc = gm > T(0) ? 2147483648.0 / ((double)L * (double)gm) : 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                if (e * 32 + lane < L) atomicAdd(hist + bucket_of(v[e]), static_cast<unsigned>((double)g[e] * sc));
            }
            __syncwarp();
            // ---- bracket: warp scan of the buckets (lane owns PB consecutive buckets) ----
            unsigned fm = 0;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
                const int bb = lane * PB + i;
                if (bb < B) fm += hist[bb];
            }
            unsigned em = fm;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned a = __shfl_up_sync(kFull, em, o);
                if (lane >= o) em += a;
            }
            em -= fm;
            // truncation lost < 1 unit per entry, < L before any bucket
            const double R = (double)r * sc, RL = R - (double)L;
            int blo = -1, bhi = -1;
#pragma unroll
            for (int i = 0; i < PB; ++i) {
                const int bb = lane * PB + i;
                if (bb < B) {
                    if ((double)em <= RL) blo = bb;
                    if ((double)em < R) bhi = bb;
                    em += hist[bb];
                }
            }
            const int lo_b = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(blo + 1)));
            const int hi_b = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(bhi + 1))) - 1;
            const int bl = lo_b > 0 ? lo_b - 1 : 0; // the first entry is always reached (rem > 0)
            // ---- below the bracket: exact base; the bracket: compacted one per lane ----
            T bs = T(0);
            int K = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int pos = e * 32 + lane;
                const int bb = pos < L ? bucket_of(v[e]) : B;
                if (bb < bl) {
                    bs = N::add(bs, g[e]);
                    acc = N::add(acc, N::mul(v[e], g[e]));
                }
                const bool in = bb >= bl && bb <= hi_b;
                const unsigned m = __ballot_sync(kFull, in);
                const int slot = K + __popc(m & lt);
                if (in && slot < 32) {
                    ckey[slot] = static_cast<unsigned long long>(order_key<T>(v[e], kPess));
                    cg[slot] = g[e];
                    cv[slot] = v[e];
                }
                K += __popc(m);
            }
            if (K > 32) {
                // too many entries in the bracket (ties, clustered values): selection kernel
                if (lane == 0) fallback[atomicAdd(nfallback, 1)] = c;
                __syncwarp();
                continue;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) bs = N::add(bs, __shfl_xor_sync(kFull, bs, o));
            __syncwarp();
            // ---- the greedy inside the bracket (slot order = position order) ----
            const bool ok = lane < K;
            Bits key = ok ? static_cast<Bits>(ckey[lane]) : ~Bits(0);
            const T gl = ok ? cg[lane] : T(0), vl = ok ? cv[lane] : T(0);
            T consumed = bs;
            T avail = N::sub(r, consumed);
            for (int nsel = 0; avail > T(0) && nsel < K; ++nsel) {
                const int sel = warp_argmin_sentinel(key);
                const T gs = __shfl_sync(kFull, gl, sel);
                if (lane == sel) {
                    add = N::mul(vl, gl < avail ? gl : avail);
                    key = ~Bits(0);
                }
                consumed = N::add(consumed, gs);
                avail = N::sub(r, consumed);
            }
            __syncwarp(); // candidates and histogram are rewritten by the next column
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            acc = N::add(acc, __shfl_xor_sync(kFull, acc, o));
            add = N::add(add, __shfl_xor_sync(kFull, add, o));
        }
        if (lane == 0) q[c] = N::add(acc, add);
    }
}

// ---------------------------------------------------------------------------
// Action reduction + reach/avoid/discount update + residual + stop test
// (bellman.hpp:88-115, solver.hpp:107-134).  Each block folds its max of
// |V_k - V_{k-1}| into ctl with one atomicMax; the launch flagged `finalize`
// (the last kernel of the iteration) counts block arrivals and its last block
// evaluates the stop test, so the residual needs no extra pass and the host
// needs no per-iteration synchronisation.
// Peer exchange of a state-sharded solve: every
// shard owns an exchange window in its HBM holding the double-buffered value
// vector, one residual slot per source rank per iteration parity and one
// iteration flag per source rank.  The window pointers of all ranks (peer
// device memory over NVLink: CUDA IPC or peer access) live in this table.
constexpr int kMaxWorld = 8;
struct PeerTable {
    int world, rank;
    void* v[kMaxWorld][2];                  // rank p's value buffers (V_k in buffer k & 1)
    unsigned long long* res[kMaxWorld];     // rank p's residual slots [2][kMaxWorld] (parity, source)
    unsigned long long* flag[kMaxWorld];    // rank p's flags [kMaxWorld]: last iteration published by each source
};

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

struct ActionArgs {
    int n;                         // local states
    int state_begin;               // shard offset of local state 0 in the global value vector
    const int* stateptr;           // local columns of local states
    const unsigned char* frozen;   // local [n] or null
    const int* forced;             // null, [n], or [horizon][n]
    int forced_td;
    int* chosen;                   // [n] or [horizon][n]
    int chosen_td;
    int maximize;
    int finite;
    long long horizon;
    long long max_iterations;
    long long k;                   // the iteration this launch computes (1-based)
    int record_only;               // sharded solves: the driver owns the stop test
    int finalize;                  // this launch is the iteration's last: run the stop test
    unsigned* work;                // work counters [2 slots][kWorkKinds], slot k & 1
    const PeerTable* peers;        // sharded solve with peer exchange, else null
};

constexpr int kWorkSorted = 4;     // work counters of the many-pick size classes 2^6 .. 2^13 (bucket / exact kernels)
constexpr int kWorkDot = 12;       // ... and of the float32 exact route's exact_dotg per class
constexpr int kWorkKinds = 20;     // 0: omax_short (q path), 1: bellman_short, 2/3: omax_medium E = 2/4, 4..19: classes

__device__ __forceinline__ const int* forced_row(const ActionArgs& a) {
    return a.forced ? a.forced + (a.forced_td ? (a.horizon - a.k) * (long long)a.n : 0) : nullptr;
}
__device__ __forceinline__ int* chosen_row(const ActionArgs& a) {
    return a.chosen ? a.chosen + (a.chosen_td ? (a.horizon - a.k) * (long long)a.n : 0) : nullptr;
}

// Block-wide residual fold and, for the finalizing launch, the stop test.
// Every thread of the block must call this exactly once.
template <class T>
__device__ void iteration_epilogue(unsigned long long my, const ActionArgs& a, T eps, Ctl* ctl) {
    using N = Num<T>;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, my, o);
        my = other > my ? other : my;
    }
    __shared__ unsigned long long wmax[32];
    __shared__ bool last;
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = wmax[i] > m ? wmax[i] : m;
        if (m) atomicMax(&ctl->res_bits[a.k & 1], m);
        last = false;
        if (a.finalize) {
            // peer exchange: this block's stores into the peers' value buffers are visible system-wide
            // before it counts as arrived
            if (a.peers) __threadfence_system();
            else __threadfence();
            last = atomicAdd(&ctl->arrive, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        const unsigned long long rb = atomicAdd(&ctl->res_bits[a.k & 1], 0ull);
        if (a.peers) {
            // publish this shard's residual and iteration k to every rank (itself included); the stop test
            // runs in peer_sync_stop once every rank has published
            const PeerTable& pt = *a.peers;
            for (int p = 0; p < pt.world; ++p)
                *reinterpret_cast<volatile unsigned long long*>(pt.res[p] + (a.k & 1) * kMaxWorld + pt.rank) = rb;
            __threadfence_system();
            for (int p = 0; p < pt.world; ++p) st_release_sys(pt.flag[p] + pt.rank, static_cast<unsigned long long>(a.k));
        }
        const T res = N::from_res_bits(rb);
        ctl->k = a.k;
        ctl->res_last = static_cast<double>(res);
        ctl->res_bits[(a.k + 1) & 1] = 0ull;
        if (a.work)
            for (int i = 0; i < kWorkKinds; ++i) a.work[((a.k + 1) & 1) * kWorkKinds + i] = 0u;
        ctl->arrive = 0u;
        if (a.record_only) {
            // the global residual is reduced across ranks by the sharded driver
        } else if (a.finite) {
            if (a.k >= a.horizon) ctl->done = 1;
        } else if (res <= eps) {
            ctl->done = 1;
        } else if (a.k >= a.max_iterations) {
            ctl->done = 1;
            ctl->status = 1;
        }
        __threadfence();
    }
}

// Barrier-free variant for kernels whose warps finish at different times:
// warps fold into shared memory and the last warp of the block to arrive
// carries the block's result to ctl (and, when finalizing, the stop test).
// `s_res` / `s_arrived` must be zeroed before the block's first __syncthreads.
template <class T>
__device__ void warp_epilogue(unsigned long long my, const ActionArgs& a, T eps, Ctl* ctl,
                              unsigned long long* s_res, unsigned* s_arrived) {
    using N = Num<T>;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, my, o);
        my = other > my ? other : my;
    }
    if ((threadIdx.x & 31) != 0) return;
    if (my) atomicMax(s_res, my);
    __threadfence_block();
    if (atomicAdd(s_arrived, 1u) != (blockDim.x >> 5) - 1) return;
    __threadfence_block();
    const unsigned long long m = *reinterpret_cast<volatile unsigned long long*>(s_res);
    if (m) atomicMax(&ctl->res_bits[a.k & 1], m);
    if (!a.finalize) return;
    __threadfence();
    if (atomicAdd(&ctl->arrive, 1u) != gridDim.x - 1) return;
    __threadfence();
    const unsigned long long rb = atomicAdd(&ctl->res_bits[a.k & 1], 0ull);
    const T res = N::from_res_bits(rb);
    ctl->k = a.k;
    ctl->res_last = static_cast<double>(res);
    ctl->res_bits[(a.k + 1) & 1] = 0ull;
    if (a.work)
        for (int i = 0; i < kWorkKinds; ++i) a.work[((a.k + 1) & 1) * kWorkKinds + i] = 0u;
    ctl->arrive = 0u;
    if (a.record_only) {
    } else if (a.finite) {
        if (a.k >= a.horizon) ctl->done = 1;
    } else if (res <= eps) {
        ctl->done = 1;
    } else if (a.k >= a.max_iterations) {
        ctl->done = 1;
        ctl->status = 1;
    }
    __threadfence();
}

// One thread per state of `states` (or of all local states when null), from
// the per-column expectations q.
template <class T>
__global__ void __launch_bounds__(256)
action_reduce(ActionArgs a, int nstates, const int* __restrict__ states, const T* __restrict__ q,
              const T* __restrict__ vin, T* __restrict__ vout, const T* __restrict__ rewards, T discount, T eps,
              Ctl* __restrict__ ctl) {
    using N = Num<T>;
    pdl_enter();
    if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
    const int* forced = forced_row(a);
    int* chosen = chosen_row(a);
    unsigned long long my = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nstates; i += gridDim.x * blockDim.x) {
        const int s = states ? states[i] : i;
        const T prev = vin[a.state_begin + s];
        T best;
        int best_c = -1;
        if (a.frozen && a.frozen[s]) {
            best = prev;
        } else {
            int cb = a.stateptr[s], ce = a.stateptr[s + 1];
            if (forced && forced[s] >= 0) {
                cb = forced[s];
                ce = cb + 1;
            }
            best = cb < ce ? q[cb] : prev; // a state without columns keeps its value
            best_c = cb < ce ? cb : -1;
            for (int c = cb + 1; c < ce; ++c) {
                const T x = q[c];
                if (a.maximize ? (x > best) : (x < best)) { // ties keep the lowest column
                    best = x;
                    best_c = c;
                }
            }
        }
        if (rewards) best = N::add(rewards[s], N::mul(discount, best));
        vout[a.state_begin + s] = best;
        if (a.peers) { // the new value goes straight into every peer's V_k buffer (NVLink stores)
            const PeerTable& pt = *a.peers;
            for (int p = 0; p < pt.world; ++p)
                if (p != pt.rank) static_cast<T*>(pt.v[p][a.k & 1])[a.state_begin + s] = best;
        }
        if (chosen) chosen[s] = best_c;
        const unsigned long long rb = N::res_bits(fabs(N::sub(best, prev)));
        my = rb > my ? rb : my;
    }
    iteration_epilogue<T>(my, a, eps, ctl);
}

// ---------------------------------------------------------------------------
// Fused Bellman step for "short states": states whose columns all have <= 32
// entries, packed by the host scheduler into state-aligned batches of <= 16
// columns (slots padded with -1).  Per batch the warp runs the column O-max
// of omax_short (same 3-deep pipeline), sums each column in row order, then
// lane j reduces state j over its columns, applies frozen / forced /
// reward, writes V_k and the chosen column and folds the residual — one
// kernel per iteration, no q round trip.
template <class T, bool kPess, int kBlocks>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kBlocks)
bellman_short(int nbatch, const int* __restrict__ slots, const int2* __restrict__ bstates,
              const long long* __restrict__ colptr, const int* __restrict__ rows, const T* __restrict__ lower,
              const T* __restrict__ gap, const T* __restrict__ rem, const T* __restrict__ vin, T* __restrict__ vout,
              const T* __restrict__ rewards, T discount, T eps, ActionArgs a, Ctl* __restrict__ ctl) {
    using N = Num<T>;
    using Bits = typename N::Bits;
    pdl_enter();
    if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
    __shared__ T xs[kWarpsPerBlock][kShortBatch][kShortLen + 1];
    __shared__ unsigned long long s_res;
    __shared__ unsigned s_arrived;
    if (threadIdx.x == 0) {
        s_res = 0ull;
        s_arrived = 0u;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarpsPerBlock + w, nw = gridDim.x * kWarpsPerBlock;
    unsigned* work = a.work + (a.k & 1) * kWorkKinds + 1;
    const int* forced = forced_row(a);
    int* chosen = chosen_row(a);
    const int* __restrict__ stateptr = a.stateptr;
    unsigned long long myres = 0;

    auto next_batch = [&]() -> int {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(work, 1u);
        return nw + static_cast<int>(__shfl_sync(kFull, t, 0));
    };
    int bt = gw;
    if (bt < nbatch) {
        int nbt = next_batch();
        // window: lane j < 16 -> slot j of batch bt, lane 16 + j -> slot j of batch nbt
        int mc = -1, mlen = 0, ms0 = 0, mns = 0;
        long long mbeg = 0;
        T mrem = T(0);
        auto load_meta = [&](int b) {
            mc = -1;
            mlen = 0;
            mbeg = 0;
            mrem = T(0);
            ms0 = 0;
            mns = 0;
            if (b < nbatch) {
                const int2 bi = __ldg(bstates + b);
                ms0 = bi.x;
                mns = bi.y;
                mc = __ldg(slots + b * kShortBatch + (lane & (kShortBatch - 1)));
                if (mc >= 0) {
                    mbeg = __ldg(colptr + mc);
                    mlen = static_cast<int>(__ldg(colptr + mc + 1) - mbeg);
                    mrem = __ldg(rem + mc);
                }
            }
        };
        load_meta(lane < kShortBatch ? bt : nbt);
        // state-side prefetch for the current batch (used at its end)
        int s0 = 0, ns = 0, cs = 0, ce = 0, fz = 0, fc = -1;
        T prev = T(0), rw = T(0);
        auto load_states = [&]() {
            s0 = __shfl_sync(kFull, ms0, 0);
            ns = __shfl_sync(kFull, mns, 0);
            if (lane < ns) {
                const int s = s0 + lane;
                cs = __ldg(stateptr + s);
                ce = __ldg(stateptr + s + 1);
                prev = __ldg(vin + a.state_begin + s);
                fz = a.frozen ? a.frozen[s] : 0;
                fc = forced ? __ldg(forced + s) : -1;
                rw = rewards ? __ldg(rewards + s) : T(0);
            }
        };
        load_states();

        // pipeline prologue: data of slot 0, rows of slot 1
        long long bn = __shfl_sync(kFull, mbeg, 0), bnn = __shfl_sync(kFull, mbeg, 1);
        int Ln = __shfl_sync(kFull, mlen, 0), Lnn = __shfl_sync(kFull, mlen, 1);
        int rowA = lane < Ln ? __ldg(rows + bn + lane) : 0;
        T lc = T(0), gc = T(0), vc = T(0);
        int Lc = Ln;
        if (lane < Ln) {
            lc = __ldg(lower + bn + lane);
            gc = __ldg(gap + bn + lane);
            vc = __ldg(vin + rowA);
        }
        bn = bnn;
        Ln = Lnn;
        rowA = lane < Ln ? __ldg(rows + bn + lane) : 0;
        bnn = __shfl_sync(kFull, mbeg, 2);
        Lnn = __shfl_sync(kFull, mlen, 2);

        for (;;) {
#pragma unroll 2
            for (int s = 0; s < kShortBatch; ++s) {
                T ln = T(0), gn = T(0), vn = T(0);
                if (lane < Ln) {
                    ln = __ldg(lower + bn + lane);
                    gn = __ldg(gap + bn + lane);
                    vn = __ldg(vin + rowA);
                }
                const int rowB = lane < Lnn ? __ldg(rows + bnn + lane) : 0;
                const T r = __shfl_sync(kFull, mrem, s);
                const bool valid = lane < Lc;
                Bits key = valid ? order_key<T>(vc, kPess) : ~Bits(0);
                T p = lc;
                T avail = r, consumed = T(0);
                for (int nsel = 0; avail > T(0) && nsel < Lc; ++nsel) {
                    const int sel = warp_argmin_sentinel(key);
                    const T gs = __shfl_sync(kFull, gc, sel);
                    {
                        const bool me = lane == sel;
                        const T pn = N::add(lc, gc < avail ? gc : avail);
                        p = me ? pn : p;
                        key = me ? ~Bits(0) : key;
                    }
                    consumed = N::add(consumed, gs);
                    avail = N::sub(r, consumed);
                }
                if (valid) xs[w][s][lane] = N::mul(vc, p);
                lc = ln;
                gc = gn;
                vc = vn;
                Lc = Ln;
                rowA = rowB;
                bn = bnn;
                Ln = Lnn;
                bnn = __shfl_sync(kFull, mbeg, s + 3);
                Lnn = __shfl_sync(kFull, mlen, s + 3);
            }
            __syncwarp();
            // column expectations in row order (omax.hpp:169-173): lane t -> slot t
            T qv = T(0);
            if (lane < kShortBatch && mc >= 0) {
                for (int i = 0; i < mlen; ++i) qv = N::add(qv, xs[w][lane][i]);
            }
            __syncwarp();
            // action reduction: lane j -> state s0 + j (bellman.hpp:88-115)
            {
                const int c0 = __shfl_sync(kFull, mc, 0);
                const int lo = cs - c0, na = ce - cs;
                const int maxa = __reduce_max_sync(kFull, lane < ns ? na : 0);
                T best = __shfl_sync(kFull, qv, lane < ns ? lo : 0);
                int bestc = lo;
                for (int j = 1; j < maxa; ++j) {
                    const T x = __shfl_sync(kFull, qv, lane < ns && j < na ? lo + j : 0);
                    if (j < na && (a.maximize ? (x > best) : (x < best))) { // ties keep the lowest column
                        best = x;
                        bestc = lo + j;
                    }
                }
                const T fq = __shfl_sync(kFull, qv, fc >= 0 && lane < ns ? fc - c0 : 0);
                if (lane < ns) {
                    const int s = s0 + lane;
                    int bc;
                    if (fz) {
                        best = prev;
                        bc = -1;
                    } else if (fc >= 0) {
                        best = fq;
                        bc = fc;
                    } else if (na <= 0) {
                        best = prev;
                        bc = -1;
                    } else {
                        bc = c0 + bestc;
                    }
                    if (rewards) best = N::add(rw, N::mul(discount, best));
                    vout[a.state_begin + s] = best;
                    if (chosen) chosen[s] = bc;
                    const unsigned long long rb = N::res_bits(fabs(N::sub(best, prev)));
                    myres = rb > myres ? rb : myres;
                }
            }
            bt = nbt;
            if (bt >= nbatch) break;
            nbt = next_batch();
            const int c2 = __shfl_down_sync(kFull, mc, kShortBatch);
            const long long b2 = __shfl_down_sync(kFull, mbeg, kShortBatch);
            const int l2 = __shfl_down_sync(kFull, mlen, kShortBatch);
            const T r2 = __shfl_down_sync(kFull, mrem, kShortBatch);
            const int s02 = __shfl_down_sync(kFull, ms0, kShortBatch);
            const int ns2 = __shfl_down_sync(kFull, mns, kShortBatch);
            if (lane < kShortBatch) {
                mc = c2;
                mbeg = b2;
                mlen = l2;
                mrem = r2;
                ms0 = s02;
                mns = ns2;
            } else {
                load_meta(nbt);
            }
            load_states();
        }
    }
    warp_epilogue<T>(myres, a, eps, ctl, &s_res, &s_arrived);
}

// Stop test of a sharded iteration k (external_stop; solver.hpp:127-134).
// After the all-gather every shard holds both iterates V_k and V_{k-1} in
// full, so the global residual max |V_k - V_{k-1}| is computed here on each
// shard over the whole vector (n x 2 x 8 B read) instead of by a collective;
// the last block to finish evaluates the stop test.
template <class T>
__global__ void __launch_bounds__(256)
global_stop_test(int n, const T* __restrict__ vk, const T* __restrict__ vk1, Ctl* ctl, long long k, int finite,
                 long long horizon, long long max_iterations, T eps) {
    using N = Num<T>;
    if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
    unsigned long long my = 0;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
        const unsigned long long rb = N::res_bits(fabs(N::sub(vk[s], vk1[s])));
        my = rb > my ? rb : my;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(kFull, my, o);
        my = other > my ? other : my;
    }
    __shared__ unsigned long long wmax[8];
    __shared__ bool last;
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = my;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = wmax[i] > m ? wmax[i] : m;
        if (m) atomicMax(&ctl->res_bits[k & 1], m);
        __threadfence();
        last = atomicAdd(&ctl->arrive_stop, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    ctl->arrive_stop = 0u;
    const T res = N::from_res_bits(atomicAdd(&ctl->res_bits[k & 1], 0ull));
    ctl->res_last = static_cast<double>(res);
    if (finite) {
        if (k >= horizon) ctl->done = 1;
    } else if (res <= eps) {
        ctl->done = 1;
    } else if (k >= max_iterations) {
        ctl->done = 1;
        ctl->status = 1;
    }
    __threadfence();
}

// Stop test of iteration k of a peer-exchange sharded solve (solver.hpp:127-134).
// One warp: lane p waits until rank p has published iteration k into this
// shard's window (its V_k slice stores precede the flag: system-scope
// release / acquire), then the max of the published residuals decides, so
// every rank takes the same decision from the same numbers.  A rank that
// already stopped returns at once (every rank stops at the same k, so no
// flag of a later iteration is ever awaited).  Launched without PDL early
// release, so the next iteration's kernels start only after it.
template <class T>
__global__ void __launch_bounds__(32)
peer_sync_stop(Ctl* ctl, const PeerTable* __restrict__ pt, long long k, int finite, long long horizon,
               long long max_iterations, T eps) {
    using N = Num<T>;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (*reinterpret_cast<const volatile int*>(&ctl->done)) return;
    const int lane = threadIdx.x;
    const int world = pt->world;
    const unsigned long long* flags = pt->flag[pt->rank];
    const unsigned long long* res = pt->res[pt->rank] + (k & 1) * kMaxWorld;
    unsigned long long m = 0;
    if (lane < world) {
        while (ld_acquire_sys(flags + lane) < static_cast<unsigned long long>(k)) __nanosleep(64);
        m = *reinterpret_cast<const volatile unsigned long long*>(res + lane);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(kFull, m, o);
        m = x > m ? x : m;
    }
    if (lane != 0) return;
    const T r = N::from_res_bits(m);
    ctl->res_last = static_cast<double>(r);
    if (finite) {
        if (k >= horizon) ctl->done = 1;
    } else if (r <= eps) {
        ctl->done = 1;
    } else if (k >= max_iterations) {
        ctl->done = 1;
        ctl->status = 1;
    }
    __threadfence();
}

template <class T>
__global__ void residual_vector(int n, const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out) {
    using N = Num<T>;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
        out[s] = fabs(N::sub(a[s], b[s]));
}

} // namespace rimdp_dev
