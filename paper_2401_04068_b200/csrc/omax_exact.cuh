// Bit-exact many-pick long columns (33 .. 8192 entries) for float32 models.
//
// Why: at float32 one ulp of the values (1-2e-6 near 10-20) is of the order
// of the stop tolerance (1e-6), so the stop test is met only at an exact
// float32 fixed point and the iteration count depends on every rounding.  The
// tree-order kernels (omax_bucket / omax_wbucket / omax_select) make the
// reference's greedy decisions but sum in a different order; the kernels
// below reproduce the reference's three sequential chains exactly:
//   value_ordering (omax.hpp:41-58)        sort by (key(V[row]), position)
//   omaximize_sequential (omax.hpp:98-112) consumed += gap along that order
//   omax_expectation (omax.hpp:164-174)    dot += V[row] * p in row order
//
// Two passes per size class 2^LG:
//
//  exact_sort   one CTA per column.  The (key, position) sort is a counting
//               sort over B = 2^LG equal-width buckets of the column's own
//               key range (bucket index monotone in the key, so buckets are
//               contiguous in the order and ties share a bucket), then each
//               entry's rank inside its bucket is counted exactly against the
//               bucket's other members (unique composite keys, any scatter
//               order): O(L) work for spread-out values.  Writes, indexed by
//               the column's store offset (global scratch, no host sizes):
//                 S[sorted j]  = gap of the j-th entry in the order
//                 POS[i]       = sorted position of entry i (row order)
//                 VS[i]        = V[row_i]
//               A column with a bucket of more than kExactMaxBucket entries
//               (heavy ties / clustered values) goes to a fallback list for
//               the bitonic omax_sorted<.., kExact = true>.
//  exact_dot    one warp per column.  Lane 0 walks S sequentially (the
//               reference's `consumed` chain) and turns every picked slot into
//               its extra share min(gap, avail); then the warp forms the
//               products V_i * (l_i + extra) of 128 row-order entries at a time
//               (coalesced loads, the extra gathered by POS) into shared
//               memory and lane 0 adds them sequentially, while the next
//               chunk's loads are in flight.  Only the two dependent chains are
//               serial; everything else is 32-wide.
#pragma once

#include "omax_kernels.cuh"

namespace rimdp_dev {

constexpr int kExactMaxBucket = 32;

template <int LG>
struct ExactShape {
    static constexpr int N = 1 << LG;  // class capacity (and bucket count)
    static constexpr int NT = N / 8 < 64 ? 64 : (N / 8 > 512 ? 512 : N / 8);
    static constexpr int E = N / NT;   // entries per thread
    static constexpr int NW = NT / 32;
    static constexpr size_t smem() { return ((N + 1) * 4 + 15) / 16 * 16 + (size_t)N * 8; }
};

// Exclusive scan in place of cnt[0 .. NT*E), cnt[NT*E] = total.  Thread t owns
// the E consecutive counters [t*E, t*E+E).  Contains two block barriers.
template <int NT, int E>
__device__ __forceinline__ void block_exclusive_scan(unsigned* cnt, unsigned* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned v[E];
    unsigned run = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        v[e] = cnt[tid * E + e];
        run += v[e];
    }
    unsigned incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    unsigned base = incl - run;
    for (int w = 0; w < wid; ++w) base += wsum[w];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        cnt[tid * E + e] = base;
        base += v[e];
    }
    if (tid == NT - 1) cnt[NT * E] = base;
    __syncthreads();
}

template <bool kPess, int LG>
__global__ void __launch_bounds__(ExactShape<LG>::NT)
exact_sort(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
           const int* __restrict__ rows, const float* __restrict__ gap, const float* __restrict__ V,
           float* __restrict__ S, unsigned short* __restrict__ POS, float* __restrict__ VS,
           int* __restrict__ fb_list, int* __restrict__ fb_count, int* __restrict__ fb_other,
           const Ctl* __restrict__ ctl, const unsigned long long* __restrict__ vrange, unsigned* __restrict__ work) {
    using Sh = ExactShape<LG>;
    constexpr int N = Sh::N, NT = Sh::NT, E = Sh::E;
    pdl_enter_class(ctl);
    // the other launch parity's fallback count is cleared even by a no-op launch after the stop: the host
    // flips the parity for every launch
    if (blockIdx.x == 0 && threadIdx.x == 0 && fb_other) *fb_other = 0;
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned* cnt = reinterpret_cast<unsigned*>(smem_raw);                                       // N + 1
    unsigned long long* tmp = reinterpret_cast<unsigned long long*>(smem_raw + ((N + 1) * 4 + 15) / 16 * 16);
    __shared__ unsigned wsum[32];
    __shared__ int over;
    const int tid = threadIdx.x;
    // equal-width buckets over the value vector's range (value_range, one launch per iteration), in
    // adversary order (w = V pessimistic, -V optimistic): fl(w - w_min) * scale truncated is
    // non-decreasing in w, so buckets are contiguous in the (key, position) order and equal values share
    // one.  (Buckets over the order keys would not do: the keys of float values are logarithmic, so half
    // of [0, 1) would land in 1/24 of them.)  A column sampling random states spreads over about the
    // whole range, ~1 entry per bucket.
    const float vlo = value_of_key<float>(static_cast<unsigned>(__ldg(vrange)), true);
    const float vhi = value_of_key<float>(static_cast<unsigned>(__ldg(vrange + 1)), true);
    const float wmin = kPess ? vlo : -vhi, wmax = kPess ? vhi : -vlo;
    const float width = __fsub_rn(wmax, wmin);
    const float scale = width > 0.f && width < 3.0e38f ? __fdiv_rn(static_cast<float>(N), width) : 0.f;
    // columns are taken dynamically (work counter; the first one per CTA is blockIdx.x): thread 0 claims
    // the CTA's next column at the start of this one, every thread reads it behind the histogram barrier
    __shared__ int next_slot[2];
    int next_item = nlist, par = 0;
    for (int item = blockIdx.x; item < nlist; item = next_item, par ^= 1) {
        if (tid == 0) next_slot[par] = work ? static_cast<int>(gridDim.x + atomicAdd(work, 1u)) : item + static_cast<int>(gridDim.x);
        const int c = list[item];
        const long long b0 = colptr[c];
        const int L = static_cast<int>(colptr[c + 1] - b0);
        for (int k = tid; k <= N; k += NT) cnt[k] = 0u;
        __syncthreads();
        // every read of the previous column's flag happened before the barrier above (racecheck-clean)
        if (tid == 0) over = 0;
        unsigned key[E];
        float g[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = tid + e * NT;
            key[e] = ~0u;
            g[e] = 0.f;
            if (j < L) {
                const float v = __ldg(V + __ldg(rows + b0 + j));
                VS[b0 + j] = v;
                g[e] = __ldg(gap + b0 + j);
                key[e] = static_cast<unsigned>(order_key<float>(v, kPess));
            }
        }
        int bk[E];
        unsigned slot[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = tid + e * NT;
            bk[e] = 0;
            slot[e] = 0;
            if (j < L) {
                const float v = value_of_key<float>(key[e], kPess);
                const float x = __fmul_rn(__fsub_rn(kPess ? v : -v, wmin), scale);
                bk[e] = x < static_cast<float>(N - 1) ? static_cast<int>(x) : N - 1;
                slot[e] = atomicAdd(&cnt[bk[e]], 1u);
            }
        }
        __syncthreads();
        next_item = next_slot[par];
        block_exclusive_scan<NT, E>(cnt, wsum);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = tid + e * NT;
            if (j < L) tmp[cnt[bk[e]] + slot[e]] = (static_cast<unsigned long long>(key[e]) << 13) | j;
        }
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = tid + e * NT;
            if (j < L) {
                const unsigned s0 = cnt[bk[e]], s1 = cnt[bk[e] + 1];
                if (s1 - s0 > static_cast<unsigned>(kExactMaxBucket)) {
                    over = 1;
                } else {
                    const unsigned long long mine = (static_cast<unsigned long long>(key[e]) << 13) | j;
                    unsigned r = 0;
                    for (unsigned k = s0; k < s1; ++k) r += tmp[k] < mine;
                    const unsigned sp = s0 + r;
                    S[b0 + sp] = g[e];
                    POS[b0 + j] = static_cast<unsigned short>(sp);
                }
            }
        }
        __syncthreads();
        if (tid == 0) {
            if (over) fb_list[atomicAdd(fb_count, 1)] = c;
        }
    }
}

constexpr int kExactDotWarps = 8;

// Lane 0's share of the greedy over 128 sorted gaps staged in sb: four steps
// per shared-memory vector load, the `consumed` chain as the only serial
// dependency (a step after the stop only makes avail smaller, so the chain
// runs unconditionally and `alive` decides what counts).  Returns the number
// of picks in the chunk; sb[k] becomes min(gap_k, avail_k) for each pick.
__device__ __forceinline__ int exact_walk_chunk(float* sb, int m, float r, float& consumed) {
    using N_ = Num<float>;
    float4* s4 = reinterpret_cast<float4*>(sb);
    bool alive = true;
    int picks = 0;
    const int m4 = m & ~3;
    float4 nxt = m4 > 0 ? s4[0] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < m4; k += 4) {
        const float4 gq = nxt;
        if (k + 4 < m4) nxt = s4[(k >> 2) + 1];
        float4 e;
        float a = N_::sub(r, consumed);
        alive = alive && a > 0.f;
        picks += alive;
        e.x = gq.x < a ? gq.x : a;
        consumed = N_::add(consumed, gq.x);
        a = N_::sub(r, consumed);
        alive = alive && a > 0.f;
        picks += alive;
        e.y = gq.y < a ? gq.y : a;
        consumed = N_::add(consumed, gq.y);
        a = N_::sub(r, consumed);
        alive = alive && a > 0.f;
        picks += alive;
        e.z = gq.z < a ? gq.z : a;
        consumed = N_::add(consumed, gq.z);
        a = N_::sub(r, consumed);
        alive = alive && a > 0.f;
        picks += alive;
        e.w = gq.w < a ? gq.w : a;
        consumed = N_::add(consumed, gq.w);
        s4[k >> 2] = e;
        if (!alive) return picks;
    }
    for (int k = m4; k < m; ++k) {
        const float a = N_::sub(r, consumed);
        if (!(a > 0.f)) return picks;
        const float gk = sb[k];
        sb[k] = gk < a ? gk : a;
        consumed = N_::add(consumed, gk);
        ++picks;
    }
    return picks;
}

__global__ void __launch_bounds__(kExactDotWarps * 32)
exact_dot(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
          const float* __restrict__ lower, const float* __restrict__ rem, float* __restrict__ S,
          const unsigned short* __restrict__ POS, const float* __restrict__ VS, float* __restrict__ q,
          const Ctl* __restrict__ ctl, unsigned* __restrict__ /*work: static assignment*/) {
    using N_ = Num<float>;
    pdl_enter();
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    __shared__ __align__(16) float buf[kExactDotWarps][128];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float* sb = buf[w];
    for (int item = blockIdx.x * kExactDotWarps + w; item < nlist; item += gridDim.x * kExactDotWarps) {
        const int c = list[item];
        const long long b0 = colptr[c];
        const int L = static_cast<int>(colptr[c + 1] - b0);
        const float r = rem[c];
        // ---- the greedy (omax.hpp:102-110) along the sorted gaps, 128 at a time ----
        // lane k of the warp holds sorted entries k, k+32, k+64, k+96 of the chunk; the next chunk is
        // loaded while lane 0 walks the current one
        float consumed = 0.f;
        int J = L;
        float gv[4], gn[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = u * 32 + lane;
            gv[u] = j < L ? S[b0 + j] : 0.f;
        }
        // exact (f64) sum of the sorted gaps walked so far: the chunk sums of <= 128 float32 gaps of one column
        // are exact in double
        double P = 0.0;
        for (int j0 = 0; j0 < L; j0 += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u) sb[u * 32 + lane] = gv[u];
            double cs = (double)gv[0] + (double)gv[1] + (double)gv[2] + (double)gv[3];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + 128 + u * 32 + lane;
                gn[u] = j < L ? S[b0 + j] : 0.f;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(kFull, cs, o);
            const int m = L - j0 < 128 ? L - j0 : 128;
            // fast chunk: the sequential float32 `consumed` after any entry of the chunk is at most the exact
            // prefix times (1 + 1.01 (j0 + m) 2^-24) (positive terms); below rem it stays below rem, so every
            // entry is a full pick (extra = gap, already in S) and the walk continues: only the chain runs
            P += cs;
            const bool fast = P * (1.0 + 1.02 * (double)(j0 + m) * 0x1p-24) < (double)r; // 2% slack: f64 rounding of P
            __syncwarp();
            int picks = m;
            if (fast) {
                if (lane == 0) {
                    const float4* s4 = reinterpret_cast<const float4*>(sb);
                    const int m4 = m >> 2;
#pragma unroll 8
                    for (int k = 0; k < m4; ++k) {
                        const float4 g4 = s4[k];
                        consumed = N_::add(consumed, g4.x);
                        consumed = N_::add(consumed, g4.y);
                        consumed = N_::add(consumed, g4.z);
                        consumed = N_::add(consumed, g4.w);
                    }
                    for (int k = m4 * 4; k < m; ++k) consumed = N_::add(consumed, sb[k]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) gv[u] = gn[u];
                __syncwarp();
                continue;
            }
            if (lane == 0) picks = exact_walk_chunk(sb, m, r, consumed);
            picks = __shfl_sync(kFull, picks, 0);
            __syncwarp();
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = u * 32 + lane;
                if (k < picks) S[b0 + j0 + k] = sb[k];
                gv[u] = gn[u];
            }
            __syncwarp();
            if (picks < m) {
                J = j0 + picks;
                break;
            }
        }
        // ---- row-order expectation (omax.hpp:169-173), 128 products at a time ----
        float dot = 0.f;
        int sp[4];
        float lw[4], vw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = u * 32 + lane;
            sp[u] = i < L ? POS[b0 + i] : 0x7fffffff;
            lw[u] = i < L ? __ldg(lower + b0 + i) : 0.f;
            vw[u] = i < L ? VS[b0 + i] : 0.f;
        }
        for (int i0 = 0; i0 < L; i0 += 128) {
            float ex[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) ex[u] = sp[u] < J ? S[b0 + sp[u]] : 0.f;
            float x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = N_::mul(vw[u], sp[u] < J ? N_::add(lw[u], ex[u]) : lw[u]);
            // the next chunk's row-order data is in flight during the serial sum
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + 128 + u * 32 + lane;
                sp[u] = i < L ? POS[b0 + i] : 0x7fffffff;
                lw[u] = i < L ? __ldg(lower + b0 + i) : 0.f;
                vw[u] = i < L ? VS[b0 + i] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) sb[u * 32 + lane] = x[u];
            __syncwarp();
            if (lane == 0) {
                const int m = L - i0 < 128 ? L - i0 : 128;
                const float4* s4 = reinterpret_cast<const float4*>(sb);
                const int m4 = m >> 2;
#pragma unroll 8
                for (int k = 0; k < m4; ++k) {
                    const float4 v = s4[k];
                    dot = N_::add(dot, v.x);
                    dot = N_::add(dot, v.y);
                    dot = N_::add(dot, v.z);
                    dot = N_::add(dot, v.w);
                }
                for (int k = m4 * 4; k < m; ++k) dot = N_::add(dot, sb[k]);
            }
            __syncwarp();
        }
        if (lane == 0) q[c] = dot;
    }
}

// exact_dot with G columns per warp (G = 2: lanes 0-15 take list item 2p,
// lanes 16-31 item 2p + 1), each lane holding 8 entries of its group's
// chunk of CH = 8 x 32/G entries.  The serial chains (the walk's `consumed`,
// the row-order dot) run on the G group leaders side by side, so every
// serial warp instruction advances G columns — the single-column kernel is
// issue-bound (80% issue-active) on exactly those chains.  The class lists
// are sorted by length, so the columns of a warp need about as many chunks.
// Same arithmetic in the same order as exact_dot: the same bits.
template <int G>
__global__ void __launch_bounds__(kExactDotWarps * 32)
exact_dotg(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
           const float* __restrict__ lower, const float* __restrict__ rem, float* __restrict__ S,
           const unsigned short* __restrict__ POS, const float* __restrict__ VS, float* __restrict__ q,
           const Ctl* __restrict__ ctl, unsigned* __restrict__ work) {
    using N_ = Num<float>;
    constexpr int U = 8;       // entries per lane per chunk
    constexpr int LPC = 32 / G; // lanes per column
    constexpr int CH = U * LPC; // chunk
    pdl_enter();
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    __shared__ __align__(16) float buf[kExactDotWarps][G][CH];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, h = lane / LPC, hl = lane % LPC;
    float* sb = buf[w][h];
    const int ngroups = (nlist + G - 1) / G;
    // column groups are taken dynamically (work counter; the first one per warp is its index): lane 0
    // claims the warp's next group at the start of this one, the warp reads it after the walk
    const int nwarps = gridDim.x * kExactDotWarps;
    int next_pr = ngroups;
    for (int pr = blockIdx.x * kExactDotWarps + w; pr < ngroups; pr = next_pr) {
        unsigned claim = 0;
        if (lane == 0) claim = work ? static_cast<unsigned>(nwarps) + atomicAdd(work, 1u) : static_cast<unsigned>(pr + nwarps);
        const int item = G * pr + h;
        const bool valid = item < nlist;
        const int c = valid ? list[item] : 0;
        const long long b0 = valid ? colptr[c] : 0;
        const int L = valid ? static_cast<int>(colptr[c + 1] - b0) : 0;
        const float r = valid ? rem[c] : 0.f;
        // ---- the greedy (omax.hpp:102-110) along the sorted gaps, CH at a time per group ----
        float consumed = 0.f;
        int J = L;
        float gv[U], gn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = u * LPC + hl;
            gv[u] = j < L ? S[b0 + j] : 0.f;
        }
        double P = 0.0;
        bool walking = L > 0;
        for (int j0 = 0; __any_sync(kFull, walking); j0 += CH) {
#pragma unroll
            for (int u = 0; u < U; ++u) sb[u * LPC + hl] = gv[u];
            double cs = 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) cs += (double)gv[u];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = j0 + CH + u * LPC + hl;
                gn[u] = walking && j < L ? S[b0 + j] : 0.f;
            }
#pragma unroll
            for (int o = LPC / 2; o > 0; o >>= 1) cs += __shfl_xor_sync(kFull, cs, o);
            const int m = L - j0 < CH ? L - j0 : CH;
            P += cs;
            // fast chunk (see exact_dot): every entry is a full pick, only the chain runs
            const bool fast = walking && P * (1.0 + 1.02 * (double)(j0 + m) * 0x1p-24) < (double)r;
            __syncwarp();
            int picks = m;
            if (walking && hl == 0) {
                if (fast) {
                    const float4* s4 = reinterpret_cast<const float4*>(sb);
                    const int m4 = m >> 2;
#pragma unroll 8
                    for (int k = 0; k < m4; ++k) {
                        const float4 g4 = s4[k];
                        consumed = N_::add(consumed, g4.x);
                        consumed = N_::add(consumed, g4.y);
                        consumed = N_::add(consumed, g4.z);
                        consumed = N_::add(consumed, g4.w);
                    }
                    for (int k = m4 * 4; k < m; ++k) consumed = N_::add(consumed, sb[k]);
                } else {
                    picks = exact_walk_chunk(sb, m, r, consumed);
                }
            }
            picks = __shfl_sync(kFull, picks, h * LPC);
            __syncwarp();
            if (walking && !fast) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = u * LPC + hl;
                    if (k < picks) S[b0 + j0 + k] = sb[k];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) gv[u] = gn[u];
            __syncwarp();
            if (walking && picks < m) {
                J = j0 + picks;
                walking = false;
            } else if (walking && j0 + CH >= L) {
                walking = false;
            }
        }
        next_pr = static_cast<int>(__shfl_sync(kFull, claim, 0));
        // ---- row-order expectation (omax.hpp:169-173), CH products at a time per group ----
        int Lmax = L;
#pragma unroll
        for (int o = LPC; o < 32; o <<= 1) Lmax = max(Lmax, __shfl_xor_sync(kFull, Lmax, o));
        float dot = 0.f;
        int sp[U];
        float lw[U], vw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = u * LPC + hl;
            sp[u] = i < L ? POS[b0 + i] : 0x7fffffff;
            lw[u] = i < L ? __ldg(lower + b0 + i) : 0.f;
            vw[u] = i < L ? VS[b0 + i] : 0.f;
        }
        for (int i0 = 0; i0 < Lmax; i0 += CH) {
            float x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const float ex = sp[u] < J ? S[b0 + sp[u]] : 0.f;
                x[u] = N_::mul(vw[u], sp[u] < J ? N_::add(lw[u], ex) : lw[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + CH + u * LPC + hl;
                sp[u] = i < L ? POS[b0 + i] : 0x7fffffff;
                lw[u] = i < L ? __ldg(lower + b0 + i) : 0.f;
                vw[u] = i < L ? VS[b0 + i] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) sb[u * LPC + hl] = x[u];
            __syncwarp();
            if (hl == 0 && i0 < L) {
                const int m = L - i0 < CH ? L - i0 : CH;
                const float4* s4 = reinterpret_cast<const float4*>(sb);
                const int m4 = m >> 2;
#pragma unroll 8
                for (int k = 0; k < m4; ++k) {
                    const float4 v = s4[k];
                    dot = N_::add(dot, v.x);
                    dot = N_::add(dot, v.y);
                    dot = N_::add(dot, v.z);
                    dot = N_::add(dot, v.w);
                }
                for (int k = m4 * 4; k < m; ++k) dot = N_::add(dot, sb[k]);
            }
            __syncwarp();
        }
        if (hl == 0 && valid) q[c] = dot;
    }
}

// ---------------------------------------------------------------------------
// Columns of 33 .. 256 entries in one pass, one warp per column
// (exact_warp): the same sort, greedy walk and row-order dot as exact_sort +
// exact_dot, but everything stays in the warp's shared-memory slice — no
// block barriers, no global scratch, no second launch.  For these short
// classes the two-pass route paid its per-column fixed costs twice (29 ns
// per transition on C5 f32 against ~8 for the long classes).
template <int LG>
struct ExactWarpShape {
    static constexpr int N = 1 << LG;   // 64 .. 256
    static constexpr int E = N / 32;    // entries per lane
    static constexpr int W = 8;         // warps per block
#ifndef RIMDP_EXACT_WARP_MINBLOCKS
#define RIMDP_EXACT_WARP_MINBLOCKS 3
#endif
    // 256 entries: 3 blocks per SM (<= 85 registers) instead of the 2 that 90 registers allow
    static constexpr int MinBlocks = LG >= 8 ? RIMDP_EXACT_WARP_MINBLOCKS : 1;
    // per warp: tmp u64[N] (then the dot's staging buffer) | cnt u32[N + 4] | S f32[N]; each lane keeps its
    // entries' V, lower, gap and sorted position in registers
    static constexpr size_t warp_bytes = (size_t)N * 8 + (size_t)(N + 4) * 4 + (size_t)N * 4;
    static constexpr size_t smem() { return W * ((warp_bytes + 15) / 16 * 16); }
};

template <bool kPess, int LG>
__global__ void __launch_bounds__(ExactWarpShape<LG>::W * 32, ExactWarpShape<LG>::MinBlocks)
exact_warp(int nlist, const int* __restrict__ list, const long long* __restrict__ colptr,
           const int* __restrict__ rows, const float* __restrict__ lower, const float* __restrict__ gap,
           const float* __restrict__ rem, const float* __restrict__ V, float* __restrict__ q,
           int* __restrict__ fb_list, int* __restrict__ fb_count, int* __restrict__ fb_other,
           const Ctl* __restrict__ ctl) {
    using Sh = ExactWarpShape<LG>;
    using N_ = Num<float>;
    constexpr int N = Sh::N, E = Sh::E, W = Sh::W;
    pdl_enter_class(ctl);
    if (blockIdx.x == 0 && threadIdx.x == 0 && fb_other) *fb_other = 0; // the other parity's count (see exact_sort)
    if (ctl && *reinterpret_cast<const volatile int*>(&ctl->done)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* base = smem_raw + (size_t)w * ((Sh::warp_bytes + 15) / 16 * 16);
    unsigned long long* tmp = reinterpret_cast<unsigned long long*>(base);
    float* xb = reinterpret_cast<float*>(base);                       // dot staging, after the sort
    unsigned* cnt = reinterpret_cast<unsigned*>(base + (size_t)N * 8);
    float* S = reinterpret_cast<float*>(base + (size_t)N * 8 + (size_t)(N + 4) * 4);
    // static assignment (a dynamic claim per column, as exact_sort, measured no better for warp kernels)
    for (int item = blockIdx.x * W + w; item < nlist; item += gridDim.x * W) {
        const int c = list[item];
        const long long b0 = colptr[c];
        const int L = static_cast<int>(colptr[c + 1] - b0);
        const float r = rem[c];
        // ---- load, keys, the column's value range ----
        unsigned key[E];
        float g[E], v[E], lo[E];
        float wlo = 3.0e38f, whi = -3.0e38f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            key[e] = ~0u;
            g[e] = v[e] = lo[e] = 0.f;
            if (j < L) {
                v[e] = __ldg(V + __ldg(rows + b0 + j));
                g[e] = __ldg(gap + b0 + j);
                lo[e] = __ldg(lower + b0 + j);
                key[e] = static_cast<unsigned>(order_key<float>(v[e], kPess));
                const float wv = kPess ? __fadd_rn(v[e], 0.f) : -__fadd_rn(v[e], 0.f);
                wlo = fminf(wlo, wv);
                whi = fmaxf(whi, wv);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wlo = fminf(wlo, __shfl_xor_sync(kFull, wlo, o));
            whi = fmaxf(whi, __shfl_xor_sync(kFull, whi, o));
        }
        const float width = __fsub_rn(whi, wlo);
        const float scale = width > 0.f && width < 3.0e38f ? __fdiv_rn(static_cast<float>(N), width) : 0.f;
        // ---- counting sort by (key, position): N buckets of the value range, then ranks inside buckets ----
#pragma unroll
        for (int e = 0; e < (N + 4) / 32 + 1; ++e)
            if (lane + 32 * e < N + 4) cnt[lane + 32 * e] = 0u;
        __syncwarp();
        int bk[E];
        unsigned slot[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            bk[e] = 0;
            slot[e] = 0;
            if (j < L) {
                const float wv = kPess ? __fadd_rn(v[e], 0.f) : -__fadd_rn(v[e], 0.f);
                const float x = __fmul_rn(__fsub_rn(wv, wlo), scale);
                bk[e] = x < static_cast<float>(N - 1) ? static_cast<int>(x) : N - 1;
                slot[e] = atomicAdd(&cnt[bk[e]], 1u);
            }
        }
        __syncwarp();
        {   // exclusive scan of cnt[0 .. N): lane l owns counters [l E, l E + E)
            unsigned cv[E], run = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                cv[e] = cnt[lane * E + e];
                run += cv[e];
            }
            unsigned incl = run;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += y;
            }
            unsigned bse = incl - run;
            __syncwarp();
#pragma unroll
            for (int e = 0; e < E; ++e) {
                cnt[lane * E + e] = bse;
                bse += cv[e];
            }
            if (lane == 31) cnt[N] = bse;
        }
        __syncwarp();
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            if (j < L) tmp[cnt[bk[e]] + slot[e]] = (static_cast<unsigned long long>(key[e]) << 13) | j;
        }
        __syncwarp();
        bool over = false;
        int sp[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int j = lane + 32 * e;
            sp[e] = N;
            if (j < L) {
                const unsigned s0 = cnt[bk[e]], s1 = cnt[bk[e] + 1];
                if (s1 - s0 > static_cast<unsigned>(kExactMaxBucket)) {
                    over = true;
                } else {
                    const unsigned long long mine = (static_cast<unsigned long long>(key[e]) << 13) | j;
                    unsigned rk = 0;
                    for (unsigned k = s0; k < s1; ++k) rk += tmp[k] < mine;
                    sp[e] = static_cast<int>(s0 + rk);
                    S[sp[e]] = g[e];
                }
            }
        }
        if (__any_sync(kFull, over)) { // heavy ties: the bitonic exact kernel takes the column
            if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = c;
            __syncwarp();
            continue;
        }
        __syncwarp();
        // ---- the greedy (omax.hpp:102-110) along S, provably-full chunks as in exact_dot ----
        float consumed = 0.f;
        int J = L;
        double P = 0.0;
        for (int j0 = 0; j0 < L; j0 += 128) {
            const int m = L - j0 < 128 ? L - j0 : 128;
            double cs = 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = u * 32 + lane;
                cs += k < m ? (double)S[j0 + k] : 0.0;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cs += __shfl_xor_sync(kFull, cs, o);
            P += cs;
            const bool fast = P * (1.0 + 1.02 * (double)(j0 + m) * 0x1p-24) < (double)r;
            int picks = m;
            if (lane == 0) {
                if (fast) {
                    const float4* s4 = reinterpret_cast<const float4*>(S + j0);
                    int k = 0;
                    for (; k + 4 <= m; k += 4) {
                        const float4 g4 = s4[k >> 2];
                        consumed = N_::add(consumed, g4.x);
                        consumed = N_::add(consumed, g4.y);
                        consumed = N_::add(consumed, g4.z);
                        consumed = N_::add(consumed, g4.w);
                    }
                    for (; k < m; ++k) consumed = N_::add(consumed, S[j0 + k]);
                } else {
                    picks = exact_walk_chunk(S + j0, m, r, consumed);
                }
            }
            picks = __shfl_sync(kFull, picks, 0);
            __syncwarp();
            if (picks < m) {
                J = j0 + picks;
                break;
            }
        }
        // ---- row-order expectation (omax.hpp:169-173): 32 products staged, lane 0 adds them in order ----
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i0 = 32 * e;
            if (i0 >= L) break;
            // entry i0 + lane is this lane's entry e: its V, lower and sorted position are in registers
            xb[lane] = lane + i0 < L ? N_::mul(v[e], sp[e] < J ? N_::add(lo[e], S[sp[e]]) : lo[e]) : 0.f;
            __syncwarp();
            if (lane == 0) {
                const int m = L - i0 < 32 ? L - i0 : 32;
                if (m == 32) {
                    const float4* x4 = reinterpret_cast<const float4*>(xb);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const float4 y = x4[k];
                        dot = N_::add(dot, y.x);
                        dot = N_::add(dot, y.y);
                        dot = N_::add(dot, y.z);
                        dot = N_::add(dot, y.w);
                    }
                } else {
                    for (int k = 0; k < m; ++k) dot = N_::add(dot, xb[k]);
                }
            }
            __syncwarp();
        }
        if (lane == 0) q[c] = dot;
        __syncwarp();
    }
}

} // namespace rimdp_dev
