// Host runtime of the B200 engine: device transition store, solve loop and
// the extern "C" boundary declared in include/rimdp_b200.h.
//
// Replaces, for Value = double|float:
//   IntervalMDP / IntervalProbabilities storage   imdp.hpp:26-181, interval.hpp:34-304
//   detail::make_plan outputs (V0, frozen, ...)   solver.hpp:40-80 (built by the caller)
//   detail::iterate                              solver.hpp:85-137
//   detail::bellman_step_impl / bellman_step     bellman.hpp:75-133
//   parallel_for_index (per-step thread fork)    parallel.hpp:27-68  -> CUDA grid
#include "rimdp_b200.h"

#include "generator.cuh"
#include "omax_exact.cuh"
#include "omax_kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <charconv>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

using namespace rimdp_dev;

namespace {

thread_local std::string g_err_msg;
thread_local rimdp_error_info g_err_info{};
thread_local int g_shard_col_offset = 0; // rimdp_multi_create: global index of the shard being created's column 0

struct Fail {
    int status;
};

int fail(int status, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err_msg = buf;
    g_err_info = rimdp_error_info{};
    g_err_info.status = status;
    return status;
}

#define CK(expr)                                                                                          \
    do {                                                                                                  \
        cudaError_t e_ = (expr);                                                                          \
        if (e_ != cudaSuccess) {                                                                          \
            fail(e_ == cudaErrorMemoryAllocation ? RIMDP_ERR_OUT_OF_MEMORY : RIMDP_ERR_CUDA, "%s: %s (%s:%d)", \
                 #expr, cudaGetErrorString(e_), __FILE__, __LINE__);                                     \
            throw Fail{g_err_info.status};                                                                \
        }                                                                                                 \
    } while (0)

size_t elem_size(rimdp_dtype t) { return t == RIMDP_F64 ? 8 : 4; }

// Device memory comes from the device's default stream-ordered pool with an
// unlimited release threshold: memory a destroyed model gives back stays
// mapped in the pool and serves the next model's allocations without driver
// calls (cudaMalloc of fresh pages measured 1-14 ms per model and up to
// 330 ms on a fresh box; model destroy 26 ms with cudaFree).
void* dev_alloc(size_t b) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    {
        static std::mutex mu;
        static bool configured[64] = {};
        std::lock_guard<std::mutex> lk(mu);
        if (!configured[dev & 63]) {
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, dev));
            unsigned long long thr = ~0ull;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
            configured[dev & 63] = true;
        }
    }
    void* p = nullptr;
    CK(cudaMallocAsync(&p, b, 0));
    CK(cudaStreamSynchronize(0)); // usable from every stream from here on
    return p;
}

// Returns an allocation to the pool once every stream of its device is idle
// (the memory may still be in use by queued work on any of them).
void dev_free(void* p, int dev) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != dev) cudaSetDevice(dev);
    cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    if (cur >= 0 && cur != dev) cudaSetDevice(cur);
}

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    ~DevBuf() { release(); }
    void release() {
        if (p) dev_free(p, dev);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        release();
        CK(cudaGetDevice(&dev));
        p = dev_alloc(b > 0 ? b : 16);
        bytes = b;
    }
    template <class U>
    U* as() const { return static_cast<U*>(p); }
};

// Column classes of the scheduler: <= 32 entries ->
// warp kernel (omax_short); longer columns whose greedy stops after a few
// picks -> pipelined warp kernel with 2 or 4 entries per lane (omax_medium,
// <= 64 / <= 128 entries) or the exact warp kernel (omax_long, any length);
// the rest -> one CTA per column, sorted (omax_sorted), by power-of-two size
// class 2^6 .. 2^13.
// tiny classes: <= 4, <= 8, <= 16 entries (4 / 8 / 16 lanes per column), and single entries (1 lane)
constexpr int kTinyClasses = 4;
constexpr int kSortedMinLog = 6, kSortedMaxLog = 13, kSortedClasses = kSortedMaxLog - kSortedMinLog + 1;
constexpr double kExactPickBudget = 4.0;

struct ColumnLists {
    DevBuf short_list, exact_list, medium_list[2], tiny_list[kTinyClasses], sorted_list[kSortedClasses];
    int n_short = 0, n_exact = 0, n_medium[2] = {}, n_tiny[kTinyClasses] = {}, n_sorted[kSortedClasses] = {};
    // tiny classes packed in list order (pack_columns): begins [n + 1], rem [n], rows / lower / gap
    DevBuf tiny_beg[kTinyClasses], tiny_rem[kTinyClasses], tiny_rows[kTinyClasses], tiny_lower[kTinyClasses],
        tiny_gap[kTinyClasses];
    bool tiny_packed[kTinyClasses] = {};
    std::vector<int> tiny_host[kTinyClasses]; // the lists on the host, until packed
    int total_sorted() const {
        int t = 0;
        for (int i = 0; i < kSortedClasses; ++i) t += n_sorted[i];
        return t;
    }
};

struct Infeasible {
    int col;
    int kind;
    double sum;
};

struct SolveState {
    DevBuf v[2], q, chosen, frozen, rewards, forced, res, ctl, work;
    void* vb[2] = {nullptr, nullptr}; // the value double buffer of the solve: v[0..1], or the exchange window
    bool has_frozen = false, has_rewards = false, has_forced = false;
    int forced_td = 0;
    int pess = 1, maxi = 1, finite = 1;
    long long horizon = 0, max_iterations = 0;
    double eps = 0, discount = 0;
    int chosen_td = 0;
    long long launched = 0; // iterations enqueued so far
    int launches_last = 0;  // kernels the last enqueued iteration launched (gpu_launches in bench.py)
    bool active = false;
    bool record_only = false;
    // kernel timing (rimdp_profile_*)
    bool profile = false;
    std::vector<cudaEvent_t> events;
    size_t events_used = 0;
    ~SolveState() {
        for (cudaEvent_t e : events) cudaEventDestroy(e);
    }
    std::vector<int> host_frozen_copy; // for infeasible-column checks
};

} // namespace

constexpr int kMaxSideStreams = 8;

struct rimdp_model {
    rimdp_dtype dtype = RIMDP_F64;
    int device = 0;
    cudaStream_t stream = nullptr;
    int n = 0;         // states owned by this store (local)
    int n_global = 0;  // length of the value vector
    long long value_capacity = 0; // allocated entries of the value buffers (>= n_global)
    int state_begin = 0;
    int ncols = 0;
    long long nnz = 0;
    int maxlen = 0;
    DevBuf stateptr, colptr, rows, lower, gap, rem, maxgap, infeasible, quoted, scratch;
    DevBuf batch_slots, batch_states, long_states;
    ColumnLists all;                          // every column by class (rimdp_column_values)
    ColumnLists qp;                           // columns of the q-path states (iterations)
    bool all_is_qp = false;                   // every column is on the q path: `all` is `qp`
    const ColumnLists& all_lists() const { return all_is_qp ? qp : all; }
    int nbatch = 0, nlong_states = 0;         // fused short-state batches / q-path states
    bool all_states_q = true;                 // every state on the q path, in order: no state list
    bool short_pair = true;                   // 17-32-entry class on omax_pair (nearly full columns)
    std::vector<int> h_stateptr;
    std::vector<Infeasible> infeasible_cols;
    long long device_bytes = 0;
    long long pack_bytes = 0; // the packed tiny classes (pack_tiny)
    int sm_count = 148;
    int short_blocks_per_sm = 4;
    bool bitonic = false;                     // many-pick long columns: bitonic sort instead of selection
    bool long_exact = false;                  // few-pick long columns: row-order omax_long (RIMDP_LONG=exact)
    bool exact_sorted = false;                // many-pick long columns: sorted + sequential sums (float32 default)
    bool bucket = true;                       // columns > 256 entries: value buckets first (RIMDP_BUCKET=0: off)
    DevBuf fallback[kSortedClasses];          // per size class: [count A, count B, columns...] omax_bucket -> omax_select
    int fallback_parity[kSortedClasses] = {}; // which count the next omax_bucket launch of the class uses
    // merged fallback list of one column pass (see begin_merged_fallback): [count A, count B, columns...]
    DevBuf fb_all;
    int fb_all_parity = 0;
    bool fb_merge = false;                    // the class launchers append to fb_* and launch no fallback kernel
    unsigned* work_cur = nullptr;             // the column pass's work counters (launch_columns)
    int* fbm_list = nullptr;
    int* fbm_count = nullptr;
    int* fbm_other = nullptr;
    int fbm_cap = 0;                          // columns the merged list can hold (the pass's many-pick columns)
    int fb_maxlg = 0;                         // largest size class that appended (0: no fallback kernel)
    int medium_blocks_per_sm = 3;             // omax_medium occupancy variant (RIMDP_MEDIUM_BLOCKS=4: <= 64 registers)
    int nstreams = 1;                         // column classes fanned out over this many streams (RIMDP_STREAMS)
    cudaStream_t side[kMaxSideStreams] = {};  // fork/join streams for concurrent column classes
    cudaEvent_t fork_ev = nullptr, join_ev[kMaxSideStreams] = {};
    cudaStream_t ls = nullptr;                // stream the next class launch goes to
    size_t l2_persist = 0;                    // bytes of L2 set aside for the value vector (0: none)
    bool pdl_now = false;                     // launches of the current iteration use PDL (launch_iteration)
    bool gate_needed = false;                 // early class kernels: a plain launch must open the column phase
    bool early_now = false;                   // the current iteration's class kernels start early (class_early)
    // PDL for kernels that wait for their predecessor's output (selection / exact_dot / fallback passes,
    // action_reduce): not behind an early-starting class kernel, whose immediate trigger would let their
    // blocks sit resident at griddepcontrol.wait and take the running class kernel's SMs
    bool pdl_wait_ok() const { return pdl_now && !early_now; }
    DevBuf xs_gap, xs_pos, xs_val;            // exact_sort -> exact_dot scratch (float32 exact route), by store offset
    DevBuf vrange;                            // value_range slots [2][min, max] (order keys), for omax_bucket
    int vrange_parity = 0;
    const unsigned long long* vrange_cur = nullptr; // slot filled for the current launch_columns
    SolveState s;
    // peer exchange of a state-sharded solve (rimdp_exchange_*): this shard's window (cudaMalloc, IPC
    // exportable) = [V buffer 0 | V buffer 1 | residual slots [2][kMaxWorld] | flags [kMaxWorld]]
    struct Exchange {
        void* win = nullptr;
        size_t vbytes = 0;               // bytes of one value buffer (capacity x element, 256-aligned)
        long long cap = 0;               // value buffer capacity in entries
        bool connected = false;
        bool shared_device = false;      // some peer window lives on this shard's device (tests on one GPU)
        int world = 1, rank = 0;
        std::vector<void*> opened;       // IPC-opened peer windows
        DevBuf table;                    // PeerTable
        unsigned long long* res() const { return reinterpret_cast<unsigned long long*>(static_cast<char*>(win) + 2 * vbytes); }
        unsigned long long* flags() const { return res() + 2 * kMaxWorld; }
        static size_t tail() { return 3 * kMaxWorld * sizeof(unsigned long long); }
    } x;
    int col_offset = 0;                       // multi-GPU shard: global index of local column 0 (error reports)
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const Fail& e) {
        return e.status;
    } catch (const std::bad_alloc&) {
        return fail(RIMDP_ERR_OUT_OF_MEMORY, "host allocation failed");
    } catch (...) {
        return fail(RIMDP_ERR_INTERNAL, "unexpected exception");
    }
}

// ---------------------------------------------------------------------------
// Large host->device uploads from pageable memory (the caller's CSC arrays):
// a process-wide pool of worker threads, each with its own stream and two
// pinned staging chunks, copies disjoint parts in parallel — memcpy into a
// pinned chunk, DMA it, reuse the chunk once its event has completed.  A
// single pageable cudaMemcpy is staged by the driver on one thread (~9 GB/s
// measured for config 2's 260 MB); this runs the host copies on several
// cores.  RIMDP_UPLOAD_THREADS=0 falls back to plain cudaMemcpyAsync.
struct UploadJob {
    void* dst;
    const void* src;
    size_t bytes;
};

struct StagingPool {
    std::mutex mu;
    int device = -1;
    int workers = 0;
    static constexpr size_t kChunk = 4u << 20;
    std::vector<void*> bufs;          // 2 per worker, pinned
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;  // 2 per worker
};

StagingPool& staging_pool(int device) {
    static std::mutex mu;
    static std::vector<std::unique_ptr<StagingPool>> pools;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)pools.size() <= device) pools.resize(device + 1);
    if (!pools[device]) pools[device].reset(new StagingPool);
    return *pools[device];
}

int upload_threads() {
    static const int t = [] {
        if (const char* e = getenv("RIMDP_UPLOAD_THREADS")) return std::max(0, std::min(atoi(e), 32));
        const int hw = (int)std::thread::hardware_concurrency();
        return std::max(1, std::min(8, hw / 2));
    }();
    return t;
}

// True when the whole range [p, p + bytes) is page-locked host memory (cudaHostAlloc / cudaHostRegister):
// the copy engines then read it directly, no staging.
bool pinned_host(const void* p, size_t bytes) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    if (a.type != cudaMemoryTypeHost || bytes == 0) return a.type == cudaMemoryTypeHost;
    // a pinned allocation covers the last byte too (separately pinned neighbours would also pass, and are
    // just as good for the DMA)
    if (cudaPointerGetAttributes(&a, static_cast<const char*>(p) + bytes - 1) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void upload_many(int device, cudaStream_t stream, const std::vector<UploadJob>& jobs) {
    size_t total = 0;
    bool all_pinned = true;
    for (const auto& j : jobs) {
        total += j.bytes;
        if (j.bytes && all_pinned) all_pinned = pinned_host(j.src, j.bytes);
    }
    const int W = upload_threads();
    if (W == 0 || total < (32u << 20) || all_pinned) {
        for (const auto& j : jobs)
            if (j.bytes) CK(cudaMemcpyAsync(j.dst, j.src, j.bytes, cudaMemcpyHostToDevice, stream));
        return;
    }
    StagingPool& P = staging_pool(device);
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.workers < W) {
        for (int w = P.workers; w < W; ++w) {
            cudaStream_t st;
            CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            P.streams.push_back(st);
            for (int k = 0; k < 2; ++k) {
                void* b = nullptr;
                CK(cudaHostAlloc(&b, StagingPool::kChunk, cudaHostAllocDefault));
                P.bufs.push_back(b);
                cudaEvent_t ev;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                P.events.push_back(ev);
            }
        }
        P.workers = W;
        P.device = device;
    }
    // earlier work on `stream` (allocations, memsets) is ordered before the copies
    CK(cudaStreamSynchronize(stream));
    std::atomic<int> err{0};
    std::vector<std::thread> th;
    const size_t per = (total + W - 1) / W;
    for (int w = 0; w < W; ++w) {
        th.emplace_back([&, w] {
            if (cudaSetDevice(device) != cudaSuccess) {
                err = 1;
                return;
            }
            const size_t lo = std::min(total, per * w), hi = std::min(total, per * (w + 1));
            size_t base = 0, i = 0;
            for (const auto& j : jobs) {
                const size_t a = std::max(lo, base), b = std::min(hi, base + j.bytes);
                for (size_t off = a; off < b; off += StagingPool::kChunk, ++i) {
                    const size_t n = std::min(StagingPool::kChunk, b - off);
                    const int slot = 2 * w + (int)(i & 1);
                    if (i >= 2 && cudaEventSynchronize(P.events[slot]) != cudaSuccess) err = 1;
                    std::memcpy(P.bufs[slot], static_cast<const char*>(j.src) + (off - base), n);
                    if (cudaMemcpyAsync(static_cast<char*>(j.dst) + (off - base), P.bufs[slot], n,
                                        cudaMemcpyHostToDevice, P.streams[w]) != cudaSuccess ||
                        cudaEventRecord(P.events[slot], P.streams[w]) != cudaSuccess)
                        err = 1;
                }
                base += j.bytes;
            }
            if (cudaStreamSynchronize(P.streams[w]) != cudaSuccess) err = 1;
        });
    }
    for (auto& t : th) t.join();
    if (err) {
        fail(RIMDP_ERR_CUDA, "staged upload failed: %s", cudaGetErrorString(cudaGetLastError()));
        throw Fail{RIMDP_ERR_CUDA};
    }
}

// Kernels of the iteration loop are launched with programmatic stream
// serialization (PDL): a kernel's blocks become resident while its
// predecessor drains and start with griddepcontrol.wait (pdl_enter), so the
// launch latency between the column kernels and the action kernel is hidden.
// It is used when an iteration is at most kPdlMaxKernels launches (C2-C4:
// 2 launches, 3-4% per iteration on C2); with the dozen column classes of a
// power-law model it measured slower (C5 f64 4.24 vs 3.25 ms per iteration),
// so those launch plainly.  RIMDP_PDL=0 launches everything plainly.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("RIMDP_PDL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

// Kernel launches issued by this thread (every launch of the iteration loop goes through launch_pdl or
// counts itself), so launch_iteration can report how many kernels one iteration really launched.
thread_local long long g_launches = 0;

template <class... KArgs, class... Args>
void launch_pdl(bool on, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
    ++g_launches;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = on && pdl_enabled() ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// RIMDP_TRACE=1: host-side phase times of model upload and solve on stderr.
struct PhaseTrace {
    const char* what;
    bool on;
    std::chrono::steady_clock::time_point t0, last;
    explicit PhaseTrace(const char* w) : what(w) {
        static const bool env_on = [] {
            const char* e = getenv("RIMDP_TRACE");
            return e && atoi(e) != 0;
        }();
        on = env_on;
        t0 = last = std::chrono::steady_clock::now();
    }
    void mark(const char* phase) {
        if (!on) return;
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[rimdp] %s %s %.2f ms\n", what, phase,
                std::chrono::duration<double, std::milli>(t - last).count());
        last = t;
    }
    ~PhaseTrace() {
        if (on)
            fprintf(stderr, "[rimdp] %s total %.2f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

int grid_for(long long work, int per_block, int sm_count, int blocks_per_sm) {
    long long g = (work + per_block - 1) / per_block;
    g = std::min<long long>(g, (long long)sm_count * blocks_per_sm);
    return (int)std::max<long long>(g, 1);
}

template <class U>
void upload_list(rimdp_model* m, DevBuf& buf, const std::vector<U>& v) {
    buf.ensure(sizeof(U) * std::max<size_t>(1, v.size()));
    if (!v.empty()) CK(cudaMemcpyAsync(buf.p, v.data(), sizeof(U) * v.size(), cudaMemcpyHostToDevice, m->stream));
}

// Routing mode for long columns (tests): RIMDP_LONG=exact (every long column
// on the exact warp kernel), sorted (every one on the bitonic CTA kernel),
// select (every one on the selection kernels, no value buckets).
// 17-32-entry columns: two per warp step (omax_pair) by default; RIMDP_PAIR=0 -> one per step (omax_short)
bool pair_mode() {
    static const bool on = [] {
        const char* e = getenv("RIMDP_PAIR");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

bool env_flag(const char* name) {
    const char* e = getenv(name);
    return e && atoi(e) != 0;
}

int long_mode() {
    const char* e = getenv("RIMDP_LONG");
    if (!e) return 0;
    if (!strcmp(e, "exact")) return 1;
    if (!strcmp(e, "sorted")) return 2;
    if (!strcmp(e, "select")) return 3;
    return 0;
}

// Class of one column given its length, remainder and largest gap.
//   0: short   1: exact long   2: medium (E = 2)   3: medium (E = 4)
//   4 + i: sorted, size class 2^(kSortedMinLog + i)
//   kClassTiny + i: <= 4 << i entries (i = 0, 1, 2), several columns per warp; kClassTiny + 3: one entry
constexpr int kClassMedium = 2, kClassSorted = 4, kClassTiny = 16;
__host__ __device__ int column_class(long long len, double rem, double maxgap, int mode) {
    if (len == 1) return kClassTiny + 3; // one lane per column (32 per warp step)
    if (len <= 4) return kClassTiny;
    if (len <= 8) return kClassTiny + 1;
    if (len <= 16) return kClassTiny + 2;
    if (len <= kShortLen) return 0;
    if (len > (1ll << kSortedMaxLog)) return 1; // beyond the largest CTA sort: exact warp kernel
    bool sorted;
    if (mode) {
        sorted = mode >= 2;
    } else {
        // the greedy needs at least rem / maxgap picks; few picks -> exact argmin kernels
        sorted = rem > 0 && (maxgap <= 0 || rem > kExactPickBudget * maxgap);
    }
    if (!sorted) {
        if (mode == 1) return 1;
        if (len <= 2 * kShortLen) return kClassMedium;
        if (len <= 4 * kShortLen) return kClassMedium + 1;
        return 1;
    }
    int lg = kSortedMinLog;
    while ((1ll << lg) < len) ++lg;
    return kClassSorted + (lg - kSortedMinLog);
}

// by_length: sort each many-pick class list by decreasing length (longest first balances the persistent
// grids of the float32 exact route)
// cols == nullptr: every column, in order
// The partition is parallel over host threads (per-thread class counts, then each thread writes its part
// of every list at its offset: the lists keep increasing column order); the length sort is a stable
// counting sort (a class spans at most 2^kSortedMaxLog lengths).
void fill_lists(rimdp_model* m, ColumnLists& L, const std::vector<int>* cols, const std::vector<signed char>& cls,
                const long long* by_length = nullptr) {
    constexpr int K = 32;
    const long long n = cols ? (long long)cols->size() : (long long)cls.size();
    const int nt = (int)std::max<long long>(1, std::min<long long>({16, (long long)std::max(1u, std::thread::hardware_concurrency()),
                                                                     n / 65536 + 1}));
    std::vector<std::array<long long, K>> cnt(nt);
    auto col_at = [&](long long i) -> int { return cols ? (*cols)[i] : (int)i; };
    auto part = [&](int t, long long& b, long long& e) {
        b = n * t / nt;
        e = n * (t + 1) / nt;
    };
    auto run = [&](auto&& f) {
        std::vector<std::thread> th;
        for (int t = 1; t < nt; ++t) th.emplace_back(f, t);
        f(0);
        for (auto& x : th) x.join();
    };
    run([&](int t) {
        long long b, e;
        part(t, b, e);
        cnt[t].fill(0);
        for (long long i = b; i < e; ++i) ++cnt[t][cls[col_at(i)] & (K - 1)];
    });
    std::vector<int> out[K];
    std::vector<std::array<long long, K>> off(nt);
    for (int k = 0; k < K; ++k) {
        long long a = 0;
        for (int t = 0; t < nt; ++t) {
            off[t][k] = a;
            a += cnt[t][k];
        }
        out[k].resize(a);
    }
    run([&](int t) {
        long long b, e;
        part(t, b, e);
        std::array<long long, K> o = off[t];
        for (long long i = b; i < e; ++i) {
            const int c = col_at(i);
            const int k = cls[c] & (K - 1);
            out[k][o[k]++] = c;
        }
    });
    L.n_short = (int)out[0].size();
    L.n_exact = (int)out[1].size();
    upload_list(m, L.short_list, out[0]);
    upload_list(m, L.exact_list, out[1]);
    for (int i = 0; i < 2; ++i) {
        L.n_medium[i] = (int)out[kClassMedium + i].size();
        upload_list(m, L.medium_list[i], out[kClassMedium + i]);
    }
    for (int i = 0; i < kTinyClasses; ++i) {
        L.n_tiny[i] = (int)out[kClassTiny + i].size();
        upload_list(m, L.tiny_list[i], out[kClassTiny + i]);
        L.tiny_host[i] = std::move(out[kClassTiny + i]);
    }
    for (int i = 0; i < kSortedClasses; ++i) {
        std::vector<int>& so = out[kClassSorted + i];
        if (by_length && so.size() > 1) {
            // stable counting sort by decreasing length
            long long lo = LLONG_MAX, hi = 0;
            for (int c : so) {
                const long long len = by_length[c + 1] - by_length[c];
                lo = std::min(lo, len);
                hi = std::max(hi, len);
            }
            std::vector<long long> pos(hi - lo + 2, 0);
            for (int c : so) ++pos[hi - (by_length[c + 1] - by_length[c]) + 1];
            for (size_t x = 1; x < pos.size(); ++x) pos[x] += pos[x - 1];
            std::vector<int> sorted(so.size());
            for (int c : so) sorted[pos[hi - (by_length[c + 1] - by_length[c])]++] = c;
            so.swap(sorted);
        }
        L.n_sorted[i] = (int)so.size();
        upload_list(m, L.sorted_list[i], so);
    }
}

// Column scheduler:
//  * every column is classified by length and by how many greedy picks it
//    can need (column_class); the lists of all columns serve
//    rimdp_column_values;
//  * for iterations, with RIMDP_FUSED=1, runs of consecutive "short states"
//    (<= 16 columns, all columns <= 32 entries) are packed into state-aligned
//    batches of <= 16 column slots for the fused bellman_short kernel; the
//    remaining states take the q path (column kernels + action_reduce).
// Tiny classes of power-law models are packed in list order at upload (pack_tiny): the kernels then stream
// contiguous runs.  RIMDP_TINY_PACK=0 keeps them reading the store in place.
bool tiny_pack_enabled() {
    static const bool on = [] {
        const char* e = getenv("RIMDP_TINY_PACK");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

template <class T>
void pack_tiny(rimdp_model* m, ColumnLists& L, const long long* h_colptr) {
    for (int i = 0; i < kTinyClasses; ++i) {
        std::vector<int>& lst = L.tiny_host[i];
        L.tiny_packed[i] = false;
        if (lst.empty() || !tiny_pack_enabled()) {
            lst.clear();
            continue;
        }
        const int n = (int)lst.size();
        std::vector<long long> beg(n + 1, 0);
        for (int k = 0; k < n; ++k) beg[k + 1] = beg[k] + (h_colptr[lst[k] + 1] - h_colptr[lst[k]]);
        const size_t z = (size_t)std::max<long long>(beg[n], 1);
        const size_t need = sizeof(long long) * (n + 1) + sizeof(T) * n + (sizeof(int) + 2 * sizeof(T)) * z;
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        if (need + (size_t(2) << 30) > free_b) { // a copy is an optimisation: never trade the headroom for it
            lst.clear();
            continue;
        }
        L.tiny_beg[i].ensure(sizeof(long long) * (n + 1));
        L.tiny_rem[i].ensure(sizeof(T) * n);
        L.tiny_rows[i].ensure(sizeof(int) * z);
        L.tiny_lower[i].ensure(sizeof(T) * z);
        L.tiny_gap[i].ensure(sizeof(T) * z);
        CK(cudaMemcpyAsync(L.tiny_beg[i].p, beg.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, m->stream));
        pack_columns<T><<<grid_for(n, 256, m->sm_count, 8), 256, 0, m->stream>>>(
            n, L.tiny_list[i].as<int>(), m->colptr.as<long long>(), L.tiny_beg[i].as<long long>(), m->rows.as<int>(),
            m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), L.tiny_rows[i].as<int>(), L.tiny_lower[i].as<T>(),
            L.tiny_gap[i].as<T>(), L.tiny_rem[i].as<T>());
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(m->stream)); // `beg` is a host temporary
        L.tiny_packed[i] = true;
        m->pack_bytes += (long long)need;
        lst.clear();
        lst.shrink_to_fit();
    }
}

// column_class of every column on the device (rem / maxgap are device-computed, so the host would need
// them copied back: 16 B per column against the 1-byte class), plus the longest column and the count and
// total length of the short class (omax_pair's test): stat = [max length, short count, short entries]
template <class T>
__global__ void __launch_bounds__(256)
classify_columns(int ncols, const long long* __restrict__ colptr, const T* __restrict__ rem,
                 const T* __restrict__ maxgap, int mode, int any_long, signed char* __restrict__ cls,
                 unsigned long long* __restrict__ stat) {
    unsigned long long mx = 0, cnt = 0, tot = 0;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const long long len = colptr[c + 1] - colptr[c];
        const int k = column_class(len, any_long ? (double)rem[c] : 0.0, any_long ? (double)maxgap[c] : 0.0, mode);
        cls[c] = static_cast<signed char>(k);
        mx = static_cast<unsigned long long>(len) > mx ? static_cast<unsigned long long>(len) : mx;
        if (k == 0) {
            ++cnt;
            tot += static_cast<unsigned long long>(len);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(stat, mx);
        atomicAdd(stat + 1, cnt);
        atomicAdd(stat + 2, tot);
    }
}

template <class T>
void build_schedule(rimdp_model* m, const long long* h_colptr) {
    PhaseTrace tr("schedule");
    m->pack_bytes = 0;
    // the pick-count test (rem vs maxgap) only matters for columns longer than a warp: models without such
    // columns (config 2) skip the device -> host copy of rem / maxgap
    bool any_long = false;
    for (int c = 0; c < m->ncols && !any_long; ++c) any_long = h_colptr[c + 1] - h_colptr[c] > kShortLen;
    const int mode = long_mode();
    m->bitonic = mode == 2;
    m->long_exact = mode == 1;
    // float32: one ulp of the values is of the order of the stop tolerance, so a tree-order sum can move
    // the iteration at which max residual <= eps; every float32 column therefore takes a row-order kernel
    // (bit-identical to the reference) unless RIMDP_F32_FAST=1 (tree-order, within a few ulps)
    if (std::is_same<T, float>::value && !env_flag("RIMDP_F32_FAST")) {
        m->long_exact = m->long_exact || mode == 0;
        m->exact_sorted = mode == 0 || mode == 1;
    }
    {
        // RIMDP_LONG=select (tests) keeps every many-pick column on the selection kernels
        const char* eb = getenv("RIMDP_BUCKET");
        m->bucket = !(eb && atoi(eb) == 0) && mode != 3;
    }
    // classes on the device, one byte per column back to the host
    std::vector<signed char> cls(m->ncols);
    unsigned long long stat[3] = {0, 0, 0};
    if (m->ncols > 0) {
        DevBuf dcls, dstat;
        dcls.ensure(m->ncols);
        dstat.ensure(sizeof stat);
        CK(cudaMemsetAsync(dstat.p, 0, sizeof stat, m->stream));
        classify_columns<T><<<grid_for(m->ncols, 256, m->sm_count, 8), 256, 0, m->stream>>>(
            m->ncols, m->colptr.as<long long>(), m->rem.as<T>(), m->maxgap.as<T>(), mode, any_long ? 1 : 0,
            dcls.as<signed char>(), dstat.as<unsigned long long>());
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(cls.data(), dcls.p, m->ncols, cudaMemcpyDeviceToHost, m->stream));
        CK(cudaMemcpyAsync(stat, dstat.p, sizeof stat, cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
    }
    tr.mark("d2h");
    const int maxlen = static_cast<int>(stat[0]);
    std::vector<int> allc, qc;
    const std::vector<int>& sp = m->h_stateptr;
    const char* fz = getenv("RIMDP_FUSED");
    const bool fused = fz && atoi(fz) != 0;
    auto short_state = [&](int s) {
        if (!fused) return false;
        const int na = sp[s + 1] - sp[s];
        if (na < 1 || na > kShortBatch) return false;
        for (int c = sp[s]; c < sp[s + 1]; ++c)
            if (cls[c] != 0 && cls[c] < kClassTiny) return false;
        return true;
    };
    std::vector<int> slots, lstates;
    std::vector<int2> bstates;
    int s0 = -1, used = 0;
    // the default (no fused short-state batches): every state is a q-path state and every column a q-path
    // column, in order — the action kernel then walks the states directly (no state list)
    m->all_states_q = !fused;
    auto close_batch = [&]() {
        if (s0 < 0) return;
        for (int j = used; j < kShortBatch; ++j) slots.push_back(-1);
        s0 = -1;
        used = 0;
    };
    for (int s = 0; s < m->n && fused; ++s) {
        if (!short_state(s)) {
            close_batch();
            lstates.push_back(s);
            for (int c = sp[s]; c < sp[s + 1]; ++c) qc.push_back(c);
            continue;
        }
        const int na = sp[s + 1] - sp[s];
        if (s0 >= 0 && (used + na > kShortBatch || s - s0 >= kShortBatch)) close_batch();
        if (s0 < 0) {
            s0 = s;
            bstates.push_back(make_int2(s, 0));
        }
        for (int c = sp[s]; c < sp[s + 1]; ++c) slots.push_back(c);
        used += na;
        bstates.back().y += 1;
    }
    close_batch();
    if (fused) {
        allc.resize(m->ncols);
        for (int c = 0; c < m->ncols; ++c) allc[c] = c;
    }
    tr.mark("classify");
    m->maxlen = maxlen;
    {   // omax_pair pays off when the two columns of a step are nearly full (config 2: all 32 entries); with
        // the mixed 17-32 lengths of a power-law model (mean ~24) the pair's loop runs the longer column's
        // picks for both and measured 2% slower than omax_short
        const unsigned long long cnt = stat[1], tot = stat[2];
        m->short_pair = cnt == 0 || tot >= 28 * cnt;
    }
    // every column on the q path (the default: no fused short-state batches): the two sets of lists are the
    // same, so `all` is not built separately
    m->all_is_qp = !fused || qc.size() == allc.size();
    const long long* by_len = m->exact_sorted ? h_colptr : nullptr;
    if (!m->all_is_qp) fill_lists(m, m->all, &allc, cls, by_len);
    fill_lists(m, m->qp, fused ? &qc : nullptr, cls, by_len);
    tr.mark("fill");
    if (!m->all_is_qp) pack_tiny<T>(m, m->all, h_colptr);
    pack_tiny<T>(m, m->qp, h_colptr);
    tr.mark("lists");
    m->nbatch = (int)bstates.size();
    m->nlong_states = m->all_states_q ? m->n : (int)lstates.size();
    upload_list(m, m->batch_slots, slots);
    upload_list(m, m->batch_states, bstates);
    upload_list(m, m->long_states, lstates);
    CK(cudaStreamSynchronize(m->stream));
}

// Reference text of a float (NumericTraits::to_string, numeric.hpp:30-35: std::to_chars shortest form).
template <class T>
std::string num_text(T v) {
    char buf[64];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

// The first violation validate_entries found, as the reference's ModelError (errors.hpp:44-55,
// Violation::to_string :155-162): "<Kind> column=<j> row=<r>: <message>".
template <class T>
void report_violation(rimdp_model* m, const unsigned long long* hf) {
    const bool structural = hf[0] != ~0ull;
    const unsigned long long key = structural ? hf[0] : hf[1];
    const int col = (int)(key >> 32);
    const unsigned low = (unsigned)key;
    const long long k = structural ? (low >> 1) : (low >> 2);
    long long b = 0;
    CK(cudaMemcpy(&b, m->colptr.as<long long>() + col, sizeof b, cudaMemcpyDeviceToHost));
    int row = 0;
    T l{}, u{};
    CK(cudaMemcpy(&row, m->rows.as<int>() + b + k, sizeof row, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&l, m->lower.as<T>() + b + k, sizeof l, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&u, m->gap.as<T>() + b + k, sizeof u, cudaMemcpyDeviceToHost)); // still the upper bounds here
    std::string kind, msg;
    int vk;
    if (structural) {
        kind = "StructuralError";
        vk = 7;
        msg = (low & 1) ? "row indices not strictly increasing within column" : "row index out of range";
    } else if ((low & 3) == 2) {
        kind = "BoundOrderViolation";
        vk = 2;
        msg = "lower bound " + num_text(l) + " exceeds upper bound " + num_text(u);
    } else {
        kind = "EntryOutOfRange";
        vk = 1;
        msg = std::string((low & 3) == 0 ? "lower" : "upper") + " bound " + num_text((low & 3) == 0 ? l : u) +
              " outside [0,1]";
    }
    // Violation::to_string prints row= only for row >= 0 (errors.hpp:155-162)
    const std::string where = row >= 0 ? " row=" + std::to_string(row) : std::string();
    fail(RIMDP_ERR_INVALID_MODEL, "%s column=%d%s: %s", kind.c_str(), col + m->col_offset, where.c_str(), msg.c_str());
    g_err_info.column = col + m->col_offset;
    g_err_info.row = row;
    g_err_info.violation_kind = vk;
}

template <class T>
void prepare(rimdp_model* m) {
    m->rem.ensure(sizeof(T) * std::max(1, m->ncols));
    m->infeasible.ensure(std::max(1, m->ncols));
    m->quoted.ensure(sizeof(T) * std::max(1, m->ncols));
    m->maxgap.ensure(sizeof(T) * std::max(1, m->ncols));
    m->scratch.ensure(64);
    CK(cudaMemsetAsync(m->scratch.p, 0, 64, m->stream));
    int* counters = m->scratch.as<int>();
    unsigned long long* first = reinterpret_cast<unsigned long long*>(m->scratch.as<char>() + 16);
    const unsigned long long none[2] = {~0ull, ~0ull};
    CK(cudaMemcpyAsync(first, none, sizeof none, cudaMemcpyHostToDevice, m->stream));
    if (m->ncols > 0)
        validate_entries<T><<<grid_for(m->ncols, 8, m->sm_count, 8), 256, 0, m->stream>>>(
            m->ncols, m->colptr.as<long long>(), m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(), m->n_global, first);
    unsigned long long hf[2];
    CK(cudaMemcpyAsync(hf, first, sizeof hf, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    if (hf[0] != ~0ull || hf[1] != ~0ull) {
        report_violation<T>(m, hf);
        throw Fail{RIMDP_ERR_INVALID_MODEL};
    }
    if (m->ncols > 0)
        prepare_columns<T><<<grid_for(m->ncols, 8, m->sm_count, 8), 256, 0, m->stream>>>(
            m->ncols, m->colptr.as<long long>(), m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(),
            m->infeasible.as<unsigned char>(), m->quoted.as<T>(), m->maxgap.as<T>(), counters);
    CK(cudaGetLastError());
    int h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, counters, sizeof h, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    m->infeasible_cols.clear();
    if (h[0]) {
        std::vector<unsigned char> flags(m->ncols);
        std::vector<T> sums(m->ncols);
        CK(cudaMemcpy(flags.data(), m->infeasible.p, m->ncols, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sums.data(), m->quoted.p, sizeof(T) * m->ncols, cudaMemcpyDeviceToHost));
        for (int c = 0; c < m->ncols; ++c)
            if (flags[c]) m->infeasible_cols.push_back({c, flags[c], (double)sums[c]});
    }
}

void init_common(rimdp_model* m, int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        fail(RIMDP_ERR_NO_DEVICE, "no CUDA device visible");
        throw Fail{RIMDP_ERR_NO_DEVICE};
    }
    if (device < 0 || device >= count) {
        fail(RIMDP_ERR_INVALID_ARGUMENT, "device %d out of range (%d visible)", device, count);
        throw Fail{RIMDP_ERR_INVALID_ARGUMENT};
    }
    m->device = device;
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
    if (const char* e = getenv("RIMDP_SHORT_BLOCKS")) m->short_blocks_per_sm = atoi(e) == 5 ? 5 : 4;
    if (const char* e = getenv("RIMDP_MEDIUM_BLOCKS")) m->medium_blocks_per_sm = atoi(e) == 4 ? 4 : 3;
    if (const char* e = getenv("RIMDP_STREAMS")) m->nstreams = std::min(std::max(atoi(e), 1), kMaxSideStreams);
    if (m->nstreams > 1) {
        for (int i = 0; i < m->nstreams; ++i) CK(cudaStreamCreateWithFlags(&m->side[i], cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&m->fork_ev, cudaEventDisableTiming));
        for (int i = 0; i < m->nstreams; ++i) CK(cudaEventCreateWithFlags(&m->join_ev[i], cudaEventDisableTiming));
    }
}

// L2 residency of the gathered value vector: when
// V is large (config 4: 80 MB) the stream of column data evicts it from L2
// and every V[row] gather costs a 32-byte DRAM sector.  An access-policy
// window marks the buffer the iteration reads as persisting in a set-aside
// part of L2 (cudaLimitPersistingL2CacheSize); the window follows the double
// buffer from iteration to iteration.  Opt-in (RIMDP_L2_PERSIST=1): on
// config 4 it cuts DRAM reads from 188 to 110 GB per iteration but the
// kernel gets slower (45 vs 38 ms: profiles/round1/ncu_c4_omax_medium_*),
// so the default relies on the per-load evict-first / evict-last hints.
void setup_l2_persistence(rimdp_model* m, size_t value_bytes) {
    m->l2_persist = 0;
    const char* e = getenv("RIMDP_L2_PERSIST");
    if (!e || atoi(e) == 0) return;
    if (value_bytes < (8u << 20)) return; // small V stays in L2 anyway
    int max_persist = 0;
    if (cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, m->device) != cudaSuccess ||
        max_persist <= 0)
        return;
    // RIMDP_L2_PERSIST=1: the whole vector; =P with 2 <= P <= 100: P percent of it
    const int pct = atoi(e) >= 2 ? std::min(atoi(e), 100) : 100;
    const size_t want = std::min<size_t>((size_t)max_persist, value_bytes * (size_t)pct / 100);
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    m->l2_persist = want;
}

void set_value_window(rimdp_model* m, const void* v, size_t bytes) {
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<void*>(v);
    a.accessPolicyWindow.num_bytes = bytes;
    a.accessPolicyWindow.hitRatio = std::min(1.0f, (float)m->l2_persist / (float)std::max<size_t>(bytes, 1));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    CK(cudaStreamSetAttribute(m->stream, cudaStreamAttributeAccessPolicyWindow, &a));
}

// ---------------------------------------------------------------------------
// Solve loop

int kernels_per_iteration(const rimdp_model* m);
constexpr int kPdlMaxKernels = 3;

// Iterations of many class kernels launch them with PDL and early start (pdl_enter_class).  Measured on C5:
// float32 (exact route) 3.74 -> 3.66 ms, float64 2.38 -> 2.90 ms (the co-resident bucket kernels slow each
// other down), so it is the float32 default only.  RIMDP_CLASS_EARLY=0 / 1 forces it off / on.
bool class_early(const rimdp_model* m) {
    static const int forced = [] {
        const char* e = getenv("RIMDP_CLASS_EARLY");
        return e ? (atoi(e) != 0 ? 1 : 0) : -1;
    }();
    const bool want = forced >= 0 ? forced == 1 : m->dtype == RIMDP_F32;
    return want && pdl_enabled() && kernels_per_iteration(m) > kPdlMaxKernels && !m->l2_persist &&
           m->nstreams == 1 && m->nbatch == 0 && !(m->x.connected && m->x.shared_device);
}

template <class T>
void upload_plan(rimdp_model* m, const rimdp_plan* p) {
    SolveState& s = m->s;
    const int N = m->n_global, n = m->n;
    s.pess = p->pessimistic != 0;
    s.maxi = p->maximize != 0;
    s.finite = p->finite != 0;
    s.horizon = p->horizon;
    s.max_iterations = p->max_iterations;
    s.eps = p->eps;
    s.discount = p->discount;
    long long cap = std::max<long long>(N, m->value_capacity);
    if (m->x.connected) {
        // the exchange window holds the double buffer; its residual slots and flags restart at 0 (the driver
        // synchronises all ranks after begin, before any rank enqueues iteration 1)
        cap = m->x.cap;
        s.vb[0] = m->x.win;
        s.vb[1] = static_cast<char*>(m->x.win) + m->x.vbytes;
        CK(cudaMemsetAsync(m->x.res(), 0, rimdp_model::Exchange::tail(), m->stream));
    } else {
        s.v[0].ensure(sizeof(T) * cap);
        s.v[1].ensure(sizeof(T) * cap);
        s.vb[0] = s.v[0].p;
        s.vb[1] = s.v[1].p;
    }
    setup_l2_persistence(m, sizeof(T) * (size_t)N);
    if (cap > N) {
        CK(cudaMemsetAsync(static_cast<T*>(s.vb[0]) + N, 0, sizeof(T) * (cap - N), m->stream));
        CK(cudaMemsetAsync(static_cast<T*>(s.vb[1]) + N, 0, sizeof(T) * (cap - N), m->stream));
    }
    s.q.ensure(sizeof(T) * std::max(1, m->ncols));
    s.res.ensure(sizeof(T) * N);
    s.ctl.ensure(sizeof(Ctl));
    if (!p->initial) {
        fail(RIMDP_ERR_INVALID_ARGUMENT, "plan.initial is required");
        throw Fail{RIMDP_ERR_INVALID_ARGUMENT};
    }
    CK(cudaMemcpyAsync(s.vb[0], p->initial, sizeof(T) * N, cudaMemcpyHostToDevice, m->stream));
    CK(cudaMemcpyAsync(s.vb[1], s.vb[0], sizeof(T) * N, cudaMemcpyDeviceToDevice, m->stream));
    s.has_frozen = p->frozen != nullptr;
    s.host_frozen_copy.clear();
    if (s.has_frozen) {
        s.frozen.ensure(n);
        CK(cudaMemcpyAsync(s.frozen.p, p->frozen + m->state_begin, n, cudaMemcpyHostToDevice, m->stream));
        s.host_frozen_copy.assign(p->frozen + m->state_begin, p->frozen + m->state_begin + n);
    }
    s.has_rewards = p->rewards != nullptr;
    if (s.has_rewards) {
        s.rewards.ensure(sizeof(T) * n);
        CK(cudaMemcpyAsync(s.rewards.p, static_cast<const T*>(p->rewards) + m->state_begin, sizeof(T) * n,
                           cudaMemcpyHostToDevice, m->stream));
    }
    s.has_forced = p->forced != nullptr;
    s.forced_td = p->forced_time_dependent != 0;
    if (s.has_forced) {
        const long long rows = s.forced_td ? std::max<long long>(p->horizon, 1) : 1;
        s.forced.ensure(sizeof(int) * n * rows);
        // local slice of each row
        for (long long t = 0; t < rows; ++t)
            CK(cudaMemcpyAsync(s.forced.as<int>() + t * n, p->forced + t * N + m->state_begin, sizeof(int) * n,
                               cudaMemcpyHostToDevice, m->stream));
    }
    Ctl c{};
    c.class_early = class_early(m) ? 1 : 0;
    CK(cudaMemcpyAsync(s.ctl.p, &c, sizeof c, cudaMemcpyHostToDevice, m->stream));
    s.work.ensure(2 * kWorkKinds * sizeof(unsigned));
    CK(cudaMemsetAsync(s.work.p, 0, 2 * kWorkKinds * sizeof(unsigned), m->stream));
    s.launched = 0;
    s.active = true;
    s.record_only = p->external_stop != 0 || m->x.connected; // sharded: the stop test is global
}

template <class T, bool P, int LG, bool X = false>
void launch_sorted_class(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    using Sh = SortedShape<LG>;
    auto k = omax_sorted<T, P, LG, X>;
    const size_t smem = Sh::template smem<T>();
    static bool configured[64] = {};
    static int per_sm[64] = {};
    const int dev = m->device & 63;
    if (!configured[dev]) {
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, Sh::threads, smem));
        per_sm[dev] = std::max(per_sm[dev], 1);
        configured[dev] = true;
    }
    const int blocks = grid_for(count, 1, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_wait_ok(), k, blocks, Sh::threads, smem, m->ls, count, list.as<int>(), m->colptr.as<long long>(), m->rows.as<int>(),
                                                m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), V, q, (const Ctl*)ctl,
                                                (const int*)nullptr);
}

template <class T, bool P, int LG>
void launch_select_class(rimdp_model* m, int count, const int* list, const T* V, T* q, Ctl* ctl,
                         const int* count_dev = nullptr) {
    using Sh = SelectShape<LG>;
    auto k = omax_select<T, P, LG>;
    const size_t smem = Sh::template smem<T>();
    static bool configured[64] = {};
    static int per_sm[64] = {};
    const int dev = m->device & 63;
    if (!configured[dev]) {
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, Sh::Block, smem));
        per_sm[dev] = std::max(per_sm[dev], 1);
        configured[dev] = true;
    }
    const int blocks = grid_for(count, Sh::Groups, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_wait_ok(), k, blocks, Sh::Block, smem, m->ls, count, list, m->colptr.as<long long>(), m->rows.as<int>(),
                                              m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), V, q, ctl,
                                              count_dev);
}

// Many-pick columns of a float32 model, bit-exact (omax_exact.cuh): the
// bucket counting sort per column, then the sequential greedy and row-order
// dot per column, then the bitonic exact kernel over the columns whose
// buckets overflowed.
struct FallbackSlots;
FallbackSlots fallback_slots(rimdp_model* m, int cls, int count);

template <class T, bool P, int LG>
void launch_exact_class(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl);

// Fallback list of one size class: [count A, count B, columns...].  The
// bucket kernels count into one counter and clear the other, alternating
// between launches, so no memset sits between the kernels of an iteration.
struct FallbackSlots {
    int* list;
    int* count;
    int* other;
};

FallbackSlots fallback_slots(rimdp_model* m, int cls, int count) {
    if (m->fb_merge) {
        m->fb_maxlg = std::max(m->fb_maxlg, cls + kSortedMinLog);
        return FallbackSlots{m->fbm_list, m->fbm_count, m->fbm_other};
    }
    DevBuf& fbuf = m->fallback[cls];
    const size_t need = sizeof(int) * (size_t)(std::max(count, 1) + 2);
    if (fbuf.bytes < need) {
        fbuf.ensure(need);
        CK(cudaMemsetAsync(fbuf.p, 0, 2 * sizeof(int), m->ls));
    }
    int& par = m->fallback_parity[cls];
    FallbackSlots f{fbuf.as<int>() + 2, fbuf.as<int>() + par, fbuf.as<int>() + (par ^ 1)};
    par ^= 1;
    return f;
}

// columns per warp of the exact route's walk + dot: 2 (exact_dotg<2>, default) or RIMDP_EXACT_DOT=1 (exact_dot).
// Four per warp measured slower (C5 f32 3.89 vs 3.50 ms: 64-entry chunks, a quarter of the loading lanes)
int exact_dot_group() {
    static const int g = [] {
        const char* e = getenv("RIMDP_EXACT_DOT");
        return e && atoi(e) == 1 ? 1 : 2;
    }();
    return g;
}
using ExactDotKernel = void (*)(int, const int*, const long long*, const float*, const float*, float*,
                                const unsigned short*, const float*, float*, const Ctl*, unsigned*);
ExactDotKernel exact_dot_kernel() {
    const int g = exact_dot_group();
    return g == 1 ? exact_dot : exact_dotg<2>;
}

// The float32 exact route's fallback: the bitonic exact kernel over the listed columns (<= 2^LG entries)
template <bool P, int LG>
void launch_exact_fallback(rimdp_model* m, int count, const int* list, const int* count_dev, const float* V,
                           float* q, Ctl* ctl) {
    using SS = SortedShape<LG>;
    auto kf = omax_sorted<float, P, LG, true>;
    static bool fconf[64] = {};
    const int dev = m->device & 63;
    if (!fconf[dev]) {
        CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS::template smem<float>()));
        fconf[dev] = true;
    }
    launch_pdl(m->pdl_wait_ok(), kf, std::min(count, m->sm_count), SS::threads, SS::template smem<float>(), m->ls, count,
               list, m->colptr.as<long long>(), m->rows.as<int>(), m->lower.as<float>(), m->gap.as<float>(),
               m->rem.as<float>(), V, q, (const Ctl*)ctl, count_dev);
}

template <class T, bool P, int LG>
void launch_exact_class(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    if constexpr (std::is_same<T, float>::value && LG <= 8) {
        // <= 256 entries: one pass per column, one warp (exact_warp)
        using Sh = ExactWarpShape<LG>;
        auto k = exact_warp<P, LG>;
        static bool configured[64] = {};
        static int per_sm[64] = {};
        const int dev = m->device & 63;
        if (!configured[dev]) {
            CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem()));
            CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, Sh::W * 32, Sh::smem()));
            per_sm[dev] = std::max(per_sm[dev], 1);
            configured[dev] = true;
        }
        const FallbackSlots f = fallback_slots(m, LG - kSortedMinLog, count);
        launch_pdl(m->pdl_now, k, grid_for(count, Sh::W, m->sm_count, per_sm[dev]), Sh::W * 32, Sh::smem(), m->ls,
                   count, list.as<int>(), m->colptr.as<long long>(), m->rows.as<int>(), m->lower.as<float>(),
                   m->gap.as<float>(), m->rem.as<float>(), V, q, f.list, f.count, f.other, (const Ctl*)ctl);
        if (!m->fb_merge) launch_exact_fallback<P, LG>(m, count, f.list, f.count, V, q, ctl);
    } else if constexpr (std::is_same<T, float>::value) {
        using Sh = ExactShape<LG>;
        auto ks = exact_sort<P, LG>;
        static bool configured[64] = {};
        static int per_sm[64] = {}, dot_per_sm[64] = {};
        const int dev = m->device & 63;
        if (!configured[dev]) {
            CK(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::smem()));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], ks, Sh::NT, Sh::smem()));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&dot_per_sm[dev], exact_dot_kernel(), kExactDotWarps * 32, 0));
            per_sm[dev] = std::max(per_sm[dev], 1);
            dot_per_sm[dev] = std::max(dot_per_sm[dev], 1);
            configured[dev] = true;
        }
        const size_t nz = (size_t)std::max<long long>(m->nnz, 1);
        if (m->xs_gap.bytes < sizeof(float) * nz) {
            m->xs_gap.ensure(sizeof(float) * nz);
            m->xs_val.ensure(sizeof(float) * nz);
            m->xs_pos.ensure(sizeof(unsigned short) * nz);
        }
        const FallbackSlots f = fallback_slots(m, LG - kSortedMinLog, count);
        launch_pdl(m->pdl_now, ks, grid_for(count, 1, m->sm_count, per_sm[dev]), Sh::NT, Sh::smem(), m->ls, count,
                   list.as<int>(), m->colptr.as<long long>(), m->rows.as<int>(), m->gap.as<float>(), V,
                   m->xs_gap.as<float>(), m->xs_pos.as<unsigned short>(), m->xs_val.as<float>(), f.list, f.count,
                   f.other, (const Ctl*)ctl, m->vrange_cur,
                   m->work_cur ? m->work_cur + kWorkSorted + (LG - kSortedMinLog) : nullptr);
        const int G = exact_dot_group();
        launch_pdl(m->pdl_wait_ok(), exact_dot_kernel(), grid_for((count + G - 1) / G, kExactDotWarps, m->sm_count, dot_per_sm[dev]),
                   kExactDotWarps * 32, 0, m->ls, count, list.as<int>(), m->colptr.as<long long>(),
                   m->lower.as<float>(), m->rem.as<float>(), m->xs_gap.as<float>(),
                   (const unsigned short*)m->xs_pos.as<unsigned short>(), (const float*)m->xs_val.as<float>(), q,
                   (const Ctl*)ctl, m->work_cur ? m->work_cur + kWorkDot + (LG - kSortedMinLog) : nullptr);
        // overflowed columns: the bitonic exact kernel (after exact_dot, which wrote placeholders for them)
        if (!m->fb_merge) launch_exact_fallback<P, LG>(m, count, f.list, f.count, V, q, ctl);
    } else {
        launch_sorted_class<T, P, LG, true>(m, count, list, V, q, ctl);
    }
}

// Columns of more than 256 entries: value-bucket kernel, then the selection
// kernel over the columns it could not bracket tightly (fallback list).
template <class T, bool P, int LG>
void launch_bucket_class(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    using Sh = BucketShape<LG, T>;
    auto k = omax_bucket<T, P, LG>;
    const size_t smem = Sh::template smem<T>();
    static bool configured[64] = {};
    static int per_sm[64] = {};
    const int dev = m->device & 63;
    if (!configured[dev]) {
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, Sh::NT, smem));
        per_sm[dev] = std::max(per_sm[dev], 1);
        configured[dev] = true;
    }
    const FallbackSlots f = fallback_slots(m, LG - kSortedMinLog, count);
    const int blocks = grid_for(count, 1, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_now, k, blocks, Sh::NT, smem, m->ls, count, list.as<int>(), m->colptr.as<long long>(),
               m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), m->maxgap.as<T>(), V, q, ctl,
               f.list, f.count, f.other, m->vrange_cur,
               m->work_cur ? m->work_cur + kWorkSorted + (LG - kSortedMinLog) : nullptr);
    if (!m->fb_merge) launch_select_class<T, P, LG>(m, count, f.list, V, q, ctl, f.count);
}

// Many-pick columns of 33 .. 256 entries: warp-per-column value buckets,
// then the selection kernel over the fallback list.
template <class T, bool P, int LG>
void launch_wbucket_class(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    using Sh = WBucketShape<LG>;
    auto k = omax_wbucket<T, P, LG>;
    static int per_sm[64] = {};
    const int dev = m->device & 63;
    if (!per_sm[dev]) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, Sh::W * 32, 0));
        per_sm[dev] = std::max(per_sm[dev], 1);
    }
    const FallbackSlots f = fallback_slots(m, LG - kSortedMinLog, count);
    const int blocks = grid_for(count, Sh::W, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_now, k, blocks, Sh::W * 32, 0, m->ls, count, list.as<int>(), m->colptr.as<long long>(),
               m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), m->maxgap.as<T>(), V, q, ctl,
               f.list, f.count, f.other, m->vrange_cur);
    if (!m->fb_merge) launch_select_class<T, P, LG>(m, count, f.list, V, q, ctl, f.count);
}

// Many-pick long columns by size class: weighted quickselect (omax_select,
// default) or the bitonic-sort kernel (omax_sorted, RIMDP_LONG=sorted).
template <class T, bool P, int LG = kSortedMinLog>
void launch_sorted(rimdp_model* m, const ColumnLists& L, const T* V, T* q, Ctl* ctl) {
    if constexpr (LG <= kSortedMaxLog) {
        const int i = LG - kSortedMinLog;
        if (L.n_sorted[i] > 0) {
            if (m->exact_sorted)
                launch_exact_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (m->bitonic)
                launch_sorted_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (LG >= 9 && m->bucket)
                launch_bucket_class<T, P, (LG >= 9 ? LG : 9)>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (LG <= 8 && m->bucket)
                launch_wbucket_class<T, P, (LG <= 8 ? LG : 8)>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else
                launch_select_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i].as<int>(), V, q, ctl);
        }
        launch_sorted<T, P, LG + 1>(m, L, V, q, ctl);
    }
}

template <class T, int E>
void launch_medium(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl, bool pess,
                   unsigned* work) {
    using Sh = MediumShape<E>;
    const bool four = m->medium_blocks_per_sm == 4;
    auto k = four ? (pess ? omax_medium<T, true, E, 4> : omax_medium<T, false, E, 4>)
                  : (pess ? omax_medium<T, true, E> : omax_medium<T, false, E>);
    static int per_sm[2][64] = {};
    const int dev = m->device & 63;
    if (!per_sm[four][dev]) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[four][dev], k, Sh::W * 32, 0));
        per_sm[four][dev] = std::max(per_sm[four][dev], 1);
    }
    const int blocks = grid_for(count, Sh::B * Sh::W, m->sm_count, per_sm[four][dev]);
    launch_pdl(m->pdl_now, k, blocks, Sh::W * 32, 0, m->ls, count, list.as<int>(), m->colptr.as<long long>(), m->rows.as<int>(),
                                             m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), V, q, ctl, work);
}

// omax_tiny_rank (ranks + one replay of the consumed chain) by default; RIMDP_TINY=loop: omax_tiny's
// repeated segment argmins.  Same bits either way.
bool tiny_rank_enabled() {
    static const bool on = [] {
        const char* e = getenv("RIMDP_TINY");
        return !(e && strcmp(e, "loop") == 0);
    }();
    return on;
}

template <class T, int SEG>
void launch_tiny(rimdp_model* m, const ColumnLists& L, int i, const T* V, T* q, Ctl* ctl, bool pess) {
    const int count = L.n_tiny[i];
    const bool pk = L.tiny_packed[i];
    auto k = tiny_rank_enabled()
                 ? (pk ? (pess ? omax_tiny_rank<T, true, SEG, true> : omax_tiny_rank<T, false, SEG, true>)
                       : (pess ? omax_tiny_rank<T, true, SEG> : omax_tiny_rank<T, false, SEG>))
                 : (pk ? (pess ? omax_tiny<T, true, SEG, true> : omax_tiny<T, false, SEG, true>)
                       : (pess ? omax_tiny<T, true, SEG> : omax_tiny<T, false, SEG>));
    static int per_sm[64] = {};
    const int dev = m->device & 63;
    if (!per_sm[dev]) {
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, 256, 0));
        per_sm[dev] = std::max(per_sm[dev], 1);
    }
    const int steps = (count + 32 / SEG - 1) / (32 / SEG);
    const int blocks = grid_for(steps, 8 * 4, m->sm_count, per_sm[dev]); // >= 4 steps per warp
    if (pk)
        launch_pdl(m->pdl_now, k, blocks, 256, 0, m->ls, count, L.tiny_list[i].as<int>(), L.tiny_beg[i].as<long long>(),
                   L.tiny_rows[i].as<int>(), L.tiny_lower[i].as<T>(), L.tiny_gap[i].as<T>(), L.tiny_rem[i].as<T>(), V,
                   q, ctl);
    else
        launch_pdl(m->pdl_now, k, blocks, 256, 0, m->ls, count, L.tiny_list[i].as<int>(), m->colptr.as<long long>(),
                   m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), V, q, ctl);
}

template <class T, bool P, bool VS>
void launch_long_v(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    auto k = omax_long<T, P, VS>;
    const size_t smem = VS ? sizeof(T) * (size_t)m->n_global : 0;
    static int per_sm[64] = {};
    static size_t configured_smem[64] = {};
    const int dev = m->device & 63;
    if (!per_sm[dev] || configured_smem[dev] != smem) {
        if (VS) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, kWarpsPerBlock * 32, smem));
        per_sm[dev] = std::max(per_sm[dev], 1);
        configured_smem[dev] = smem;
    }
    const int blocks = grid_for(count, kWarpsPerBlock * kLongGroup, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_now, k, blocks, kWarpsPerBlock * 32, smem, m->ls, count, list.as<int>(), m->colptr.as<long long>(),
                                                          m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(),
                                                          m->rem.as<T>(), V, m->n_global, q, ctl);
}

template <class T, bool P, bool VS>
void launch_long_tree_v(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl) {
    auto k = omax_long_tree<T, P, VS>;
    const size_t smem = VS ? sizeof(T) * (size_t)m->n_global : 0;
    static int per_sm[64] = {};
    static size_t configured_smem[64] = {};
    const int dev = m->device & 63;
    if (!per_sm[dev] || configured_smem[dev] != smem) {
        if (VS) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k, kWarpsPerBlock * 32, smem));
        per_sm[dev] = std::max(per_sm[dev], 1);
        configured_smem[dev] = smem;
    }
    const int blocks = grid_for(count, kWarpsPerBlock, m->sm_count, per_sm[dev]);
    launch_pdl(m->pdl_now, k, blocks, kWarpsPerBlock * 32, smem, m->ls, count, list.as<int>(), m->colptr.as<long long>(),
                                                     m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(),
                                                     m->rem.as<T>(), V, m->n_global, q, ctl);
}

// Few-pick long columns: the single-pass tree-order kernel by default, the
// row-order (bit-exact) omax_long with RIMDP_LONG=exact.  The value vector
// is staged in shared memory when it is small (kLongVsMaxBytes) and the
// columns are long enough to amortise it.
template <class T>
void launch_long(rimdp_model* m, int count, const DevBuf& list, const T* V, T* q, Ctl* ctl, bool pess) {
    const bool vs = sizeof(T) * (size_t)m->n_global <= (size_t)kLongVsMaxBytes &&
                    (long long)count * 64 >= (long long)m->n_global;
    if (!m->long_exact) {
        if (pess) {
            if (vs) launch_long_tree_v<T, true, true>(m, count, list, V, q, ctl);
            else launch_long_tree_v<T, true, false>(m, count, list, V, q, ctl);
        } else {
            if (vs) launch_long_tree_v<T, false, true>(m, count, list, V, q, ctl);
            else launch_long_tree_v<T, false, false>(m, count, list, V, q, ctl);
        }
        return;
    }
    if (pess) {
        if (vs) launch_long_v<T, true, true>(m, count, list, V, q, ctl);
        else launch_long_v<T, true, false>(m, count, list, V, q, ctl);
    } else {
        if (vs) launch_long_v<T, false, true>(m, count, list, V, q, ctl);
        else launch_long_v<T, false, false>(m, count, list, V, q, ctl);
    }
}

// Fork/join over the side streams: independent column classes (they write
// disjoint entries of q) run concurrently, so the latency-bound phases and
// launch tails of one class overlap the loads of another.
struct ClassFanout {
    rimdp_model* m;
    int used = 0, next = 0;
    bool on;
    ClassFanout(rimdp_model* mm, int classes) : m(mm), on(mm->nstreams > 1 && classes > 1) {
        m->ls = m->stream;
        if (on) CK(cudaEventRecord(m->fork_ev, m->stream));
    }
    void pick() {
        if (!on) return;
        const int i = next++ % m->nstreams;
        if (i >= used) {
            CK(cudaStreamWaitEvent(m->side[i], m->fork_ev, 0));
            used = i + 1;
        }
        m->ls = m->side[i];
    }
    ~ClassFanout() noexcept(false) {
        if (on)
            for (int i = 0; i < used; ++i) {
                CK(cudaEventRecord(m->join_ev[i], m->side[i]));
                CK(cudaStreamWaitEvent(m->stream, m->join_ev[i], 0));
            }
        m->ls = m->stream;
    }
};

int column_classes(const ColumnLists& L) {
    int k = (L.n_short > 0) + (L.n_exact > 0) + (L.n_medium[0] > 0) + (L.n_medium[1] > 0);
    for (int i = 0; i < kTinyClasses; ++i) k += L.n_tiny[i] > 0;
    for (int i = 0; i < kSortedClasses; ++i) k += L.n_sorted[i] > 0;
    return k;
}

template <class T, bool P, int LG = kSortedMaxLog>
void launch_sorted_fanout(rimdp_model* m, const ColumnLists& L, const T* V, T* q, Ctl* ctl, ClassFanout& f) {
    // longest classes first: they dominate and should start earliest
    if constexpr (LG >= kSortedMinLog) {
        const int i = LG - kSortedMinLog;
        if (L.n_sorted[i] > 0) {
            f.pick();
            if (m->exact_sorted)
                launch_exact_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (m->bitonic)
                launch_sorted_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (LG >= 9 && m->bucket)
                launch_bucket_class<T, P, (LG >= 9 ? LG : 9)>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else if (LG <= 8 && m->bucket)
                launch_wbucket_class<T, P, (LG <= 8 ? LG : 8)>(m, L.n_sorted[i], L.sorted_list[i], V, q, ctl);
            else
                launch_select_class<T, P, LG>(m, L.n_sorted[i], L.sorted_list[i].as<int>(), V, q, ctl);
        }
        launch_sorted_fanout<T, P, LG - 1>(m, L, V, q, ctl, f);
    }
}

// Per-column expectations q for the columns of one set of class lists.
// Range of V for the value buckets of omax_bucket and exact_sort: one small
// launch per column pass, only when such a class is scheduled.
template <class T>
void launch_value_range(rimdp_model* m, const ColumnLists& L, const T* V) {
    bool need = false;
    for (int i = 0; i < kSortedClasses; ++i) need = need || L.n_sorted[i] > 0;
    m->vrange_cur = nullptr;
    if (!need || m->bitonic || !(m->exact_sorted || m->bucket)) return;
    if (!m->vrange.p) {
        m->vrange.ensure(4 * sizeof(unsigned long long));
        const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
        CK(cudaMemcpyAsync(m->vrange.p, init, sizeof init, cudaMemcpyHostToDevice, m->stream));
        CK(cudaStreamSynchronize(m->stream));
    }
    unsigned long long* slot = m->vrange.as<unsigned long long>() + 2 * m->vrange_parity;
    unsigned long long* other = m->vrange.as<unsigned long long>() + 2 * (m->vrange_parity ^ 1);
    m->vrange_parity ^= 1;
    const int n = m->n_global;
    value_range<T><<<grid_for(n, 256 * 8, m->sm_count, 4), 256, 0, m->stream>>>(n, V, slot, other);
    ++g_launches;
    m->vrange_cur = slot;
}

// Merged fallback of one column pass.  Every many-pick class kernel (bucket, wbucket, exact) appends the
// columns it could not finish to one list, and a single fallback kernel sized for the largest class that
// ran (omax_select, or the bitonic exact kernel on the float32 route) processes them after all classes:
// one launch instead of one per class (C5: 7, each a full wait on its predecessor; they find the list
// empty almost always).  The counters alternate between passes like the per-class ones.
void begin_merged_fallback(rimdp_model* m, const ColumnLists& L) {
    long long total = 0;
    for (int i = 0; i < kSortedClasses; ++i) total += L.n_sorted[i];
    m->fb_maxlg = 0;
    m->fb_merge = total > 0 && !m->bitonic && (m->bucket || m->exact_sorted);
    if (!m->fb_merge) return;
    const size_t need = sizeof(int) * (size_t)(total + 2);
    if (m->fb_all.bytes < need) {
        m->fb_all.ensure(need);
        CK(cudaMemsetAsync(m->fb_all.p, 0, 2 * sizeof(int), m->ls));
    }
    int* base = m->fb_all.as<int>();
    m->fbm_list = base + 2;
    m->fbm_count = base + m->fb_all_parity;
    m->fbm_other = base + (m->fb_all_parity ^ 1);
    m->fbm_cap = (int)total;
    m->fb_all_parity ^= 1;
}

template <class T, bool P, int LG = kSortedMinLog>
void launch_merged_fallback_lg(rimdp_model* m, const T* V, T* q, Ctl* ctl) {
    if constexpr (LG <= kSortedMaxLog) {
        if (m->fb_maxlg == LG) {
            if constexpr (std::is_same<T, float>::value) {
                if (m->exact_sorted) {
                    launch_exact_fallback<P, LG>(m, m->fbm_cap, m->fbm_list, m->fbm_count, V, q, ctl);
                    return;
                }
            }
            launch_select_class<T, P, LG>(m, m->fbm_cap, m->fbm_list, V, q, ctl, m->fbm_count);
            return;
        }
        launch_merged_fallback_lg<T, P, LG + 1>(m, V, q, ctl);
    }
}

template <class T>
void end_merged_fallback(rimdp_model* m, bool pess, const T* V, T* q, Ctl* ctl) {
    if (m->fb_merge && m->fb_maxlg > 0) {
        if (pess)
            launch_merged_fallback_lg<T, true>(m, V, q, ctl);
        else
            launch_merged_fallback_lg<T, false>(m, V, q, ctl);
    }
    m->fb_merge = false;
}

template <class T>
void launch_columns(rimdp_model* m, const ColumnLists& L, const T* V, T* q, Ctl* ctl, bool pess, unsigned* work) {
    m->work_cur = work;
    launch_value_range<T>(m, L, V);
    if (m->gate_needed && !m->vrange_cur) { // value_range (plain launch) is the gate when it runs
        pdl_gate<<<1, 32, 0, m->stream>>>();
        ++g_launches;
    }
    m->gate_needed = false;
    ClassFanout f(m, column_classes(L));
    if (f.on) {
        if (pess)
            launch_sorted_fanout<T, true>(m, L, V, q, ctl, f);
        else
            launch_sorted_fanout<T, false>(m, L, V, q, ctl, f);
    }
    if (L.n_short > 0) {
        f.pick();
        const bool pair = pair_mode() && m->short_pair;
        const int blocks = grid_for(L.n_short, kShortBatch * kWarpsPerBlock, m->sm_count, pair ? 4 : 5);
        auto k = pair ? (pess ? omax_pair<T, true> : omax_pair<T, false>)
                      : (pess ? omax_short<T, true> : omax_short<T, false>);
        launch_pdl(m->pdl_now, k, blocks, kWarpsPerBlock * 32, 0, m->ls, L.n_short, L.short_list.as<int>(), m->colptr.as<long long>(),
                                                      m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(),
                                                      m->rem.as<T>(), V, q, ctl, work);
    }
    if (L.n_medium[0] > 0) { f.pick(); launch_medium<T, 2>(m, L.n_medium[0], L.medium_list[0], V, q, ctl, pess, work + 2); }
    if (L.n_medium[1] > 0) { f.pick(); launch_medium<T, 4>(m, L.n_medium[1], L.medium_list[1], V, q, ctl, pess, work + 3); }
    if (L.n_exact > 0) { f.pick(); launch_long<T>(m, L.n_exact, L.exact_list, V, q, ctl, pess); }
    if (L.n_tiny[2] > 0) { f.pick(); launch_tiny<T, 16>(m, L, 2, V, q, ctl, pess); }
    if (L.n_tiny[1] > 0) { f.pick(); launch_tiny<T, 8>(m, L, 1, V, q, ctl, pess); }
    if (L.n_tiny[0] > 0) { f.pick(); launch_tiny<T, 4>(m, L, 0, V, q, ctl, pess); }
    if (L.n_tiny[3] > 0) { f.pick(); launch_tiny<T, 1>(m, L, 3, V, q, ctl, pess); }
    if (!f.on) {
        begin_merged_fallback(m, L);
        if (pess)
            launch_sorted<T, true>(m, L, V, q, ctl);
        else
            launch_sorted<T, false>(m, L, V, q, ctl);
        end_merged_fallback<T>(m, pess, V, q, ctl);
    }
}

// One Bellman iteration: [q path for long states: column kernels] ->
// [fused bellman_short over the short-state batches] -> [action_reduce over
// the long states].  The last launch of the three runs the stop test.

template <class T>
void launch_iteration(rimdp_model* m, long long k, int* chosen, int chosen_td) {
    SolveState& s = m->s;
    const long long launches0 = g_launches;
    const T* vin = static_cast<const T*>(s.vb[(k - 1) & 1]);
    T* vout = static_cast<T*>(s.vb[k & 1]);
    Ctl* ctl = s.ctl.as<Ctl>();
    unsigned* work = s.work.as<unsigned>() + (k & 1) * kWorkKinds;
    cudaEvent_t* ev = nullptr;
    if (s.profile) {
        while (s.events.size() < s.events_used + 4) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            s.events.push_back(e);
        }
        ev = &s.events[s.events_used];
        s.events_used += 4;
        CK(cudaEventRecord(ev[0], m->stream));
    }
    ActionArgs a{};
    a.n = m->n;
    a.state_begin = m->state_begin;
    a.stateptr = m->stateptr.as<int>();
    a.frozen = s.has_frozen ? s.frozen.as<unsigned char>() : nullptr;
    a.forced = s.has_forced ? s.forced.as<int>() : nullptr;
    a.forced_td = s.forced_td;
    a.chosen = chosen;
    a.chosen_td = chosen_td;
    a.maximize = s.maxi;
    a.finite = s.finite;
    a.horizon = s.horizon;
    a.max_iterations = s.max_iterations;
    a.k = k;
    a.record_only = s.record_only;
    a.work = s.work.as<unsigned>();
    a.peers = m->x.connected ? m->x.table.as<PeerTable>() : nullptr;
    const T* rw = s.has_rewards ? s.rewards.as<T>() : nullptr;
    // PDL lets the next kernel's blocks become resident early; with two shards on one device (tests) those
    // blocks could take the SMs the other shard needs to publish the flag this shard waits for
    const bool early = class_early(m);
    m->pdl_now = (kernels_per_iteration(m) <= kPdlMaxKernels && !m->l2_persist && m->nstreams == 1 &&
                  !(m->x.connected && m->x.shared_device)) ||
                 early;
    m->gate_needed = early; // launch_columns puts a plain-launched gate before the first class kernel
    m->early_now = early;
    if (m->nbatch > 0) {
        a.finalize = m->nlong_states == 0;
        // occupancy variant: 4 resident blocks (64 registers) or 5 (48 registers)
        const int bps = m->short_blocks_per_sm;
        const int blocks = grid_for((long long)m->nbatch, kWarpsPerBlock, m->sm_count, bps);
        auto kern = bps == 5 ? (s.pess ? bellman_short<T, true, 5> : bellman_short<T, false, 5>)
                             : (s.pess ? bellman_short<T, true, 4> : bellman_short<T, false, 4>);
        launch_pdl(m->pdl_now, kern, blocks, kWarpsPerBlock * 32, 0, m->stream,
            m->nbatch, m->batch_slots.as<int>(), m->batch_states.as<int2>(), m->colptr.as<long long>(),
            m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>(), m->rem.as<T>(), vin, vout, rw, (T)s.discount,
            (T)s.eps, a, ctl);
    }
    if (ev) CK(cudaEventRecord(ev[1], m->stream));
    if (m->l2_persist) set_value_window(m, vin, sizeof(T) * (size_t)m->n_global);
    launch_columns<T>(m, m->qp, vin, s.q.as<T>(), ctl, s.pess, work);
    if (ev) CK(cudaEventRecord(ev[2], m->stream));
    if (m->nlong_states > 0 || m->nbatch == 0) {
        // a shard that owns no states still runs one block: its epilogue advances ctl->k and the residual
        // slots, so the sharded stop test and the solve outputs see iteration k
        a.finalize = 1;
        launch_pdl(m->pdl_wait_ok(), action_reduce<T>, grid_for(m->nlong_states, 256, m->sm_count, 8), 256, 0, m->stream,
            a, m->nlong_states, m->all_states_q ? nullptr : m->long_states.as<int>(), s.q.as<T>(), vin, vout, rw,
            (T)s.discount, (T)s.eps, ctl);
    }
    if (m->x.connected) {
        // the global stop test once every rank has published iteration k (peer_sync_stop)
        peer_sync_stop<T><<<1, 32, 0, m->stream>>>(ctl, m->x.table.as<PeerTable>(), k, s.finite, s.horizon,
                                                   std::max(1LL, s.max_iterations), (T)s.eps);
        ++g_launches;
    }
    if (ev) CK(cudaEventRecord(ev[3], m->stream));
    m->pdl_now = false;
    m->early_now = false;
    s.launches_last = (int)(g_launches - launches0);
    CK(cudaGetLastError());
}

int kernels_per_iteration(const rimdp_model* m) {
    int k = (m->nbatch > 0) + (m->qp.n_short > 0) + (m->qp.n_exact > 0) + (m->nlong_states > 0) +
            (m->qp.n_medium[0] > 0) + (m->qp.n_medium[1] > 0);
    for (int i = 0; i < kTinyClasses; ++i) k += m->qp.n_tiny[i] > 0;
    for (int i = 0; i < kSortedClasses; ++i) k += m->qp.n_sorted[i] > 0;
    return k + (m->x.connected ? 1 : 0);
}

// First infeasible column that a step would evaluate (bellman.hpp:88-112:
// frozen states are skipped, forced states evaluate one column; the lowest
// state index wins, parallel.hpp:41-67).
// only_it >= 0: only iteration only_it + 1's row (multi-GPU solves scan the rows across shards in order)
const Infeasible* first_evaluated_infeasible(rimdp_model* m, const rimdp_plan* p, long long only_it = -1) {
    if (m->infeasible_cols.empty()) return nullptr;
    std::vector<char> bad(m->ncols, 0);
    for (const auto& f : m->infeasible_cols) bad[f.col] = 1;
    const int n = m->n, N = m->n_global;
    auto lookup = [&](int c) -> const Infeasible* {
        for (const auto& f : m->infeasible_cols)
            if (f.col == c) return &f;
        return nullptr;
    };
    const long long rows = (p->forced && p->forced_time_dependent) ? std::max<long long>(p->horizon, 1) : 1;
    // iteration k = 1 uses row horizon - 1, k = 2 row horizon - 2, ...
    for (long long it = only_it >= 0 ? only_it : 0; it < (only_it >= 0 ? std::min(rows, only_it + 1) : rows); ++it) {
        const long long t = (p->forced && p->forced_time_dependent) ? p->horizon - 1 - it : 0;
        for (int s = 0; s < n; ++s) {
            if (p->frozen && p->frozen[m->state_begin + s]) continue;
            int cb = m->h_stateptr[s], ce = m->h_stateptr[s + 1];
            if (p->forced) {
                const int f = p->forced[t * N + m->state_begin + s];
                if (f >= 0) {
                    cb = f;
                    ce = f + 1;
                }
            }
            for (int c = cb; c < ce; ++c)
                if (bad[c]) return lookup(c);
        }
    }
    return nullptr;
}

int report_infeasible(const Infeasible* f, rimdp_dtype dtype, int col_offset = 0) {
    char num[64];
    // shortest round-trip text, as NumericTraits::to_string (numeric.hpp:30-35)
    for (int prec = 1; prec <= 17; ++prec) {
        snprintf(num, sizeof num, "%.*g", prec, f->sum);
        const double back = strtod(num, nullptr);
        if (dtype == RIMDP_F32 ? ((float)back == (float)f->sum) : (back == f->sum)) break;
    }
    fail(RIMDP_ERR_INFEASIBLE_COLUMN, "InfeasibleColumn: %s bounds sum to %s %s", f->kind == 1 ? "lower" : "upper",
         num, f->kind == 1 ? "> 1" : "< 1");
    g_err_info.column = f->col + col_offset;
    g_err_info.infeasible_kind = f->kind;
    g_err_info.infeasible_sum = f->sum;
    return RIMDP_ERR_INFEASIBLE_COLUMN;
}

template <class T>
int solve_begin_t(rimdp_model* m, const rimdp_plan* p) {
    upload_plan<T>(m, p);
    // a connected shard's window (V_0 in both buffers, zeroed flags) must be in place before the driver's
    // barrier lets any peer store iteration 1 into it
    if (m->x.connected) CK(cudaStreamSynchronize(m->stream));
    return RIMDP_OK;
}

template <class T>
void advance_t(rimdp_model* m, long long iters) {
    SolveState& s = m->s;
    int* chosen = nullptr;
    int chosen_td = 0;
    if (s.chosen.p) {
        chosen = s.chosen.as<int>();
        chosen_td = s.chosen_td;
    }
    for (long long i = 0; i < iters; ++i) {
        const long long k = s.launched + 1;
        if (s.finite && k > s.horizon) break;
        if (!s.finite && k > std::max(1LL, s.max_iterations)) break; // iterate() always runs step 1
        launch_iteration<T>(m, k, chosen, chosen_td);
        s.launched = k;
    }
}

Ctl read_ctl(rimdp_model* m) {
    Ctl c{};
    CK(cudaMemcpyAsync(&c, m->s.ctl.p, sizeof c, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return c;
}

template <class T>
void finish_t(rimdp_model* m, const rimdp_outputs* o, long long k) {
    SolveState& s = m->s;
    const int N = m->n_global;
    if (o->values)
        CK(cudaMemcpyAsync(o->values, s.vb[k & 1], sizeof(T) * N, cudaMemcpyDeviceToHost, m->stream));
    if (o->residual) {
        if (k == 0) {
            CK(cudaMemsetAsync(s.res.p, 0, sizeof(T) * N, m->stream));
        } else {
            residual_vector<T><<<grid_for(N, 256, m->sm_count, 8), 256, 0, m->stream>>>(N, static_cast<T*>(s.vb[k & 1]),
                                                                                        static_cast<T*>(s.vb[(k - 1) & 1]),
                                                                                        s.res.as<T>());
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(o->residual, s.res.p, sizeof(T) * N, cudaMemcpyDeviceToHost, m->stream));
    }
    if (o->chosen && s.chosen.p) {
        const long long rows = s.chosen_td ? std::max<long long>(s.horizon, 0) : 1;
        if (rows > 0)
            CK(cudaMemcpyAsync(o->chosen, s.chosen.p, sizeof(int) * (size_t)m->n * rows, cudaMemcpyDeviceToHost,
                               m->stream));
    }
    if (o->iterations) *o->iterations = k;
    CK(cudaStreamSynchronize(m->stream));
}

void prepare_chosen(rimdp_model* m, const rimdp_outputs* o, const rimdp_plan* p) {
    SolveState& s = m->s;
    s.chosen_td = 0;
    if (o && o->chosen) {
        s.chosen_td = o->record_all_steps && p->finite;
        const long long rows = s.chosen_td ? std::max<long long>(p->horizon, 1) : 1;
        s.chosen.ensure(sizeof(int) * (size_t)m->n * rows);
        CK(cudaMemsetAsync(s.chosen.p, 0xff, sizeof(int) * (size_t)m->n * rows, m->stream));
    } else if (s.chosen.p) {
        // do not record
        s.chosen.release();
    }
}

// How many iterations to enqueue before the next poll.  Finite horizons are
// capped exactly by advance_t.  For infinite horizons the residual decays
// geometrically near convergence (contraction), so the rate measured between
// two polls predicts the iteration at which max residual <= eps; enqueueing
// up to that prediction (+1) keeps the no-op launches after the device stop
// test (kernels return at their first instruction once `done` is set) to a
// handful instead of a whole doubling chunk.
struct ChunkPlanner {
    bool finite;
    double eps;
    long long chunk = 8, last_k = 0;
    double last_res = -1.0;
    explicit ChunkPlanner(const rimdp_plan* p) : finite(p->finite != 0), eps(p->eps) {}
    long long next() const { return chunk; }
    void observe(long long k, double res) {
        long long want = std::min<long long>(chunk * 2, kMaxChunk);
        if (!finite && last_res > 0.0 && res > 0.0 && res < last_res && k > last_k && eps > 0.0) {
            const double rate = std::log(res / last_res) / (double)(k - last_k); // log rho < 0
            const double need = std::log(eps / res) / rate;                        // iterations to eps
            if (std::isfinite(need)) want = std::max<long long>(1, std::min<long long>((long long)need + 1, want));
        }
        chunk = want;
        last_k = k;
        last_res = res;
    }
    static constexpr long long kMaxChunk = 64;
};

template <class T>
int solve_t(rimdp_model* m, const rimdp_plan* p, const rimdp_outputs* o) {
    const bool will_step = p->finite ? p->horizon > 0 : true;
    if (will_step) {
        if (const Infeasible* f = first_evaluated_infeasible(m, p)) return report_infeasible(f, m->dtype);
    }
    PhaseTrace tr("solve");
    m->s.record_only = false;
    upload_plan<T>(m, p);
    prepare_chosen(m, o, p);
    tr.mark("plan");
    const long long total = p->finite ? p->horizon : std::max<long long>(1, p->max_iterations);
    long long k = 0;
    Ctl c{};
    if (o && o->on_iteration) {
        std::vector<T> hv(m->n_global);
        while (k < total) {
            advance_t<T>(m, 1);
            c = read_ctl(m);
            k = c.k;
            CK(cudaMemcpy(hv.data(), m->s.vb[k & 1], sizeof(T) * m->n_global, cudaMemcpyDeviceToHost));
            o->on_iteration(k, hv.data(), o->user);
            if (c.done) break;
        }
    } else {
        ChunkPlanner cp(p);
        while (!c.done && m->s.launched < total) {
            advance_t<T>(m, cp.next());
            c = read_ctl(m);
            cp.observe(c.k, c.res_last);
        }
        k = c.k;
    }
    tr.mark("iterations");
    // omax_long (RIMDP_LONG=exact) tracks at most kMaxPartial positions that received a partial share;
    // more than one needs avail > 0 to survive a consumed += gap >= avail step through rounding, so the
    // overflow is only reachable by adversarial bounds, and it is reported instead of summed wrongly
    if (c.status == 2) return fail(RIMDP_ERR_INTERNAL, "partial-assignment overflow in a long column");
    finish_t<T>(m, o, k);
    tr.mark("finish");
    m->s.active = false;
    if (c.status == 1) {
        fail(RIMDP_ERR_NON_CONVERGENCE, "no convergence after %lld iterations (max residual %f)", k, c.res_last);
        g_err_info.iterations = k;
        g_err_info.residual = c.res_last;
        return RIMDP_ERR_NON_CONVERGENCE;
    }
    return RIMDP_OK;
}

template <class T>
int step_t(rimdp_model* m, const void* v_in, int pess, int maxi, const uint8_t* frozen, const int32_t* forced,
           void* v_out, int32_t* chosen_out) {
    rimdp_plan p{};
    p.pessimistic = pess;
    p.maximize = maxi;
    p.finite = 1;
    p.horizon = 1;
    p.initial = v_in;
    p.frozen = frozen;
    p.forced = forced;
    if (const Infeasible* f = first_evaluated_infeasible(m, &p)) return report_infeasible(f, m->dtype);
    rimdp_outputs o{};
    o.values = v_out;
    o.chosen = chosen_out;
    m->s.record_only = false;
    upload_plan<T>(m, &p);
    prepare_chosen(m, &o, &p);
    advance_t<T>(m, 1);
    finish_t<T>(m, &o, 1);
    return RIMDP_OK;
}

template <class T>
int column_values_t(rimdp_model* m, const void* v_in, int pess, void* q_out) {
    // every column is evaluated: the first infeasible one throws (omax.hpp:72-80)
    if (!m->infeasible_cols.empty()) return report_infeasible(&m->infeasible_cols[0], m->dtype);
    SolveState& s = m->s;
    s.v[0].ensure(sizeof(T) * m->n_global);
    s.q.ensure(sizeof(T) * std::max(1, m->ncols));
    CK(cudaMemcpyAsync(s.v[0].p, v_in, sizeof(T) * m->n_global, cudaMemcpyHostToDevice, m->stream));
    s.work.ensure(2 * kWorkKinds * sizeof(unsigned));
    CK(cudaMemsetAsync(s.work.p, 0, 2 * kWorkKinds * sizeof(unsigned), m->stream));
    launch_columns<T>(m, m->all_lists(), s.v[0].as<T>(), s.q.as<T>(), nullptr, pess != 0, s.work.as<unsigned>());
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(q_out, s.q.p, sizeof(T) * m->ncols, cudaMemcpyDeviceToHost, m->stream));
    CK(cudaStreamSynchronize(m->stream));
    return RIMDP_OK;
}

#define DISPATCH(m, fn, ...) ((m)->dtype == RIMDP_F64 ? fn<double>(__VA_ARGS__) : fn<float>(__VA_ARGS__))

} // namespace

// ---------------------------------------------------------------------------
// C ABI

extern "C" {

const char* rimdp_last_error(void) { return g_err_msg.c_str(); }

int rimdp_last_error_info(rimdp_error_info* out) {
    if (!out) return RIMDP_ERR_INVALID_ARGUMENT;
    *out = g_err_info;
    return RIMDP_OK;
}

int rimdp_abi_version(void) { return RIMDP_B200_ABI_VERSION; }

/* Error hook for the host-only translation units (native_io.cpp). */
int rimdp_internal_fail(int status, const char* msg) { return fail(status, "%s", msg); }

int rimdp_device_count(int* count) {
    if (!count) return fail(RIMDP_ERR_INVALID_ARGUMENT, "count is null");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
    *count = c;
    return RIMDP_OK;
}

static int model_create_impl(const rimdp_model_desc* d, int state_begin, int num_global, rimdp_model** out);

int rimdp_model_create(const rimdp_model_desc* d, rimdp_model** out) {
    if (!d) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    return model_create_impl(d, 0, d->num_states, out);
}

int rimdp_model_create_shard(const rimdp_model_desc* d, int32_t state_begin, int32_t num_global, rimdp_model** out) {
    if (!d) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (state_begin < 0 || num_global < 0 || (long long)state_begin + d->num_states > num_global)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "shard [%d, %lld) outside [0, %d)", state_begin,
                    (long long)state_begin + d->num_states, num_global);
    return model_create_impl(d, state_begin, num_global, out);
}

static int model_create_impl(const rimdp_model_desc* d, int state_begin, int num_global, rimdp_model** out) {
    return guarded([&]() -> int {
        if (!d || !out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
        if (d->dtype != RIMDP_F64 && d->dtype != RIMDP_F32) return fail(RIMDP_ERR_INVALID_ARGUMENT, "unknown dtype");
        if (d->num_states < 0 || d->num_cols < 0 || d->nnz < 0 || !d->stateptr || !d->colptr)
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad model sizes");
        if (d->nnz > 0 && (!d->rowval || !d->lower || !d->upper))
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "null CSC arrays");
        // structural checks of the pointer arrays (csc.hpp:76-106, imdp.hpp:129-168)
        if (d->colptr[0] != 0 || d->colptr[d->num_cols] != d->nnz)
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "colptr must run from 0 to nnz");
        for (int c = 0; c < d->num_cols; ++c)
            if (d->colptr[c + 1] < d->colptr[c]) return fail(RIMDP_ERR_INVALID_ARGUMENT, "colptr not monotone at %d", c);
        if (d->stateptr[0] != 0 || d->stateptr[d->num_states] != d->num_cols)
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "stateptr must run from 0 to num_cols");
        for (int s = 0; s < d->num_states; ++s)
            if (d->stateptr[s + 1] < d->stateptr[s])
                return fail(RIMDP_ERR_INVALID_ARGUMENT, "stateptr not monotone at %d", s);
        PhaseTrace tr("model_create");
        std::unique_ptr<rimdp_model> m(new rimdp_model);
        m->dtype = d->dtype;
        m->col_offset = g_shard_col_offset;
        init_common(m.get(), d->device);
        tr.mark("init");
        DeviceGuard g(m->device);
        m->n = d->num_states;
        m->n_global = num_global;
        m->state_begin = state_begin;
        m->ncols = d->num_cols;
        m->nnz = d->nnz;
        m->h_stateptr.assign(d->stateptr, d->stateptr + d->num_states + 1);
        const size_t es = elem_size(d->dtype);
        m->stateptr.ensure(sizeof(int) * (d->num_states + 1));
        m->colptr.ensure(sizeof(long long) * (d->num_cols + 1));
        m->rows.ensure(sizeof(int) * std::max<long long>(1, d->nnz));
        m->lower.ensure(es * std::max<long long>(1, d->nnz));
        m->gap.ensure(es * std::max<long long>(1, d->nnz));
        tr.mark("alloc");
        CK(cudaMemcpyAsync(m->stateptr.p, d->stateptr, sizeof(int) * (d->num_states + 1), cudaMemcpyHostToDevice,
                           m->stream));
        CK(cudaMemcpyAsync(m->colptr.p, d->colptr, sizeof(long long) * (d->num_cols + 1), cudaMemcpyHostToDevice,
                           m->stream));
        if (d->nnz > 0)
            upload_many(m->device, m->stream,
                        {{m->rows.p, d->rowval, sizeof(int) * (size_t)d->nnz},
                         {m->lower.p, d->lower, es * (size_t)d->nnz},
                         {m->gap.p, d->upper, es * (size_t)d->nnz}});
        tr.mark("upload");
        DISPATCH(m, prepare, m.get());
        tr.mark("prepare");
        DISPATCH(m, build_schedule, m.get(), reinterpret_cast<const long long*>(d->colptr));
        tr.mark("schedule");
        m->device_bytes = (long long)(m->stateptr.bytes + m->colptr.bytes + m->rows.bytes + m->lower.bytes +
                                      m->gap.bytes + m->rem.bytes + m->infeasible.bytes + m->quoted.bytes +
                                      m->maxgap.bytes + m->pack_bytes);
        *out = m.release();
        return RIMDP_OK;
    });
}

int rimdp_model_destroy(rimdp_model* m) {
    if (!m) return RIMDP_OK;
    {
        DeviceGuard g(m->device);
        if (m->stream) cudaStreamSynchronize(m->stream);
        m->s.~SolveState();
        new (&m->s) SolveState();
        for (int i = 0; i < kMaxSideStreams; ++i) {
            if (m->side[i]) cudaStreamDestroy(m->side[i]);
            if (m->join_ev[i]) cudaEventDestroy(m->join_ev[i]);
        }
        if (m->fork_ev) cudaEventDestroy(m->fork_ev);
        for (void* w : m->x.opened) cudaIpcCloseMemHandle(w);
        m->x.table.release();
        if (m->x.win) cudaFree(m->x.win);
        if (m->stream) cudaStreamDestroy(m->stream);
        m->stream = nullptr;
    }
    delete m;
    return RIMDP_OK;
}

int rimdp_model_info_get(rimdp_model* m, rimdp_model_info* o) {
    if (!m || !o) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    *o = rimdp_model_info{};
    o->dtype = m->dtype;
    o->device = m->device;
    o->num_states = m->n;
    o->num_cols = m->ncols;
    o->nnz = m->nnz;
    o->state_begin = m->state_begin;
    o->state_end = m->state_begin + m->n;
    o->max_column_length = m->maxlen;
    o->num_infeasible_columns = (int)m->infeasible_cols.size();
    o->device_bytes = m->device_bytes;
    const ColumnLists& all = m->all_lists();
    o->short_columns = all.n_short + all.n_tiny[0] + all.n_tiny[1] + all.n_tiny[2] + all.n_tiny[3];
    o->mid_columns = all.n_exact + all.n_medium[0] + all.n_medium[1];
    o->long_columns = all.total_sorted();
    return RIMDP_OK;
}

int rimdp_model_stream(rimdp_model* m, void** s) {
    if (!m || !s) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    *s = m->stream;
    return RIMDP_OK;
}

static int check_plan(rimdp_model* m, const rimdp_plan* p) {
    if (!m || !p) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (!p->initial) return fail(RIMDP_ERR_INVALID_ARGUMENT, "plan.initial is required");
    if (p->finite && p->horizon < 0) return fail(RIMDP_ERR_INVALID_ARGUMENT, "negative horizon");
    if (p->forced) {
        const long long rows = p->forced_time_dependent ? p->horizon : 1;
        for (long long t = 0; t < rows; ++t)
            for (int s = 0; s < m->n; ++s) {
                const int f = p->forced[t * m->n_global + m->state_begin + s];
                if (f >= 0 && (f < m->h_stateptr[s] || f >= m->h_stateptr[s + 1]))
                    return fail(RIMDP_ERR_INVALID_ARGUMENT, "forced column %d is not a column of state %d", f,
                                m->state_begin + s);
            }
    }
    return RIMDP_OK;
}

// A shard connected to peers only iterates together with them (begin / advance / poll / finish on every
// rank, or rimdp_multi_solve): a lone solve or step would wait forever for the peers' flags.
static int reject_connected(rimdp_model* m, const char* what) {
    if (m && m->x.connected && m->x.world > 1)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "%s: this model is a connected shard of a %d-rank solve", what,
                    m->x.world);
    return RIMDP_OK;
}

int rimdp_solve(rimdp_model* m, const rimdp_plan* p, const rimdp_outputs* o) {
    if (int st = check_plan(m, p)) return st;
    if (int st = reject_connected(m, "rimdp_solve")) return st;
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        rimdp_outputs none{};
        return DISPATCH(m, solve_t, m, p, o ? o : &none);
    });
}

int rimdp_solve_begin(rimdp_model* m, const rimdp_plan* p) {
    if (int st = check_plan(m, p)) return st;
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        // the same InfeasibleColumn report as rimdp_solve (omax.hpp:72-80): the first column a step evaluates
        if (!p->finite || p->horizon > 0)
            if (const Infeasible* f = first_evaluated_infeasible(m, p)) return report_infeasible(f, m->dtype);
        m->s.record_only = false;
        rimdp_outputs none{};
        prepare_chosen(m, &none, p);
        return DISPATCH(m, solve_begin_t, m, p);
    });
}

int rimdp_solve_advance(rimdp_model* m, int64_t iters) {
    if (!m || !m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        if (m->dtype == RIMDP_F64)
            advance_t<double>(m, iters);
        else
            advance_t<float>(m, iters);
        return RIMDP_OK;
    });
}

int rimdp_solve_poll(rimdp_model* m, int64_t* k, int32_t* finished, double* res) {
    if (!m || !m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        Ctl c = read_ctl(m);
        if (k) *k = c.k;
        if (finished) *finished = c.done;
        if (res) *res = c.res_last;
        return RIMDP_OK;
    });
}

int rimdp_solve_finish(rimdp_model* m, const rimdp_outputs* o) {
    if (!m || !m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        Ctl c = read_ctl(m);
        rimdp_outputs none{};
        if (m->dtype == RIMDP_F64)
            finish_t<double>(m, o ? o : &none, c.k);
        else
            finish_t<float>(m, o ? o : &none, c.k);
        m->s.active = false;
        return RIMDP_OK;
    });
}

int rimdp_profile_enable(rimdp_model* m, int32_t on) {
    if (!m) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null model");
    m->s.profile = on != 0;
    return RIMDP_OK;
}

int rimdp_profile_read(rimdp_model* m, double* fused_ms, double* columns_ms, double* action_ms, int64_t* iterations,
                       int32_t* kernels) {
    if (!m) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null model");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        CK(cudaStreamSynchronize(m->stream));
        double f = 0, c = 0, a = 0;
        long long it = 0;
        for (size_t i = 0; i + 4 <= m->s.events_used; i += 4) {
            float x = 0, y = 0, z = 0;
            CK(cudaEventElapsedTime(&x, m->s.events[i], m->s.events[i + 1]));
            CK(cudaEventElapsedTime(&y, m->s.events[i + 1], m->s.events[i + 2]));
            CK(cudaEventElapsedTime(&z, m->s.events[i + 2], m->s.events[i + 3]));
            f += x;
            c += y;
            a += z;
            ++it;
        }
        m->s.events_used = 0;
        if (fused_ms) *fused_ms = f;
        if (columns_ms) *columns_ms = c;
        if (action_ms) *action_ms = a;
        if (iterations) *iterations = it;
        if (kernels) *kernels = m->s.launches_last > 0 ? m->s.launches_last : kernels_per_iteration(m);
        return RIMDP_OK;
    });
}

int rimdp_solve_residual_slots(rimdp_model* m, void** slots) {
    if (!m || !m->s.active || !slots) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    *slots = m->s.ctl.as<Ctl>()->res_bits;
    return RIMDP_OK;
}

int rimdp_solve_stop_test(rimdp_model* m) {
    if (!m || !m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        SolveState& s = m->s;
        if (s.launched == 0) return RIMDP_OK;
        const long long k = s.launched;
        const int blocks = grid_for(m->n_global, 256, m->sm_count, 4);
        if (m->dtype == RIMDP_F64)
            global_stop_test<double><<<blocks, 256, 0, m->stream>>>(
                m->n_global, static_cast<double*>(s.vb[k & 1]), static_cast<double*>(s.vb[(k - 1) & 1]), s.ctl.as<Ctl>(), k, s.finite,
                s.horizon, s.max_iterations, (double)s.eps);
        else
            global_stop_test<float><<<blocks, 256, 0, m->stream>>>(
                m->n_global, static_cast<float*>(s.vb[k & 1]), static_cast<float*>(s.vb[(k - 1) & 1]), s.ctl.as<Ctl>(), k, s.finite,
                s.horizon, s.max_iterations, (float)s.eps);
        CK(cudaGetLastError());
        return RIMDP_OK;
    });
}

int rimdp_model_set_value_capacity(rimdp_model* m, int64_t entries) {
    if (!m || entries < 0) return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad argument");
    m->value_capacity = entries;
    return RIMDP_OK;
}

// ---- peer exchange (state-sharded solves) ----------

static int exchange_alloc(rimdp_model* m) {
    if (m->x.win) return RIMDP_OK;
    const size_t es = elem_size(m->dtype);
    m->x.cap = std::max<long long>(m->n_global, m->value_capacity);
    m->x.vbytes = ((size_t)m->x.cap * es + 255) / 256 * 256;
    const size_t bytes = 2 * m->x.vbytes + rimdp_model::Exchange::tail();
    CK(cudaMalloc(&m->x.win, bytes)); // plain cudaMalloc: IPC-exportable, unlike the stream-ordered pool
    CK(cudaMemset(m->x.win, 0, bytes));
    return RIMDP_OK;
}

// Builds and uploads the PeerTable from the ranks' window base pointers (in this process's address space).
static void exchange_table(rimdp_model* m, int rank, int world, const std::vector<char*>& bases,
                           const std::vector<size_t>& vbytes) {
    PeerTable t{};
    t.world = world;
    t.rank = rank;
    for (int p = 0; p < world; ++p) {
        t.v[p][0] = bases[p];
        t.v[p][1] = bases[p] + vbytes[p];
        t.res[p] = reinterpret_cast<unsigned long long*>(bases[p] + 2 * vbytes[p]);
        t.flag[p] = t.res[p] + 2 * kMaxWorld;
    }
    m->x.table.ensure(sizeof(PeerTable));
    CK(cudaMemcpy(m->x.table.p, &t, sizeof t, cudaMemcpyHostToDevice));
    m->x.world = world;
    m->x.rank = rank;
    m->x.connected = true;
}

static int check_exchange(rimdp_model* m, int rank, int world) {
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "rank %d / world %d outside 1..%d", rank, world, kMaxWorld);
    if (m->nbatch > 0)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "the fused short-state path (RIMDP_FUSED) has no peer exchange");
    if (m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "a solve is active");
    return RIMDP_OK;
}

int rimdp_exchange_export(rimdp_model* m, void* handle_out) {
    if (!m) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null model");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        exchange_alloc(m);
        if (handle_out) {
            cudaIpcMemHandle_t h;
            CK(cudaIpcGetMemHandle(&h, m->x.win));
            std::memcpy(handle_out, &h, sizeof h);
        }
        return RIMDP_OK;
    });
}

int rimdp_exchange_connect(rimdp_model* m, int32_t rank, int32_t world, const void* handles) {
    if (!m || !handles) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (int st = check_exchange(m, rank, world)) return st;
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        exchange_alloc(m);
        const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
        std::vector<char*> bases(world);
        std::vector<size_t> vb(world, m->x.vbytes); // every rank sizes its window for the same capacity
        for (void* w : m->x.opened) cudaIpcCloseMemHandle(w);
        m->x.opened.clear();
        m->x.shared_device = false;
        for (int p = 0; p < world; ++p) {
            if (p == rank) {
                bases[p] = static_cast<char*>(m->x.win);
                continue;
            }
            void* ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, hs[p], cudaIpcMemLazyEnablePeerAccess));
            m->x.opened.push_back(ptr);
            bases[p] = static_cast<char*>(ptr);
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.device == m->device) m->x.shared_device = true;
        }
        exchange_table(m, rank, world, bases, vb);
        return RIMDP_OK;
    });
}

int rimdp_exchange_connect_local(rimdp_model* const* shards, int32_t world) {
    if (!shards || world < 1) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    for (int r = 0; r < world; ++r) {
        if (!shards[r]) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null shard %d", r);
        if (int st = check_exchange(shards[r], r, world)) return st;
        if (shards[r]->dtype != shards[0]->dtype || shards[r]->n_global != shards[0]->n_global)
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "shard %d does not belong to the same model", r);
    }
    return guarded([&]() -> int {
        std::vector<char*> bases(world);
        std::vector<size_t> vb(world);
        for (int r = 0; r < world; ++r) {
            DeviceGuard g(shards[r]->device);
            exchange_alloc(shards[r]);
            bases[r] = static_cast<char*>(shards[r]->x.win);
            vb[r] = shards[r]->x.vbytes;
        }
        for (int r = 0; r < world; ++r) {
            DeviceGuard g(shards[r]->device);
            bool shared = false;
            for (int p = 0; p < world; ++p) {
                if (p == r) continue;
                if (shards[p]->device == shards[r]->device) {
                    shared = true;
                } else {
                    int can = 0;
                    CK(cudaDeviceCanAccessPeer(&can, shards[r]->device, shards[p]->device));
                    if (!can) {
                        fail(RIMDP_ERR_CUDA, "device %d cannot access device %d (no P2P)", shards[r]->device,
                             shards[p]->device);
                        throw Fail{RIMDP_ERR_CUDA};
                    }
                    const cudaError_t e = cudaDeviceEnablePeerAccess(shards[p]->device, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                    cudaGetLastError();
                }
            }
            shards[r]->x.shared_device = shared;
            exchange_table(shards[r], r, world, bases, vb);
        }
        return RIMDP_OK;
    });
}

int rimdp_solve_value_buffers(rimdp_model* m, void** b0, void** b1) {
    if (!m || !m->s.active) return fail(RIMDP_ERR_INVALID_ARGUMENT, "no active solve");
    if (b0) *b0 = m->s.vb[0];
    if (b1) *b1 = m->s.vb[1];
    return RIMDP_OK;
}

int rimdp_bellman_step(rimdp_model* m, const void* v_in, int32_t pess, int32_t maxi, const uint8_t* frozen,
                       const int32_t* forced, void* v_out, int32_t* chosen_out) {
    if (!m || !v_in || !v_out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    rimdp_plan p{};
    p.initial = v_in;
    p.forced = forced;
    p.finite = 1;
    p.horizon = 1;
    if (int st = check_plan(m, &p)) return st;
    if (int st = reject_connected(m, "rimdp_bellman_step")) return st;
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        return DISPATCH(m, step_t, m, v_in, pess, maxi, frozen, forced, v_out, chosen_out);
    });
}

int rimdp_column_values(rimdp_model* m, const void* v_in, int32_t pess, void* q_out) {
    if (!m || !v_in || !q_out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        return DISPATCH(m, column_values_t, m, v_in, pess, q_out);
    });
}

} // extern "C"

// ---------------------------------------------------------------------------
// Synthetic stores generated in HBM (generator.cuh)

namespace {

__global__ void gen_lengths(rimdp_gen::Params p, long long col0, int ncols, const unsigned long long* cdf,
                            int* len) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x)
        len[c] = rimdp_gen::column_length(p, reinterpret_cast<const uint64_t*>(cdf), col0 + c);
}

template <class T>
__global__ void gen_columns(rimdp_gen::Params p, long long col0, int ncols, const long long* colptr, int* rows,
                            T* lower, T* upper) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const long long b = colptr[c];
        const int k = static_cast<int>(colptr[c + 1] - b);
        rimdp_gen::write_column<T>(p, col0 + c, k, rows + b, lower + b, upper + b);
    }
}

struct GenSetup {
    rimdp_gen::Params p{};
    int sb = 0, se = 0, ncols = 0;
    long long col0 = 0;
    std::vector<unsigned long long> cdf;
};

int gen_setup(const rimdp_gen_config* cfg, GenSetup& g) {
    if (!cfg) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null config");
    if (cfg->dtype != RIMDP_F64 && cfg->dtype != RIMDP_F32) return fail(RIMDP_ERR_INVALID_ARGUMENT, "unknown dtype");
    if (cfg->num_states <= 0 || cfg->actions <= 0) return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad model size");
    if ((long long)cfg->num_states * cfg->actions > INT32_MAX)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "more than 2^31-1 columns");
    g.sb = cfg->state_begin;
    g.se = cfg->state_end;
    if (g.sb == 0 && g.se == 0) g.se = cfg->num_states;
    if (g.sb < 0 || g.se > cfg->num_states || g.sb > g.se)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad shard [%d, %d)", g.sb, g.se);
    g.p.num_states = cfg->num_states;
    g.p.actions = cfg->actions;
    g.p.law = cfg->law;
    g.p.support = cfg->support;
    g.p.kmax = cfg->kmax;
    g.p.lower_scale = cfg->lower_scale;
    g.p.upper_scale = cfg->upper_scale;
    g.p.seed = cfg->seed;
    if (cfg->law == 0) {
        if (cfg->support <= 0) return fail(RIMDP_ERR_INVALID_ARGUMENT, "law 0 needs support > 0");
    } else if (cfg->law == 1) {
        if (cfg->kmax <= 0 || cfg->kmax > rimdp_gen::kMaxK)
            return fail(RIMDP_ERR_INVALID_ARGUMENT, "kmax must be in [1, %d]", rimdp_gen::kMaxK);
        const std::vector<uint64_t> cdf = rimdp_gen::power_law_cdf(cfg->kmax, cfg->alpha);
        g.cdf.assign(cdf.begin(), cdf.end());
    } else {
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "unknown law %d", cfg->law);
    }
    g.ncols = (g.se - g.sb) * cfg->actions;
    g.col0 = (long long)g.sb * cfg->actions;
    return RIMDP_OK;
}

template <class T>
void generate_t(rimdp_model* m, const GenSetup& g) {
    const int nc = g.ncols;
    DevBuf d_cdf, d_len;
    std::vector<long long> h_colptr(nc + 1, 0);
    if (g.p.law == 1) {
        d_cdf.ensure(sizeof(unsigned long long) * g.cdf.size());
        CK(cudaMemcpyAsync(d_cdf.p, g.cdf.data(), sizeof(unsigned long long) * g.cdf.size(), cudaMemcpyHostToDevice,
                           m->stream));
        d_len.ensure(sizeof(int) * std::max(1, nc));
        if (nc > 0)
            gen_lengths<<<grid_for(nc, 256, m->sm_count, 8), 256, 0, m->stream>>>(g.p, g.col0, nc,
                                                                                d_cdf.as<unsigned long long>(),
                                                                                d_len.as<int>());
        CK(cudaGetLastError());
        std::vector<int> len(nc);
        if (nc > 0) CK(cudaMemcpyAsync(len.data(), d_len.p, sizeof(int) * nc, cudaMemcpyDeviceToHost, m->stream));
        CK(cudaStreamSynchronize(m->stream));
        for (int c = 0; c < nc; ++c) h_colptr[c + 1] = h_colptr[c] + len[c];
    } else {
        const int k = std::min(g.p.support, g.p.num_states);
        for (int c = 0; c < nc; ++c) h_colptr[c + 1] = h_colptr[c] + k;
    }
    const long long nnz = h_colptr[nc];
    m->nnz = nnz;
    m->ncols = nc;
    m->n = g.se - g.sb;
    m->n_global = g.p.num_states;
    m->state_begin = g.sb;
    m->h_stateptr.resize(m->n + 1);
    for (int s = 0; s <= m->n; ++s) m->h_stateptr[s] = s * g.p.actions;
    m->stateptr.ensure(sizeof(int) * (m->n + 1));
    m->colptr.ensure(sizeof(long long) * (nc + 1));
    m->rows.ensure(sizeof(int) * std::max<long long>(1, nnz));
    m->lower.ensure(sizeof(T) * std::max<long long>(1, nnz));
    m->gap.ensure(sizeof(T) * std::max<long long>(1, nnz));
    CK(cudaMemcpyAsync(m->stateptr.p, m->h_stateptr.data(), sizeof(int) * (m->n + 1), cudaMemcpyHostToDevice,
                       m->stream));
    CK(cudaMemcpyAsync(m->colptr.p, h_colptr.data(), sizeof(long long) * (nc + 1), cudaMemcpyHostToDevice,
                       m->stream));
    if (nc > 0)
        gen_columns<T><<<grid_for(nc, 128, m->sm_count, 16), 128, 0, m->stream>>>(
            g.p, g.col0, nc, m->colptr.as<long long>(), m->rows.as<int>(), m->lower.as<T>(), m->gap.as<T>());
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(m->stream));
    prepare<T>(m);
    build_schedule<T>(m, h_colptr.data());
    m->device_bytes = (long long)(m->stateptr.bytes + m->colptr.bytes + m->rows.bytes + m->lower.bytes +
                                  m->gap.bytes + m->rem.bytes + m->infeasible.bytes + m->quoted.bytes +
                                  m->maxgap.bytes + m->pack_bytes);
}

template <class T>
int generate_host_t(const GenSetup& g, int32_t* num_cols, int64_t* nnz_out, int32_t* stateptr, int64_t* colptr,
                    int32_t* rowval, void* lower, void* upper) {
    const int nc = g.ncols;
    std::vector<long long> cp(nc + 1, 0);
    for (int c = 0; c < nc; ++c)
        cp[c + 1] = cp[c] + rimdp_gen::column_length(g.p, reinterpret_cast<const uint64_t*>(g.cdf.data()), g.col0 + c);
    if (num_cols) *num_cols = nc;
    if (nnz_out) *nnz_out = cp[nc];
    if (!colptr) return RIMDP_OK;
    for (int c = 0; c <= nc; ++c) colptr[c] = cp[c];
    if (stateptr)
        for (int s = 0; s <= g.se - g.sb; ++s) stateptr[s] = s * g.p.actions;
    if (rowval && lower && upper)
        for (int c = 0; c < nc; ++c)
            rimdp_gen::write_column<T>(g.p, g.col0 + c, (int)(cp[c + 1] - cp[c]), rowval + cp[c],
                                       static_cast<T*>(lower) + cp[c], static_cast<T*>(upper) + cp[c]);
    return RIMDP_OK;
}

} // namespace

extern "C" {

int rimdp_model_generate(const rimdp_gen_config* cfg, rimdp_model** out) {
    return guarded([&]() -> int {
        if (!out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
        GenSetup g;
        if (int st = gen_setup(cfg, g)) return st;
        std::unique_ptr<rimdp_model> m(new rimdp_model);
        m->dtype = cfg->dtype;
        init_common(m.get(), cfg->device);
        DeviceGuard dg(m->device);
        if (m->dtype == RIMDP_F64)
            generate_t<double>(m.get(), g);
        else
            generate_t<float>(m.get(), g);
        *out = m.release();
        return RIMDP_OK;
    });
}

int rimdp_generate_host(const rimdp_gen_config* cfg, int32_t* num_cols, int64_t* nnz, int32_t* stateptr,
                        int64_t* colptr, int32_t* rowval, void* lower, void* upper) {
    return guarded([&]() -> int {
        GenSetup g;
        if (int st = gen_setup(cfg, g)) return st;
        return cfg->dtype == RIMDP_F64 ? generate_host_t<double>(g, num_cols, nnz, stateptr, colptr, rowval, lower, upper)
                                       : generate_host_t<float>(g, num_cols, nnz, stateptr, colptr, rowval, lower, upper);
    });
}

int rimdp_model_read_columns(rimdp_model* m, int32_t cb, int32_t ce, int64_t* colptr_out, int32_t* rowval_out,
                             void* lower_out, void* gap_out) {
    if (!m || !colptr_out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (cb < 0 || ce > m->ncols || cb > ce) return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad column range");
    return guarded([&]() -> int {
        DeviceGuard g(m->device);
        std::vector<long long> cp(ce - cb + 1);
        CK(cudaMemcpy(cp.data(), m->colptr.as<long long>() + cb, sizeof(long long) * cp.size(), cudaMemcpyDeviceToHost));
        const long long b = cp[0], cnt = cp.back() - cp[0];
        for (size_t i = 0; i < cp.size(); ++i) colptr_out[i] = cp[i] - b;
        const size_t es = elem_size(m->dtype);
        if (cnt > 0) {
            if (rowval_out)
                CK(cudaMemcpy(rowval_out, m->rows.as<int>() + b, sizeof(int) * cnt, cudaMemcpyDeviceToHost));
            if (lower_out)
                CK(cudaMemcpy(lower_out, m->lower.as<char>() + b * es, es * cnt, cudaMemcpyDeviceToHost));
            if (gap_out) CK(cudaMemcpy(gap_out, m->gap.as<char>() + b * es, es * cnt, cudaMemcpyDeviceToHost));
        }
        return RIMDP_OK;
    });
}

} // extern "C"

// ---------------------------------------------------------------------------
// Multi-GPU solves in one process: the model's states cut into
// contiguous, transition-balanced shards, one per device, exchanging V over
// peer memory every iteration (rimdp_exchange_connect_local).  The drop-in
// layer reaches it through rimdp_b200::SolverOptions::gpus.

struct rimdp_multi {
    std::vector<rimdp_model*> shards;
    std::vector<int> sbeg, cbeg; // state / column begin of each shard (world + 1 entries)
    int n = 0, ncols = 0;
    rimdp_dtype dtype = RIMDP_F64;
    ~rimdp_multi() {
        for (rimdp_model* m : shards) rimdp_model_destroy(m);
    }
};

namespace {

template <class T>
int multi_solve_t(rimdp_multi* mm, const rimdp_plan* p, const rimdp_outputs* o) {
    const int W = (int)mm->shards.size(), N = mm->n;
    // per-shard plans: forced columns are global column indices, the shards' stores are local
    std::vector<std::vector<int>> fl(W);
    std::vector<rimdp_plan> pl(W, *p);
    const long long rows = (p->forced && p->forced_time_dependent) ? std::max<long long>(p->horizon, 1) : 1;
    if (p->forced) {
        for (int r = 0; r < W; ++r) {
            fl[r].assign(p->forced, p->forced + rows * N);
            for (long long t = 0; t < rows; ++t)
                for (int s = mm->sbeg[r]; s < mm->sbeg[r + 1]; ++s) {
                    int& f = fl[r][t * N + s];
                    if (f >= 0) f -= mm->cbeg[r];
                }
            pl[r].forced = fl[r].data();
        }
    }
    for (int r = 0; r < W; ++r)
        if (int st = check_plan(mm->shards[r], &pl[r])) return st;
    if (p->finite ? p->horizon > 0 : true) {
        // the first infeasible column a step evaluates: iteration rows first, then states in order
        for (long long it = 0; it < rows; ++it)
            for (int r = 0; r < W; ++r)
                if (const Infeasible* f = first_evaluated_infeasible(mm->shards[r], &pl[r], it))
                    return report_infeasible(f, mm->dtype, mm->shards[r]->col_offset);
    }
    for (int r = 0; r < W; ++r) {
        rimdp_model* m = mm->shards[r];
        DeviceGuard g(m->device);
        upload_plan<T>(m, &pl[r]);
        prepare_chosen(m, o, &pl[r]);
    }
    for (rimdp_model* m : mm->shards) { // every window reset before any rank publishes iteration 1
        DeviceGuard g(m->device);
        CK(cudaStreamSynchronize(m->stream));
    }
    // one iteration per shard in turn: a launch that blocks on a full launch queue (a shard's kernels wait in
    // peer_sync_stop for the other shards' flags) then always finds the other shards' same iteration
    // already enqueued, so they can progress and drain it
    auto advance_all = [&](long long it) {
        for (long long i = 0; i < it; ++i)
            for (rimdp_model* m : mm->shards) {
                DeviceGuard g(m->device);
                advance_t<T>(m, 1);
            }
    };
    auto poll_all = [&]() {
        Ctl c0{};
        for (int r = W - 1; r >= 0; --r) {
            DeviceGuard g(mm->shards[r]->device);
            const Ctl c = read_ctl(mm->shards[r]);
            if (r == 0) c0 = c;
        }
        return c0;
    };
    rimdp_model* m0 = mm->shards[0];
    const long long total = p->finite ? p->horizon : std::max<long long>(1, p->max_iterations);
    long long k = 0;
    Ctl c{};
    if (o && o->on_iteration) {
        std::vector<T> hv(N);
        while (k < total) {
            advance_all(1);
            c = poll_all();
            k = c.k;
            DeviceGuard g(m0->device);
            CK(cudaMemcpy(hv.data(), m0->s.vb[k & 1], sizeof(T) * N, cudaMemcpyDeviceToHost));
            o->on_iteration(k, hv.data(), o->user);
            if (c.done) break;
        }
    } else {
        ChunkPlanner cp(p);
        while (!c.done && m0->s.launched < total) {
            advance_all(cp.next());
            c = poll_all();
            cp.observe(c.k, c.res_last);
        }
        k = c.k;
    }
    for (rimdp_model* m : mm->shards) {
        DeviceGuard g(m->device);
        if (read_ctl(m).status == 2) return fail(RIMDP_ERR_INTERNAL, "partial-assignment overflow in a long column");
    }
    {
        DeviceGuard g(m0->device);
        rimdp_outputs o0{};
        if (o) {
            o0.values = o->values;
            o0.residual = o->residual;
            o0.iterations = o->iterations;
        }
        finish_t<T>(m0, &o0, k);
    }
    if (o && o->chosen) {
        const long long crow = (o->record_all_steps && p->finite) ? std::max<long long>(p->horizon, 0) : 1;
        for (int r = 0; r < W; ++r) {
            rimdp_model* m = mm->shards[r];
            if (!m->s.chosen.p || m->n == 0) continue;
            DeviceGuard g(m->device);
            std::vector<int> loc((size_t)m->n * crow);
            CK(cudaMemcpy(loc.data(), m->s.chosen.p, sizeof(int) * loc.size(), cudaMemcpyDeviceToHost));
            for (long long t = 0; t < crow; ++t)
                for (int s = 0; s < m->n; ++s) {
                    const int ch = loc[t * m->n + s];
                    o->chosen[t * N + mm->sbeg[r] + s] = ch >= 0 ? ch + mm->cbeg[r] : ch;
                }
        }
    }
    for (rimdp_model* m : mm->shards) m->s.active = false;
    if (c.status == 1) {
        fail(RIMDP_ERR_NON_CONVERGENCE, "no convergence after %lld iterations (max residual %f)", k, c.res_last);
        g_err_info.iterations = k;
        g_err_info.residual = c.res_last;
        return RIMDP_ERR_NON_CONVERGENCE;
    }
    return RIMDP_OK;
}

} // namespace

extern "C" {

int rimdp_multi_create(const rimdp_model_desc* d, int32_t world, const int32_t* devices, rimdp_multi** out) {
    if (!d || !out) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (world < 1 || world > kMaxWorld) return fail(RIMDP_ERR_INVALID_ARGUMENT, "world %d outside 1..%d", world, kMaxWorld);
    if (d->num_states < 0 || d->num_cols < 0 || d->nnz < 0 || !d->stateptr || !d->colptr)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "bad model sizes");
    if (d->stateptr[0] != 0 || d->stateptr[d->num_states] != d->num_cols || d->colptr[0] != 0 ||
        d->colptr[d->num_cols] != d->nnz)
        return fail(RIMDP_ERR_INVALID_ARGUMENT, "stateptr / colptr must run from 0 to num_cols / nnz");
    return guarded([&]() -> int {
        std::unique_ptr<rimdp_multi> mm(new rimdp_multi);
        mm->n = d->num_states;
        mm->ncols = d->num_cols;
        mm->dtype = d->dtype;
        const int n = d->num_states;
        const int64_t* cp = d->colptr;
        const int32_t* sp = d->stateptr;
        // transition-balanced cut: shard r starts at the first state whose columns begin at >= r/world of nnz
        mm->sbeg.assign(world + 1, n);
        mm->sbeg[0] = 0;
        for (int r = 1; r < world; ++r) {
            const long long target = (long long)((__int128)d->nnz * r / world);
            int lo = mm->sbeg[r - 1], hi = n;
            while (lo < hi) {
                const int mid = lo + (hi - lo) / 2;
                if (cp[sp[mid]] >= target) hi = mid;
                else lo = mid + 1;
            }
            mm->sbeg[r] = lo;
        }
        mm->cbeg.resize(world + 1);
        for (int r = 0; r <= world; ++r) mm->cbeg[r] = sp[mm->sbeg[r]];
        const size_t es = elem_size(d->dtype);
        for (int r = 0; r < world; ++r) {
            const int sb = mm->sbeg[r], se = mm->sbeg[r + 1], cb = mm->cbeg[r], ce = mm->cbeg[r + 1];
            const int64_t zb = cp[cb], ze = cp[ce];
            std::vector<int32_t> lsp(se - sb + 1);
            std::vector<int64_t> lcp(ce - cb + 1);
            for (int s = sb; s <= se; ++s) lsp[s - sb] = sp[s] - cb;
            for (int c = cb; c <= ce; ++c) lcp[c - cb] = cp[c] - zb;
            rimdp_model_desc ld = *d;
            ld.device = devices ? devices[r] : r;
            ld.num_states = se - sb;
            ld.num_cols = ce - cb;
            ld.nnz = ze - zb;
            ld.stateptr = lsp.data();
            ld.colptr = lcp.data();
            ld.rowval = d->rowval ? d->rowval + zb : nullptr;
            ld.lower = d->lower ? static_cast<const char*>(d->lower) + zb * es : nullptr;
            ld.upper = d->upper ? static_cast<const char*>(d->upper) + zb * es : nullptr;
            rimdp_model* m = nullptr;
            g_shard_col_offset = cb; // violations found at upload name global columns
            const int st = rimdp_model_create_shard(&ld, sb, n, &m);
            g_shard_col_offset = 0;
            if (st) return st;
            mm->shards.push_back(m);
            m->col_offset = cb;
            m->value_capacity = n;
        }
        if (int st = rimdp_exchange_connect_local(mm->shards.data(), world)) return st;
        *out = mm.release();
        return RIMDP_OK;
    });
}

int rimdp_multi_solve(rimdp_multi* mm, const rimdp_plan* p, const rimdp_outputs* o) {
    if (!mm || !p) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    if (!p->initial) return fail(RIMDP_ERR_INVALID_ARGUMENT, "plan.initial is required");
    return guarded([&]() -> int {
        rimdp_outputs none{};
        return mm->dtype == RIMDP_F64 ? multi_solve_t<double>(mm, p, o ? o : &none)
                                      : multi_solve_t<float>(mm, p, o ? o : &none);
    });
}

int rimdp_multi_info(rimdp_multi* mm, int32_t* world, int32_t* state_begin, int32_t* devices) {
    if (!mm) return fail(RIMDP_ERR_INVALID_ARGUMENT, "null argument");
    const int W = (int)mm->shards.size();
    if (world) *world = W;
    for (int r = 0; r < W; ++r) {
        if (state_begin) state_begin[r] = mm->sbeg[r];
        if (devices) devices[r] = mm->shards[r]->device;
    }
    if (state_begin) state_begin[W] = mm->n;
    return RIMDP_OK;
}

int rimdp_multi_destroy(rimdp_multi* mm) {
    delete mm;
    return RIMDP_OK;
}

} // extern "C"
