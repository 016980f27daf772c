// Native IMDPCSC1 model containers -> the engine's CSC arrays (SURVEY §8f
// rank 2): the on-disk form of the device store, read without building the
// reference's host objects, then uploaded with rimdp_model_create and checked
// on the device (rimdp_model_validate).
//
// Follows read_native_model (io/native.hpp:457-561):
//   * container: magic "IMDPCSC1", u32 attribute count, (u32 len, key, u32
//     len, value)*, u32 variable count, (u32 len, key, u8 dtype, u64 count,
//     payload)* with dtype 1 int32, 2 f64, 3 f32, 4 string, 5 rational
//     (native.hpp:15-41, 295-347);
//   * attributes model = imc|imdp, format = sparse_csc, rows = to,
//     cols = from | from/action, num_states > 0 (native.hpp:486-500);
//   * variables lower/upper colptr/rowval (int32) and nzval (f64 or f32: an
//     f64 store accepts either, an f32 store only f32 — NativeValueCodec,
//     native.hpp:206-225); stateptr + action_vals for imdp; imc promotes to
//     one action "0" per state (native.hpp:519-532);
//   * row bounds (native.hpp:536-541), CscMatrix::structural_violation of
//     both matrices (csc.hpp:75-107), the pattern merge of
//     IntervalProbabilities::align (interval.hpp:218-252) and the removal of
//     [0, 0] entries (interval.hpp:261-279);
//   * IntervalMDP::validate's structure checks (imdp.hpp:129-168).
//   * the entry and column-sum checks of IntervalProbabilities::validate
//     (interval.hpp:132-179) on the aligned pattern, before [0,0] removal.
// 64-bit extension: the reference's int32 colptr caps a
// container at 2^31-1 transitions (native.hpp:514-517), so BASELINE config 4
// (5.12e9) cannot be stored.  Variables of dtype 6 = int64 are accepted for
// lower_colptr / upper_colptr (the reference's reader rejects dtype 6 as
// unknown, so such files are engine files); rimdp_native_write emits them
// when the model needs them (or when asked), and int32 otherwise — then the
// file is byte-identical to the reference's write_native_model.
// Every failure is a SchemaViolation whose message is "schema violation:
// <path>: <reason>" as in the reference (errors.hpp:92-95).  The JSON debug
// variant of the container is not read here (text parsing is out of scope).
#include "rimdp_b200.h"

#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

extern "C" int rimdp_internal_fail(int status, const char* msg);

namespace {

struct SchemaError : std::runtime_error {
    int status;
    SchemaError(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

struct Var {
    uint8_t dtype = 0;
    std::vector<int32_t> i32;
    std::vector<int64_t> i64; // dtype 6: 64-bit column pointers (engine extension)
    std::vector<double> f64;
    std::vector<float> f32;
    std::vector<std::string> str;
    uint64_t count = 0;
};

class Reader {
public:
    Reader(const std::string& path) : path_(path), in_(path, std::ios::binary) {
        if (!in_) throw SchemaError(RIMDP_ERR_MISSING_FILE, "missing file: " + path); // errors.hpp MissingFile
    }
    // SchemaViolation (errors.hpp:92-95) thrown as path + ": " + reason (native.hpp:459-461)
    [[noreturn]] void fail(const std::string& why) {
        throw SchemaError(RIMDP_ERR_SCHEMA, "schema violation: " + path_ + ": " + why);
    }
    // a ModelError caught by read_native_model (native.hpp:557-559): Violation::to_string (errors.hpp:156-163)
    [[noreturn]] void model_error(const char* kind, const std::string& msg, long long state = -1,
                                  long long column = -1, long long row = -1) {
        std::string v = kind;
        if (state >= 0) v += " state=" + std::to_string(state);
        if (column >= 0) v += " column=" + std::to_string(column);
        if (row >= 0) v += " row=" + std::to_string(row);
        fail(v + ": " + msg);
    }
    void bytes(void* p, size_t n) {
        in_.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
        if (static_cast<size_t>(in_.gcount()) != n) fail("unexpected end of file");
    }
    uint8_t u8() { uint8_t v; bytes(&v, 1); return v; }
    uint32_t u32() { uint32_t v; bytes(&v, 4); return v; }
    uint64_t u64() { uint64_t v; bytes(&v, 8); return v; }
    std::string str() {
        const uint32_t n = u32();
        if (n > (1u << 28)) fail("string length implausibly large");
        std::string s(n, '\0');
        if (n) bytes(s.data(), n);
        return s;
    }

private:
    std::string path_;
    std::ifstream in_;
};

// NumericTraits<V>::to_string (numeric.hpp:31-35): shortest round-trip form
template <class V>
std::string num(V v) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

template <class V>
struct Model {
    int32_t num_states = 0;
    int32_t num_cols = 0;
    bool imdp = true;
    std::vector<int32_t> stateptr;
    std::vector<int64_t> colptr;
    std::vector<int32_t> rowval;
    std::vector<V> lower, upper;
    std::vector<std::string> labels;
};

template <class V>
std::unique_ptr<Model<V>> read_model(const std::string& path) {
    Reader in(path);
    char magic[8];
    {
        std::ifstream probe(path, std::ios::binary);
        probe.read(magic, 8);
        if (probe.gcount() != 8 || std::memcmp(magic, "IMDPCSC1", 8) != 0)
            in.fail("not an IMDPCSC1 binary container (the JSON debug variant is read by the reference "
                    "tools only)");
    }
    in.bytes(magic, 8);
    std::map<std::string, std::string> attrs;
    std::map<std::string, Var> vars;
    const uint32_t na = in.u32();
    for (uint32_t i = 0; i < na; ++i) {
        std::string k = in.str();
        attrs[k] = in.str();
    }
    const uint32_t nv = in.u32();
    for (uint32_t i = 0; i < nv; ++i) {
        std::string key = in.str();
        Var v;
        v.dtype = in.u8();
        v.count = in.u64();
        if (v.count > (1ull << 33)) in.fail("variable " + key + " implausibly large");
        switch (v.dtype) {
        case 1: v.i32.resize(v.count); if (v.count) in.bytes(v.i32.data(), 4 * v.count); break;
        case 6: v.i64.resize(v.count); if (v.count) in.bytes(v.i64.data(), 8 * v.count); break;
        case 2: v.f64.resize(v.count); if (v.count) in.bytes(v.f64.data(), 8 * v.count); break;
        case 3: v.f32.resize(v.count); if (v.count) in.bytes(v.f32.data(), 4 * v.count); break;
        case 4: v.str.resize(v.count); for (auto& s : v.str) s = in.str(); break;
        case 5: {
            std::vector<int64_t> skip(2 * v.count);
            if (v.count) in.bytes(skip.data(), 16 * v.count);
            break;
        }
        default: in.fail("unknown dtype " + std::to_string(v.dtype) + " for variable " + key);
        }
        vars[key] = std::move(v);
    }
    auto attr = [&](const char* k) -> const std::string& {
        auto it = attrs.find(k);
        if (it == attrs.end()) in.fail(std::string("missing attribute ") + k);
        return it->second;
    };
    const std::string model = attr("model");
    if (model != "imc" && model != "imdp") in.fail("model must be imc or imdp");
    if (attr("format") != "sparse_csc") in.fail("format must be sparse_csc");
    if (attr("rows") != "to") in.fail("rows must be to");
    const std::string expected_cols = model == "imc" ? "from" : "from/action";
    if (attr("cols") != expected_cols) in.fail("cols must be " + expected_cols + " for model " + model);
    long long ns = -1;
    {
        const std::string& s = attr("num_states");
        auto r = std::from_chars(s.data(), s.data() + s.size(), ns);
        if (r.ec != std::errc() || r.ptr != s.data() + s.size()) ns = -1;
    }
    if (ns <= 0 || ns > INT32_MAX) in.fail("bad num_states");
    auto var = [&](const char* k) -> Var& {
        auto it = vars.find(k);
        if (it == vars.end()) in.fail(std::string("missing variable ") + k);
        return it->second;
    };
    auto ints = [&](const char* k) -> std::vector<int32_t>& {
        Var& v = var(k);
        if (v.dtype != 1) in.fail(std::string("variable ") + k + " must be int32");
        return v.i32;
    };
    auto values = [&](const char* k) -> std::vector<V> {
        Var& v = var(k);
        std::vector<V> out;
        if constexpr (sizeof(V) == 8) {
            if (v.dtype == 2) out.assign(v.f64.begin(), v.f64.end());
            else if (v.dtype == 3) out.assign(v.f32.begin(), v.f32.end());
            else in.fail(std::string("variable ") + k + " is not floating point");
        } else {
            if (v.dtype != 3) in.fail(std::string("variable ") + k + " is not float32; convert explicitly");
            out.assign(v.f32.begin(), v.f32.end());
        }
        return out;
    };
    // column pointers: int32 (the reference) or int64 (dtype 6)
    auto ptrs = [&](const char* k) -> std::vector<int64_t> {
        Var& v = var(k);
        if (v.dtype == 1) return std::vector<int64_t>(v.i32.begin(), v.i32.end());
        if (v.dtype == 6) return std::move(v.i64);
        in.fail(std::string("variable ") + k + " must be int32 or int64");
    };
    const std::vector<int64_t> lcp = ptrs("lower_colptr");
    const std::vector<int32_t>& lrv = ints("lower_rowval");
    const std::vector<int64_t> ucp = ptrs("upper_colptr");
    const std::vector<int32_t>& urv = ints("upper_rowval");
    const std::vector<V> lnz = values("lower_nzval");
    const std::vector<V> unz = values("upper_nzval");
    if (ucp.empty()) in.fail("empty upper_colptr");
    const int64_t ncols = static_cast<int64_t>(ucp.size()) - 1;
    if (static_cast<int64_t>(lcp.size()) - 1 != ncols) in.fail("lower and upper matrices must have the same column count");

    auto m = std::make_unique<Model<V>>();
    m->num_states = static_cast<int32_t>(ns);
    m->num_cols = static_cast<int32_t>(ncols);
    m->imdp = model == "imdp";
    if (m->imdp) {
        m->stateptr = ints("stateptr");
        Var& lab = var("action_vals");
        if (lab.dtype != 4) in.fail("variable action_vals must be strings");
        m->labels = std::move(lab.str);
    } else {
        if (ncols != ns) in.fail("imc requires one column per state");
        m->stateptr.resize(ns + 1);
        for (int32_t s = 0; s <= ns; ++s) m->stateptr[s] = s;
        m->labels.assign(ns, "0");
    }
    for (int32_t r : lrv)
        if (r < 0 || r >= ns) in.fail("IndexOutOfBounds: lower_rowval entry");
    for (int32_t r : urv)
        if (r < 0 || r >= ns) in.fail("IndexOutOfBounds: upper_rowval entry");
    // CscMatrix::from_csc -> structural_violation (csc.hpp:75-107); ModelError -> SchemaViolation
    auto structural = [&](const std::vector<int64_t>& cp, const std::vector<int32_t>& rv, size_t nz) {
        const char* SE = "StructuralError";
        if (cp.front() != 0) in.model_error(SE, "colptr must start at 0");
        if (cp.back() != static_cast<int64_t>(rv.size()) || rv.size() != nz)
            in.model_error(SE, "value arrays do not match colptr");
        for (int64_t j = 0; j < ncols; ++j) {
            if (cp[j] > cp[j + 1]) in.model_error(SE, "colptr not monotone", -1, j);
            if (cp[j + 1] > static_cast<int64_t>(rv.size())) {
                // a later pointer decreases (front/back are checked): report that column instead of
                // reading past the row array (the reference's loop would read out of bounds here)
                int64_t d = j + 1;
                while (d < ncols && cp[d] <= cp[d + 1]) ++d;
                in.model_error(SE, "colptr not monotone", -1, d);
            }
            for (int64_t k = cp[j]; k < cp[j + 1]; ++k)
                if (k > cp[j] && rv[k] <= rv[k - 1])
                    in.model_error(SE, "row indices not strictly increasing within column", -1, j, rv[k]);
        }
    };
    structural(lcp, lrv, lnz.size());
    structural(ucp, urv, unz.size());
    // align (interval.hpp:218-252), check every entry and column sum of the
    // aligned pattern (IntervalProbabilities::validate, interval.hpp:132-179,
    // first violation wins as in check_or_throw :255-258), then drop [0, 0]
    // entries (:261-279).  Done column by column: the report is column-major.
    const V tol = sizeof(V) == 8 ? V(1e-9) : V(1e-5f); // NumericTraits feasibility_tolerance (numeric.hpp:53-81)
    m->colptr.reserve(ncols + 1);
    m->colptr.push_back(0);
    m->rowval.reserve(urv.size());
    m->lower.reserve(urv.size());
    m->upper.reserve(urv.size());
    for (int64_t j = 0; j < ncols; ++j) {
        int64_t a = lcp[j], ae = lcp[j + 1], b = ucp[j], be = ucp[j + 1];
        V lo_sum(0), up_sum(0);
        while (a < ae || b < be) {
            const int32_t ra = a < ae ? lrv[a] : INT32_MAX, rb = b < be ? urv[b] : INT32_MAX;
            int32_t r;
            V lo, up;
            if (ra < rb) { r = ra; lo = lnz[a++]; up = V(0); }
            else if (rb < ra) { r = rb; lo = V(0); up = unz[b++]; }
            else { r = ra; lo = lnz[a++]; up = unz[b++]; }
            if (!std::isfinite(lo) || lo < V(0) || lo > V(1))
                in.model_error("EntryOutOfRange", "lower bound " + num(lo) + " outside [0,1]", -1, j, r);
            if (!std::isfinite(up) || up < V(0) || up > V(1))
                in.model_error("EntryOutOfRange", "upper bound " + num(up) + " outside [0,1]", -1, j, r);
            if (lo > up)
                in.model_error("BoundOrderViolation", "lower bound " + num(lo) + " exceeds upper bound " + num(up),
                               -1, j, r);
            lo_sum += lo;
            up_sum += up;
            if (lo == V(0) && up == V(0)) continue;
            m->rowval.push_back(r);
            m->lower.push_back(lo);
            m->upper.push_back(up);
        }
        if (lo_sum > V(1) + tol) in.model_error("InfeasibleColumn", "lower bounds sum to " + num(lo_sum) + " > 1", -1, j);
        if (up_sum < V(1) - tol) in.model_error("InfeasibleColumn", "upper bounds sum to " + num(up_sum) + " < 1", -1, j);
        m->colptr.push_back(static_cast<int64_t>(m->rowval.size()));
    }
    // IntervalMDP structure (imdp.hpp:129-168): the first violation of the report
    const auto& sp = m->stateptr;
    const char* SE = "StructuralError";
    if (sp.empty() || sp.front() != 0) in.model_error(SE, "stateptr must start at 0");
    const int64_t nst = static_cast<int64_t>(sp.size()) - 1;
    if (nst != ns)
        in.model_error("DestinationCountMismatch", "transition matrix has " + std::to_string(ns) +
                                                       " destinations for " + std::to_string(nst) + " states");
    if (sp.back() != ncols)
        in.model_error(SE, "stateptr must end at the column count (" + std::to_string(sp.back()) + " != " +
                               std::to_string(ncols) + ")");
    if (static_cast<int64_t>(m->labels.size()) != ncols) in.model_error(SE, "one action label required per column");
    for (int64_t s = 0; s < nst; ++s) {
        if (sp[s + 1] <= sp[s]) in.model_error("EmptyActionSet", "state has no actions", s);
        if (sp[s + 1] > static_cast<int64_t>(m->labels.size())) continue;
        std::unordered_set<std::string> seen;
        for (int32_t c = sp[s]; c < sp[s + 1]; ++c)
            if (!seen.insert(m->labels[c]).second)
                in.model_error("DuplicateActionLabel", "action \"" + m->labels[c] + "\" occurs twice", s, c);
    }
    return m;
}

struct Handle {
    int dtype;
    std::unique_ptr<Model<double>> d;
    std::unique_ptr<Model<float>> f;
};

template <class V>
void sizes_of(const Model<V>& m, rimdp_native_sizes* s) {
    s->num_states = m.num_states;
    s->num_cols = m.num_cols;
    s->nnz = static_cast<int64_t>(m.rowval.size());
    s->imdp = m.imdp;
    int64_t lb = 0;
    for (const auto& l : m.labels) lb += static_cast<int64_t>(l.size()) + 1;
    s->label_bytes = lb;
}

template <class V>
void take(const Model<V>& m, int32_t* sp, int64_t* cp, int32_t* rv, void* lo, void* up, char* labels) {
    if (sp) std::memcpy(sp, m.stateptr.data(), sizeof(int32_t) * m.stateptr.size());
    if (cp) std::memcpy(cp, m.colptr.data(), sizeof(int64_t) * m.colptr.size());
    if (rv) std::memcpy(rv, m.rowval.data(), sizeof(int32_t) * m.rowval.size());
    if (lo) std::memcpy(lo, m.lower.data(), sizeof(V) * m.lower.size());
    if (up) std::memcpy(up, m.upper.data(), sizeof(V) * m.upper.size());
    if (labels)
        for (const auto& l : m.labels) {
            std::memcpy(labels, l.c_str(), l.size() + 1);
            labels += l.size() + 1;
        }
}

// ---- writer: the engine's aligned CSC arrays -> an IMDPCSC1 container ------
// Mirrors write_native_model (native.hpp:424-455) + write_container_binary
// (:251-292): attributes and variables in key order (std::map), both bound
// matrices with their zero entries stripped (IntervalProbabilities::lower_csc
// / upper_csc, interval.hpp:125-129), stateptr and action labels.

class Writer {
public:
    explicit Writer(const std::string& path) : path_(path), out_(path, std::ios::binary | std::ios::trunc) {
        if (!out_) throw SchemaError(RIMDP_ERR_INVALID_ARGUMENT, "cannot open " + path + " for writing");
    }
    template <class U>
    void le(U v) {
        char b[sizeof(U)];
        for (size_t i = 0; i < sizeof(U); ++i) b[i] = static_cast<char>((static_cast<uint64_t>(v) >> (8 * i)) & 0xff);
        out_.write(b, sizeof(U));
    }
    void u8(uint8_t v) { out_.put(static_cast<char>(v)); }
    void str(const std::string& s) {
        le<uint32_t>(static_cast<uint32_t>(s.size()));
        out_.write(s.data(), static_cast<std::streamsize>(s.size()));
    }
    template <class U>
    void raw(const std::vector<U>& v) {
        out_.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(U) * v.size()));
    }
    void finish() {
        out_.flush();
        if (!out_) throw SchemaError(RIMDP_ERR_INVALID_ARGUMENT, "write to " + path_ + " failed");
    }

private:
    std::string path_;
    std::ofstream out_;
};

template <class V>
void write_model(const char* path, int32_t ns, int32_t nc, const int32_t* sp, const int64_t* cp, const int32_t* rv,
                 const V* lower, const V* upper, const char* labels, int32_t index64) {
    // the two matrices, zero entries stripped
    std::vector<int64_t> lcp{0}, ucp{0};
    std::vector<int32_t> lrv, urv;
    std::vector<V> lnz, unz;
    for (int32_t c = 0; c < nc; ++c) {
        for (int64_t k = cp[c]; k < cp[c + 1]; ++k) {
            if (lower[k] != V(0)) { lrv.push_back(rv[k]); lnz.push_back(lower[k]); }
            if (upper[k] != V(0)) { urv.push_back(rv[k]); unz.push_back(upper[k]); }
        }
        lcp.push_back(static_cast<int64_t>(lrv.size()));
        ucp.push_back(static_cast<int64_t>(urv.size()));
    }
    const bool wide = index64 != 0 || lcp.back() > INT32_MAX || ucp.back() > INT32_MAX;
    std::vector<std::string> labs;
    if (labels) {
        const char* q = labels;
        for (int32_t c = 0; c < nc; ++c) {
            labs.emplace_back(q);
            q += labs.back().size() + 1;
        }
    } else { // positional labels "0", "1", ... within each state
        for (int32_t st = 0; st < ns; ++st)
            for (int32_t c = sp[st]; c < sp[st + 1]; ++c) labs.push_back(std::to_string(c - sp[st]));
    }
    Writer w(path);
    w.raw(std::vector<char>{'I', 'M', 'D', 'P', 'C', 'S', 'C', '1'});
    w.le<uint32_t>(5);
    const std::pair<const char*, std::string> attrs[5] = {
        {"cols", "from/action"}, {"format", "sparse_csc"}, {"model", "imdp"}, {"num_states", std::to_string(ns)},
        {"rows", "to"}};
    for (const auto& [k, v] : attrs) {
        w.str(k);
        w.str(v);
    }
    w.le<uint32_t>(8);
    const uint8_t vdt = sizeof(V) == 8 ? 2 : 3;
    auto ptr_var = [&](const char* key, const std::vector<int64_t>& p) {
        w.str(key);
        w.u8(wide ? 6 : 1);
        w.le<uint64_t>(p.size());
        if (wide) {
            w.raw(p);
        } else {
            std::vector<int32_t> n(p.begin(), p.end());
            w.raw(n);
        }
    };
    auto var = [&](const char* key, uint8_t dt, const auto& v) {
        w.str(key);
        w.u8(dt);
        w.le<uint64_t>(v.size());
        w.raw(v);
    };
    w.str("action_vals");
    w.u8(4);
    w.le<uint64_t>(labs.size());
    for (const auto& l : labs) w.str(l);
    ptr_var("lower_colptr", lcp);
    var("lower_nzval", vdt, lnz);
    var("lower_rowval", 1, lrv);
    var("stateptr", 1, std::vector<int32_t>(sp, sp + ns + 1));
    ptr_var("upper_colptr", ucp);
    var("upper_nzval", vdt, unz);
    var("upper_rowval", 1, urv);
    w.finish();
}

} // namespace

extern "C" {

int rimdp_native_write(const char* path, int32_t dtype, int32_t num_states, int32_t num_cols, const int32_t* stateptr,
                       const int64_t* colptr, const int32_t* rowval, const void* lower, const void* upper,
                       const char* labels, int32_t index64) {
    if (!path || !stateptr || !colptr || num_states < 0 || num_cols < 0 || (dtype != RIMDP_F64 && dtype != RIMDP_F32) ||
        (colptr[num_cols] > 0 && (!rowval || !lower || !upper)))
        return rimdp_internal_fail(RIMDP_ERR_INVALID_ARGUMENT, "rimdp_native_write: bad argument");
    try {
        if (dtype == RIMDP_F64)
            write_model<double>(path, num_states, num_cols, stateptr, colptr, rowval, static_cast<const double*>(lower),
                                static_cast<const double*>(upper), labels, index64);
        else
            write_model<float>(path, num_states, num_cols, stateptr, colptr, rowval, static_cast<const float*>(lower),
                               static_cast<const float*>(upper), labels, index64);
        return RIMDP_OK;
    } catch (const SchemaError& e) {
        return rimdp_internal_fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return rimdp_internal_fail(RIMDP_ERR_OUT_OF_MEMORY, "host allocation failed");
    }
}


int rimdp_native_read(const char* path, int32_t dtype, rimdp_native_sizes* sizes, void** handle) {
    if (!path || !sizes || !handle || (dtype != RIMDP_F64 && dtype != RIMDP_F32))
        return rimdp_internal_fail(RIMDP_ERR_INVALID_ARGUMENT, "rimdp_native_read: bad argument");
    try {
        auto h = std::make_unique<Handle>();
        h->dtype = dtype;
        if (dtype == RIMDP_F64) {
            h->d = read_model<double>(path);
            sizes_of(*h->d, sizes);
        } else {
            h->f = read_model<float>(path);
            sizes_of(*h->f, sizes);
        }
        *handle = h.release();
        return RIMDP_OK;
    } catch (const SchemaError& e) {
        return rimdp_internal_fail(e.status, e.what());
    } catch (const std::bad_alloc&) {
        return rimdp_internal_fail(RIMDP_ERR_OUT_OF_MEMORY, "host allocation failed");
    }
}

int rimdp_native_take(void* handle, int32_t* stateptr, int64_t* colptr, int32_t* rowval, void* lower, void* upper,
                      char* labels) {
    if (!handle) return rimdp_internal_fail(RIMDP_ERR_INVALID_ARGUMENT, "rimdp_native_take: null handle");
    Handle* h = static_cast<Handle*>(handle);
    if (h->dtype == RIMDP_F64)
        take(*h->d, stateptr, colptr, rowval, lower, upper, labels);
    else
        take(*h->f, stateptr, colptr, rowval, lower, upper, labels);
    return RIMDP_OK;
}

void rimdp_native_free(void* handle) { delete static_cast<Handle*>(handle); }

} // extern "C"
