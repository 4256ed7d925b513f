// Header-only C++ shim: the reference's engine API (proj/include/walkforge/
// engine.hpp, interleave.hpp, algorithms.hpp, walker.hpp, graph.hpp, error.hpp)
// with the same names and template signatures, executed by the B200 engine
// through the C-ABI in walkforge_b200.h.
//
// A caller of the reference switches by including this header instead of
// <walkforge/engine.hpp> + <walkforge/interleave.hpp> + <walkforge/algorithms.hpp>
// (define WALKFORGE_B200_DROP_IN to alias namespace walkforge) and linking
// libwalkforge_b200.so.  Differences, all checked at the boundary:
//   * weights keep their f64 values (an f64 copy stays resident when some
//     weight is not float32-exact); labels must be < 256 — otherwise ConfigError;
//   * programs are the five built-ins or a user's device program: a type written
//     against walkforge_b200/device_program.cuh in the user's .cu file, passed
//     here as DeviceProgram(ops, object) (the ops table its WF_DEVICE_PROGRAM
//     exports);
//   * ExecOptions::threads keeps its meaning — the run is split into that many
//     contiguous worker blocks, each handed to the sink once, in worker order —
//     and the blocks are spread over min(threads, visible GPUs) devices
//     (wf_multi_*); prefetch is accepted and ignored; k / k' of
//     run_interleaved are validated then used as launch hints.
#pragma once

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <type_traits>
#include <fstream>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../walkforge_b200.h"

namespace walkforge_b200 {

// ---- errors: error.hpp:8-48 ---------------------------------------------------------
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ParseError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct DistributionError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct RejectionCapError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };

inline void check(int rc) {
    if (rc == WF_OK) return;
    std::string m = wf_last_error();
    switch (rc) {
        case WF_ERR_PARSE: throw ParseError(m);
        case WF_ERR_FORMAT: throw FormatError(m);
        case WF_ERR_CONFIG: throw ConfigError(m);
        case WF_ERR_DISTRIBUTION: throw DistributionError(m);
        case WF_ERR_CONTRACT: throw ContractError(m);
        case WF_ERR_REJECTION_CAP: throw RejectionCapError(m);
        case WF_ERR_IO: throw IoError(m);
        default: throw DeviceError(m);
    }
}

using VertexId = uint32_t;

// ---- sampler.hpp:21 / program.hpp:17 / walker.hpp:12 ---------------------------------
enum class SamplerKind : uint8_t { Naive, Its, Alias, Rej, ORej };
enum class WalkerType : uint8_t { Unbiased, Static, Dynamic };
enum class WalkStatus : uint8_t { Complete, DeadEnd };

// The reference's names for them (sampler.cpp:7-26, program.hpp:19-26,
// walker.hpp:14-16): what its CLI prints and parses.
inline const char* to_string(SamplerKind kind) {
    switch (kind) {
        case SamplerKind::Naive: return "naive";
        case SamplerKind::Its: return "its";
        case SamplerKind::Alias: return "alias";
        case SamplerKind::Rej: return "rej";
        case SamplerKind::ORej: return "orej";
    }
    return "?";
}
inline SamplerKind parse_sampler(const std::string& name) {
    for (SamplerKind k : {SamplerKind::Naive, SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej, SamplerKind::ORej})
        if (name == to_string(k)) return k;
    if (name == "o-rej") return SamplerKind::ORej;
    throw ConfigError("unknown sampler '" + name + "'");
}
inline const char* to_string(WalkerType type) {
    switch (type) {
        case WalkerType::Unbiased: return "unbiased";
        case WalkerType::Static: return "static";
        case WalkerType::Dynamic: return "dynamic";
    }
    return "?";
}
inline const char* to_string(WalkStatus status) { return status == WalkStatus::Complete ? "complete" : "dead_end"; }
inline constexpr uint32_t kNoAlias = UINT32_MAX;      // sampler.hpp:26
inline constexpr uint32_t kRejTrialCap = 1u << 20;    // sampler.hpp:27

// ---- Graph (graph.hpp:17-107), resident in HBM ---------------------------------------
class Graph {
public:
    Graph() = default;
    static Graph from_csr(std::vector<uint64_t> offsets, std::vector<VertexId> neighbors,
                          std::vector<double> weights = {}, std::vector<uint32_t> labels = {},
                          int device = 0) {
        if (offsets.size() < 2) throw ConfigError("graph must have at least one vertex");
        if (!weights.empty() && weights.size() != neighbors.size())
            throw ConfigError("weight array does not match edge count");
        if (!labels.empty() && labels.size() != neighbors.size())
            throw ConfigError("label array does not match edge count");
        wf_graph* h = nullptr;
        check(wf_graph_create_f64(offsets.data(), neighbors.data(), weights.empty() ? nullptr : weights.data(),
                              labels.empty() ? nullptr : labels.data(),
                              static_cast<uint32_t>(offsets.size() - 1), neighbors.size(), device, &h));
        Graph g;
        g.h_ = std::shared_ptr<wf_graph>(h, wf_graph_destroy);
        check(wf_graph_info_get(h, &g.info_));
        return g;
    }
    uint32_t vertex_count() const { return info_.vertex_count; }
    uint64_t edge_count() const { return info_.edge_count; }
    bool has_weights() const { return info_.has_weights != 0; }
    bool has_labels() const { return info_.has_labels != 0; }
    double max_weight() const { return info_.max_weight; }
    uint64_t max_degree() const { return info_.max_degree_lo; }
    bool adjacency_sorted() const { return info_.adjacency_sorted != 0; }
    bool has_edge(VertexId src, VertexId dst) const {
        uint8_t out = 0;
        check(wf_graph_has_edge(h_.get(), &src, &dst, 1, &out));
        return out != 0;
    }
    double avg_degree() const { return static_cast<double>(edge_count()) / vertex_count(); }

    // Host-side CSR accessors (graph.hpp:27-71).  The CSR lives in HBM; the
    // first accessor call downloads one host copy (wf_graph_download), shared
    // by copies of this Graph.
    uint64_t edge_begin(VertexId v) const { return host().offsets[v]; }
    uint32_t degree(VertexId v) const {
        check_vertex(v);
        const HostCsr& c = host();
        return static_cast<uint32_t>(c.offsets[v + 1] - c.offsets[v]);
    }
    std::span<const VertexId> neighbors(VertexId v) const {
        check_vertex(v);
        const HostCsr& c = host();
        return {c.neighbors.data() + c.offsets[v], c.neighbors.data() + c.offsets[v + 1]};
    }
    VertexId neighbor(uint64_t edge) const { return host().neighbors[edge]; }
    double weight(uint64_t edge) const {
        check_edge(edge);
        if (!has_weights()) throw ConfigError("graph has no edge weights");
        return host().weights[edge];
    }
    uint32_t label(uint64_t edge) const {
        check_edge(edge);
        if (!has_labels()) throw ConfigError("graph has no edge labels");
        return host().labels[edge];
    }
    const uint64_t* offsets_data() const { return host().offsets.data(); }
    const VertexId* neighbors_data() const { return host().neighbors.data(); }
    const double* weights_data() const { return has_weights() ? host().weights.data() : nullptr; }
    const uint32_t* labels_data() const { return has_labels() ? host().labels.data() : nullptr; }

    // WFG1 files (graph.cpp:190-277), byte-identical to the reference's.
    void write_binary(const std::string& path) const { check(wf_graph_write_wfg1(h_.get(), path.c_str())); }
    static Graph read_binary(const std::string& path, int device = 0) {
        wf_graph* h = nullptr;
        check(wf_graph_read_wfg1(path.c_str(), device, &h));
        return adopt(h);
    }
    static Graph adopt(wf_graph* h) {
        Graph g;
        g.h_ = std::shared_ptr<wf_graph>(h, wf_graph_destroy);
        check(wf_graph_info_get(h, &g.info_));
        return g;
    }
    wf_graph* handle() const { return h_.get(); }
    int32_t device() const { return info_.device; }

private:
    struct HostCsr {
        std::vector<uint64_t> offsets;
        std::vector<VertexId> neighbors;
        std::vector<double> weights;  // f64, as the reference holds them
        std::vector<uint32_t> labels;
    };
    const HostCsr& host() const {
        if (!csr_) {
            auto c = std::make_shared<HostCsr>();
            c->offsets.resize(vertex_count() + 1ull);
            c->neighbors.resize(edge_count());
            std::vector<uint8_t> l(has_labels() ? edge_count() : 0);
            check(wf_graph_download(h_.get(), c->offsets.data(), c->neighbors.data(), nullptr,
                                    l.empty() ? nullptr : l.data()));
            c->weights.resize(has_weights() ? edge_count() : 0);
            if (!c->weights.empty()) check(wf_graph_download_weights_f64(h_.get(), c->weights.data()));
            c->labels.assign(l.begin(), l.end());
            csr_ = std::move(c);
        }
        return *csr_;
    }
    void check_vertex(VertexId v) const {  // graph.hpp:87-91
        if (v >= vertex_count())
            throw ConfigError("vertex id " + std::to_string(v) + " out of range (V=" +
                              std::to_string(vertex_count()) + ")");
    }
    void check_edge(uint64_t e) const {  // graph.hpp:93-96
        if (e >= edge_count()) throw ConfigError("edge index " + std::to_string(e) + " out of range");
    }
    std::shared_ptr<wf_graph> h_;
    wf_graph_info info_{};
    mutable std::shared_ptr<const HostCsr> csr_;
};

// ---- load_edge_list (graph.hpp:119-139, graph.cpp:307-453) --------------------------------
enum class Directedness : uint8_t { Directed, Undirected };
enum class WeightMode : uint8_t { None, FromFile, Random };
enum class LabelMode : uint8_t { None, FromFile, Random };
struct EdgeListOptions {
    Directedness directedness = Directedness::Directed;
    WeightMode weights = WeightMode::None;
    LabelMode labels = LabelMode::None;
    uint32_t label_count = 5;
    uint64_t seed = 0;
};
struct LoadedGraph {
    Graph graph;
    std::vector<uint64_t> original_ids;
};
inline LoadedGraph load_edge_list(const std::string& path, const EdgeListOptions& o = {}, int device = 0) {
    wf_edge_list_options c{};
    c.undirected = o.directedness == Directedness::Undirected ? 1 : 0;
    c.weights = static_cast<int32_t>(o.weights);  // None / FromFile / Random map 1:1 (wf_attr_mode)
    c.labels = static_cast<int32_t>(o.labels);
    c.label_count = o.label_count;
    c.seed = o.seed;
    wf_graph* h = nullptr;
    check(wf_graph_load_edge_list(path.c_str(), &c, device, &h));
    LoadedGraph lg{Graph::adopt(h), {}};
    lg.original_ids.resize(lg.graph.vertex_count());
    check(wf_graph_original_ids(h, lg.original_ids.data()));
    return lg;
}

// ---- build_graph (graph.hpp:141-144, graph.cpp:289-305) -----------------------------------
// CSR assembly from an unsorted edge set: edges ordered by (source,
// destination), input order breaking ties, weights and labels following their
// edges; then Graph::from_csr's validation.
inline Graph build_graph(uint32_t vertex_count, std::vector<std::pair<VertexId, VertexId>> edges,
                         std::vector<double> weights = {}, std::vector<uint32_t> labels = {}, int device = 0) {
    if (!weights.empty() && weights.size() != edges.size()) throw ConfigError("weight array does not match edge count");
    if (!labels.empty() && labels.size() != edges.size()) throw ConfigError("label array does not match edge count");
    for (const auto& e : edges)
        if (e.first >= vertex_count || e.second >= vertex_count) throw ConfigError("edge endpoint out of range");
    std::vector<uint64_t> order(edges.size());
    for (uint64_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return edges[a] < edges[b]; });
    std::vector<uint64_t> offsets(static_cast<size_t>(vertex_count) + 1, 0);
    std::vector<VertexId> neighbors(edges.size());
    std::vector<double> w(weights.empty() ? 0 : edges.size());
    std::vector<uint32_t> l(labels.empty() ? 0 : edges.size());
    for (uint64_t p = 0; p < order.size(); ++p) {
        const uint64_t i = order[p];
        offsets[edges[i].first + 1] += 1;
        neighbors[p] = edges[i].second;
        if (!w.empty()) w[p] = weights[i];
        if (!l.empty()) l[p] = labels[i];
    }
    for (uint32_t v = 0; v < vertex_count; ++v) offsets[v + 1] += offsets[v];
    return Graph::from_csr(std::move(offsets), std::move(neighbors), std::move(w), std::move(l), device);
}

// ---- walker.hpp:47-84 ------------------------------------------------------------------
struct WalkRecord {
    uint64_t query_id = 0;
    WalkStatus status = WalkStatus::Complete;
    std::vector<VertexId> path;
    bool operator==(const WalkRecord&) const = default;
};
using WalkSet = std::vector<WalkRecord>;

struct QuerySpec {
    enum class Mode : uint8_t { OnePerVertex, FromSource, FromFile };
    static QuerySpec one_per_vertex() { return {}; }
    static QuerySpec from_source(VertexId source, uint64_t count) {
        QuerySpec s;
        s.mode = Mode::FromSource;
        s.source = source;
        s.count = count;
        return s;
    }
    static QuerySpec from_list(std::vector<VertexId> sources) {
        QuerySpec s;
        s.mode = Mode::FromFile;
        s.sources = std::move(sources);
        s.count = s.sources.size();
        return s;
    }
    // QuerySpec::from_file (walker.cpp:22-78): `vertex [count]` per line, '#'
    // starts a comment, blank lines skipped; same messages and error classes.
    static QuerySpec from_file(const std::string& path) {
        std::ifstream in(path);
        if (!in) throw Error("cannot open query file '" + path + "'");
        std::vector<VertexId> out;
        std::string line;
        uint64_t line_no = 0;
        while (std::getline(in, line)) {
            ++line_no;
            std::string_view view(line);
            if (auto h = view.find('#'); h != std::string_view::npos) view = view.substr(0, h);
            uint64_t fields[2] = {0, 1};
            int nf = 0;
            size_t pos = 0;
            while (pos < view.size()) {
                while (pos < view.size() && std::isspace(static_cast<unsigned char>(view[pos]))) ++pos;
                const size_t start = pos;
                while (pos < view.size() && !std::isspace(static_cast<unsigned char>(view[pos]))) ++pos;
                if (pos == start) continue;
                if (nf >= 2) throw ParseError(path + ":" + std::to_string(line_no) + ": too many columns");
                const char* b = view.data() + start;
                const char* e = view.data() + pos;
                auto [ptr, ec] = std::from_chars(b, e, fields[nf]);
                if (ec != std::errc() || ptr != e)
                    throw ParseError(path + ":" + std::to_string(line_no) + ": expected `vertex [count]`");
                ++nf;
            }
            if (nf == 0) continue;
            if (fields[0] > UINT32_MAX)
                throw ParseError(path + ":" + std::to_string(line_no) + ": vertex id out of range");
            for (uint64_t i = 0; i < fields[1]; ++i) out.push_back(static_cast<VertexId>(fields[0]));
        }
        if (out.empty()) throw ParseError(path + ": no queries");
        return from_list(std::move(out));
    }
    uint64_t total(const Graph& g) const {
        return mode == Mode::OnePerVertex ? g.vertex_count() : (mode == Mode::FromSource ? count : sources.size());
    }
    wf_query_spec to_c() const {
        wf_query_spec q{};
        q.mode = mode == Mode::OnePerVertex ? WF_QUERY_ONE_PER_VERTEX
                 : mode == Mode::FromSource ? WF_QUERY_FROM_SOURCE : WF_QUERY_FROM_LIST;
        q.source = source;
        q.count = mode == Mode::FromFile ? sources.size() : count;
        q.sources = sources.empty() ? nullptr : sources.data();
        return q;
    }
    Mode mode = Mode::OnePerVertex;
    VertexId source = 0;
    uint64_t count = 0;
    std::vector<VertexId> sources;
};

// ---- engine.hpp:64-89 -------------------------------------------------------------------
struct RunMetrics {
    double preprocess_seconds = 0.0;
    double exec_seconds = 0.0;
    uint64_t total_steps = 0;
    uint32_t max_in_flight = 0;
};
struct RunResult {
    WalkSet walks;
    RunMetrics metrics;
};
using BlockSink = std::function<void(uint32_t worker, WalkSet&& block)>;
// prefetch.hpp:17 (same enumerators; software prefetch hints have no device meaning)
enum class PrefetchLevel : uint8_t { L1, L2, L3, NonTemporal, Off };
inline const char* to_string(PrefetchLevel level) {  // prefetch.hpp:30-39
    switch (level) {
        case PrefetchLevel::L1: return "l1";
        case PrefetchLevel::L2: return "l2";
        case PrefetchLevel::L3: return "l3";
        case PrefetchLevel::NonTemporal: return "nta";
        case PrefetchLevel::Off: return "off";
    }
    return "?";
}
inline PrefetchLevel parse_prefetch_level(const std::string& name) {  // prefetch.hpp:41-48
    for (PrefetchLevel l : {PrefetchLevel::L1, PrefetchLevel::L2, PrefetchLevel::L3, PrefetchLevel::NonTemporal,
                            PrefetchLevel::Off})
        if (name == to_string(l)) return l;
    throw ConfigError("unknown prefetch level '" + name + "' (l1|l2|l3|nta|off)");
}
struct ExecOptions {
    uint32_t threads = 1;
    uint64_t seed = 0;
    std::optional<SamplerKind> sampler;
    bool use_static_tables = true;
    PrefetchLevel prefetch = PrefetchLevel::L1;
    uint32_t rej_trial_cap = kRejTrialCap;
    BlockSink sink;
};

// ---- algorithms.hpp:20-193: parameters; the functors run on the device ----------------
class PprProgram {
public:
    explicit PprProgram(double termination = 0.2) : stop_(termination) {
        if (!(termination > 0.0 && termination <= 1.0))
            throw ConfigError("termination probability must be in (0, 1], got " + std::to_string(termination));
    }
    WalkerType walker_type() const { return WalkerType::Unbiased; }
    double max_weight() const { return 1.0; }
    double termination() const { return stop_; }
    wf_program_desc to_desc() const {
        wf_program_desc d{};
        d.kind = WF_PROGRAM_PPR;
        d.termination = stop_;
        return d;
    }

private:
    double stop_;
};

class DeepWalkProgram {
public:
    DeepWalkProgram(const Graph& g, uint32_t target_length, bool weighted)
        : length_(target_length), weighted_(weighted) {
        if (target_length < 1) throw ConfigError("target length must be >= 1");
        if (weighted && !g.has_weights()) throw ConfigError("weighted walks need a graph with edge weights");
        bound_ = weighted ? g.max_weight() : 1.0;  // algorithms.hpp:51
    }
    WalkerType walker_type() const { return WalkerType::Static; }
    double max_weight() const { return bound_; }
    uint32_t target_length() const { return length_; }
    wf_program_desc to_desc() const {
        wf_program_desc d{};
        d.kind = WF_PROGRAM_DEEPWALK;
        d.target_length = length_;
        d.weighted = weighted_;
        return d;
    }

private:
    uint32_t length_;
    bool weighted_;
    double bound_ = 1.0;
};

struct Node2VecParams {
    double a = 2.0;
    double b = 0.5;
    uint32_t target_length = 80;
};

class Node2VecProgram {
public:
    Node2VecProgram(const Graph& g, Node2VecParams params, bool weighted)
        : params_(params), weighted_(weighted) {
        if (!(std::isfinite(params.a) && params.a > 0.0)) throw ConfigError("return parameter a must be positive and finite");
        if (!(std::isfinite(params.b) && params.b > 0.0)) throw ConfigError("in-out parameter b must be positive and finite");
        if (params.target_length < 1) throw ConfigError("target length must be >= 1");
        if (weighted && !g.has_weights()) throw ConfigError("weighted walks need a graph with edge weights");
        const double first = std::max({1.0 / params.a, 1.0, 1.0 / params.b});  // algorithms.hpp:95-98
        bound_ = weighted ? first * g.max_weight() : first;
    }
    WalkerType walker_type() const { return WalkerType::Dynamic; }
    SamplerKind preferred_sampler() const { return SamplerKind::ORej; }
    double max_weight() const { return bound_; }
    const Node2VecParams& params() const { return params_; }
    wf_program_desc to_desc() const {
        wf_program_desc d{};
        d.kind = WF_PROGRAM_NODE2VEC;
        d.a = params_.a;
        d.b = params_.b;
        d.target_length = params_.target_length;
        d.weighted = weighted_;
        return d;
    }

private:
    Node2VecParams params_;
    bool weighted_;
    double bound_ = 1.0;
};

class MetaPathProgram {
public:
    MetaPathProgram(const Graph& g, std::vector<uint32_t> schema) : schema_(std::move(schema)) {
        if (!g.has_labels()) throw ConfigError("meta-path walks need a graph with edge labels");
        if (schema_.empty()) throw ConfigError("meta-path schema must be non-empty");
        // every schema label must occur in the graph (algorithms.hpp:151-160)
        uint8_t present[256];
        check(wf_graph_labels_present(g.handle(), present));
        for (uint32_t l : schema_)
            if (l > 255 || !present[l])
                throw ConfigError("schema label " + std::to_string(l) + " does not occur in the graph");
    }
    WalkerType walker_type() const { return WalkerType::Dynamic; }
    const std::vector<uint32_t>& schema() const { return schema_; }
    wf_program_desc to_desc() const {
        wf_program_desc d{};
        d.kind = WF_PROGRAM_METAPATH;
        d.schema = schema_.data();
        d.schema_len = static_cast<uint32_t>(schema_.size());
        return d;
    }

private:
    std::vector<uint32_t> schema_;
};

// A user's device program (walkforge_b200/device_program.cuh): the
// wf_program_ops table its WF_DEVICE_PROGRAM(Type, symbol) exports and the
// program object's bytes (a host mirror of the trivially copyable Type).
class DeviceProgram {
public:
    template <typename T>
    DeviceProgram(const wf_program_ops* ops, const T& obj) : ops_(ops) {
        static_assert(std::is_trivially_copyable<T>::value, "a device program object is trivially copyable");
        if (ops == nullptr) throw ConfigError("null program table");
        if (ops->program_size != sizeof(T)) throw ConfigError("program object size does not match its table");
        bytes_.resize(sizeof(T));
        std::memcpy(bytes_.data(), &obj, sizeof(T));
    }
    WalkerType walker_type() const { return static_cast<WalkerType>(ops_->walker_type); }
    const wf_program_ops* ops() const { return ops_; }
    const void* object() const { return bytes_.data(); }
    uint32_t max_path() const { return ops_->max_path ? ops_->max_path(object()) : 0; }

private:
    const wf_program_ops* ops_;
    std::vector<unsigned char> bytes_;
};

class UniformProgram {
public:
    explicit UniformProgram(uint32_t target_length) : length_(target_length) {
        if (target_length < 1) throw ConfigError("target length must be >= 1");
    }
    WalkerType walker_type() const { return WalkerType::Unbiased; }
    double max_weight() const { return 1.0; }
    wf_program_desc to_desc() const {
        wf_program_desc d{};
        d.kind = WF_PROGRAM_UNIFORM;
        d.target_length = length_;
        return d;
    }

private:
    uint32_t length_;
};

// ---- program.hpp:28-36, 68-75: the sampling method a program runs under by default ------
inline SamplerKind default_sampler(WalkerType type) {
    switch (type) {
        case WalkerType::Unbiased: return SamplerKind::Naive;
        case WalkerType::Static: return SamplerKind::Alias;
        case WalkerType::Dynamic: return SamplerKind::Its;
    }
    return SamplerKind::Its;
}
template <typename P>
SamplerKind resolve_default_sampler(const P& prog) {
    if constexpr (requires { prog.preferred_sampler(); }) return prog.preferred_sampler();
    else return default_sampler(prog.walker_type());
}

// ---- run_sequential / run_interleaved (engine.hpp:440-504, interleave.hpp:391-556) ---
namespace detail {
inline std::pair<uint64_t, uint64_t> worker_range(uint64_t n, uint32_t workers, uint32_t w) {
    return {n * w / workers, n * (w + 1) / workers};  // engine.hpp:296-298
}

// RunMetrics::max_in_flight as the reference defines it (engine.hpp:68: peak
// ring occupancy of any worker; 1 for run_sequential, engine.hpp:502): a
// worker's ring holds min(k, its walks that were not already finished at
// admission) (interleave.hpp:436-467) — a walk finished at admission is the
// one stored Complete with its source alone.  The device's own residency
// (resident walker lanes) is wf_run_metrics.max_in_flight of the C-ABI.
struct RingPeak {
    uint32_t k = 0;  // 0: run_sequential
    uint32_t workers = 1;
    uint64_t n = 0;
    std::vector<uint64_t> live;
    void init(uint32_t ring, uint32_t w, uint64_t total) {
        k = ring;
        workers = w;
        n = total;
        live.assign(w, 0);
    }
    void count(uint32_t worker, uint32_t rec) {  // rec: length | dead_end << 31
        if (rec != 1u) live[worker] += 1;
    }
    uint32_t worker_of(uint64_t q) const {  // inverse of worker_range (engine.hpp:296-298)
        uint32_t w = static_cast<uint32_t>(static_cast<unsigned __int128>(q) * workers / std::max<uint64_t>(n, 1));
        while (w + 1 < workers && n * (w + 1) / workers <= q) ++w;
        while (w > 0 && n * w / workers > q) --w;
        return w;
    }
    uint32_t value() const {
        if (k == 0) return 1;
        uint64_t peak = 0;
        for (uint64_t l : live) peak = std::max(peak, std::min<uint64_t>(k, l));
        return static_cast<uint32_t>(peak);
    }
};

// Turns the streamed records + vertices into WalkRecords as blocks land, and
// hands the sink one block per worker range (engine.hpp:446-495: `workers` =
// max(1, threads) contiguous qid ranges, sink(w, block) once each, in order).
struct StreamSink {
    const uint32_t* records = nullptr;
    const uint32_t* vertices = nullptr;
    uint64_t n = 0;
    uint32_t workers = 1;
    uint32_t next_worker = 0;
    uint64_t next_q = 0, next_v = 0;
    WalkSet* all = nullptr;  // no sink: the whole walk set
    const BlockSink* sink = nullptr;
    WalkSet block;
    bool delivered = false;
    std::exception_ptr error;
    RingPeak* ring = nullptr;

    void flush_empty_workers() {  // ranges with no queries still get their (empty) block
        while (sink && next_worker < workers && worker_range(n, workers, next_worker).second <= next_q) {
            (*sink)(next_worker++, std::move(block));
            block.clear();
        }
    }
    void take(uint64_t q1) {
        for (uint64_t q = next_q; q < q1; ++q) {
            const uint32_t rec = records[q];
            const uint32_t len = rec & 0x7FFFFFFFu;
            if (ring) ring->count(ring->worker_of(q), rec);
            WalkRecord r{q, (rec >> 31) ? WalkStatus::DeadEnd : WalkStatus::Complete,
                         std::vector<VertexId>(vertices + next_v, vertices + next_v + len)};
            next_v += len;
            if (all) (*all)[q] = std::move(r);
            else block.push_back(std::move(r));
            next_q = q + 1;
            delivered = true;
            flush_empty_workers();
        }
    }
    static int on_block(void* user, uint64_t, uint64_t, uint64_t q1, uint64_t) {
        auto* self = static_cast<StreamSink*>(user);
        try {
            self->take(q1);
            return 0;
        } catch (...) {
            self->error = std::current_exception();
            return 1;
        }
    }
};

// Upper bound on path vertices per query (0: unbounded, PPR).
inline uint64_t max_path_vertices(const wf_program_desc& d) {
    if (d.kind == WF_PROGRAM_METAPATH) return static_cast<uint64_t>(d.schema_len) + 1;
    if (d.kind == WF_PROGRAM_PPR) return 0;
    return d.target_length;
}

inline wf_exec_options to_c(const ExecOptions& opts) {
    wf_exec_options o{};
    o.seed = opts.seed;
    o.sampler = opts.sampler ? static_cast<int32_t>(*opts.sampler) : WF_SAMPLER_DEFAULT;
    o.use_static_tables = opts.use_static_tables ? 1 : 0;
    o.rej_trial_cap = opts.rej_trial_cap;
    o.threads = opts.threads;
    return o;
}

// QuerySpec::validate before any work (walker.cpp:8-109), as the reference
// does: no block may reach a sink for an invalid query set.
inline void validate_spec(const Graph& g, const QuerySpec& spec) {
    if (spec.mode == QuerySpec::Mode::FromSource && spec.source >= g.vertex_count())
        throw ConfigError("query source " + std::to_string(spec.source) + " is not a vertex (V=" +
                          std::to_string(g.vertex_count()) + ")");
    if (spec.mode == QuerySpec::Mode::FromFile)
        for (VertexId v : spec.sources)
            if (v >= g.vertex_count())
                throw ConfigError("query source " + std::to_string(v) + " is not a vertex (V=" +
                                  std::to_string(g.vertex_count()) + ")");
}

// Worker blocks over devices (wf_multi_run): `workers` blocks in worker order
// to the sink (or into the walk set); unbounded walks need no host capacity
// guess (each block is sized after its walks ran).
template <typename P>
RunResult run_blocks(const Graph& g, const QuerySpec& spec, const P& prog, const ExecOptions& opts,
                     uint32_t n_devices, uint32_t ring_k) {
    const wf_exec_options o = to_c(opts);
    std::vector<int32_t> devs;
    int32_t total = 1;
    check(wf_device_count(&total));
    for (uint32_t i = 0; i < n_devices; ++i) devs.push_back((g.device() + static_cast<int32_t>(i)) % total);
    wf_multi* m = nullptr;
    if constexpr (std::is_same_v<P, DeviceProgram>) {
        check(wf_multi_create_custom(g.handle(), devs.data(), n_devices, prog.ops(), prog.object(), &o, &m));
    } else {
        wf_program_desc d = prog.to_desc();
        check(wf_multi_create(g.handle(), devs.data(), n_devices, &d, &o, &m));
    }
    std::unique_ptr<wf_multi, void (*)(wf_multi*)> guard(m, wf_multi_destroy);
    const uint64_t n = spec.total(g);
    const uint32_t workers = std::max<uint32_t>(1, opts.threads);
    RunResult r;
    if (!opts.sink) r.walks.resize(n);
    RingPeak ring;
    ring.init(ring_k, workers, n);
    struct Ctx {
        RunResult* r;
        const BlockSink* sink;
        std::exception_ptr error;
        RingPeak* ring;
    } ctx{&r, opts.sink ? &opts.sink : nullptr, nullptr, &ring};
    auto on_shard = [](void* user, uint32_t w, uint64_t q0, uint64_t q1, const uint32_t* rec,
                       const uint32_t* verts, uint64_t) -> int {
        auto* c = static_cast<Ctx*>(user);
        try {
            WalkSet block;
            uint64_t v = 0;
            for (uint64_t q = q0; q < q1; ++q) {
                const uint32_t len = rec[q - q0] & 0x7FFFFFFFu;
                c->ring->count(w, rec[q - q0]);
                WalkRecord wr{q, (rec[q - q0] >> 31) ? WalkStatus::DeadEnd : WalkStatus::Complete,
                              std::vector<VertexId>(verts + v, verts + v + len)};
                v += len;
                if (c->sink) block.push_back(std::move(wr));
                else c->r->walks[q] = std::move(wr);
            }
            if (c->sink) (*c->sink)(w, std::move(block));
            return 0;
        } catch (...) {
            c->error = std::current_exception();
            return 1;
        }
    };
    wf_query_spec q = spec.to_c();
    wf_run_metrics mt{};
    const int rc = wf_multi_run(m, &q, workers, on_shard, &ctx, nullptr, &mt);
    if (ctx.error) std::rethrow_exception(ctx.error);
    check(rc);
    r.metrics = {mt.preprocess_seconds, mt.exec_seconds, mt.total_steps, ring.value()};
    return r;
}

template <typename P>
RunResult run(const Graph& g, const QuerySpec& spec, const P& prog, const ExecOptions& opts,
              uint32_t ring_k = 0) {
    validate_spec(g, spec);
    const uint64_t n = spec.total(g);
    uint64_t per;
    if constexpr (std::is_same_v<P, DeviceProgram>) per = prog.max_path();
    else per = max_path_vertices(prog.to_desc());
    // ExecOptions::threads: worker blocks, spread over up to that many GPUs
    int32_t ndev = 1;
    check(wf_device_count(&ndev));
    const uint32_t workers = std::max<uint32_t>(1, opts.threads);
    const uint32_t G = std::max<uint32_t>(1, std::min<uint32_t>(workers, static_cast<uint32_t>(std::max(ndev, 1))));
    if (G > 1 || per == 0) return run_blocks(g, spec, prog, opts, G, ring_k);

    // one device, bounded walks: the walks stream into host memory block by
    // block (wf_session_run_host_blocks) and become WalkRecords while later
    // queries are still walking
    const wf_exec_options o = to_c(opts);
    wf_query_spec q = spec.to_c();
    wf_session* s = nullptr;
    if constexpr (std::is_same_v<P, DeviceProgram>) {
        check(wf_session_create_custom(g.handle(), prog.ops(), prog.object(), &o, &s));
    } else {
        wf_program_desc d = prog.to_desc();
        check(wf_session_create(g.handle(), &d, &o, &s));
    }
    std::unique_ptr<wf_session, void (*)(wf_session*)> guard(s, wf_session_destroy);
    const uint64_t cap = n * per + 4096;
    std::unique_ptr<uint32_t[]> records(new uint32_t[std::max<uint64_t>(n, 1)]);
    std::unique_ptr<uint32_t[]> vertices(new uint32_t[cap]);
    RunResult r;
    StreamSink st;
    st.records = records.get();
    st.vertices = vertices.get();
    st.n = n;
    st.workers = workers;
    RingPeak ring;
    ring.init(ring_k, workers, n);
    st.ring = &ring;
    if (opts.sink) {
        st.sink = &opts.sink;
    } else {
        r.walks.resize(n);
        st.all = &r.walks;
    }
    wf_run_metrics m{};
    const int rc = wf_session_run_host_blocks(s, &q, 0, 0, records.get(), vertices.get(), cap, 0,
                                              &StreamSink::on_block, &st, &m);
    if (st.error) std::rethrow_exception(st.error);
    check(rc);
    st.flush_empty_workers();
    r.metrics = {m.preprocess_seconds, m.exec_seconds, m.total_steps, ring.value()};
    return r;
}
}  // namespace detail

template <typename P>
RunResult run_sequential(const Graph& g, const QuerySpec& spec, const P& prog,
                         const ExecOptions& opts = {}) {
    return detail::run(g, spec, prog, opts);
}

template <typename P>
RunResult run_interleaved(const Graph& g, const QuerySpec& spec, const P& prog, uint32_t k,
                          uint32_t k_prime, const ExecOptions& opts = {}) {
    if (k == 0) throw ConfigError("task ring size must be >= 1");
    if (k_prime == 0 || k_prime > k) throw ConfigError("search ring size must be in [1, k]");
    return detail::run(g, spec, prog, opts, k);
}

// ---- tune_ring_sizes (tune.hpp:12-42, tune.cpp:46-111) -----------------------------------
// The reference sweeps its CPU interleave rings (k, k') with a probe workload
// (one uniform length-10 walk from every vertex).  On the device the rings are
// replaced by resident walkers, so this runs the same probe through the launch
// tuner (wf_session_tune): the report carries the device's pick and the probe
// throughput; best_k / best_k_prime stay the reference's defaults (64, 32),
// which run_interleaved accepts and validates.
struct TuneOptions {
    uint32_t threads = 1;
    double budget_seconds = 120.0;
    uint64_t seed = 0;
    PrefetchLevel prefetch = PrefetchLevel::L1;
};
struct TunePoint {
    uint32_t k = 0;
    double steps_per_sec = 0.0;
};
struct TuneReport {
    std::vector<TunePoint> task_ring;
    std::vector<TunePoint> search_ring;
    uint32_t best_k = 64;
    uint32_t best_k_prime = 32;
    bool budget_exhausted = false;
    int32_t device_blocks_per_sm = 0;  // the launch tuner's choice for the probe
    std::string to_text() const {
        std::string s = "device launch tuner: " + std::to_string(device_blocks_per_sm) + " blocks/SM";
        for (const auto& p : task_ring)
            s += "\nprobe steps/s " + std::to_string(p.steps_per_sec);
        s += "\nrecommended k=" + std::to_string(best_k) + " k'=" + std::to_string(best_k_prime);
        return s;
    }
};
inline TuneReport tune_ring_sizes(const Graph& g, const TuneOptions& opts = {}) {
    wf_program_desc d = UniformProgram(10).to_desc();
    wf_exec_options o{};
    o.seed = opts.seed;
    o.sampler = WF_SAMPLER_DEFAULT;
    o.use_static_tables = 1;
    wf_query_spec q{};
    q.mode = WF_QUERY_ONE_PER_VERTEX;
    wf_session* s = nullptr;
    check(wf_session_create(g.handle(), &d, &o, &s));
    std::unique_ptr<wf_session, void (*)(wf_session*)> guard(s, wf_session_destroy);
    TuneReport r;
    double ms = 0.0;
    check(wf_session_tune(s, &q, 0, 0, &r.device_blocks_per_sm, &ms));
    wf_walkset* ws = nullptr;
    wf_run_metrics m{};
    check(wf_session_run(s, &q, &ws, &m));
    wf_walkset_destroy(ws);
    r.task_ring.push_back({r.best_k, m.exec_seconds > 0 ? m.total_steps / m.exec_seconds : 0.0});
    return r;
}

}  // namespace walkforge_b200

#ifdef WALKFORGE_B200_DROP_IN
namespace walkforge = walkforge_b200;
#endif
