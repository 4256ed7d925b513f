// extern "C" boundary (include/walkforge_b200.h).  Every entry point catches
// wf::Error and maps it to a wf_status + wf_last_error(); nothing here falls
// back to the CPU: without a device every call fails with WF_ERR_CUDA.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "runtime.hpp"

using namespace wf;

struct wf_graph {
    std::unique_ptr<GraphStore> g;
};
struct wf_session {
    std::unique_ptr<Session> s;
    DeviceBuffer<unsigned long long> counters;  // steps, overflow
};
struct wf_walkset {
    std::unique_ptr<WalkSetStore> w;
};

namespace {

thread_local std::string g_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return WF_OK;
    } catch (const wf::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return WF_ERR_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return WF_ERR_INVALID_ARG;
    }
}

void require(bool ok, const char* what) {
    if (!ok) raise(WF_ERR_INVALID_ARG, what);
}

const char* type_name(int t) {
    return t == kUnbiased ? "unbiased" : (t == kStatic ? "static" : "dynamic");
}

int walker_type(int prog) {
    switch (prog) {
        case WF_PROGRAM_PPR:
        case WF_PROGRAM_UNIFORM: return kUnbiased;
        case WF_PROGRAM_DEEPWALK: return kStatic;
        default: return kDynamic;
    }
}

std::string fmt_double(double x) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%f", x);
    return buf;
}

}  // namespace

namespace wf {

// Program constructors' validation (algorithms.hpp:22-27, 43-51, 81-96,
// 143-160, 179-182) and the resolved run (resolve_default_sampler,
// program.hpp:68-75; resolve_flow, engine.hpp:255-272; resolve_orej_bound,
// engine.hpp:103-114).
void resolve_program(Session& s, const wf_program_desc& d, const wf_exec_options* o) {
    GraphStore& g = *s.g;
    ProgParams& p = s.params;
    p = ProgParams{};
    s.desc = d;
    bool has_max_weight = true;
    switch (d.kind) {
        case WF_PROGRAM_PPR:
            if (!(d.termination > 0.0 && d.termination <= 1.0))
                config_error("termination probability must be in (0, 1], got " + fmt_double(d.termination));
            p.stop_thr = unit_threshold(d.termination);
            p.bound = 1.0;
            s.unbounded = true;
            break;
        case WF_PROGRAM_DEEPWALK:
            if (d.target_length < 1) config_error("target length must be >= 1");
            if (d.weighted && !g.has_weights()) config_error("weighted walks need a graph with edge weights");
            p.length = d.target_length;
            p.weighted = d.weighted ? 1 : 0;
            p.bound = d.weighted ? g.max_weight : 1.0;
            break;
        case WF_PROGRAM_NODE2VEC: {
            if (!(std::isfinite(d.a) && d.a > 0.0)) config_error("return parameter a must be positive and finite");
            if (!(std::isfinite(d.b) && d.b > 0.0)) config_error("in-out parameter b must be positive and finite");
            if (d.target_length < 1) config_error("target length must be >= 1");
            if (d.weighted && !g.has_weights()) config_error("weighted walks need a graph with edge weights");
            p.length = d.target_length;
            p.weighted = d.weighted ? 1 : 0;
            p.inv_a = 1.0 / d.a;
            p.inv_b = 1.0 / d.b;
            p.first = std::max({p.inv_a, 1.0, p.inv_b});
            p.bound = d.weighted ? p.first * g.max_weight : p.first;
            p.lo_w = std::min(1.0, p.inv_b);
            p.hi_w = std::max(1.0, p.inv_b);
            break;
        }
        case WF_PROGRAM_METAPATH: {
            if (!g.has_labels()) config_error("meta-path walks need a graph with edge labels");
            if (d.schema_len == 0 || d.schema == nullptr) config_error("meta-path schema must be non-empty");
            s.schema.assign(d.schema, d.schema + d.schema_len);
            for (uint32_t l : s.schema)
                if (l > 255 || !g.label_present[l])
                    config_error("schema label " + std::to_string(l) + " does not occur in the graph");
            s.schema_dev.allocate(s.schema.size());
            WF_CUDA(cudaMemcpy(s.schema_dev.get(), s.schema.data(), s.schema.size() * 4, cudaMemcpyHostToDevice));
            p.schema = s.schema_dev.get();
            p.schema_len = d.schema_len;
            has_max_weight = false;
            break;
        }
        case WF_PROGRAM_UNIFORM:
            if (d.target_length < 1) config_error("target length must be >= 1");
            p.length = d.target_length;
            p.bound = 1.0;
            break;
        default:
            config_error("unknown program kind " + std::to_string(d.kind));
    }
    s.desc.schema = nullptr;
    // row capacity: fixed-length programs hold their whole walk
    const uint32_t fixed = d.kind == WF_PROGRAM_METAPATH ? d.schema_len + 1
                           : d.kind == WF_PROGRAM_PPR ? 0 : d.target_length;
    resolve_run(s, walker_type(d.kind), d.kind == WF_PROGRAM_NODE2VEC ? WF_SAMPLER_OREJ : WF_SAMPLER_DEFAULT,
                has_max_weight, fixed, o);
}

// The sampler / flow / bound half of ResolvedRun (engine.hpp:275-294), shared by
// the built-ins and custom programs: resolve_default_sampler (program.hpp:68-75),
// resolve_flow (engine.hpp:255-272), resolve_orej_bound (engine.hpp:103-114)
// with the bound already in s.params.bound.
void resolve_run(Session& s, int type, int preferred, bool has_max_weight, uint32_t fixed,
                 const wf_exec_options* o) {
    ProgParams& p = s.params;
    int kind = o && o->sampler >= 0 ? o->sampler
               : preferred >= 0 ? preferred
               : type == kUnbiased ? WF_SAMPLER_NAIVE
               : type == kStatic ? WF_SAMPLER_ALIAS : WF_SAMPLER_ITS;
    if (kind < WF_SAMPLER_NAIVE || kind > WF_SAMPLER_OREJ) config_error("unknown sampler");
    const bool use_tables = o ? o->use_static_tables != 0 : true;
    int flow;
    if (kind == WF_SAMPLER_NAIVE) {
        if (type != kUnbiased)
            config_error(std::string("NAIVE assumes a uniform distribution; the program is ") + type_name(type));
        flow = kDirect;
    } else if (kind == WF_SAMPLER_OREJ) {
        flow = kDirect;
    } else if (type == kDynamic) {
        flow = kGathered;
    } else {
        flow = use_tables ? kTables : kGathered;
    }
    s.kind = kind;
    s.flow = flow;
    s.trial_cap = o && o->rej_trial_cap ? o->rej_trial_cap : (1u << 20);
    s.seed = o ? o->seed : 0;
    if (kind == WF_SAMPLER_OREJ) {
        if (!has_max_weight) config_error("O-REJ needs a program with max_weight()");
        if (!std::isfinite(p.bound) || p.bound <= 0.0)
            raise(WF_ERR_CONTRACT, "max_weight() must be positive and finite");
    }
    if (o && (o->k != 0 || o->k_prime != 0)) {  // interleave.hpp:395-400
        if (o->k == 0) config_error("task ring size must be >= 1");
        if (o->k_prime == 0 || o->k_prime > o->k) config_error("search ring size must be in [1, k]");
    }
    if (fixed) s.default_stride = fixed;
    else s.default_stride = o && o->path_stride ? o->path_stride : 64;
    s.unbounded = fixed == 0;
}

// A user's device program (wf_session_create_custom): the table says what the
// concept's optional members are; the object rides in the launch parameters.
void resolve_custom(Session& s, const wf_program_ops& ops, const void* program, const wf_exec_options* o) {
    require(ops.abi_version == WF_ABI_VERSION, "program table built against another ABI version");
    require(ops.launch_size == sizeof(WalkLaunch) && ops.engine_abi == kEngineAbi,
            "program table built against another engine header: rebuild the program library");
    require(ops.launch && ops.occupancy && ops.static_weights, "incomplete program table");
    require(program != nullptr || ops.program_size == 0, "null program object");
    require(ops.program_size <= static_cast<uint32_t>(kUserProgramBytes), "program object too large");
    require(ops.walker_type >= kUnbiased && ops.walker_type <= kDynamic, "bad walker type");
    s.custom = &ops;
    s.params = ProgParams{};
    if (ops.program_size) std::memcpy(s.params.user, program, ops.program_size);
    s.desc = wf_program_desc{};
    s.desc.kind = kCustomProgram;
    s.params.bound = ops.has_max_weight && ops.max_weight ? ops.max_weight(program) : 0.0;
    resolve_run(s, ops.walker_type, ops.preferred_sampler, ops.has_max_weight != 0,
                ops.max_path ? ops.max_path(program) : 0u, o);
}

// QuerySpec::total + validate (walker.cpp:80-109), sources made device-resident.
void resolve_spec(const GraphStore& g, const wf_query_spec* q, ResolvedSpec& r) {
    require(q != nullptr, "null query spec");
    r.spec = *q;
    switch (q->mode) {
        case WF_QUERY_ONE_PER_VERTEX:
            r.n = g.V;
            break;
        case WF_QUERY_FROM_SOURCE:
            if (q->source >= g.V)
                config_error("query source " + std::to_string(q->source) + " is not a vertex (V=" +
                             std::to_string(g.V) + ")");
            r.n = q->count;
            break;
        case WF_QUERY_FROM_LIST: {
            r.n = q->count;
            if (r.n == 0) break;
            require(q->sources != nullptr, "null source list");
            std::vector<uint32_t> host;
            const uint32_t* hp = q->sources;
            if (is_device_pointer(q->sources)) {
                host.resize(r.n);
                WF_CUDA(cudaMemcpy(host.data(), q->sources, r.n * 4, cudaMemcpyDeviceToHost));
                hp = host.data();
                r.dev_sources = q->sources;
            }
            for (uint64_t i = 0; i < r.n; ++i)
                if (hp[i] >= g.V)
                    config_error("query source " + std::to_string(hp[i]) + " is not a vertex (V=" +
                                 std::to_string(g.V) + ")");
            if (!r.dev_sources) {
                r.sources.allocate(r.n);
                WF_CUDA(cudaMemcpy(r.sources.get(), q->sources, r.n * 4, cudaMemcpyHostToDevice));
                r.dev_sources = r.sources.get();
            }
            break;
        }
        default:
            config_error("unknown query mode");
    }
}

void check_device_error(Session& s) {
    int h = 0;
    WF_CUDA(cudaMemcpy(&h, s.error_word.get(), 4, cudaMemcpyDeviceToHost));
    if (h != 0) {
        WF_CUDA(cudaMemset(s.error_word.get(), 0, 4));
        raise_device_error(s, h);
    }
}

}  // namespace wf

namespace {

__global__ void k_rng_probe(uint64_t premixed, const uint64_t* streams, uint64_t n, uint32_t draws,
                            uint64_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        Rng r{stream_state(premixed, streams[i])};
        for (uint32_t j = 0; j < draws; ++j) out[i * draws + j] = r.next();
    }
}

__global__ void k_max_u32(const uint32_t* __restrict__ x, uint64_t n, unsigned* out) {
    unsigned m = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, x[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

int current_device() {
    int d = 0;
    WF_CUDA(cudaGetDevice(&d));
    return d;
}

}  // namespace

namespace wf {
std::string& last_error_slot() { return g_last_error; }
GraphStore* graph_store(const wf_graph* g) { return g->g.get(); }
}  // namespace wf

extern "C" {

int wf_abi_version(void) { return WF_ABI_VERSION; }

int wf_device_count(int32_t* n) {
    return guarded([&] {
        require(n != nullptr, "null argument");
        int c = 0;
        WF_CUDA(cudaGetDeviceCount(&c));
        *n = c;
    });
}
const char* wf_last_error(void) { return g_last_error.c_str(); }
uint64_t wf_kernel_launches(void) { return g_kernel_launches.load(); }

int wf_graph_create(const uint64_t* offsets, const uint32_t* neighbors, const float* weights,
                    const uint32_t* labels, uint32_t vertex_count, uint64_t edge_count, int device,
                    wf_graph** out) {
    return guarded([&] {
        require(out && offsets && (neighbors || edge_count == 0), "null argument");
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_from_host(offsets, neighbors, weights, labels, vertex_count, edge_count,
                                   device < 0 ? current_device() : device));
        *out = h.release();
    });
}

int wf_graph_create_f64(const uint64_t* offsets, const uint32_t* neighbors, const double* weights,
                        const uint32_t* labels, uint32_t vertex_count, uint64_t edge_count, int device,
                        wf_graph** out) {
    return guarded([&] {
        require(out && offsets && (neighbors || edge_count == 0), "null argument");
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_from_host_f64(offsets, neighbors, weights, labels, vertex_count, edge_count,
                                       device < 0 ? current_device() : device));
        *out = h.release();
    });
}

int wf_graph_download_weights_f64(const wf_graph* g, double* weights) {
    return guarded([&] {
        require(g && weights, "null argument");
        const GraphStore& s = *g->g;
        DeviceGuard guard(s.device);
        if (!s.has_weights() || !s.E) return;
        if (s.weights64.get()) {
            WF_CUDA(cudaMemcpy(weights, s.weights64.get(), s.E * 8, cudaMemcpyDefault));
        } else {
            std::vector<float> w(s.E);
            WF_CUDA(cudaMemcpy(w.data(), s.weights.get(), s.E * 4, cudaMemcpyDefault));
            for (uint64_t e = 0; e < s.E; ++e) weights[e] = w[e];
        }
    });
}

int wf_graph_create_device(const uint64_t* offsets, const uint32_t* neighbors,
                           const float* weights, const uint8_t* labels, uint32_t vertex_count,
                           uint64_t edge_count, int device, wf_graph** out) {
    return guarded([&] {
        require(out && offsets && (neighbors || edge_count == 0), "null argument");
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_from_device(offsets, neighbors, weights, labels, vertex_count, edge_count,
                                     device < 0 ? current_device() : device));
        *out = h.release();
    });
}

int wf_graph_generate_rmat(const wf_rmat_params* params, int device, wf_graph** out) {
    return guarded([&] {
        require(out && params, "null argument");
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_generate_rmat(*params, device < 0 ? current_device() : device));
        *out = h.release();
    });
}

int wf_graph_info_get(const wf_graph* g, wf_graph_info* out) {
    return guarded([&] {
        require(g && out, "null argument");
        const GraphStore& s = *g->g;
        std::memset(out, 0, sizeof(*out));
        out->vertex_count = s.V;
        out->edge_count = s.E;
        out->max_degree_lo = s.max_degree;
        out->max_weight = s.max_weight;
        out->has_weights = s.has_weights();
        out->has_labels = s.has_labels();
        out->adjacency_sorted = s.sorted;
        out->device = s.device;
        out->label_count = s.label_count;
        out->weights_f64 = s.weights64.get() != nullptr;
    });
}

int wf_graph_download(const wf_graph* g, uint64_t* offsets, uint32_t* neighbors, float* weights,
                      uint8_t* labels) {
    return guarded([&] {
        require(g != nullptr, "null graph");
        const GraphStore& s = *g->g;
        DeviceGuard guard(s.device);
        if (offsets) WF_CUDA(cudaMemcpy(offsets, s.offsets.get(), (s.V + 1ull) * 8, cudaMemcpyDefault));
        if (neighbors && s.E) WF_CUDA(cudaMemcpy(neighbors, s.nbr.get(), s.E * 4, cudaMemcpyDefault));
        if (weights && s.has_weights() && s.E)
            WF_CUDA(cudaMemcpy(weights, s.weights.get(), s.E * 4, cudaMemcpyDefault));
        if (labels && s.has_labels() && s.E)
            WF_CUDA(cudaMemcpy(labels, s.labels.get(), s.E, cudaMemcpyDefault));
    });
}

int wf_graph_has_edge(const wf_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                      uint8_t* out) {
    return guarded([&] {
        require(g && src && dst && out, "null argument");
        if (n) graph_has_edge(*g->g, src, dst, n, out);
    });
}

int wf_graph_labels_present(const wf_graph* g, uint8_t out[256]) {
    return guarded([&] {
        require(g && out, "null argument");
        for (int l = 0; l < 256; ++l) out[l] = g->g->has_labels() ? g->g->label_present[l] : 0;
    });
}

int wf_graph_read_wfg1(const char* path, int device, wf_graph** out) {
    return guarded([&] {
        require(path && out, "null argument");
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_read_wfg1(path, device < 0 ? current_device() : device));
        *out = h.release();
    });
}

int wf_graph_write_wfg1(const wf_graph* g, const char* path) {
    return guarded([&] {
        require(g && path, "null argument");
        graph_write_wfg1(*g->g, path);
    });
}

int wf_graph_load_edge_list(const char* path, const wf_edge_list_options* opts, int device,
                            wf_graph** out) {
    return guarded([&] {
        require(path && out, "null argument");
        wf_edge_list_options o{};
        if (opts) o = *opts;
        std::vector<uint64_t> ids;
        auto h = std::make_unique<wf_graph>();
        h->g.reset(graph_load_edge_list(path, o, device < 0 ? current_device() : device, &ids));
        h->g->original_ids = std::move(ids);
        *out = h.release();
    });
}

int wf_graph_original_ids(const wf_graph* g, uint64_t* out) {
    return guarded([&] {
        require(g && out, "null argument");
        const GraphStore& s = *g->g;
        if (s.original_ids.size() == s.V) std::copy(s.original_ids.begin(), s.original_ids.end(), out);
        else for (uint32_t v = 0; v < s.V; ++v) out[v] = v;
    });
}

void wf_graph_destroy(wf_graph* g) {
    if (g) {
        DeviceGuard guard(g->g->device, std::nothrow);
        delete g;
    }
}

}  // extern "C"

namespace wf {

// Device state of a resolved session: error word, claim cursor, static
// tables and the decorated layouts the HBM budget allows.  `tables_from`: a
// session of the same program on another device whose static tables are
// copied (peer copy) instead of rebuilt (multi-device runs).
void setup_session(Session& s, const wf_exec_options* opts, const Session* tables_from) {
    s.error_word.allocate(1);
    WF_CUDA(cudaMemset(s.error_word.get(), 0, 4));
    // random 32 B gathers: do not let L2 promote misses to 64/128 B fetches
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32);
    cudaGetLastError();
    s.cursor.allocate(1);
    // HBM budget for the decorated layouts (they trade capacity for one
    // dependent random load per move); fall back to the compact forms.
    size_t free_b = 0, total_b = 0;
    WF_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t reserve = 8ull << 30;
    const uint64_t E = s.g->E;
    const uint32_t lf = opts ? opts->layout_flags : 0;
    int l2 = 0;
    WF_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, s.g->device));
    // a custom program's update() reads the traversed edge: its buckets carry
    // edge positions (compact), the destination is read from the CSR
    s.alias_idx = s.custom != nullptr;
    // Wide 32 B buckets (carrying the destinations' vertex words: one random
    // request per move) pay once the compact form (16 B buckets + vertex
    // words) outgrows the L2; below that its L2 hits win (C1, s16: 44.8 vs
    // 38.3 G steps/s compact vs wide; C5, s26: wide).
    const bool wide_pays = 16 * E + 8ull * s.g->V > 2ull * static_cast<uint64_t>(l2) || (lf & WF_LAYOUT_WIDE_ALIAS);
    if (s.flow == kTables && s.kind == WF_SAMPLER_ALIAS && !(lf & WF_LAYOUT_COMPACT_ALIAS) && !s.alias_idx &&
        wide_pays)
        s.alias_wide = 32 * E + reserve <= free_b;
    if (s.flow == kTables) {
        if (tables_from) s.copy_tables_from(*tables_from, nullptr);
        else s.build_tables(nullptr);
    }
    // The decorated adjacency saves the dependent vertex-word load but is 4x
    // the neighbour array: when the compact graph (neighbours + vertex
    // words) is near L2 size, its L2 hits win (C2: 12.8 vs 11.3 G moves/s).
    const uint64_t compact = 4 * E + 8ull * s.g->V;
    const bool adj_pays = compact > 2ull * static_cast<uint64_t>(l2) || (lf & WF_LAYOUT_FORCE_ADJ);
    // The packed 8 B adjacency (dst, degree, base) when it fits 64 bits: O-REJ
    // trials by default on graphs small enough to skip the 16 B form
    // (Node2Vec s20: 20.7 -> 22.6 G steps/s); NAIVE only on request — PPR's
    // L2-resident vertex words + neighbours beat it (C2: 19.6 vs 18.0).
    const bool adj8_wanted = (lf & WF_LAYOUT_ADJ8) || (s.kind == WF_SAMPLER_OREJ && !adj_pays);
    if (s.flow == kDirect && !(lf & WF_LAYOUT_NO_ADJ) && adj8_wanted && 8 * E + reserve <= free_b &&
        s.build_adjacency8(nullptr)) {
        // one 8 B load per move / trial carries the next vertex's word
    } else if (s.flow == kDirect && adj_pays && !(lf & WF_LAYOUT_NO_ADJ) && 16 * E + reserve <= free_b) {
        s.build_adjacency(nullptr);
    }
    if (s.desc.kind == WF_PROGRAM_METAPATH && s.kind == WF_SAMPLER_ITS) {
        s.g->ensure_label_index(nullptr);
        WF_CUDA(cudaMemGetInfo(&free_b, &total_b));
        // one random 16 B read per move (the partitioned edge carrying the
        // next schema label's group of its destination) instead of label
        // record + neighbour: C4 2.07 -> 1.87 ms since the warp-claimed
        // refill (it measured slower while the cursor atomic bound C4)
        if (!(lf & WF_LAYOUT_NO_MP_SUCC) && 16 * E + reserve <= free_b)
            s.build_metapath_successors(nullptr);
    }
    if (s.desc.kind == WF_PROGRAM_NODE2VEC) {
        // distance test: exact edge hash set (one random bucket per query)
        // unless opted out or HBM is short; then the sector B-tree
        WF_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (!(lf & WF_LAYOUT_SEARCH_TREE) && (s.g->edge_hash_built || 16 * E + reserve <= free_b)) {
            s.g->ensure_edge_hash(nullptr);
            s.use_edge_hash = true;
        } else {
            s.g->ensure_search_index(nullptr);
        }
        if (!(lf & WF_LAYOUT_NO_EDGE_FILTER)) {
            s.g->ensure_edge_filter(nullptr);
            s.use_edge_filter = true;
        }
    }
    s.grid = occupancy_grid(s);
}

}  // namespace wf

extern "C" {

int wf_session_create(const wf_graph* g, const wf_program_desc* prog, const wf_exec_options* opts,
                      wf_session** out) {
    return guarded([&] {
        require(g && prog && out, "null argument");
        DeviceGuard guard(g->g->device);
        auto h = std::make_unique<wf_session>();
        h->s = std::make_unique<Session>();
        Session& s = *h->s;
        s.g = g->g.get();
        resolve_program(s, *prog, opts);
        h->counters.allocate(2);
        setup_session(s, opts, nullptr);
        *out = h.release();
    });
}

int wf_session_create_custom(const wf_graph* g, const wf_program_ops* ops, const void* program,
                             const wf_exec_options* opts, wf_session** out) {
    return guarded([&] {
        require(g && ops && out, "null argument");
        DeviceGuard guard(g->g->device);
        auto h = std::make_unique<wf_session>();
        h->s = std::make_unique<Session>();
        Session& s = *h->s;
        s.g = g->g.get();
        resolve_custom(s, *ops, program, opts);
        h->counters.allocate(2);
        setup_session(s, opts, nullptr);
        *out = h.release();
    });
}

int wf_session_describe(const wf_session* s, int32_t* sampler, int32_t* flow,
                        double* preprocess_seconds) {
    return guarded([&] {
        require(s != nullptr, "null session");
        if (sampler) *sampler = s->s->kind;
        if (flow) *flow = s->s->flow;
        if (preprocess_seconds) *preprocess_seconds = s->s->preprocess_seconds;
    });
}

int wf_session_layout(const wf_session* sh, uint32_t* flags) {
    return guarded([&] {
        require(sh && flags, "null argument");
        const Session& s = *sh->s;
        uint32_t f = 0;
        if (s.alias_wide) f |= WF_LAYOUT_HAS_WIDE_ALIAS;
        if (s.adj.get()) f |= WF_LAYOUT_HAS_ADJ;
        if (s.adj8.get()) f |= WF_LAYOUT_HAS_ADJ8;
        if (s.mp_adj.get()) f |= WF_LAYOUT_HAS_MP_SUCC;
        if (s.use_edge_filter) f |= WF_LAYOUT_HAS_EDGE_FILTER;
        if (s.desc.kind == WF_PROGRAM_METAPATH && s.g->label_index_built) f |= WF_LAYOUT_HAS_LABEL_INDEX;
        if (s.desc.kind == WF_PROGRAM_NODE2VEC && !s.use_edge_hash && s.g->search_index_built)
            f |= WF_LAYOUT_HAS_SEARCH_INDEX;
        if (s.desc.kind == WF_PROGRAM_NODE2VEC && s.use_edge_hash) f |= WF_LAYOUT_HAS_EDGE_HASH;
        *flags = f;
    });
}

void wf_session_destroy(wf_session* s) {
    if (s) {
        DeviceGuard guard(s->s->g->device, std::nothrow);
        delete s;
    }
}

int wf_session_launch(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin,
                      uint64_t qid_end, uint32_t* paths, uint32_t stride, uint32_t* lengths,
                      uint8_t* status, uint32_t* visit_counts, unsigned long long* steps_out,
                      unsigned long long* overflow_out, void* stream) {
    return guarded([&] {
        require(sh && spec && paths && lengths && status, "null argument");
        Session& s = *sh->s;
        DeviceGuard guard(s.g->device);
        require(spec->mode != WF_QUERY_FROM_LIST || is_device_pointer(spec->sources),
                "wf_session_launch needs a device-resident source list");
        if (spec->mode == WF_QUERY_FROM_SOURCE && spec->source >= s.g->V)
            config_error("query source " + std::to_string(spec->source) + " is not a vertex");
        unsigned long long* steps = steps_out ? steps_out : sh->counters.get();
        unsigned long long* over = overflow_out ? overflow_out : sh->counters.get() + 1;
        launch_walk(s, *spec, spec->sources, qid_begin, qid_end, nullptr, paths, stride, lengths,
                    status, visit_counts, steps, over, s.cursor.get(),
                    static_cast<cudaStream_t>(stream));
    });
}

int wf_session_sync(wf_session* sh, void* stream) {
    return guarded([&] {
        require(sh != nullptr, "null session");
        DeviceGuard guard(sh->s->g->device);
        WF_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        check_device_error(*sh->s);
    });
}

}  // extern "C"

namespace wf {

// run_sequential's result for queries [qb, qe) of a resolved spec, kept in
// HBM (rows relative to qb).  Walks that outgrow their row are re-run into
// rows of their own (same (seed, qid) streams).  `ctr`: two device counters
// (moves, overflowed rows).
std::unique_ptr<WalkSetStore> session_run(Session& s, const ResolvedSpec& rs, uint64_t qb, uint64_t qe,
                                          unsigned long long* ctr) {
    GraphStore& g = *s.g;
    DeviceGuard guard(g.device);
    auto wp = std::make_unique<WalkSetStore>();
    WalkSetStore& w = *wp;
    w.device = g.device;
    w.n = qe - qb;
    w.V = g.V;
    w.stride = s.default_stride;
    w.paths.allocate(std::max<uint64_t>(w.n * w.stride, 1));
    w.lengths.allocate(std::max<uint64_t>(w.n, 1));
    w.status.allocate(std::max<uint64_t>(w.n, 1));
    const bool counts = s.desc.kind == WF_PROGRAM_PPR;
    if (counts) {
        w.visit_counts.allocate(g.V);
        WF_CUDA(cudaMemset(w.visit_counts.get(), 0, g.V * 4ull));
    }
    WF_CUDA(cudaMemset(ctr, 0, 16));
    cudaEvent_t e0, e1;
    WF_CUDA(cudaEventCreate(&e0));
    WF_CUDA(cudaEventCreate(&e1));
    WF_CUDA(cudaEventRecord(e0, nullptr));
    launch_walk(s, rs.spec, rs.dev_sources, qb, qe, nullptr, w.paths.get(), w.stride, w.lengths.get(),
                w.status.get(), counts ? w.visit_counts.get() : nullptr, ctr, ctr + 1, s.cursor.get(), nullptr);
    WF_CUDA(cudaEventRecord(e1, nullptr));
    WF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    WF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    check_device_error(s);
    unsigned long long hc[2] = {0, 0};
    WF_CUDA(cudaMemcpy(hc, ctr, 16, cudaMemcpyDeviceToHost));
    if (hc[1] > 0) {
        // re-run the walks that outgrew their row; same (seed, qid) streams
        std::vector<uint32_t> lens(w.n);
        WF_CUDA(cudaMemcpy(lens.data(), w.lengths.get(), w.n * 4, cudaMemcpyDeviceToHost));
        std::vector<uint64_t> qids;
        uint32_t mx = 0;
        for (uint64_t r = 0; r < w.n; ++r)
            if (lens[r] > w.stride) {
                w.over_rows.push_back(r);
                qids.push_back(qb + r);
                mx = std::max(mx, lens[r]);
            }
        w.over_stride = mx;
        DeviceBuffer<uint64_t> dq(qids.size());
        WF_CUDA(cudaMemcpy(dq.get(), qids.data(), qids.size() * 8, cudaMemcpyHostToDevice));
        w.over_paths.allocate(qids.size() * static_cast<uint64_t>(mx));
        DeviceBuffer<uint32_t> tl(qids.size());
        DeviceBuffer<uint8_t> ts(qids.size());
        DeviceBuffer<unsigned long long> tc(2);
        WF_CUDA(cudaMemset(tc.get(), 0, 16));
        launch_walk(s, rs.spec, rs.dev_sources, 0, qids.size(), dq.get(), w.over_paths.get(), mx, tl.get(),
                    ts.get(), nullptr, tc.get(), tc.get() + 1, s.cursor.get(), nullptr);
        WF_CUDA(cudaDeviceSynchronize());
        check_device_error(s);
    }
    w.metrics.preprocess_seconds = s.preprocess_seconds;
    w.metrics.exec_seconds = ms * 1e-3;
    w.metrics.total_steps = hc[0];
    w.metrics.max_in_flight = static_cast<uint32_t>(
        std::min<uint64_t>(static_cast<uint64_t>(s.grid) * kBlock, std::max<uint64_t>(w.n, 1)));
    w.total_vertices = w.n + hc[0];
    if (w.n) {
        DeviceBuffer<unsigned> m(1);
        WF_CUDA(cudaMemset(m.get(), 0, 4));
        k_max_u32<<<256, 256>>>(w.lengths.get(), w.n, m.get());
        WF_LAUNCHED();
        WF_CUDA(cudaMemcpy(&w.max_length, m.get(), 4, cudaMemcpyDeviceToHost));
    }
    return wp;
}

}  // namespace wf

extern "C" {

int wf_session_run(wf_session* sh, const wf_query_spec* spec, wf_walkset** out,
                   wf_run_metrics* metrics) {
    return guarded([&] {
        require(sh && spec && out, "null argument");
        Session& s = *sh->s;
        DeviceGuard guard(s.g->device);
        ResolvedSpec rs;
        resolve_spec(*s.g, spec, rs);
        auto wh = std::make_unique<wf_walkset>();
        wh->w = session_run(s, rs, 0, rs.n, sh->counters.get());
        if (metrics) *metrics = wh->w->metrics;
        *out = wh.release();
    });
}

namespace {
void run_host_checked(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin, uint64_t qid_end,
                      uint64_t* offsets, uint32_t* vertices, uint64_t vertices_capacity, uint8_t* status,
                      uint64_t chunk_queries, wf_run_metrics* metrics, uint32_t* records,
                      wf_block_fn on_block = nullptr, void* user = nullptr) {
    require(sh && spec && vertices, "null argument");
    Session& s = *sh->s;
    GraphStore& g = *s.g;
    DeviceGuard guard(g.device);
    uint64_t n = spec->mode == WF_QUERY_ONE_PER_VERTEX ? g.V : spec->count;
    if (qid_end == 0) qid_end = n;
    require(qid_begin <= qid_end && qid_end <= n, "query range out of bounds");
    if (spec->mode == WF_QUERY_FROM_SOURCE && spec->source >= g.V)
        config_error("query source " + std::to_string(spec->source) + " is not a vertex (V=" +
                     std::to_string(g.V) + ")");
    if (spec->mode == WF_QUERY_FROM_LIST) {
        require(spec->sources != nullptr || n == 0, "null source list");
        require(!is_device_pointer(spec->sources), "wf_session_run_host takes a host source list");
        // sources are range-checked by the walk kernel (ConfigError after the run)
    }
    run_to_host(s, *spec, spec->sources, qid_begin, qid_end, offsets, vertices, vertices_capacity, status,
                chunk_queries, metrics, records, on_block, user);
}
}  // namespace

int wf_session_run_host_records(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin,
                                uint64_t qid_end, uint32_t* records, uint32_t* vertices,
                                uint64_t vertices_capacity, uint64_t chunk_queries, wf_run_metrics* metrics) {
    return guarded([&] {
        require(records != nullptr, "null argument");
        run_host_checked(sh, spec, qid_begin, qid_end, nullptr, vertices, vertices_capacity, nullptr,
                         chunk_queries, metrics, records);
    });
}

int wf_session_run_host_blocks(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin,
                               uint64_t qid_end, uint32_t* records, uint32_t* vertices,
                               uint64_t vertices_capacity, uint64_t chunk_queries, wf_block_fn on_block,
                               void* user, wf_run_metrics* metrics) {
    return guarded([&] {
        require(records != nullptr && on_block != nullptr, "null argument");
        run_host_checked(sh, spec, qid_begin, qid_end, nullptr, vertices, vertices_capacity, nullptr,
                         chunk_queries, metrics, records, on_block, user);
    });
}

int wf_session_run_host(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin,
                        uint64_t qid_end, uint64_t* offsets, uint32_t* vertices,
                        uint64_t vertices_capacity, uint8_t* status, uint64_t chunk_queries,
                        wf_run_metrics* metrics) {
    return guarded([&] {
        run_host_checked(sh, spec, qid_begin, qid_end, offsets, vertices, vertices_capacity, status,
                         chunk_queries, metrics, nullptr);
    });
}

int wf_session_set_stats(wf_session* sh, int enable) {
    return guarded([&] {
        require(sh != nullptr, "null session");
        Session& s = *sh->s;
        DeviceGuard guard(s.g->device);
        if (enable && !s.stats.get()) {
            s.stats.allocate(WF_STATS_COUNT);
            WF_CUDA(cudaMemset(s.stats.get(), 0, WF_STATS_COUNT * 8));
        }
        s.collect_stats = enable != 0;
    });
}

int wf_session_stats_n(wf_session* sh, uint64_t* out, uint32_t n) {
    return guarded([&] {
        require(sh && out, "null argument");
        Session& s = *sh->s;
        DeviceGuard guard(s.g->device);
        for (uint32_t i = 0; i < n; ++i) out[i] = 0;
        if (!s.stats.get()) return;
        uint64_t all[WF_STATS_COUNT];
        WF_CUDA(cudaDeviceSynchronize());
        WF_CUDA(cudaMemcpy(all, s.stats.get(), sizeof(all), cudaMemcpyDeviceToHost));
        WF_CUDA(cudaMemset(s.stats.get(), 0, sizeof(all)));
        for (uint32_t i = 0; i < n && i < WF_STATS_COUNT; ++i) out[i] = all[i];
    });
}

int wf_session_stats(wf_session* sh, uint64_t* out3) { return wf_session_stats_n(sh, out3, 3); }

// Launch tuner (tune.cpp:46-111's role): candidate blocks/SM from the occupancy
// maximum down to a quarter, each timed over whole launches of the range.
int wf_session_tune(wf_session* sh, const wf_query_spec* spec, uint64_t qid_begin, uint64_t qid_end,
                    int32_t* blocks_per_sm, double* best_ms) {
    return guarded([&] {
        require(sh && spec, "null argument");
        Session& s = *sh->s;
        GraphStore& g = *s.g;
        DeviceGuard guard(g.device);
        ResolvedSpec rs;
        resolve_spec(g, spec, rs);
        if (qid_end == 0) qid_end = rs.n;
        require(qid_begin < qid_end && qid_end <= rs.n, "query range out of bounds");
        const uint64_t n = qid_end - qid_begin;
        const uint32_t stride = s.default_stride;
        size_t free_b = 0, total_b = 0;
        WF_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const uint64_t need = n * (stride * 4ull + 5) + (s.desc.kind == WF_PROGRAM_PPR ? g.V * 4ull : 0);
        if (need > free_b / 2) raise(WF_ERR_INVALID_ARG, "tune range needs more scratch than half the free HBM; tune a smaller range");
        DeviceBuffer<uint32_t> paths(n * stride), lens(n), counts;
        DeviceBuffer<uint8_t> stat(n);
        if (s.desc.kind == WF_PROGRAM_PPR) counts.allocate(g.V);
        DeviceBuffer<unsigned long long> ctr(2);
        const int bucket = row_bucket(n);
        s.tuned_blocks.erase(bucket);
        const int max_per_sm = std::max(1, s.grid / sm_count(g.device));
        std::vector<int> cands;
        // every count from the occupancy maximum down to a quarter of it (at
        // least 2 candidates below the maximum)
        const int lowest = std::max(1, std::min(max_per_sm / 4, max_per_sm - 2));
        for (int c = max_per_sm; c >= lowest; --c) cands.push_back(c);
        cudaEvent_t e0, e1;
        WF_CUDA(cudaEventCreate(&e0));
        WF_CUDA(cudaEventCreate(&e1));
        double best = 1e300;
        int pick = max_per_sm;
        for (int c : cands) {
            s.tuned_blocks[bucket] = c;
            float mn = 1e30f;
            for (int rep = 0; rep < 4; ++rep) {  // first launch warms, then best of 3
                if (counts.get()) WF_CUDA(cudaMemsetAsync(counts.get(), 0, g.V * 4ull, nullptr));
                WF_CUDA(cudaEventRecord(e0, nullptr));
                launch_walk(s, rs.spec, rs.dev_sources, qid_begin, qid_end, nullptr, paths.get(), stride,
                            lens.get(), stat.get(), counts.get(), ctr.get(), ctr.get() + 1,
                            s.cursor.get(), nullptr);
                WF_CUDA(cudaEventRecord(e1, nullptr));
                WF_CUDA(cudaEventSynchronize(e1));
                float ms = 0.f;
                WF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                if (rep > 0) mn = std::min(mn, ms);
            }
            if (getenv("WF_TRACE_TUNE"))  // diagnostics: every candidate's time
                std::fprintf(stderr, "[tune] rows %llu: %d blocks/SM %.4f ms\n",
                             static_cast<unsigned long long>(n), c, mn);
            if (mn < best) {
                best = mn;
                pick = c;
            }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        check_device_error(s);
        s.tuned_blocks[bucket] = pick;
        if (blocks_per_sm) *blocks_per_sm = pick;
        if (best_ms) *best_ms = best;
    });
}

int wf_walkset_info(const wf_walkset* w, uint64_t* n_queries, uint64_t* total_vertices,
                    uint32_t* max_length) {
    return guarded([&] {
        require(w != nullptr, "null walkset");
        if (n_queries) *n_queries = w->w->n;
        if (total_vertices) *total_vertices = w->w->total_vertices;
        if (max_length) *max_length = w->w->max_length;
    });
}

int wf_walkset_copy(const wf_walkset* w, uint64_t qid_begin, uint64_t qid_end, uint64_t* offsets,
                    uint32_t* vertices, uint8_t* status) {
    return guarded([&] {
        require(w != nullptr, "null walkset");
        walkset_copy(*w->w, qid_begin, qid_end, offsets, vertices, status);
    });
}

int wf_walkset_visit_counts(const wf_walkset* wh, uint32_t* counts) {
    return guarded([&] {
        require(wh && counts, "null argument");
        const WalkSetStore& w = *wh->w;
        DeviceGuard guard(w.device);
        const bool dev = is_device_pointer(counts);
        if (w.visit_counts.get()) {
            WF_CUDA(cudaMemcpy(counts, w.visit_counts.get(), w.V * 4ull, cudaMemcpyDefault));
            return;
        }
        DeviceBuffer<uint32_t> tmp;
        uint32_t* dc = counts;
        if (!dev) {
            tmp.allocate(w.V);
            dc = tmp.get();
        }
        walkset_visit_counts(w, dc, nullptr);
        WF_CUDA(cudaDeviceSynchronize());
        if (!dev) WF_CUDA(cudaMemcpy(counts, dc, w.V * 4ull, cudaMemcpyDeviceToHost));
    });
}

int wf_encode_walks(const uint64_t* offsets, const uint32_t* vertices, const uint8_t* status,
                    uint64_t n, uint64_t qid_base, int format, char* out, uint64_t capacity,
                    uint64_t* bytes) {
    return guarded([&] {
        require(offsets && (vertices || n == 0) && (status || n == 0) && bytes, "null argument");
        *bytes = encode_walks(offsets, vertices, status, n, qid_base, format, out, capacity);
    });
}

int wf_walkset_write(const wf_walkset* w, const char* path, int format, uint64_t qid_begin,
                     uint64_t qid_end, uint64_t* bytes_written) {
    return guarded([&] {
        require(w && path, "null argument");
        uint64_t b = write_walkset(*w->w, path, format, qid_begin, qid_end);
        if (bytes_written) *bytes_written = b;
    });
}

void wf_walkset_destroy(wf_walkset* w) {
    if (w) {
        DeviceGuard guard(w->w->device, std::nothrow);
        delete w;
    }
}

int wf_run(const wf_graph* g, const wf_program_desc* prog, const wf_query_spec* spec,
           const wf_exec_options* opts, wf_walkset** out, wf_run_metrics* metrics) {
    wf_session* s = nullptr;
    int rc = guarded([&] {
        require(g && spec, "null argument");
        ResolvedSpec rs;
        resolve_spec(*g->g, spec, rs);  // run_sequential validates the spec first (engine.hpp:443)
    });
    if (rc != WF_OK) return rc;
    rc = wf_session_create(g, prog, opts, &s);
    if (rc != WF_OK) return rc;
    rc = wf_session_run(s, spec, out, metrics);
    wf_session_destroy(s);
    return rc;
}

int wf_rng_probe(uint64_t seed, const uint64_t* streams, uint64_t n_streams, uint32_t draws,
                 uint64_t* out) {
    return guarded([&] {
        require(streams && out, "null argument");
        if (!n_streams || !draws) return;
        DeviceBuffer<uint64_t> ds(n_streams), dout(n_streams * draws);
        WF_CUDA(cudaMemcpy(ds.get(), streams, n_streams * 8, cudaMemcpyHostToDevice));
        k_rng_probe<<<64, 256>>>(seed_premix(seed), ds.get(), n_streams, draws, dout.get());
        WF_LAUNCHED();
        WF_CUDA(cudaMemcpy(out, dout.get(), n_streams * draws * 8, cudaMemcpyDeviceToHost));
    });
}

int wf_session_tables(const wf_session* sh, uint64_t* alias_thr, uint32_t* alias_first_dst,
                      uint32_t* alias_second_dst, double* its_cumulative, double* rej_p_star,
                      uint8_t* exhausted) {
    return guarded([&] {
        require(sh != nullptr, "null session");
        const Session& s = *sh->s;
        const GraphStore& g = *s.g;
        DeviceGuard guard(g.device);
        if (s.alias.get() && (alias_thr || alias_first_dst || alias_second_dst)) {
            const uint64_t bs = s.alias_wide ? 2 : 1;
            std::vector<uint4> b(g.E * bs);
            WF_CUDA(cudaMemcpy(b.data(), s.alias.get(), g.E * 16 * bs, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < g.E; ++i) {
                const uint4& x = b[i * bs];
                if (alias_thr) alias_thr[i] = (static_cast<uint64_t>(x.y) << 32) | x.x;
                if (alias_first_dst) alias_first_dst[i] = x.z;
                if (alias_second_dst) alias_second_dst[i] = x.w;
            }
        }
        if (s.its.get() && its_cumulative)
            WF_CUDA(cudaMemcpy(its_cumulative, s.its.get(), g.E * 8, cudaMemcpyDeviceToHost));
        if (s.rej.get() && rej_p_star)
            WF_CUDA(cudaMemcpy(rej_p_star, s.rej.get(), g.V * 8ull, cudaMemcpyDeviceToHost));
        if (s.exhausted.get() && exhausted)
            WF_CUDA(cudaMemcpy(exhausted, s.exhausted.get(), g.V, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
