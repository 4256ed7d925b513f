// Host-side runtime objects behind the C-ABI handles.
//
//   GraphStore   device-resident Graph (graph.hpp:17-107): CSR + packed vertex
//                words + optional label index; stats from finalize_stats
//                (graph.cpp:161-180).
//   Session      ResolvedRun (engine.hpp:275-294): program parameters, resolved
//                sampler/flow, device static tables (preprocess_static).
//   WalkSetStore RunResult (engine.hpp:71-74): device rows + lengths + status.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "walkforge_b200/device/engine.cuh"

namespace wf {

constexpr uint64_t kNbrPad = 8;  // neighbour array slack: sector-wide reads at the end

struct GraphStore {
    int device = 0;
    uint32_t V = 0;
    uint64_t E = 0;
    DeviceBuffer<uint64_t> offsets;
    DeviceBuffer<uint32_t> nbr;
    DeviceBuffer<float> weights;
    // the reference's f64 weights (graph.hpp:102), kept only when some weight
    // is not float32-exact (then `weights` holds their f32 roundings for the
    // hot-path layouts and this array is what samplers and tables read)
    DeviceBuffer<double> weights64;
    double max_weight64 = 0.0;
    DeviceBuffer<uint8_t> labels;
    DeviceBuffer<uint64_t> vword;
    bool sorted = true;
    uint32_t max_degree = 0;
    double max_weight = 0.0;
    uint32_t label_count = 0;
    std::vector<uint8_t> label_present;  // 256 flags (MetaPath constructor check)
    std::vector<uint64_t> original_ids;  // edge-list ingest: dense id -> input id

    std::mutex mu;
    bool label_index_built = false;
    DeviceBuffer<uint4> lab_rec;
    DeviceBuffer<uint32_t> lab_nbr;
    bool search_index_built = false;
    int sidx_levels = 0;
    DeviceBuffer<uint32_t> sidx[kSidxMaxLevels];  // sector B-tree levels (has_edge_indexed)
    bool edge_hash_built = false;
    uint64_t ehash_buckets = 0;
    DeviceBuffer<unsigned long long> ehash;  // edge hash set (has_edge_hashed)
    bool edge_filter_built = false;
    uint64_t efilter_sectors = 0;
    DeviceBuffer<uint4> efilter;  // blocked Bloom filter of vertex pairs (efilter_maybe)

    GraphView view() const {
        GraphView g{};
        g.V = V;
        g.E = E;
        g.offsets = offsets.get();
        g.nbr = nbr.get();
        g.weights = weights.get();
        g.weights64 = weights64.get();
        g.labels = labels.get();
        g.vword = vword.get();
        g.sorted = sorted ? 1 : 0;
        g.lab_rec = lab_rec.get();
        g.lab_nbr = lab_nbr.get();
        g.label_count = label_count;
        g.sidx_levels = sidx_levels;
        for (int l = 0; l < kSidxMaxLevels; ++l) g.sidx[l] = sidx[l].get();
        g.ehash = ehash.get();
        g.ehash_buckets = ehash_buckets;
        g.efilter = efilter.get();
        g.efilter_sectors = efilter_sectors;
        return g;
    }
    bool has_weights() const { return weights.get() != nullptr; }
    bool has_labels() const { return labels.get() != nullptr; }

    // After offsets/nbr/weights/labels are resident: validate (from_csr),
    // compute stats, build vertex words.  `labels_checked` = labels already u8.
    void finalize(cudaStream_t st);
    // takes the reference's f64 weights (device): fills the f32 mirror and
    // keeps the f64 array only when some weight is not float32-exact
    void adopt_weights64(DeviceBuffer<double>&& w64, cudaStream_t st);
    void ensure_label_index(cudaStream_t st);
    void ensure_search_index(cudaStream_t st);
    void ensure_edge_hash(cudaStream_t st);
    void ensure_edge_filter(cudaStream_t st);
};

struct HostPipe;  // stream.cu: cached streams/buffers of the host-output pipeline
void release_host_pipe(HostPipe* p);

struct Session {
    GraphStore* g = nullptr;
    const wf_program_ops* custom = nullptr;  // a user's device program (wf_session_create_custom)
    std::unique_ptr<HostPipe, void (*)(HostPipe*)> pipe{nullptr, release_host_pipe};
    wf_program_desc desc{};
    std::vector<uint32_t> schema;
    DeviceBuffer<uint32_t> schema_dev;
    ProgParams params{};
    int kind = 0;  // wf_sampler
    int flow = 0;  // Flow
    uint64_t seed = 0;
    uint32_t trial_cap = 1u << 20;
    uint32_t default_stride = 0;  // path row capacity
    bool unbounded = false;       // PPR: geometric lengths
    double preprocess_seconds = 0.0;
    DeviceBuffer<uint4> alias;
    DeviceBuffer<double> its;
    DeviceBuffer<double> rej;
    DeviceBuffer<uint8_t> exhausted;
    DeviceBuffer<uint64_t> sview;  // vertex words with exhausted vertices at degree 0
    bool any_exhausted = false;
    DeviceBuffer<int> error_word;
    DeviceBuffer<unsigned long long> cursor;
    DeviceBuffer<double> scratch;
    uint64_t scratch_stride = 0;
    int grid = 0;                       // occupancy grid (max blocks/SM x SMs)
    std::map<int, int> tuned_blocks;    // wf_session_tune: log2 row bucket -> blocks/SM
    bool collect_stats = false;
    DeviceBuffer<unsigned long long> stats;  // [trials, probes, scanned]
    bool alias_wide = false;     // 32 B buckets carrying the destinations' vertex words
    bool alias_idx = false;      // buckets carry edge positions (custom programs read the edge)
    bool use_edge_hash = false;  // Node2Vec distance test through the graph's edge hash set
    bool use_edge_filter = false;  // ... behind the graph's pair pre-filter
    DeviceBuffer<uint4> adj;     // Direct flows: decorated adjacency {dst, 0, word}
    DeviceBuffer<unsigned long long> adj8;  // ... packed in 8 B when (dst, deg, base) fit
    uint32_t adj8_vbits = 0, adj8_dbits = 0;
    DeviceBuffer<uint4> mp_adj;  // MetaPath: partitioned edges decorated with the next group

    void build_tables(cudaStream_t st);
    // the static tables of a session of the same program on another device
    // (multi-device runs: peer copies instead of a rebuild)
    void copy_tables_from(const Session& src, cudaStream_t st);
    void build_adjacency(cudaStream_t st);
    // the packed form; false when (dst, degree, base) do not fit 64 bits
    bool build_adjacency8(cudaStream_t st);
    // MetaPath with a schema whose successor label is a function of the label
    // (e.g. cyclic): returns false (no table) otherwise.
    bool build_metapath_successors(cudaStream_t st);
};

struct WalkSetStore {
    int device = 0;
    uint64_t n = 0;
    uint32_t stride = 0;
    uint32_t V = 0;
    DeviceBuffer<uint32_t> paths;
    DeviceBuffer<uint32_t> lengths;
    DeviceBuffer<uint8_t> status;
    DeviceBuffer<uint32_t> visit_counts;
    // walks longer than `stride`, re-run into their own rows
    std::vector<uint64_t> over_rows;
    uint32_t over_stride = 0;
    DeviceBuffer<uint32_t> over_paths;
    wf_run_metrics metrics{};
    uint64_t total_vertices = 0;
    uint32_t max_length = 0;
};

// Host streaming of a launch (run_to_host): see WalkLaunch's fields.
struct StreamLaunch {
    unsigned long long* tile_word = nullptr;   // device, per tile, zeroed
    unsigned long long* chunk_word = nullptr;  // device, per chunk, zeroed
    unsigned long long* chunk_flag = nullptr;  // host-mapped, per chunk, zeroed
    uint32_t tile_shift = 10;
    uint32_t chunk_tiles_shift = 6;
    const unsigned int* src_ready = nullptr;  // device, or null
    uint32_t src_shift = 16;
    uint64_t src_row0 = 0;  // rows of the list (src_ready's count) before the launch's first row
};

// capi.cu: the calling thread's wf_last_error() text; the store behind a handle
std::string& last_error_slot();
GraphStore* graph_store(const wf_graph* g);

// capi.cu: ResolvedRun (engine.hpp:275-294) and QuerySpec resolution
struct ResolvedSpec {
    wf_query_spec spec{};
    uint64_t n = 0;
    DeviceBuffer<uint32_t> sources;
    const uint32_t* dev_sources = nullptr;
};
void resolve_program(Session& s, const wf_program_desc& d, const wf_exec_options* o);
void resolve_custom(Session& s, const wf_program_ops& ops, const void* program, const wf_exec_options* o);
void resolve_run(Session& s, int type, int preferred, bool has_max_weight, uint32_t fixed,
                 const wf_exec_options* o);
void setup_session(Session& s, const wf_exec_options* opts, const Session* tables_from);
void resolve_spec(const GraphStore& g, const wf_query_spec* q, ResolvedSpec& r);
void check_device_error(Session& s);
std::unique_ptr<WalkSetStore> session_run(Session& s, const ResolvedSpec& rs, uint64_t qb, uint64_t qe,
                                          unsigned long long* ctr);

// walk.cu
void launch_walk(Session& s, const wf_query_spec& spec, const uint32_t* dev_sources,
                 uint64_t qid_begin, uint64_t qid_end, const uint64_t* qid_map, uint32_t* paths,
                 uint32_t stride, uint32_t* lengths, uint8_t* status, uint32_t* visit_counts,
                 unsigned long long* steps_out, unsigned long long* overflow_out,
                 unsigned long long* cursor, cudaStream_t st, const StreamLaunch* stream = nullptr);
int occupancy_grid(const Session& s);
int row_bucket(uint64_t n_rows);  // tuner key: ceil(log2(rows))

// graph.cu
GraphStore* graph_from_host(const uint64_t* offsets, const uint32_t* neighbors, const float* weights,
                            const uint32_t* labels, uint32_t V, uint64_t E, int device, bool finalize = true);
GraphStore* graph_from_host_f64(const uint64_t* offsets, const uint32_t* neighbors, const double* weights,
                                const uint32_t* labels, uint32_t V, uint64_t E, int device);
GraphStore* graph_from_device(const uint64_t* offsets, const uint32_t* neighbors,
                              const float* weights, const uint8_t* labels, uint32_t V, uint64_t E,
                              int device);
GraphStore* graph_generate_rmat(const wf_rmat_params& p, int device);
void graph_has_edge(const GraphStore& g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                    uint8_t* out);

// graph_io.cu
GraphStore* graph_read_wfg1(const char* path, int device);
void graph_write_wfg1(const GraphStore& g, const char* path);
GraphStore* graph_load_edge_list(const char* path, const wf_edge_list_options& o, int device,
                                 std::vector<uint64_t>* original_ids);

// u32 -> u64 widening for scans over lengths / degrees
struct WidenU64 {
    __host__ __device__ uint64_t operator()(uint32_t x) const { return x; }
};

// stream.cu: the exception of a device-side error word (error.hpp classes)
[[noreturn]] void raise_device_error(const Session& s, int code);

// stream.cu: pipelined run + copy of the walk set into host buffers
void run_to_host(Session& s, const wf_query_spec& spec, const uint32_t* host_sources, uint64_t qb,
                 uint64_t qe, uint64_t* offsets, uint32_t* vertices, uint64_t capacity, uint8_t* status,
                 uint64_t chunk, wf_run_metrics* metrics, uint32_t* records = nullptr,
                 wf_block_fn on_block = nullptr, void* user = nullptr);

// output.cu: record encoding (text / binary, byte-identical to output.cpp)
uint64_t encode_walks(const uint64_t* offsets, const uint32_t* vertices, const uint8_t* status,
                      uint64_t n, uint64_t qid_base, int fmt, char* out, uint64_t capacity);
uint64_t write_walkset(const WalkSetStore& w, const char* path, int fmt, uint64_t qb, uint64_t qe);

// walk set copy-out (walk.cu)
void walkset_visit_counts(const WalkSetStore& w, uint32_t* counts_dev, cudaStream_t st);
void walkset_copy(const WalkSetStore& w, uint64_t qb, uint64_t qe, uint64_t* offsets,
                  uint32_t* vertices, uint8_t* status);

}  // namespace wf
