/*
 * walkforge_b200.h — C-ABI of the B200-native random-walk engine.
 *
 * Drop-in boundary for the reference's step-centric Gather–Move–Update path
 * (walkforge, /root/reference/proj).  Every entry point below replaces one
 * reference interface; the citation is on each declaration.  Plain pointers and
 * sizes only — no C++ or torch types cross this line.  A header-only C++ shim
 * with the reference's own template signatures sits on top of it
 * (include/walkforge_b200/engine.hpp); a Python ctypes mirror lives in
 * paper_2107_11983_b200/engine.py.
 *
 * Error model: every function returns a wf_status.  Status codes map 1:1 onto
 * the reference exception classes (proj/include/walkforge/error.hpp:8-48); the
 * message of the last failure on the calling thread is wf_last_error().
 *
 * Threading (the reference's model, SPEC "graph read-only shared, no locks on
 * the hot path"): a wf_graph may be shared by sessions on any threads (its lazily
 * built indexes are built under a lock); a wf_session and a wf_walkset must be
 * used by one thread at a time (they own streams, staging buffers and the claim
 * cursor of their launches).
 */
#ifndef WALKFORGE_B200_H
#define WALKFORGE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WF_ABI_VERSION 1

/* ---- status codes: proj/include/walkforge/error.hpp:8-48 ------------------ */
typedef enum wf_status {
    WF_OK = 0,
    WF_ERR_PARSE = 1,         /* ParseError        error.hpp:14-16 */
    WF_ERR_FORMAT = 2,        /* FormatError       error.hpp:19-21 */
    WF_ERR_CONFIG = 3,        /* ConfigError       error.hpp:25-27 */
    WF_ERR_DISTRIBUTION = 4,  /* DistributionError error.hpp:31-33 */
    WF_ERR_CONTRACT = 5,      /* ContractError     error.hpp:36-38 */
    WF_ERR_REJECTION_CAP = 6, /* RejectionCapError error.hpp:42-44 */
    WF_ERR_IO = 7,            /* IoError           error.hpp:47-49 */
    WF_ERR_CUDA = 8,          /* device fault / no device (no reference class) */
    WF_ERR_OOM = 9,           /* device allocation failed */
    WF_ERR_INVALID_ARG = 10   /* null handle / bad pointer at the ABI */
} wf_status;

/* ---- enums mirrored from the reference ------------------------------------ */
/* SamplerKind, proj/include/walkforge/sampler.hpp:21 */
typedef enum wf_sampler {
    WF_SAMPLER_DEFAULT = -1, /* resolve_default_sampler, program.hpp:68-75 */
    WF_SAMPLER_NAIVE = 0,
    WF_SAMPLER_ITS = 1,
    WF_SAMPLER_ALIAS = 2,
    WF_SAMPLER_REJ = 3,
    WF_SAMPLER_OREJ = 4
} wf_sampler;

/* The built-in programs, proj/include/walkforge/algorithms.hpp:20-193 */
typedef enum wf_program_kind {
    WF_PROGRAM_PPR = 0,      /* PprProgram       algorithms.hpp:20-37   */
    WF_PROGRAM_DEEPWALK = 1, /* DeepWalkProgram  algorithms.hpp:41-67   */
    WF_PROGRAM_NODE2VEC = 2, /* Node2VecProgram  algorithms.hpp:79-133  */
    WF_PROGRAM_METAPATH = 3, /* MetaPathProgram  algorithms.hpp:141-173 */
    WF_PROGRAM_UNIFORM = 4   /* UniformProgram   algorithms.hpp:177-193 */
} wf_program_kind;

/* WalkStatus, proj/include/walkforge/walker.hpp:12 (0 complete, 1 dead end) */
typedef enum wf_walk_status { WF_WALK_COMPLETE = 0, WF_WALK_DEAD_END = 1 } wf_walk_status;

/* QuerySpec::Mode, proj/include/walkforge/walker.hpp:61-84 */
typedef enum wf_query_mode {
    WF_QUERY_ONE_PER_VERTEX = 0,
    WF_QUERY_FROM_SOURCE = 1,
    WF_QUERY_FROM_LIST = 2 /* QuerySpec::from_file after parsing: explicit sources */
} wf_query_mode;

/* ---- plain-data descriptors ----------------------------------------------- */

/* One program and its constructor arguments.  Validation follows each
 * reference constructor (e.g. PprProgram: termination in (0, 1],
 * algorithms.hpp:22-27; Node2Vec a, b > 0 finite, algorithms.hpp:81-96). */
typedef struct wf_program_desc {
    int32_t kind;           /* wf_program_kind */
    uint32_t target_length; /* DeepWalk / Node2Vec / Uniform: vertices per walk */
    int32_t weighted;       /* DeepWalk / Node2Vec: scale by edge weight */
    int32_t reserved0;
    double termination;     /* PPR stop probability */
    double a;               /* Node2Vec return parameter */
    double b;               /* Node2Vec in-out parameter */
    const uint32_t* schema; /* MetaPath label schema (host pointer) */
    uint32_t schema_len;
    uint32_t reserved1;
} wf_program_desc;

/* ExecOptions, proj/include/walkforge/engine.hpp:81-89.  `threads` is the
 * reference's worker count; on the device it is ignored (lanes replace
 * workers).  k / k_prime (interleave ring sizes, interleave.hpp:391-393) are
 * accepted and validated like the reference, then used as launch hints. */
typedef struct wf_exec_options {
    uint64_t seed;
    int32_t sampler;           /* wf_sampler */
    int32_t use_static_tables; /* default 1 */
    uint32_t rej_trial_cap;    /* default 1<<20 (sampler.hpp:27) */
    uint32_t threads;
    uint32_t k;
    uint32_t k_prime;
    uint32_t path_stride;      /* device row capacity for unbounded walks (0 = auto) */
    uint32_t layout_flags;     /* WF_LAYOUT_*: opt out of the decorated HBM layouts */
} wf_exec_options;

/* Decorated layouts trade HBM capacity for one fewer dependent random load per
 * move; they are used automatically when memory allows unless opted out. */
#define WF_LAYOUT_COMPACT_ALIAS 1u /* 16 B alias buckets (no destination vertex words); the default
                                      while buckets + vertex words fit twice the L2 */
#define WF_LAYOUT_NO_ADJ 2u        /* no decorated adjacency for NAIVE / O-REJ */
#define WF_LAYOUT_MP_SUCC 4u       /* MetaPath successor-decorated edges (cyclic schemas; default when HBM allows) */
#define WF_LAYOUT_FORCE_ADJ 8u     /* decorated adjacency even when the compact graph fits L2 */
#define WF_LAYOUT_SEARCH_TREE 16u  /* Node2Vec: sector B-tree instead of the edge hash set */
#define WF_LAYOUT_NO_MP_SUCC 32u   /* MetaPath: label records + partitioned neighbours only */
#define WF_LAYOUT_NO_EDGE_FILTER 64u /* Node2Vec: no pair pre-filter before the exact distance test */
#define WF_LAYOUT_WIDE_ALIAS 256u    /* 32 B alias buckets even when the compact form fits the L2 */
#define WF_LAYOUT_ADJ8 128u          /* NAIVE too: adjacency packed as (dst, degree, base) in 8 B where it fits
                                        (O-REJ uses it by default on graphs below the 16 B form's threshold) */

typedef struct wf_query_spec {
    int32_t mode; /* wf_query_mode */
    uint32_t source;
    uint64_t count;
    const uint32_t* sources; /* FROM_LIST: host or device pointer, `count` entries */
} wf_query_spec;

/* RunMetrics, proj/include/walkforge/engine.hpp:64-69 */
typedef struct wf_run_metrics {
    double preprocess_seconds;
    double exec_seconds;
    uint64_t total_steps;
    uint32_t max_in_flight;
    uint32_t reserved;
} wf_run_metrics;

typedef struct wf_graph_info {
    uint32_t vertex_count;
    uint32_t max_degree_lo; /* max degree fits in 32 bits (graph.cpp:165-168) */
    uint64_t edge_count;
    double max_weight;      /* 0 when unweighted (graph.hpp:56) */
    int32_t has_weights;
    int32_t has_labels;
    int32_t adjacency_sorted;
    int32_t device;
    uint32_t label_count; /* max label + 1 (0 if unlabeled) */
    uint32_t weights_f64; /* 1: some weight is not float32-exact; an f64 copy is resident */
} wf_graph_info;

/* Synthetic R-MAT generator (ingest; SURVEY §8 d).  Symmetrised,
 * de-duplicated, self-loops dropped, sorted adjacency.  Weights f32 =
 * synthetic_weight(seed, e) rounded to f32 and labels = synthetic_label(seed,
 * e, label_count), keyed on the final CSR edge index like the reference's
 * synthetic attributes (graph.cpp:279-287, synthetic.cpp:11-39). */
typedef struct wf_rmat_params {
    uint32_t scale;
    uint32_t edge_factor;
    double a, b, c; /* d = 1 - a - b - c */
    uint64_t seed;
    int32_t weighted;
    uint32_t label_count; /* 0 = unlabeled */
} wf_rmat_params;

typedef struct wf_graph wf_graph;     /* device-resident CSR (Graph, graph.hpp:17-107) */
typedef struct wf_session wf_session; /* program + resolved sampler + static tables (ResolvedRun, engine.hpp:275-294) */
typedef struct wf_walkset wf_walkset; /* WalkSet + RunMetrics (engine.hpp:71-74, walker.hpp:47-55) */

/* ---- library ---------------------------------------------------------------- */
int wf_abi_version(void);
const char* wf_last_error(void);
/* Visible CUDA devices (ExecOptions::threads -> device count in the C++ shim). */
int wf_device_count(int32_t* n);
/* Number of engine kernel launches since load (evidence for bench's gpu_launches). */
uint64_t wf_kernel_launches(void);

/* ---- graph residency: Graph::from_csr, graph.cpp:118-159 ---------------------
 * Validates like from_csr (monotone offsets, ids in range, finite non-negative
 * weights, matching lengths) and uploads.  Host pointers.  weights/labels may
 * be NULL (absent).  Labels must be < 256 (stored as u8 on the device). */
int wf_graph_create(const uint64_t* offsets, const uint32_t* neighbors, const float* weights,
                    const uint32_t* labels, uint32_t vertex_count, uint64_t edge_count, int device,
                    wf_graph** out);
/* Same with the reference's f64 weights (graph.hpp:102): weights that are all
 * float32-exact are stored as f32 only; otherwise an f64 copy stays resident
 * and every sampler, table and program reads it (the f32 array then mirrors
 * it for the hot-path layouts).  Walks equal the reference's either way. */
int wf_graph_create_f64(const uint64_t* offsets, const uint32_t* neighbors, const double* weights,
                        const uint32_t* labels, uint32_t vertex_count, uint64_t edge_count, int device,
                        wf_graph** out);
/* The weights as the reference holds them (f64[E], HOST). */
int wf_graph_download_weights_f64(const wf_graph* g, double* weights);
/* Same from DEVICE pointers (already resident, e.g. torch tensors); copies. */
int wf_graph_create_device(const uint64_t* offsets, const uint32_t* neighbors,
                           const float* weights, const uint8_t* labels, uint32_t vertex_count,
                           uint64_t edge_count, int device, wf_graph** out);
int wf_graph_generate_rmat(const wf_rmat_params* params, int device, wf_graph** out);
int wf_graph_info_get(const wf_graph* g, wf_graph_info* out);
/* Copies CSR arrays back to HOST buffers (any may be NULL to skip). */
int wf_graph_download(const wf_graph* g, uint64_t* offsets, uint32_t* neighbors, float* weights,
                      uint8_t* labels);
/* Membership test, Graph::has_edge (graph.cpp:182-188), batched on the device. */
int wf_graph_has_edge(const wf_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                      uint8_t* out);
/* Which labels occur on some edge: out[l] = 1 for l in [0, 256), else 0 (all 0
 * when unlabeled).  MetaPathProgram's constructor check (algorithms.hpp:151-160)
 * without a scan: the flags are computed once at graph creation. */
int wf_graph_labels_present(const wf_graph* g, uint8_t out[256]);
void wf_graph_destroy(wf_graph* g);

/* ---- graph ingest (graph.cpp:190-453) -------------------------------------- */
/* WFG1 binary files, Graph::read_binary / write_binary: magic "WFG1", u64 V,
 * u64 E, u8 flags, u64 offsets[V+1], u32 neighbors[E], f64 weights[E]?, u32
 * labels[E]?.  Reading applies the reference's FormatError checks; weights
 * keep their f64 values (wf_graph_create_f64); labels must be < 256 (device
 * storage, ConfigError). */
int wf_graph_read_wfg1(const char* path, int device, wf_graph** out);
int wf_graph_write_wfg1(const wf_graph* g, const char* path);

/* Text edge lists, load_edge_list (graph.cpp:307-453): `src dst [weight
 * [label]]` per line, '#' comments; ids remapped to dense ids in ascending
 * numeric order; CSR assembled on the device (stable sort by (src, dst), input
 * order breaking ties); random attributes keyed on the final edge index. */
typedef enum wf_attr_mode { WF_ATTR_NONE = 0, WF_ATTR_FROM_FILE = 1, WF_ATTR_RANDOM = 2 } wf_attr_mode;
typedef struct wf_edge_list_options {
    int32_t undirected; /* Directedness::Undirected: emit both directions */
    int32_t weights;    /* wf_attr_mode */
    int32_t labels;     /* wf_attr_mode */
    uint32_t label_count;
    uint64_t seed;
} wf_edge_list_options;
int wf_graph_load_edge_list(const char* path, const wf_edge_list_options* opts, int device,
                            wf_graph** out);
/* LoadedGraph::original_ids: u64[V] (identity for graphs not loaded from text). */
int wf_graph_original_ids(const wf_graph* g, uint64_t* out);

/* ---- sessions: ResolvedRun (engine.hpp:275-294) ------------------------------
 * Resolves the sampler (program default or override), checks the
 * program/sampler pairing (resolve_flow, engine.hpp:255-272), and builds the
 * static tables on the device (preprocess_static, engine.hpp:190-251). */
int wf_session_create(const wf_graph* g, const wf_program_desc* prog, const wf_exec_options* opts,
                      wf_session** out);
/* ---- custom device programs: the WalkProgram concept (program.hpp:49-93) -----
 * The reference's extension point is a C++ type with walker_type(),
 * weight(const Walker*, const EdgeRef&), update(Walker&, const EdgeRef&) and
 * optional max_weight() / preferred_sampler() / finished() (program.hpp:49-93;
 * its own tests write CountingProgram, AvoidVertexProgram and
 * NegativeWeightProgram that way, tests/test_engine.cpp:17-47).  Here such a
 * type has __device__ members and is compiled in the USER's .cu translation
 * unit against include/walkforge_b200/device_program.cuh, whose
 * WF_DEVICE_PROGRAM(Type, symbol) instantiates the walk kernel for it and
 * exports `const wf_program_ops* symbol(void)`: the table below.  The library
 * never needs to know the type; the user's code launches its own kernels on
 * the library's streams through it (kernels live where they are compiled). */
typedef struct wf_program_ops {
    uint32_t abi_version;      /* WF_ABI_VERSION of the header the table was built with */
    uint32_t launch_size;      /* sizeof(wf::WalkLaunch) it was built with (checked) */
    const char* name;          /* the program type's name */
    int32_t walker_type;       /* 0 unbiased, 1 static, 2 dynamic (WalkerType, program.hpp:17) */
    int32_t preferred_sampler; /* wf_sampler, or WF_SAMPLER_DEFAULT (SamplerPreferringProgram) */
    int32_t has_max_weight;    /* BoundedWeightProgram (required for O-REJ) */
    int32_t prechecked;        /* PreCheckedProgram: finished() before the first move */
    uint32_t program_size;     /* bytes of the program object (<= 256, trivially copyable) */
    uint32_t engine_abi;       /* wf::kEngineAbi of the device headers it was compiled with (checked) */
    /* Launches walk_kernel<Custom<Type>, sampler, flow, streaming> with `grid`
     * blocks on `stream`; `walk_launch` is the engine's launch record. */
    int (*launch)(const void* walk_launch, int32_t sampler, int32_t flow, int32_t streaming, int32_t grid,
                  void* stream);
    /* Resident blocks per SM and registers per thread of that kernel. */
    int (*occupancy)(int32_t sampler, int32_t flow, int32_t streaming, int32_t* blocks_per_sm, int32_t* regs);
    /* weight(nullptr, e) of every edge into out[E] (static tables,
     * preprocess_static, engine.hpp:190-251); *bad (device int) is set when a
     * weight is negative or not finite (check_program_weight, engine.hpp:97-101). */
    int (*static_weights)(const void* graph_view, const void* program, double* out, int32_t* bad, void* stream);
    /* max_weight() on the host (resolve_orej_bound, engine.hpp:103-114). */
    double (*max_weight)(const void* program);
    /* max_path_vertices(): an upper bound on a walk's vertices (the row
     * capacity of fixed-length programs); 0 = unbounded. */
    uint32_t (*max_path)(const void* program);
} wf_program_ops;

/* ResolvedRun for a custom program: `program` points to the program object
 * (program_size bytes, copied).  Everything else is as wf_session_create;
 * the session works with every run / launch / streaming / tune entry point. */
int wf_session_create_custom(const wf_graph* g, const wf_program_ops* ops, const void* program,
                             const wf_exec_options* opts, wf_session** out);

/* Resolved sampler and flow (0 Direct, 1 Tables, 2 Gathered). */
int wf_session_describe(const wf_session* s, int32_t* sampler, int32_t* flow,
                        double* preprocess_seconds);
/* Which HBM layouts the session uses (bitmask of WF_LAYOUT_HAS_*). */
#define WF_LAYOUT_HAS_WIDE_ALIAS 1u   /* 32 B alias buckets with destination vertex words */
#define WF_LAYOUT_HAS_ADJ 2u          /* decorated adjacency (NAIVE / O-REJ) */
#define WF_LAYOUT_HAS_MP_SUCC 4u      /* MetaPath successor-decorated partitioned edges */
#define WF_LAYOUT_HAS_LABEL_INDEX 8u  /* MetaPath label-partitioned CSR */
#define WF_LAYOUT_HAS_SEARCH_INDEX 16u /* adjacency search B-tree (Node2Vec, opt-in) */
#define WF_LAYOUT_HAS_EDGE_HASH 32u    /* exact edge hash set (Node2Vec default) */
#define WF_LAYOUT_HAS_EDGE_FILTER 64u  /* blocked Bloom pre-filter of vertex pairs (Node2Vec default) */
#define WF_LAYOUT_HAS_ADJ8 128u        /* packed 8 B decorated adjacency (NAIVE / O-REJ) */
int wf_session_layout(const wf_session* s, uint32_t* flags);
void wf_session_destroy(wf_session* s);

/* Runs every query of `spec` (run_sequential / run_interleaved,
 * engine.hpp:440-504, interleave.hpp:391-556 — identical outputs).  Result
 * owned by the returned walkset (device memory). */
int wf_session_run(wf_session* s, const wf_query_spec* spec, wf_walkset** out,
                   wf_run_metrics* metrics);

/* Low-level launch into caller-owned DEVICE buffers on a caller stream (bench
 * and streaming paths).  Queries [qid_begin, qid_end) of `spec`.
 *   paths   u32[(qid_end-qid_begin) * stride]   row r = query qid_begin + r
 *   lengths u32[(qid_end-qid_begin)]            true path length (may exceed stride)
 *   status  u8 [(qid_end-qid_begin)]            wf_walk_status
 *   visit_counts u32[V] or NULL                 += occurrences of each vertex
 *   steps_out u64[1] or NULL                    += moves (device counter)
 * Rows whose walk outgrows `stride` hold the first `stride` vertices; their
 * count is accumulated in overflow_out (u64, device, may be NULL).  Async: no
 * host synchronisation; errors flagged on the device surface at the next
 * wf_session_sync. */
int wf_session_launch(wf_session* s, const wf_query_spec* spec, uint64_t qid_begin,
                      uint64_t qid_end, uint32_t* paths, uint32_t stride, uint32_t* lengths,
                      uint8_t* status, uint32_t* visit_counts, unsigned long long* steps_out,
                      unsigned long long* overflow_out, void* stream);
/* Synchronises `stream` and raises any device-side error (RejectionCapError,
 * ContractError) recorded by launches since the last sync. */
int wf_session_sync(wf_session* s, void* stream);

/* Runs every query of `spec` and streams the walk set straight into HOST
 * buffers (the reference returns RunResult::walks in host memory,
 * engine.hpp:448-452, or streams blocks to a BlockSink, engine.hpp:76-79):
 *   offsets  u64[n+1]   path of query i = vertices[offsets[i] .. offsets[i+1])
 *   vertices u32[vertices_capacity]
 *   status   u8[n]
 * One persistent launch covers the queries (several for very large runs);
 * completed chunks of `chunk_queries` rows (0 = auto, 64 Ki; rounded up to a
 * power of two) are compacted and copied to the host while the rest still
 * run.  Pinned host memory gives full copy bandwidth, and a pinned source
 * list is streamed in while the kernel starts.  A FROM_LIST spec takes a HOST
 * source list.
 * Only queries [qid_begin, qid_end) run (qid_end 0 = all; a shard of a
 * multi-GPU job); outputs are indexed relative to qid_begin.
 * WF_ERR_INVALID_ARG if the walks need more than vertices_capacity entries. */
int wf_session_run_host(wf_session* s, const wf_query_spec* spec, uint64_t qid_begin,
                        uint64_t qid_end, uint64_t* offsets, uint32_t* vertices,
                        uint64_t vertices_capacity, uint8_t* status, uint64_t chunk_queries,
                        wf_run_metrics* metrics);

/* The same, with the walk set as records in query order — the shape of the
 * reference's WalkRecord{qid, status, path} (walker.hpp:47-55) without the
 * implicit qid:
 *   records  u32[n]   path length | status << 31  (status 1 = dead end)
 *   vertices u32[...] the paths back to back
 * 4 B per query instead of 9 (offsets + status): the lighter form to stream
 * over PCIe. */
int wf_session_run_host_records(wf_session* s, const wf_query_spec* spec, uint64_t qid_begin,
                                uint64_t qid_end, uint32_t* records, uint32_t* vertices,
                                uint64_t vertices_capacity, uint64_t chunk_queries,
                                wf_run_metrics* metrics);

/* The BlockSink form (engine.hpp:76-79: the sink gets one block per worker,
 * records in qid order, output.cpp's OrderedBlockSink merges them): as
 * wf_session_run_host_records, and `on_block(user, block, qid_begin, qid_end,
 * vertex_begin)` is called on the calling thread, in qid order, as soon as the
 * records [qid_begin, qid_end) and their vertices (from vertex_begin) have
 * landed in the host buffers — while later queries are still walking.  qids
 * are relative to the call's qid_begin; blocks are consecutive and cover the
 * run; `block` counts from 0.  Blocks holding a walk longer than the session's
 * row capacity are delivered after the run, once patched.  A non-zero return
 * stops the run with WF_ERR_IO (in-flight work is drained first). */
typedef int (*wf_block_fn)(void* user, uint64_t block, uint64_t qid_begin, uint64_t qid_end,
                           uint64_t vertex_begin);
int wf_session_run_host_blocks(wf_session* s, const wf_query_spec* spec, uint64_t qid_begin,
                               uint64_t qid_end, uint32_t* records, uint32_t* vertices,
                               uint64_t vertices_capacity, uint64_t chunk_queries, wf_block_fn on_block,
                               void* user, wf_run_metrics* metrics);

/* Instrumentation (measurement only; no reference counterpart): when enabled,
 * launches accumulate logical access counts used for the algorithmic sector
 * figure of SURVEY §8 d — out[0] rejection trials, out[1] adjacency-search
 * probes, out[2] edges scanned by per-step gathers.  Reading resets them. */
int wf_session_set_stats(wf_session* s, int enable);
int wf_session_stats(wf_session* s, uint64_t* out3);
/* All counters (n <= WF_STATS_COUNT): out[3] binary-search probes the
 * reference's Node2Vec weight() would make (ceil(log2(d_prev + 1)) per
 * adjacency test), out[4] u8-label sectors the reference's
 * MetaPath gather would scan (ceil(d_v / 32) per step), out[5] MetaPath step
 * attempts (moves + dead ends).  Reading resets them. */
#define WF_STATS_COUNT 6
int wf_session_stats_n(wf_session* s, uint64_t* out, uint32_t n);

/* Launch tuner: the device analogue of tune_ring_sizes (tune.cpp:46-111).  The
 * reference sweeps the interleave ring sizes (k, k') for its CPU; on the device
 * the knob is the number of resident walkers — blocks per SM — which trades
 * memory-level parallelism against per-move latency (Little's law: more lanes
 * in flight than the memory system can serve only lengthen every walk's chain).
 * Times whole launches of queries [qid_begin, qid_end) (host or device source
 * list; results discarded) at each candidate and keeps the fastest for launches
 * of that size (same power-of-two bucket of rows) on this session.  Walk
 * results never depend on it.  Out: the chosen blocks/SM and its time. */
int wf_session_tune(wf_session* s, const wf_query_spec* spec, uint64_t qid_begin, uint64_t qid_end,
                    int32_t* blocks_per_sm, double* best_ms);

/* ---- multi-GPU: run_*'s workers over devices --------------------------------
 * The reference splits a run into ExecOptions::threads workers, each a
 * contiguous qid block (worker_range, engine.hpp:296-298) on its own thread
 * (parallel_workers, engine.hpp:302-328), each block handed to the BlockSink
 * once, in worker order (engine.hpp:76-79).  Here the blocks are spread over
 * devices in contiguous groups: the graph is replicated on every listed device
 * (peer copies), the static tables are built once and peer-copied, one host
 * thread per device walks its blocks, and the calling thread receives the
 * blocks in worker order as they complete.  Output equals the single-device
 * run (walks depend only on (seed, qid)).  The one collective is an NCCL
 * all-reduce of the PPR visit counts (NCCL is loaded at run time); a device
 * listed twice shares nothing with NCCL, and its shards' counts are summed on
 * the device instead. */
typedef struct wf_multi wf_multi;
/* worker_range (engine.hpp:296-298): [n*w/W, n*(w+1)/W). */
int wf_worker_range(uint64_t n, uint32_t workers, uint32_t w, uint64_t* begin, uint64_t* end);
int wf_multi_create(const wf_graph* g, const int32_t* devices, uint32_t n_devices, const wf_program_desc* prog,
                    const wf_exec_options* opts, wf_multi** out);
int wf_multi_create_custom(const wf_graph* g, const int32_t* devices, uint32_t n_devices,
                           const wf_program_ops* ops, const void* program, const wf_exec_options* opts,
                           wf_multi** out);
/* collective: 1 when the visit counts are reduced with NCCL */
int wf_multi_info(const wf_multi* m, uint32_t* n_devices, int32_t* collective);
/* One worker block: records u32[qid_end - qid_begin] (length | status << 31)
 * and the paths back to back (n_vertices), valid during the call.  Non-zero
 * return stops the run (WF_ERR_IO). */
typedef int (*wf_shard_fn)(void* user, uint32_t worker, uint64_t qid_begin, uint64_t qid_end,
                           const uint32_t* records, const uint32_t* vertices, uint64_t n_vertices);
/* Runs every query of `spec` as `workers` blocks (0 = one per device);
 * visit_counts (host or device, u32[V], or NULL): PPR occurrence counts over
 * all paths, reduced over the devices. */
int wf_multi_run(wf_multi* m, const wf_query_spec* spec, uint32_t workers, wf_shard_fn on_shard, void* user,
                 uint32_t* visit_counts, wf_run_metrics* metrics);
void wf_multi_destroy(wf_multi* m);

/* One process per GPU (torchrun): each rank runs its worker_range shard with
 * the single-device API and reduces its visit counts through the library's
 * own NCCL communicator.  Rank 0 makes the id; the caller ships it to the
 * other ranks (any channel). */
#define WF_COMM_ID_BYTES 128
typedef struct wf_comm wf_comm;
int wf_comm_unique_id(uint8_t* id);
int wf_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, wf_comm** out);
/* In-place sum over the ranks of a device u32 vector, on `stream`. */
int wf_comm_allreduce_u32(wf_comm* c, uint32_t* dev_counts, uint64_t count, void* stream);
void wf_comm_destroy(wf_comm* c);
int wf_nccl_version(int32_t* version);

/* ---- walk sets: WalkSet (walker.hpp:47-55) -------------------------------- */
int wf_walkset_info(const wf_walkset* w, uint64_t* n_queries, uint64_t* total_vertices,
                    uint32_t* max_length);
/* Ragged copy-out of queries [qid_begin, qid_end): offsets u64[n+1] (relative
 * to the first), vertices u32[sum], status u8[n].  HOST or DEVICE pointers
 * (detected); any may be NULL. */
int wf_walkset_copy(const wf_walkset* w, uint64_t qid_begin, uint64_t qid_end, uint64_t* offsets,
                    uint32_t* vertices, uint8_t* status);
/* Occurrences of each vertex over all paths (sources included): u32[V]. */
int wf_walkset_visit_counts(const wf_walkset* w, uint32_t* counts);
void wf_walkset_destroy(wf_walkset* w);

/* ---- walk record encoding: OutputFormat (output.hpp:17-27, output.cpp:26-47) -
 * Text   "<qid>\t<complete|dead_end>\t<v0> <v1> ...\n"   (append_text_record)
 * Binary u64 qid | u8 status | u32 length | u32 path[length] (append_binary_record)
 * Encoded on the device; bytes are identical to the reference's writers. */
typedef enum wf_output_format { WF_OUTPUT_TEXT = 0, WF_OUTPUT_BINARY = 1 } wf_output_format;

/* Encodes n records (query ids qid_base..qid_base+n-1) from ragged arrays
 * (offsets u64[n+1] relative, vertices, status; host or device pointers) into
 * `out` (host or device, `capacity` bytes).  *bytes = encoded size; with
 * out == NULL only the size is computed.  WF_ERR_INVALID_ARG if it does not fit. */
int wf_encode_walks(const uint64_t* offsets, const uint32_t* vertices, const uint8_t* status,
                    uint64_t n, uint64_t qid_base, int format, char* out, uint64_t capacity,
                    uint64_t* bytes);

/* Writes queries [qid_begin, qid_end) of a walk set to a file in qid order
 * (DoubleBufferedWriter + OrderedBlockSink, output.cpp:49-200): blocks are
 * encoded on the device and written by a host thread while the next block is
 * encoded (double-buffered pinned memory).  qid_end 0 = all.  WF_ERR_IO on
 * file errors. */
int wf_walkset_write(const wf_walkset* w, const char* path, int format, uint64_t qid_begin,
                     uint64_t qid_end, uint64_t* bytes_written);

/* ---- convenience: run_sequential in one call -------------------------------- */
int wf_run(const wf_graph* g, const wf_program_desc* prog, const wf_query_spec* spec,
           const wf_exec_options* opts, wf_walkset** out, wf_run_metrics* metrics);

/* ---- device RNG probes (RngStream, rng.hpp:19-67), for parity tests --------- */
/* out[i*draws + j] = j-th next_u64() of RngStream(seed, streams[i]) */
int wf_rng_probe(uint64_t seed, const uint64_t* streams, uint64_t n_streams, uint32_t draws,
                 uint64_t* out);

/* ---- static tables probe (preprocess_static, engine.hpp:190-251) -------------
 * Copies the session's ALIAS buckets to HOST: thr u64[E] = ceil(split*2^53),
 * first_dst/second_dst u32[E]; exhausted u8[V].  ITS: cumulative f64[E]. REJ:
 * p_star f64[V]. Pointers may be NULL to skip. */
int wf_session_tables(const wf_session* s, uint64_t* alias_thr, uint32_t* alias_first_dst,
                      uint32_t* alias_second_dst, double* its_cumulative, double* rej_p_star,
                      uint8_t* exhausted);

#ifdef __cplusplus
}
#endif

#endif /* WALKFORGE_B200_H */
