// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// Thin extern "C" harness around the UNMODIFIED reference engine
// (/root/reference/proj).  `make -C oracle ref` compiles this file together
// with the reference's own sources, in place under /root/reference, into
// oracle/_ref/libwfref.so.  Nothing here restates an algorithm: every call
// goes to the reference's public API —
//   Graph::from_csr / build_graph        proj/src/graph.cpp:118-159, 289-304
//   make_power_law_graph / ring graph    proj/src/synthetic.cpp:46-80
//   run_sequential                       proj/include/walkforge/engine.hpp:440-504
//   run_interleaved                      proj/include/walkforge/interleave.hpp:391-556
//   detail::ResolvedRun / StepDriver     engine.hpp:275-294, 334-432 (sampled qids, the
//                                        pattern of proj/tests/test_algorithms.cpp:127-139)
//   preprocess_static                    engine.hpp:190-251
//   RngStream                            proj/include/walkforge/rng.hpp:19-67
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting library.
#include <algorithm>
#include <atomic>
#include <exception>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "walkforge/algorithms.hpp"
#include "walkforge/engine.hpp"
#include "walkforge/interleave.hpp"
#include "walkforge/output.hpp"
#include "walkforge/synthetic.hpp"

#include "../include/walkforge_b200.h"

using namespace walkforge;

namespace {

thread_local std::string g_error;

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return WF_OK;
    } catch (const ParseError& e) {
        return fail(WF_ERR_PARSE, e.what());
    } catch (const FormatError& e) {
        return fail(WF_ERR_FORMAT, e.what());
    } catch (const ConfigError& e) {
        return fail(WF_ERR_CONFIG, e.what());
    } catch (const DistributionError& e) {
        return fail(WF_ERR_DISTRIBUTION, e.what());
    } catch (const ContractError& e) {
        return fail(WF_ERR_CONTRACT, e.what());
    } catch (const RejectionCapError& e) {
        return fail(WF_ERR_REJECTION_CAP, e.what());
    } catch (const IoError& e) {
        return fail(WF_ERR_IO, e.what());
    } catch (const std::exception& e) {
        return fail(WF_ERR_INVALID_ARG, e.what());
    }
}

struct RefResult {
    WalkSet walks;
    RunMetrics metrics;
};

ExecOptions to_exec(const wf_exec_options* o) {
    ExecOptions eo;
    if (o == nullptr) {
        return eo;
    }
    eo.seed = o->seed;
    eo.threads = o->threads == 0 ? 1 : o->threads;
    if (o->sampler >= 0) {
        eo.sampler = static_cast<SamplerKind>(o->sampler);
    }
    eo.use_static_tables = o->use_static_tables != 0;
    eo.rej_trial_cap = o->rej_trial_cap == 0 ? kRejTrialCap : o->rej_trial_cap;
    return eo;
}

QuerySpec to_spec(const wf_query_spec* q) {
    switch (q->mode) {
        case WF_QUERY_ONE_PER_VERTEX:
            return QuerySpec::one_per_vertex();
        case WF_QUERY_FROM_SOURCE:
            return QuerySpec::from_source(q->source, q->count);
        default: {
            QuerySpec spec;
            spec.mode = QuerySpec::Mode::FromFile;
            spec.sources.assign(q->sources, q->sources + q->count);
            return spec;
        }
    }
}

// Instantiates the reference program named by the descriptor and hands it to fn.
template <typename Fn>
void with_program(const Graph& g, const wf_program_desc* p, Fn&& fn) {
    switch (p->kind) {
        case WF_PROGRAM_PPR:
            fn(PprProgram(p->termination));
            return;
        case WF_PROGRAM_DEEPWALK:
            fn(DeepWalkProgram(g, p->target_length, p->weighted != 0));
            return;
        case WF_PROGRAM_NODE2VEC:
            fn(Node2VecProgram(g, {.a = p->a, .b = p->b, .target_length = p->target_length},
                               p->weighted != 0));
            return;
        case WF_PROGRAM_METAPATH:
            fn(MetaPathProgram(g, std::vector<uint32_t>(p->schema, p->schema + p->schema_len)));
            return;
        case WF_PROGRAM_UNIFORM:
            fn(UniformProgram(p->target_length));
            return;
        default:
            throw ConfigError("unknown program kind");
    }
}

}  // namespace

extern "C" {

const char* wfref_last_error() { return g_error.c_str(); }

// ---- graphs -----------------------------------------------------------------

int wfref_graph_create(const uint64_t* offsets, const uint32_t* neighbors, const double* weights,
                       const uint32_t* labels, uint32_t vertex_count, uint64_t edge_count,
                       void** out) {
    return guarded([&] {
        std::vector<uint64_t> off(offsets, offsets + vertex_count + 1);
        std::vector<VertexId> nbr(neighbors, neighbors + edge_count);
        std::vector<double> w;
        std::vector<uint32_t> l;
        if (weights) w.assign(weights, weights + edge_count);
        if (labels) l.assign(labels, labels + edge_count);
        *out = new Graph(Graph::from_csr(std::move(off), std::move(nbr), std::move(w), std::move(l)));
    });
}

// Same, from f32 weights and u8 labels (the device formats), widened while
// filling the reference's vectors so no f64 copy exists outside them.
int wfref_graph_create_f32(const uint64_t* offsets, const uint32_t* neighbors, const float* weights,
                           const uint8_t* labels, uint32_t vertex_count, uint64_t edge_count,
                           void** out) {
    return guarded([&] {
        std::vector<uint64_t> off(offsets, offsets + vertex_count + 1);
        std::vector<VertexId> nbr(neighbors, neighbors + edge_count);
        std::vector<double> w;
        std::vector<uint32_t> l;
        if (weights) w.assign(weights, weights + edge_count);
        if (labels) l.assign(labels, labels + edge_count);
        *out = new Graph(Graph::from_csr(std::move(off), std::move(nbr), std::move(w), std::move(l)));
    });
}

int wfref_graph_build(uint32_t vertex_count, const uint32_t* edge_pairs, uint64_t n_edges,
                      const double* weights, const uint32_t* labels, void** out) {
    return guarded([&] {
        std::vector<std::pair<VertexId, VertexId>> edges(n_edges);
        for (uint64_t i = 0; i < n_edges; ++i) {
            edges[i] = {edge_pairs[2 * i], edge_pairs[2 * i + 1]};
        }
        std::vector<double> w;
        std::vector<uint32_t> l;
        if (weights) w.assign(weights, weights + n_edges);
        if (labels) l.assign(labels, labels + n_edges);
        *out = new Graph(build_graph(vertex_count, std::move(edges), std::move(w), std::move(l)));
    });
}

int wfref_graph_power_law(uint32_t vertex_count, uint64_t edge_count, double exponent,
                          uint64_t seed, int weighted, uint32_t label_count, void** out) {
    return guarded([&] {
        PowerLawConfig cfg;
        cfg.vertex_count = vertex_count;
        cfg.edge_count = edge_count;
        cfg.exponent = exponent;
        cfg.seed = seed;
        cfg.weighted = weighted != 0;
        cfg.label_count = label_count;
        *out = new Graph(make_power_law_graph(cfg));
    });
}

int wfref_graph_ring(uint32_t n, uint64_t seed, int weighted, uint32_t label_count, void** out) {
    return guarded([&] { *out = new Graph(make_ring_graph(n, seed, weighted != 0, label_count)); });
}

void wfref_graph_destroy(void* g) { delete static_cast<Graph*>(g); }

// load_edge_list (graph.cpp:307-453).  weights/labels: 0 none, 1 file, 2 random.
int wfref_load_edge_list(const char* path, int undirected, int weights, int labels,
                         uint32_t label_count, uint64_t seed, void** out, uint64_t* n_ids,
                         uint64_t* ids, uint64_t ids_cap) {
    return guarded([&] {
        EdgeListOptions o;
        o.directedness = undirected ? Directedness::Undirected : Directedness::Directed;
        o.weights = static_cast<WeightMode>(weights);
        o.labels = static_cast<LabelMode>(labels);
        o.label_count = label_count;
        o.seed = seed;
        LoadedGraph lg = load_edge_list(path, o);
        *n_ids = lg.original_ids.size();
        if (ids)
            for (size_t i = 0; i < lg.original_ids.size() && i < ids_cap; ++i) ids[i] = lg.original_ids[i];
        *out = new Graph(std::move(lg.graph));
    });
}

int wfref_graph_write_binary(const void* g, const char* path) {
    return guarded([&] { static_cast<const Graph*>(g)->write_binary(path); });
}

int wfref_graph_read_binary(const char* path, void** out) {
    return guarded([&] { *out = new Graph(Graph::read_binary(path)); });
}

int wfref_graph_info(const void* gp, uint32_t* v, uint64_t* e, int* has_w, int* has_l,
                     uint64_t* max_degree, double* max_weight, int* sorted) {
    const Graph& g = *static_cast<const Graph*>(gp);
    *v = g.vertex_count();
    *e = g.edge_count();
    *has_w = g.has_weights();
    *has_l = g.has_labels();
    *max_degree = g.max_degree();
    *max_weight = g.max_weight();
    *sorted = g.adjacency_sorted();
    return WF_OK;
}

int wfref_graph_export(const void* gp, uint64_t* offsets, uint32_t* neighbors, double* weights,
                       uint32_t* labels) {
    const Graph& g = *static_cast<const Graph*>(gp);
    if (offsets) std::memcpy(offsets, g.offsets_data(), (g.vertex_count() + 1) * sizeof(uint64_t));
    if (neighbors) std::memcpy(neighbors, g.neighbors_data(), g.edge_count() * sizeof(uint32_t));
    if (weights && g.has_weights())
        std::memcpy(weights, g.weights_data(), g.edge_count() * sizeof(double));
    if (labels && g.has_labels())
        std::memcpy(labels, g.labels_data(), g.edge_count() * sizeof(uint32_t));
    return WF_OK;
}

int wfref_has_edge(const void* gp, uint32_t src, uint32_t dst) {
    return static_cast<const Graph*>(gp)->has_edge(src, dst) ? 1 : 0;
}

// ---- test programs ----------------------------------------------------------
// The custom programs of the reference's own engine tests (written against its
// WalkProgram concept, program.hpp:49-93), for parity with the same programs
// written against the device program API (tests/programs/test_programs.cu).

struct TestProgramParams {  // mirrors tests/test_custom_programs_gpu.py
    uint32_t length;
    uint32_t banned;
    double stop;
    uint32_t stop_label;
    uint32_t schema_len;
    uint32_t schema[48];
};

// proj/tests/test_engine.cpp:17-27
struct CountingProgram {
    uint32_t length;
    std::atomic<uint64_t>* updates;
    WalkerType walker_type() const { return WalkerType::Unbiased; }
    double weight(const Walker*, const EdgeRef&) const { return 1.0; }
    bool update(Walker& q, const EdgeRef&) const {
        updates->fetch_add(1, std::memory_order_relaxed);
        return q.path.size() >= length;
    }
};

// proj/tests/test_engine.cpp:29-40
struct AvoidVertexProgram {
    VertexId banned;
    uint32_t length;
    WalkerType walker_type() const { return WalkerType::Static; }
    double weight(const Walker*, const EdgeRef& e) const { return e.dst() == banned ? 0.0 : 1.0; }
    bool update(Walker& q, const EdgeRef&) const { return q.path.size() >= length; }
    double max_weight() const { return 1.0; }
};

// proj/tests/test_engine.cpp:42-46
struct NegativeWeightProgram {
    WalkerType walker_type() const { return WalkerType::Static; }
    double weight(const Walker*, const EdgeRef&) const { return -1.0; }
    bool update(Walker&, const EdgeRef&) const { return true; }
};

// a weighted meta-path walk has no reference built-in; this is
// the test-local program the survey prescribes (label match ? w_e : 0).
struct LabelWeightProgram {
    std::vector<uint32_t> schema;
    WalkerType walker_type() const { return WalkerType::Dynamic; }
    double weight(const Walker* q, const EdgeRef& e) const {
        if (q == nullptr) return 0.0;
        return e.label() == schema[q->moves()] ? e.weight() : 0.0;
    }
    bool update(Walker& q, const EdgeRef&) const { return q.moves() >= schema.size(); }
    bool finished(const Walker& q) const { return q.moves() >= schema.size(); }
};

// Unbiased, unbounded: a stop coin drawn in update() plus the traversed edge's label.
struct LabelStopProgram {
    double stop;
    uint32_t stop_label;
    WalkerType walker_type() const { return WalkerType::Unbiased; }
    double weight(const Walker*, const EdgeRef&) const { return 1.0; }
    bool update(Walker& q, const EdgeRef& e) const {
        const bool coin = q.rng.uniform_real(1.0) < stop;
        return coin || e.label() == stop_label;
    }
    double max_weight() const { return 1.0; }
};

// ---- runs -------------------------------------------------------------------

// interleaved: 0 -> run_sequential, 1 -> run_interleaved(k, k').
// discard: 1 -> a no-op BlockSink, so timing excludes result assembly
// (SURVEY §8 d "CPU timing beside it").
int wfref_run(const void* gp, const wf_program_desc* prog, const wf_query_spec* q,
              const wf_exec_options* opts, int interleaved, int discard, void** out,
              wf_run_metrics* metrics) {
    return guarded([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        auto res = std::make_unique<RefResult>();
        ExecOptions eo = to_exec(opts);
        if (discard) {
            eo.sink = [](uint32_t, WalkSet&&) {};
        }
        QuerySpec spec = to_spec(q);
        uint32_t k = opts && opts->k ? opts->k : 64;
        uint32_t kp = opts && opts->k_prime ? opts->k_prime : 32;
        with_program(g, prog, [&](const auto& p) {
            RunResult r = interleaved ? run_interleaved(g, spec, p, k, kp, eo)
                                      : run_sequential(g, spec, p, eo);
            res->walks = std::move(r.walks);
            res->metrics = r.metrics;
        });
        if (metrics) {
            metrics->preprocess_seconds = res->metrics.preprocess_seconds;
            metrics->exec_seconds = res->metrics.exec_seconds;
            metrics->total_steps = res->metrics.total_steps;
            metrics->max_in_flight = res->metrics.max_in_flight;
        }
        *out = res.release();
    });
}

// Runs only the listed query ids, exactly as run_sequential's per-query loop
// (engine.hpp:466-492) does, through the reference's ResolvedRun + StepDriver.
// Lets full-size configs be checked on a sample of queries.
int wfref_run_qids(const void* gp, const wf_program_desc* prog, const wf_query_spec* q,
                   const wf_exec_options* opts, const uint64_t* qids, uint64_t n_qids,
                   void** out, wf_run_metrics* metrics) {
    return guarded([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        auto res = std::make_unique<RefResult>();
        ExecOptions eo = to_exec(opts);
        QuerySpec spec = to_spec(q);
        spec.validate(g);
        with_program(g, prog, [&](const auto& p) {
            using P = std::decay_t<decltype(p)>;
            detail::ResolvedRun<P> run(g, p, eo);
            detail::StepDriver<P> driver(g, p, run);
            TransitionContext ctx;
            Walker walker;
            uint64_t steps = 0;
            res->walks.resize(n_qids);
            for (uint64_t i = 0; i < n_qids; ++i) {
                uint64_t qid = qids[i];
                walker.id = qid;
                walker.rng = RngStream(eo.seed, qid);
                walker.path.clear();
                walker.path.push_back(spec.source_at(qid, g));
                WalkStatus status = WalkStatus::DeadEnd;
                if (walk_already_finished(p, walker)) {
                    status = WalkStatus::Complete;
                } else {
                    while (true) {
                        uint64_t edge = driver.step(walker, ctx);
                        if (edge == detail::StepDriver<P>::kNoEdge) break;
                        steps += 1;
                        if (p.update(walker, EdgeRef{&g, walker.prev(), edge})) {
                            status = WalkStatus::Complete;
                            break;
                        }
                    }
                }
                res->walks[i] = {qid, status, walker.path};
            }
            res->metrics.total_steps = steps;
            res->metrics.preprocess_seconds = run.tables.build_seconds;
        });
        if (metrics) {
            metrics->preprocess_seconds = res->metrics.preprocess_seconds;
            metrics->exec_seconds = 0;
            metrics->total_steps = res->metrics.total_steps;
            metrics->max_in_flight = 1;
        }
        *out = res.release();
    });
}

// Whole-run digest for full-size parity (C5: 2^26 walks): every query of the
// spec is walked through the reference's ResolvedRun + StepDriver (the same
// per-query loop as wfref_run_qids / engine.hpp:466-492) on `threads` host
// threads, and folded into one 64-bit digest per block of `block_qids`
// consecutive query ids instead of being stored.  A walk contributes
// mix(qid*K1 + (len << 8 | status) + K3) + sum over positions of
// mix(qid*K1 + pos*K2 + vertex) (mod 2^64); oracle.py:walk_digest is the same
// fold over a WalkSet.
static inline uint64_t digest_mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

int wfref_run_digest(const void* gp, const wf_program_desc* prog, const wf_query_spec* q,
                     const wf_exec_options* opts, uint32_t threads, uint64_t block_qids,
                     uint64_t* digests, uint64_t n_blocks, wf_run_metrics* metrics) {
    return guarded([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        ExecOptions eo = to_exec(opts);
        QuerySpec spec = to_spec(q);
        spec.validate(g);
        const uint64_t n = spec.total(g);
        if (block_qids == 0 || (n + block_qids - 1) / block_qids != n_blocks)
            throw ConfigError("wfref_run_digest: n_blocks does not cover the query count");
        with_program(g, prog, [&](const auto& p) {
            using P = std::decay_t<decltype(p)>;
            detail::ResolvedRun<P> run(g, p, eo);
            std::atomic<uint64_t> next{0}, steps{0};
            std::exception_ptr first_error;
            std::atomic<bool> failed{false};
            auto work = [&] {
                try {
                    detail::StepDriver<P> driver(g, p, run);
                    TransitionContext ctx;
                    Walker walker;
                    uint64_t my_steps = 0;
                    for (;;) {
                        const uint64_t b = next.fetch_add(1);
                        if (b >= n_blocks || failed.load()) break;
                        const uint64_t q0 = b * block_qids, q1 = std::min(n, q0 + block_qids);
                        uint64_t d = 0;
                        for (uint64_t qid = q0; qid < q1; ++qid) {
                            walker.id = qid;
                            walker.rng = RngStream(eo.seed, qid);
                            walker.path.clear();
                            walker.path.push_back(spec.source_at(qid, g));
                            WalkStatus status = WalkStatus::DeadEnd;
                            if (walk_already_finished(p, walker)) {
                                status = WalkStatus::Complete;
                            } else {
                                while (true) {
                                    uint64_t edge = driver.step(walker, ctx);
                                    if (edge == detail::StepDriver<P>::kNoEdge) break;
                                    my_steps += 1;
                                    if (p.update(walker, EdgeRef{&g, walker.prev(), edge})) {
                                        status = WalkStatus::Complete;
                                        break;
                                    }
                                }
                            }
                            const uint64_t base = qid * 0x9E3779B97F4A7C15ull;
                            const uint64_t len = walker.path.size();
                            d += digest_mix(base + ((len << 8) | static_cast<uint64_t>(status)) +
                                            0x632BE59BD9B4E019ull);
                            for (uint64_t i = 0; i < len; ++i)
                                d += digest_mix(base + i * 0xC2B2AE3D27D4EB4Full + walker.path[i]);
                        }
                        digests[b] = d;
                    }
                    steps.fetch_add(my_steps);
                } catch (...) {
                    if (!failed.exchange(true)) first_error = std::current_exception();
                }
            };
            std::vector<std::thread> pool;
            const uint32_t t = std::max<uint32_t>(1, threads);
            for (uint32_t i = 1; i < t; ++i) pool.emplace_back(work);
            work();
            for (auto& th : pool) th.join();
            if (first_error) std::rethrow_exception(first_error);
            if (metrics) {
                metrics->preprocess_seconds = run.tables.build_seconds;
                metrics->exec_seconds = 0;
                metrics->total_steps = steps.load();
                metrics->max_in_flight = t;
            }
        });
    });
}

int wfref_result_info(const void* rp, uint64_t* n, uint64_t* total_vertices) {
    const RefResult& r = *static_cast<const RefResult*>(rp);
    *n = r.walks.size();
    uint64_t t = 0;
    for (const auto& w : r.walks) t += w.path.size();
    *total_vertices = t;
    return WF_OK;
}

int wfref_result_copy(const void* rp, uint64_t* qids, uint64_t* offsets, uint32_t* vertices,
                      uint8_t* status) {
    const RefResult& r = *static_cast<const RefResult*>(rp);
    uint64_t pos = 0;
    for (size_t i = 0; i < r.walks.size(); ++i) {
        const WalkRecord& w = r.walks[i];
        if (qids) qids[i] = w.query_id;
        if (status) status[i] = static_cast<uint8_t>(w.status);
        if (offsets) offsets[i] = pos;
        if (vertices) std::memcpy(vertices + pos, w.path.data(), w.path.size() * sizeof(uint32_t));
        pos += w.path.size();
    }
    if (offsets) offsets[r.walks.size()] = pos;
    return WF_OK;
}

void wfref_result_destroy(void* r) { delete static_cast<RefResult*>(r); }

// Record encoding through the reference's own writers (output.cpp:26-47).
// out == NULL: size only.
int wfref_encode(const void* rp, int format, char* out, uint64_t capacity, uint64_t* written) {
    return guarded([&] {
        const RefResult& r = *static_cast<const RefResult*>(rp);
        std::string buf;
        for (const WalkRecord& w : r.walks) {
            if (format == 0) append_text_record(buf, w);
            else append_binary_record(buf, w);
        }
        *written = buf.size();
        if (out) {
            if (buf.size() > capacity) throw ConfigError("buffer too small");
            std::memcpy(out, buf.data(), buf.size());
        }
    });
}

// A whole walk set through DoubleBufferedWriter (output.cpp:49-131).
int wfref_write_file(const void* rp, const char* path, int format) {
    return guarded([&] {
        const RefResult& r = *static_cast<const RefResult*>(rp);
        DoubleBufferedWriter writer(path, format == 0 ? OutputFormat::Text : OutputFormat::Binary);
        writer.write_all(r.walks);
        writer.finish();
    });
}

// ---- static tables ----------------------------------------------------------

// preprocess_static for the described (static) program.  alias: split f64,
// first/second u32 (second == first when no alias), first_dst/second_dst u32.
int wfref_static_tables(const void* gp, const wf_program_desc* prog, int sampler,
                        double* alias_split, uint32_t* alias_first, uint32_t* alias_second,
                        uint32_t* alias_first_dst, uint32_t* alias_second_dst,
                        double* its_cumulative, double* rej_p_star, uint8_t* exhausted,
                        double* seconds) {
    return guarded([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        with_program(g, prog, [&](const auto& p) {
            StaticTables t = preprocess_static(g, p, static_cast<SamplerKind>(sampler));
            if (seconds) *seconds = t.build_seconds;
            if (exhausted) std::memcpy(exhausted, t.exhausted.data(), t.exhausted.size());
            for (size_t i = 0; i < t.alias.size(); ++i) {
                if (alias_split) alias_split[i] = t.alias[i].split;
                if (alias_first) alias_first[i] = t.alias[i].first;
                if (alias_second) alias_second[i] = t.alias[i].second;
                if (alias_first_dst) alias_first_dst[i] = t.alias[i].first_dst;
                if (alias_second_dst) alias_second_dst[i] = t.alias[i].second_dst;
            }
            if (its_cumulative && !t.its_cumulative.empty())
                std::memcpy(its_cumulative, t.its_cumulative.data(),
                            t.its_cumulative.size() * sizeof(double));
            if (rej_p_star && !t.rej_p_star.empty())
                std::memcpy(rej_p_star, t.rej_p_star.data(), t.rej_p_star.size() * sizeof(double));
        });
    });
}

// Pure alias_init over one weight sequence (sampler.cpp:57-69).
int wfref_alias_init(const double* weights, uint32_t n, double* split, uint32_t* first,
                     uint32_t* second) {
    return guarded([&] {
        AliasTable t = alias_init(std::span<const double>(weights, n));
        for (uint32_t i = 0; i < n; ++i) {
            split[i] = t.slots[i].split;
            first[i] = t.slots[i].first;
            second[i] = t.slots[i].second;
        }
    });
}

// ---- RNG ----------------------------------------------------------------------

int wfref_rng_probe(uint64_t seed, uint64_t stream, uint32_t draws, uint64_t* out) {
    RngStream rng(seed, stream);
    for (uint32_t i = 0; i < draws; ++i) out[i] = rng.next_u64();
    return WF_OK;
}

// One fresh stream: uniform_index(n) then uniform_real(bound).
int wfref_rng_index_real(uint64_t seed, uint64_t stream, uint32_t n, double bound, uint32_t* idx,
                         double* real) {
    RngStream rng(seed, stream);
    *idx = rng.uniform_index(n);
    *real = rng.uniform_real(bound);
    return WF_OK;
}

double wfref_synthetic_weight(uint64_t seed, uint64_t edge) { return synthetic_weight(seed, edge); }
uint32_t wfref_synthetic_label(uint64_t seed, uint64_t edge, uint32_t count) {
    return synthetic_label(seed, edge, count);
}

unsigned wfref_hardware_threads() { return std::thread::hardware_concurrency(); }

// run_sequential / run_interleaved over one of the test programs above:
// which = 0 Counting, 1 AvoidVertex, 2 NegativeWeight, 3 LabelWeight,
// 4 LabelStop.  *updates = CountingProgram's update() calls.
int wfref_run_test_program(const void* gp, int which, const TestProgramParams* tp, const wf_query_spec* q,
                           const wf_exec_options* opts, int interleaved, void** out, wf_run_metrics* metrics,
                           uint64_t* updates) {
    return guarded([&] {
        const Graph& g = *static_cast<const Graph*>(gp);
        auto res = std::make_unique<RefResult>();
        ExecOptions eo = to_exec(opts);
        QuerySpec spec = to_spec(q);
        uint32_t k = opts && opts->k ? opts->k : 64;
        uint32_t kp = opts && opts->k_prime ? opts->k_prime : 32;
        std::atomic<uint64_t> count{0};
        auto go = [&](const auto& p) {
            RunResult r = interleaved ? run_interleaved(g, spec, p, k, kp, eo) : run_sequential(g, spec, p, eo);
            res->walks = std::move(r.walks);
            res->metrics = r.metrics;
        };
        switch (which) {
            case 0: go(CountingProgram{tp->length, &count}); break;
            case 1: go(AvoidVertexProgram{tp->banned, tp->length}); break;
            case 2: go(NegativeWeightProgram{}); break;
            case 3: go(LabelWeightProgram{std::vector<uint32_t>(tp->schema, tp->schema + tp->schema_len)}); break;
            case 4: go(LabelStopProgram{tp->stop, tp->stop_label}); break;
            default: throw ConfigError("unknown test program");
        }
        if (updates) *updates = count.load();
        if (metrics) {
            metrics->preprocess_seconds = res->metrics.preprocess_seconds;
            metrics->exec_seconds = res->metrics.exec_seconds;
            metrics->total_steps = res->metrics.total_steps;
            metrics->max_in_flight = res->metrics.max_in_flight;
        }
        *out = res.release();
    });
}

}  // extern "C"
