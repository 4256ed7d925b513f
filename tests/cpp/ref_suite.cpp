// The reference's own unit suites for the hot path — "engine"
// (/root/reference/proj/tests/test_engine.cpp:62-262), "interleave"
// (/root/reference/proj/tests/test_interleave.cpp:47-191), "algorithms"
// (/root/reference/proj/tests/test_algorithms.cpp:13-215; where the reference
// evaluates a program's weight() on the host, the case measures the same
// transition through walks instead) and "graph"
// (/root/reference/proj/tests/test_graph.cpp:18-196; its two cases on the
// reference's synthetic fixture generators are not part of the drop-in) —
// re-expressed against
// the drop-in shim (WALKFORGE_B200_DROP_IN: namespace walkforge), case by case
// under the reference's case names, with the reference's call patterns:
// run_sequential / run_interleaved, ExecOptions, BlockSink, custom programs.
// No doctest here (absent from the image): a case is a function, a failed
// expectation prints its line, the process exits with the number of failed
// cases.  Inputs are small graphs built through Graph::from_csr; the
// reference's random fixtures are replaced by a seeded generator of this
// file's own (the cases check invariants, not golden values — bit-exactness
// against the reference is tests/test_engine_gpu.py's job).
// The custom programs are the device versions in tests/programs/test_programs.cu.
#define WALKFORGE_B200_DROP_IN
#include "walkforge_b200/engine.hpp"

#include "mini_check.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iterator>
#include <limits>
#include <map>
#include <mutex>
#include <optional>
#include <string>
#include <utility>
#include <vector>

using namespace walkforge;

extern "C" const wf_program_ops* wf_test_counting_program(void);
extern "C" const wf_program_ops* wf_test_avoid_vertex_program(void);
extern "C" const wf_program_ops* wf_test_negative_weight_program(void);
extern "C" unsigned long long* wf_test_counter_new(void);
extern "C" unsigned long long wf_test_counter_read(const unsigned long long*);
extern "C" void wf_test_counter_free(unsigned long long*);

namespace {
struct CountingObj {  // host mirrors of the device programs' layouts
    uint32_t length;
    unsigned long long* updates;
};
struct AvoidVertexObj {
    uint32_t banned, length;
};
struct NegativeObj {
    uint32_t unused;
};

using EdgeList = std::vector<std::pair<VertexId, VertexId>>;

// the reference's build_graph (graph.hpp:143): adjacency sorted, attributes follow their edges
Graph graph_of(uint32_t n, const EdgeList& edges, const std::vector<double>& weights = {},
               const std::vector<uint32_t>& labels = {}) {
    return build_graph(n, edges, weights, labels);
}
Graph triangle() { return graph_of(3, {{0, 1}, {1, 2}, {2, 0}}); }  // 0 -> 1 -> 2 -> 0
Graph line(uint32_t n) {                                               // 0 -> 1 -> ... -> n-1
    EdgeList e;
    for (uint32_t v = 0; v + 1 < n; ++v) e.push_back({v, v + 1});
    return graph_of(n, e);
}
Graph clique(uint32_t n) {
    EdgeList e;
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = 0; v < n; ++v)
            if (u != v) e.push_back({u, v});
    return graph_of(n, e);
}
// a skewed random multigraph (hubs at the low ids), every vertex with an out-edge
Graph skewed_graph(uint32_t n, uint32_t m, uint64_t seed, bool weighted = false, uint32_t label_count = 0) {
    uint64_t s = seed * 0x9E3779B97F4A7C15ull + 12345;
    auto next = [&] {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    auto skew = [&] {
        const double u = static_cast<double>(next() >> 11) * 0x1.0p-53;
        return static_cast<VertexId>(u * u * n);
    };
    EdgeList e;
    std::vector<double> w;
    std::vector<uint32_t> lab;
    for (uint32_t i = 0; i < m; ++i) {
        const VertexId u = i < n ? i : skew(), v = skew();
        e.push_back({u, v});
        e.push_back({v, u});
        const double x = 1.0 + static_cast<double>(next() % 4000) / 1000.0;
        const uint32_t l = label_count ? static_cast<uint32_t>(next() % label_count) : 0;
        for (int r = 0; r < 2; ++r) {
            if (weighted) w.push_back(x);
            if (label_count) lab.push_back(l);
        }
    }
    return graph_of(n, e, w, lab);
}
bool scan_edge(const Graph& g, VertexId u, VertexId v) {
    for (VertexId x : g.neighbors(u))
        if (x == v) return true;
    return false;
}
bool adjacency_holds(const Graph& g, const WalkSet& walks) {
    for (const WalkRecord& r : walks)
        for (size_t i = 0; i + 1 < r.path.size(); ++i)
            if (!scan_edge(g, r.path[i], r.path[i + 1])) return false;
    return true;
}

// ---- suite "engine" (test_engine.cpp) -------------------------------------------------------
void fixed_length_walks_hit_their_target_exactly() {  // :63
    Graph g = triangle();
    RunResult res = run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 12, false));
    EXPECT(res.walks.size() == 3);
    for (const WalkRecord& r : res.walks) {
        EXPECT(r.status == WalkStatus::Complete);
        EXPECT(r.path.size() == 12);
    }
    EXPECT(res.metrics.total_steps == 3 * 11);
    EXPECT(adjacency_holds(g, res.walks));
}
void target_length_one_completes_without_a_single_move() {  // :75
    Graph g = triangle();
    RunResult res = run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 1, false));
    EXPECT(res.walks.size() == 3);
    for (const WalkRecord& r : res.walks) {
        EXPECT(r.status == WalkStatus::Complete);
        EXPECT(r.path.size() == 1);
    }
    EXPECT(res.metrics.total_steps == 0);
}
void dead_ends_emit_the_partial_path_with_the_right_status() {  // :85
    Graph g = line(4);
    RunResult res = run_sequential(g, QuerySpec::from_source(0, 1), DeepWalkProgram(g, 10, false));
    EXPECT(res.walks.size() == 1);
    EXPECT(res.walks[0].status == WalkStatus::DeadEnd);
    EXPECT((res.walks[0].path == std::vector<VertexId>{0, 1, 2, 3}));
}
void results_are_invariant_to_thread_count() {  // :93
    Graph g = skewed_graph(300, 1200, 8);
    ExecOptions one, four;
    one.threads = 1;
    one.seed = 123;
    four.threads = 4;
    four.seed = 123;
    RunResult a = run_sequential(g, QuerySpec::one_per_vertex(), PprProgram(0.2), one);
    RunResult b = run_sequential(g, QuerySpec::one_per_vertex(), PprProgram(0.2), four);
    EXPECT(a.walks == b.walks);
    EXPECT(a.walks.size() == 300);
}
void static_tables_and_per_step_gather_agree_for_every_table_sampler() {  // :106
    Graph g = skewed_graph(200, 800, 4, true);
    DeepWalkProgram prog(g, 10, true);
    for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej}) {
        ExecOptions tables;
        tables.sampler = kind;
        tables.seed = 5;
        ExecOptions gathered = tables;
        gathered.use_static_tables = false;
        RunResult a = run_sequential(g, QuerySpec::one_per_vertex(), prog, tables);
        RunResult b = run_sequential(g, QuerySpec::one_per_vertex(), prog, gathered);
        EXPECT(a.walks == b.walks);
        EXPECT(a.metrics.preprocess_seconds >= 0.0);
    }
}
void unbiased_programs_run_under_every_sampling_method_identically_in_law() {  // :123
    Graph g = skewed_graph(100, 450, 2);
    for (SamplerKind kind : {SamplerKind::Naive, SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej,
                             SamplerKind::ORej}) {
        ExecOptions opts;
        opts.sampler = kind;
        opts.seed = 31;
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 4000), PprProgram(0.2), opts);
        const double mean = static_cast<double>(res.metrics.total_steps) / 4000.0;
        EXPECT(mean > 4.0);
        EXPECT(mean < 6.0);
    }
}
void illegal_pairings_are_refused_up_front() {  // :143
    Graph g = triangle();
    ExecOptions naive;
    naive.sampler = SamplerKind::Naive;
    EXPECT_THROWS(run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 5, false), naive), ConfigError);
    ExecOptions orej;
    orej.sampler = SamplerKind::ORej;
    unsigned long long* ctr = wf_test_counter_new();
    DeviceProgram no_bound(wf_test_counting_program(), CountingObj{5, ctr});  // no max_weight()
    EXPECT_THROWS(run_sequential(g, QuerySpec::one_per_vertex(), no_bound, orej), ConfigError);
    wf_test_counter_free(ctr);
    Graph labeled = graph_of(3, {{0, 1}, {1, 2}, {2, 0}}, {}, {0, 0, 0});
    EXPECT_THROWS(run_sequential(labeled, QuerySpec::one_per_vertex(), MetaPathProgram(labeled, {0, 0}), orej),
                  ConfigError);
}
void a_program_emitting_negative_weights_is_caught() {  // :164
    Graph g = triangle();
    DeviceProgram neg(wf_test_negative_weight_program(), NegativeObj{0});
    EXPECT_THROWS(run_sequential(g, QuerySpec::one_per_vertex(), neg), ContractError);
}
void zero_weight_edges_are_never_traversed() {  // :171
    Graph g = clique(4);
    DeviceProgram prog(wf_test_avoid_vertex_program(), AvoidVertexObj{2, 16});
    for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej}) {
        ExecOptions opts;
        opts.sampler = kind;
        opts.seed = 7;
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 200), prog, opts);
        EXPECT(res.walks.size() == 200);
        for (const WalkRecord& r : res.walks) {
            EXPECT(r.status == WalkStatus::Complete);
            EXPECT(r.path.size() == 16);
            for (VertexId v : r.path) EXPECT(v != 2);
        }
    }
}
void vertices_whose_weights_all_vanish_dead_end_their_walkers() {  // :188
    Graph g = graph_of(3, {{0, 1}, {1, 2}});
    DeviceProgram prog(wf_test_avoid_vertex_program(), AvoidVertexObj{2, 16});
    ExecOptions opts;
    opts.sampler = SamplerKind::Alias;
    RunResult res = run_sequential(g, QuerySpec::from_source(0, 4), prog, opts);
    EXPECT(res.walks.size() == 4);
    for (const WalkRecord& r : res.walks) {
        EXPECT(r.status == WalkStatus::DeadEnd);
        EXPECT((r.path == std::vector<VertexId>{0, 1}));
    }
}
void update_runs_exactly_once_per_completed_move() {  // :201
    Graph g = triangle();
    unsigned long long* ctr = wf_test_counter_new();
    DeviceProgram prog(wf_test_counting_program(), CountingObj{9, ctr});
    RunResult res = run_sequential(g, QuerySpec::one_per_vertex(), prog);
    EXPECT(wf_test_counter_read(ctr) == res.metrics.total_steps);
    EXPECT(res.metrics.total_steps == 3 * 8);
    wf_test_counter_free(ctr);
}
void sink_mode_streams_the_same_records_the_walk_set_would_hold() {  // :210
    Graph g = skewed_graph(120, 350, 3);
    ExecOptions plain;
    plain.threads = 3;
    plain.seed = 17;
    RunResult expected = run_sequential(g, QuerySpec::one_per_vertex(), PprProgram(0.3), plain);
    std::map<uint32_t, WalkSet> blocks;
    std::mutex mu;
    ExecOptions streamed = plain;
    streamed.sink = [&](uint32_t worker, WalkSet&& block) {
        std::lock_guard lock(mu);
        blocks[worker] = std::move(block);
    };
    RunResult res = run_sequential(g, QuerySpec::one_per_vertex(), PprProgram(0.3), streamed);
    EXPECT(res.walks.empty());
    EXPECT(blocks.size() == 3);
    WalkSet merged;
    for (auto& [worker, block] : blocks)
        for (WalkRecord& r : block) merged.push_back(std::move(r));
    EXPECT(merged == expected.walks);
}
void query_specs_validate_their_sources() {  // :236
    Graph g = triangle();
    EXPECT_THROWS(run_sequential(g, QuerySpec::from_source(9, 5), PprProgram(0.2)), ConfigError);
    EXPECT(QuerySpec::one_per_vertex().total(g) == 3);
    EXPECT(QuerySpec::from_source(0, 42).total(g) == 42);
}
void doubling_the_step_count_does_not_blow_past_linear_scaling() {  // :244
    Graph g = skewed_graph(400, 2000, 6);
    QuerySpec spec = QuerySpec::from_source(0, 3000);
    bool ok = false;
    for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
        auto time_for = [&](uint32_t length) {
            RunResult res = run_sequential(g, spec, DeepWalkProgram(g, length, false));
            return res.metrics.exec_seconds;
        };
        time_for(11);
        const double t1 = time_for(11), t2 = time_for(21);
        ok = t2 <= 2.5 * t1 + 1e-4;
    }
    EXPECT(ok);
}

// ---- suite "interleave" (test_interleave.cpp) ------------------------------------------------
Graph matrix_graph() {
    static Graph g = skewed_graph(160, 700, 11, true, 4);
    return g;
}
template <typename P>
void check_equivalence(const Graph& g, const P& prog, SamplerKind kind, bool use_tables = true) {  // :23
    ExecOptions opts;
    opts.sampler = kind;
    opts.seed = 99;
    opts.use_static_tables = use_tables;
    QuerySpec spec = QuerySpec::one_per_vertex();
    RunResult base = run_sequential(g, spec, prog, opts);
    EXPECT(base.metrics.max_in_flight == 1);  // engine.hpp:502
    for (uint32_t k : {1u, 3u, 8u, 64u}) {
        for (uint32_t k_prime : {1u, std::max(1u, k / 2), k}) {
            RunResult inter = run_interleaved(g, spec, prog, k, k_prime, opts);
            EXPECT(inter.walks == base.walks);
            EXPECT(inter.metrics.total_steps == base.metrics.total_steps);
            EXPECT(inter.metrics.max_in_flight <= k);
            EXPECT(inter.metrics.max_in_flight >= 1);
        }
    }
}
void interleaved_execution_replays_the_sequential_run_exactly() {  // :48
    Graph g = matrix_graph();
    {  // unbiased walks
        PprProgram ppr(0.25);
        for (SamplerKind kind : {SamplerKind::Naive, SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej,
                                 SamplerKind::ORej})
            check_equivalence(g, ppr, kind);
    }
    {  // statically weighted walks through tables
        DeepWalkProgram dw(g, 14, true);
        for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej, SamplerKind::ORej})
            check_equivalence(g, dw, kind);
    }
    {  // statically weighted walks gathered per step
        DeepWalkProgram dw(g, 14, true);
        for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej})
            check_equivalence(g, dw, kind, /*use_tables=*/false);
    }
    {  // dynamically weighted walks
        Node2VecProgram n2v(g, {.a = 2.0, .b = 0.5, .target_length = 12}, true);
        for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej, SamplerKind::ORej})
            check_equivalence(g, n2v, kind);
    }
    {  // label-constrained walks
        MetaPathProgram mp(g, {0, 1, 2, 1});
        for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej})
            check_equivalence(g, mp, kind);
    }
}
void multi_threaded_interleaving_matches_as_well() {  // :91
    Graph g = matrix_graph();
    DeepWalkProgram dw(g, 14, true);
    ExecOptions opts;
    opts.seed = 5;
    RunResult base = run_sequential(g, QuerySpec::one_per_vertex(), dw, opts);
    ExecOptions threaded = opts;
    threaded.threads = 4;
    RunResult inter = run_interleaved(g, QuerySpec::one_per_vertex(), dw, 16, 8, threaded);
    EXPECT(inter.walks == base.walks);
    EXPECT(inter.metrics.max_in_flight <= 16);
}
void ring_sizes_are_validated() {  // :104
    Graph g = triangle();
    PprProgram ppr(0.5);
    QuerySpec spec = QuerySpec::one_per_vertex();
    EXPECT_THROWS(run_interleaved(g, spec, ppr, 0, 1), ConfigError);
    EXPECT_THROWS(run_interleaved(g, spec, ppr, 4, 0), ConfigError);
    EXPECT_THROWS(run_interleaved(g, spec, ppr, 4, 8), ConfigError);
    RunResult ok = run_interleaved(g, spec, ppr, 4, 4);
    EXPECT(ok.walks.size() == 3);
}
void rings_larger_than_the_query_set_stay_correct() {  // :114
    Graph g = triangle();
    DeepWalkProgram dw(g, 6, false);
    RunResult base = run_sequential(g, QuerySpec::one_per_vertex(), dw);
    RunResult inter = run_interleaved(g, QuerySpec::one_per_vertex(), dw, 256, 128);
    EXPECT(inter.walks == base.walks);
    EXPECT(inter.metrics.max_in_flight <= 3);
}
void prefetch_level_does_not_change_results() {  // :123
    Graph g = matrix_graph();
    DeepWalkProgram dw(g, 10, true);
    std::optional<RunResult> previous;
    for (PrefetchLevel level : {PrefetchLevel::L1, PrefetchLevel::L3, PrefetchLevel::Off}) {
        ExecOptions opts;
        opts.seed = 44;
        opts.prefetch = level;
        RunResult res = run_interleaved(g, QuerySpec::one_per_vertex(), dw, 32, 16, opts);
        if (previous) EXPECT(res.walks == previous->walks);
        previous = std::move(res);
    }
}
void walks_of_target_length_one_bypass_the_rings() {  // :139
    Graph g = triangle();
    DeepWalkProgram dw(g, 1, false);
    RunResult res = run_interleaved(g, QuerySpec::one_per_vertex(), dw, 8, 4);
    EXPECT(res.walks.size() == 3);
    for (const WalkRecord& r : res.walks) {
        EXPECT(r.status == WalkStatus::Complete);
        EXPECT(r.path.size() == 1);
    }
    EXPECT(res.metrics.total_steps == 0);
    EXPECT(res.metrics.max_in_flight == 0);
}
void rejection_trial_caps_propagate() {  // :152
    // the walker circles vertex 0, where one edge sits far below the vertex
    // envelope: half of all trials reject, so a cap of 2 trips within a few steps
    Graph g = graph_of(2, {{0, 0}, {0, 1}, {1, 1}}, {1.0, 1e-6, 1.0});
    DeepWalkProgram dw(g, 50, true);
    ExecOptions opts;
    opts.sampler = SamplerKind::Rej;
    opts.rej_trial_cap = 2;
    bool threw_somewhere = false;
    for (uint64_t seed = 0; seed < 8 && !threw_somewhere; ++seed) {
        opts.seed = seed;
        try {
            run_interleaved(g, QuerySpec::one_per_vertex(), dw, 4, 2, opts);
        } catch (const RejectionCapError&) {
            threw_somewhere = true;
        }
    }
    EXPECT(threw_somewhere);
}
void sink_mode_emits_ordered_blocks_identical_to_the_walk_set() {  // :173
    Graph g = matrix_graph();
    PprProgram ppr(0.3);
    ExecOptions plain;
    plain.seed = 12;
    RunResult expected = run_interleaved(g, QuerySpec::one_per_vertex(), ppr, 16, 8, plain);
    WalkSet streamed;
    ExecOptions opts = plain;
    opts.sink = [&](uint32_t, WalkSet&& block) {
        for (WalkRecord& r : block) streamed.push_back(std::move(r));
    };
    RunResult res = run_interleaved(g, QuerySpec::one_per_vertex(), ppr, 16, 8, opts);
    EXPECT(res.walks.empty());
    EXPECT(streamed == expected.walks);
}

// ---- suite "algorithms" (test_algorithms.cpp) -------------------------------------------------
Graph ring(uint32_t n) {  // v <-> v+1 (mod n)
    EdgeList e;
    for (uint32_t v = 0; v < n; ++v) {
        e.push_back({v, (v + 1) % n});
        e.push_back({v, (v + n - 1) % n});
    }
    return graph_of(n, e);
}
Graph fan(const std::vector<double>& weights) {  // 0 -> 1..n with the given weights
    EdgeList e;
    for (uint32_t i = 0; i < weights.size(); ++i) e.push_back({0, i + 1});
    return graph_of(static_cast<uint32_t>(weights.size()) + 1, e, weights);
}
bool near(double x, double want, double rel) { return std::fabs(x - want) <= rel * std::fabs(want); }

void restart_walks_stop_geometrically() {  // :14
    Graph g = ring(64);
    {  // probability one stops after the first move
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 500), PprProgram(1.0));
        EXPECT(res.walks.size() == 500);
        for (const WalkRecord& r : res.walks) {
            EXPECT(r.status == WalkStatus::Complete);
            EXPECT(r.path.size() == 2);
        }
    }
    {  // mean step count approaches the geometric expectation
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 20000), PprProgram(0.2));
        EXPECT(near(static_cast<double>(res.metrics.total_steps) / 20000.0, 5.0, 0.03));
    }
    {  // termination probability is validated
        EXPECT_THROWS(PprProgram(0.0), ConfigError);
        EXPECT_THROWS(PprProgram(-0.5), ConfigError);
        EXPECT_THROWS(PprProgram(1.5), ConfigError);
        EXPECT_THROWS(PprProgram(std::nan("")), ConfigError);
    }
}
void fixed_length_walk_weights_follow_the_edge_weights() {  // :40
    {  // target length and weighted mode are validated
        Graph g = triangle();
        EXPECT_THROWS(DeepWalkProgram(g, 0, false), ConfigError);
        EXPECT_THROWS(DeepWalkProgram(g, 10, true), ConfigError);
    }
    {  // first-step frequencies match the weight ratio
        Graph g = fan({1.0, 3.0});
        DeepWalkProgram prog(g, 2, true);
        EXPECT(prog.max_weight() == 3.0);
        for (SamplerKind kind : {SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej}) {
            ExecOptions opts;
            opts.sampler = kind;
            opts.seed = 21;
            RunResult res = run_sequential(g, QuerySpec::from_source(0, 20000), prog, opts);
            uint64_t heavy = 0;
            for (const WalkRecord& r : res.walks) {
                EXPECT(r.path.size() == 2);
                heavy += r.path.size() == 2 && r.path[1] == 2;
            }
            EXPECT(near(static_cast<double>(heavy) / 20000.0, 0.75, 0.02));
        }
    }
    {  // unweighted mode ignores stored weights
        Graph g = fan({1.0, 99.0});
        DeepWalkProgram prog(g, 2, false);
        ExecOptions opts;
        opts.sampler = SamplerKind::Alias;
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 20000), prog, opts);
        uint64_t heavy = 0;
        for (const WalkRecord& r : res.walks) heavy += r.path[1] == 2;
        EXPECT(near(static_cast<double>(heavy) / 20000.0, 0.5, 0.05));
    }
}
// share of the walks [0, 1, y] with y == 2 among those that went 0 -> 1 first
double forward_share(const Graph& g, const Node2VecProgram& prog, SamplerKind kind, uint64_t& seen) {
    ExecOptions opts;
    opts.sampler = kind;
    opts.seed = 77;
    RunResult res = run_sequential(g, QuerySpec::from_source(0, 80000), prog, opts);
    uint64_t via1 = 0, forward = 0;
    for (const WalkRecord& r : res.walks) {
        if (r.path.size() == 3 && r.path[1] == 1) {
            via1 += 1;
            forward += r.path[2] == 2;
        }
    }
    seen = via1;
    return via1 ? static_cast<double>(forward) / static_cast<double>(via1) : 0.0;
}
void second_order_walk_weights_depend_on_the_previous_vertex() {  // :80
    // out of vertex 1 with the walk at [0, 1]: back to 0 scores 1/a = 0.5, on to
    // 2 (adjoins 0) 1, on to 3 (does not) 1/b = 2 -> 1/7, 2/7, 4/7
    Graph g = graph_of(4, {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {1, 3}});
    Node2VecProgram prog(g, {.a = 2.0, .b = 0.5, .target_length = 3}, false);
    for (SamplerKind kind : {SamplerKind::ORej, SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej}) {
        ExecOptions opts;
        opts.sampler = kind;
        opts.seed = 9;
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 80000), prog, opts);
        uint64_t via1 = 0, to[4] = {0, 0, 0, 0};
        for (const WalkRecord& r : res.walks)
            if (r.path.size() == 3 && r.path[1] == 1) {
                via1 += 1;
                to[r.path[2]] += 1;
            }
        EXPECT(via1 > 30000);  // the first move scores every edge at the shared maximum: 1/2 each
        EXPECT(near(static_cast<double>(via1) / 80000.0, 0.5, 0.03));
        EXPECT(near(static_cast<double>(to[0]) / via1, 1.0 / 7.0, 0.05));
        EXPECT(near(static_cast<double>(to[2]) / via1, 2.0 / 7.0, 0.04));
        EXPECT(near(static_cast<double>(to[3]) / via1, 4.0 / 7.0, 0.03));
    }
    EXPECT(prog.max_weight() == 2.0);  // the weight bound covers every reachable weight
    // parameters are validated
    EXPECT_THROWS(Node2VecProgram(g, {.a = 0.0, .b = 0.5}, false), ConfigError);
    EXPECT_THROWS(Node2VecProgram(g, {.a = 2.0, .b = -1.0}, false), ConfigError);
    EXPECT_THROWS(Node2VecProgram(g, {.a = std::numeric_limits<double>::infinity(), .b = 1.0}, false), ConfigError);
    EXPECT_THROWS(Node2VecProgram(g, {.target_length = 0}, false), ConfigError);
    EXPECT_THROWS(Node2VecProgram(g, {}, true), ConfigError);
}
void second_order_transitions_match_the_hand_computed_distribution() {  // :117
    // undirected triangle: from [0, 1] back to 0 (1/a = 0.5) or on to 2, a neighbor of 0 (1) -> 1/3 vs 2/3
    Graph g = graph_of(3, {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}});
    Node2VecProgram prog(g, {.a = 2.0, .b = 0.5, .target_length = 3}, false);
    for (SamplerKind kind : {SamplerKind::ORej, SamplerKind::Its}) {
        uint64_t seen = 0;
        const double share = forward_share(g, prog, kind, seen);
        EXPECT(seen > 30000);
        EXPECT(near(share, 2.0 / 3.0, 0.02));
    }
}
void weighted_second_order_walks_scale_by_the_edge_weight() {  // :145
    Graph g = graph_of(3, {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}}, {1.0, 1.0, 2.0, 4.0, 1.0, 1.0});
    Node2VecProgram prog(g, {.a = 2.0, .b = 0.5, .target_length = 3}, true);
    EXPECT(prog.max_weight() == 2.0 * 4.0);
    // from [0, 1]: back to 0 scores 0.5 * 2, on to 2 scores 1 * 4 -> 1/5 vs 4/5
    for (SamplerKind kind : {SamplerKind::ORej, SamplerKind::Its, SamplerKind::Alias}) {
        uint64_t seen = 0;
        const double share = forward_share(g, prog, kind, seen);
        EXPECT(seen > 30000);
        EXPECT(near(share, 0.8, 0.02));
    }
}
void label_constrained_walks_obey_the_schema() {  // :157
    Graph g = graph_of(4, {{0, 1}, {0, 2}, {1, 2}, {2, 3}, {3, 0}}, {}, {0, 1, 1, 2, 0});
    {  // a fully matching path completes
        MetaPathProgram prog(g, {0, 1, 2});
        RunResult res = run_sequential(g, QuerySpec::from_source(0, 50), prog);
        EXPECT(res.walks.size() == 50);
        for (const WalkRecord& r : res.walks) {
            EXPECT(r.status == WalkStatus::Complete);
            EXPECT((r.path == std::vector<VertexId>{0, 1, 2, 3}));
        }
    }
    {  // a vertex with no edge of the wanted label dead-ends
        MetaPathProgram prog(g, {0, 1, 2});
        RunResult res = run_sequential(g, QuerySpec::from_source(1, 50), prog);
        for (const WalkRecord& r : res.walks) {
            EXPECT(r.status == WalkStatus::DeadEnd);
            EXPECT((r.path == std::vector<VertexId>{1}));
        }
    }
    {  // construction is validated
        EXPECT_THROWS(MetaPathProgram(g, {}), ConfigError);
        EXPECT_THROWS(MetaPathProgram(g, {0, 9}), ConfigError);
        Graph bare = triangle();
        EXPECT_THROWS(MetaPathProgram(bare, {0}), ConfigError);
    }
    {  // the unknown label is named in the error
        bool named = false;
        try {
            MetaPathProgram prog(g, {0, 7, 2});
        } catch (const ConfigError& e) {
            named = std::string(e.what()).find('7') != std::string::npos;
        }
        EXPECT(named);
    }
}
void uniform_fixed_length_walks_need_no_weights_at_all() {  // :196
    Graph g = triangle();
    UniformProgram prog(5);
    RunResult res = run_sequential(g, QuerySpec::one_per_vertex(), prog);
    EXPECT(res.walks.size() == 3);
    for (const WalkRecord& r : res.walks) EXPECT(r.path.size() == 5);
    EXPECT_THROWS(UniformProgram(0), ConfigError);
}
void each_program_lands_on_its_expected_default_sampling_method() {  // :206
    Graph g = graph_of(4, {{0, 1}, {0, 2}, {1, 2}, {2, 3}, {3, 0}}, {}, {0, 1, 1, 2, 0});
    EXPECT(resolve_default_sampler(PprProgram(0.2)) == SamplerKind::Naive);
    EXPECT(resolve_default_sampler(DeepWalkProgram(g, 5, false)) == SamplerKind::Alias);
    EXPECT(resolve_default_sampler(Node2VecProgram(g, {}, false)) == SamplerKind::ORej);
    EXPECT(resolve_default_sampler(MetaPathProgram(g, {0, 1})) == SamplerKind::Its);
    EXPECT(resolve_default_sampler(UniformProgram(3)) == SamplerKind::Naive);
    // the names the reference CLI prints and parses (sampler.cpp:7-26, prefetch.hpp:30-48)
    for (SamplerKind k : {SamplerKind::Naive, SamplerKind::Its, SamplerKind::Alias, SamplerKind::Rej, SamplerKind::ORej})
        EXPECT(parse_sampler(to_string(k)) == k);
    EXPECT(parse_sampler("o-rej") == SamplerKind::ORej);
    EXPECT_THROWS(parse_sampler("fastest"), ConfigError);
    EXPECT(parse_prefetch_level("nta") == PrefetchLevel::NonTemporal);
    EXPECT_THROWS(parse_prefetch_level("l9"), ConfigError);
    EXPECT(std::string(to_string(WalkStatus::DeadEnd)) == "dead_end");
    EXPECT(std::string(to_string(WalkerType::Dynamic)) == "dynamic");
    EXPECT(ExecOptions{}.rej_trial_cap == kRejTrialCap);
}

// ---- suite "graph" (test_graph.cpp) ---------------------------------------------------------
std::string g_tmp;  // scratch directory (argv[1])
std::string tmp_file(const std::string& name) { return g_tmp + "/" + name; }
void write_file(const std::string& path, const std::string& bytes) {
    std::ofstream(path, std::ios::binary) << bytes;
}
std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}
Graph star(uint32_t leaves) {  // hub 0 connected both ways to leaves 1..n
    EdgeList e;
    for (uint32_t v = 1; v <= leaves; ++v) {
        e.push_back({0, v});
        e.push_back({v, 0});
    }
    return graph_of(leaves + 1, e);
}

void csr_assembly_sorts_adjacency_and_keeps_attributes_aligned() {  // :19
    Graph g = build_graph(3, {{1, 2}, {0, 2}, {0, 1}, {2, 0}}, {12.0, 2.0, 1.0, 20.0});
    EXPECT(g.vertex_count() == 3);
    EXPECT(g.edge_count() == 4);
    EXPECT(g.degree(0) == 2);
    EXPECT(g.neighbors(0)[0] == 1);
    EXPECT(g.neighbors(0)[1] == 2);
    EXPECT(g.weight(g.edge_begin(0)) == 1.0);
    EXPECT(g.weight(g.edge_begin(0) + 1) == 2.0);
    EXPECT(g.weight(g.edge_begin(1)) == 12.0);
    EXPECT(g.weight(g.edge_begin(2)) == 20.0);
    EXPECT(g.adjacency_sorted());
}
void edge_existence_via_binary_search() {  // :36
    Graph g = star(5);
    EXPECT(g.has_edge(0, 3));
    EXPECT(g.has_edge(3, 0));
    EXPECT(!g.has_edge(1, 2));
    EXPECT(!g.has_edge(2, 2));
}
void degree_zero_vertices_are_just_dead_ends_not_errors() {  // :44
    Graph g = line(4);
    EXPECT(g.degree(3) == 0);
    EXPECT(g.neighbors(3).empty());
}
void from_csr_validates_structure() {  // :50
    EXPECT_THROWS(Graph::from_csr({0}, {}), ConfigError);                   // zero vertices
    EXPECT_THROWS(Graph::from_csr({0, 2}, {0}), ConfigError);               // framing
    EXPECT_THROWS(Graph::from_csr({0, 2, 1}, {0, 0}), ConfigError);         // non-monotone
    EXPECT_THROWS(Graph::from_csr({0, 1}, {5}), ConfigError);               // id range
    EXPECT_THROWS(Graph::from_csr({0, 1}, {0}, {-1.0}), ConfigError);       // negative weight
    EXPECT_THROWS(Graph::from_csr({0, 1}, {0}, {1.0, 2.0}), ConfigError);   // length
    EXPECT_THROWS(Graph::from_csr({0, 1}, {0}, {}, {1, 2}), ConfigError);   // labels length
}
void binary_files_round_trip_bit_exactly() {  // :60
    Graph g = build_graph(4, {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {0, 2}}, {1.0, 2.5, 3.25, 4.125, 0.5},
                          {0, 1, 2, 3, 4});
    const std::string a = tmp_file("a.wfg"), b = tmp_file("b.wfg");
    g.write_binary(a);
    Graph loaded = Graph::read_binary(a);
    loaded.write_binary(b);
    EXPECT(read_file(a) == read_file(b));
    EXPECT(!read_file(a).empty());
    EXPECT(loaded.vertex_count() == 4);
    EXPECT(loaded.edge_count() == 5);
    EXPECT(loaded.weight(1) == g.weight(1));
    EXPECT(loaded.label(4) == g.label(4));
}
void binary_reader_rejects_corruption() {  // :76
    Graph g = triangle();
    const std::string path = tmp_file("g.wfg");
    g.write_binary(path);
    const std::string bytes = read_file(path);
    std::string bad_magic = bytes;
    bad_magic[0] = 'X';
    write_file(tmp_file("magic.wfg"), bad_magic);
    EXPECT_THROWS(Graph::read_binary(tmp_file("magic.wfg")), FormatError);
    write_file(tmp_file("trunc.wfg"), bytes.substr(0, bytes.size() - 3));
    EXPECT_THROWS(Graph::read_binary(tmp_file("trunc.wfg")), FormatError);
    write_file(tmp_file("trail.wfg"), bytes + "xx");
    EXPECT_THROWS(Graph::read_binary(tmp_file("trail.wfg")), FormatError);
    EXPECT_THROWS(Graph::read_binary(tmp_file("missing.wfg")), IoError);
}
void edge_list_loader_handles_comments_blanks_and_weights() {  // :97
    const std::string path = tmp_file("edges.txt");
    write_file(path, "# comment line\n0 1 2.5\n\n1 2 0.5\n2 0 1.5\n");
    EdgeListOptions options;
    options.weights = WeightMode::FromFile;
    LoadedGraph loaded = load_edge_list(path, options);
    EXPECT(loaded.graph.vertex_count() == 3);
    EXPECT(loaded.graph.edge_count() == 3);
    EXPECT(loaded.graph.has_weights());
    EXPECT(loaded.graph.weight(loaded.graph.edge_begin(0)) == 2.5);
}
void edge_list_loader_reports_the_offending_line() {  // :115
    const std::string path = tmp_file("bad.txt");
    write_file(path, "0 1\nnonsense here\n");
    bool named = false;
    try {
        load_edge_list(path);
    } catch (const ParseError& e) {
        named = std::string(e.what()).find(":2") != std::string::npos;
    }
    EXPECT(named);
    write_file(path, "0 1 1.0 2 9\n");
    EXPECT_THROWS(load_edge_list(path), ParseError);
    write_file(path, "# only comments\n");
    EXPECT_THROWS(load_edge_list(path), ParseError);
    write_file(path, "0 1\n");
    EdgeListOptions needs_weights;
    needs_weights.weights = WeightMode::FromFile;
    EXPECT_THROWS(load_edge_list(path, needs_weights), ParseError);
}
void sparse_ids_are_remapped_densely_in_ascending_order() {  // :138
    const std::string path = tmp_file("sparse.txt");
    write_file(path, "100 7\n7 42\n42 100\n");
    LoadedGraph loaded = load_edge_list(path);
    EXPECT(loaded.graph.vertex_count() == 3);
    EXPECT(loaded.original_ids.size() == 3);
    if (loaded.original_ids.size() == 3) {
        EXPECT(loaded.original_ids[0] == 7);
        EXPECT(loaded.original_ids[1] == 42);
        EXPECT(loaded.original_ids[2] == 100);
    }
    EXPECT(scan_edge(loaded.graph, 2, 0));  // 100 -> 7 becomes 2 -> 0
}
void undirected_mode_emits_both_directions() {  // :152
    const std::string path = tmp_file("undirected.txt");
    write_file(path, "0 1\n1 2\n");
    EdgeListOptions options;
    options.directedness = Directedness::Undirected;
    LoadedGraph loaded = load_edge_list(path, options);
    EXPECT(loaded.graph.edge_count() == 4);
    EXPECT(scan_edge(loaded.graph, 1, 0));
    EXPECT(scan_edge(loaded.graph, 2, 1));
}
void random_attributes_are_a_pure_function_of_the_seed() {  // :164
    const std::string path = tmp_file("edges3.txt");
    write_file(path, "0 1\n1 2\n2 0\n");
    EdgeListOptions options;
    options.weights = WeightMode::Random;
    options.labels = LabelMode::Random;
    options.label_count = 3;
    options.seed = 99;
    LoadedGraph first = load_edge_list(path, options);
    LoadedGraph second = load_edge_list(path, options);
    const std::string a = tmp_file("ra.wfg"), b = tmp_file("rb.wfg");
    first.graph.write_binary(a);
    second.graph.write_binary(b);
    EXPECT(read_file(a) == read_file(b));
    for (uint64_t e = 0; e < first.graph.edge_count(); ++e) {
        const double w = first.graph.weight(e);
        EXPECT(w >= 1.0);
        EXPECT(w < 5.0);
        EXPECT(first.graph.label(e) < 3);
    }
}
void attribute_access_on_a_bare_graph_is_refused() {  // :190
    Graph g = triangle();
    EXPECT(!g.has_weights());
    EXPECT_THROWS(g.weight(0), ConfigError);
    EXPECT_THROWS(g.label(0), ConfigError);
}
}  // namespace

int main(int argc, char** argv) {
    g_tmp = argc > 1 ? argv[1] : "/tmp";
    const std::vector<std::pair<const char*, std::function<void()>>> cases = {
        {"engine: fixed-length walks hit their target exactly", fixed_length_walks_hit_their_target_exactly},
        {"engine: target length one completes without a single move",
         target_length_one_completes_without_a_single_move},
        {"engine: dead ends emit the partial path with the right status",
         dead_ends_emit_the_partial_path_with_the_right_status},
        {"engine: results are invariant to thread count", results_are_invariant_to_thread_count},
        {"engine: static tables and per-step gather agree for every table sampler",
         static_tables_and_per_step_gather_agree_for_every_table_sampler},
        {"engine: unbiased programs run under every sampling method identically in law",
         unbiased_programs_run_under_every_sampling_method_identically_in_law},
        {"engine: illegal pairings are refused up front", illegal_pairings_are_refused_up_front},
        {"engine: a program emitting negative weights is caught", a_program_emitting_negative_weights_is_caught},
        {"engine: zero-weight edges are never traversed", zero_weight_edges_are_never_traversed},
        {"engine: vertices whose weights all vanish dead-end their walkers",
         vertices_whose_weights_all_vanish_dead_end_their_walkers},
        {"engine: update runs exactly once per completed move", update_runs_exactly_once_per_completed_move},
        {"engine: sink mode streams the same records the walk set would hold",
         sink_mode_streams_the_same_records_the_walk_set_would_hold},
        {"engine: query specs validate their sources", query_specs_validate_their_sources},
        {"engine: doubling the step count does not blow past linear scaling",
         doubling_the_step_count_does_not_blow_past_linear_scaling},
        {"interleave: interleaved execution replays the sequential run exactly",
         interleaved_execution_replays_the_sequential_run_exactly},
        {"interleave: multi-threaded interleaving matches as well", multi_threaded_interleaving_matches_as_well},
        {"interleave: ring sizes are validated", ring_sizes_are_validated},
        {"interleave: rings larger than the query set stay correct", rings_larger_than_the_query_set_stay_correct},
        {"interleave: prefetch level does not change results", prefetch_level_does_not_change_results},
        {"interleave: walks of target length one bypass the rings", walks_of_target_length_one_bypass_the_rings},
        {"interleave: rejection trial caps propagate", rejection_trial_caps_propagate},
        {"interleave: sink mode emits ordered blocks identical to the walk set",
         sink_mode_emits_ordered_blocks_identical_to_the_walk_set},
        {"algorithms: restart walks stop geometrically", restart_walks_stop_geometrically},
        {"algorithms: fixed-length walk weights follow the edge weights",
         fixed_length_walk_weights_follow_the_edge_weights},
        {"algorithms: second-order walk weights depend on the previous vertex",
         second_order_walk_weights_depend_on_the_previous_vertex},
        {"algorithms: second-order transitions match the hand-computed distribution",
         second_order_transitions_match_the_hand_computed_distribution},
        {"algorithms: weighted second-order walks scale by the edge weight",
         weighted_second_order_walks_scale_by_the_edge_weight},
        {"algorithms: label-constrained walks obey the schema", label_constrained_walks_obey_the_schema},
        {"algorithms: uniform fixed-length walks need no weights at all",
         uniform_fixed_length_walks_need_no_weights_at_all},
        {"algorithms: each program lands on its expected default sampling method",
         each_program_lands_on_its_expected_default_sampling_method},
        {"graph: csr assembly sorts adjacency and keeps attributes aligned",
         csr_assembly_sorts_adjacency_and_keeps_attributes_aligned},
        {"graph: edge existence via binary search", edge_existence_via_binary_search},
        {"graph: degree-zero vertices are just dead ends, not errors",
         degree_zero_vertices_are_just_dead_ends_not_errors},
        {"graph: from_csr validates structure", from_csr_validates_structure},
        {"graph: binary files round-trip bit-exactly", binary_files_round_trip_bit_exactly},
        {"graph: binary reader rejects corruption", binary_reader_rejects_corruption},
        {"graph: edge list loader handles comments, blanks, and weights",
         edge_list_loader_handles_comments_blanks_and_weights},
        {"graph: edge list loader reports the offending line", edge_list_loader_reports_the_offending_line},
        {"graph: sparse ids are remapped densely in ascending order",
         sparse_ids_are_remapped_densely_in_ascending_order},
        {"graph: undirected mode emits both directions", undirected_mode_emits_both_directions},
        {"graph: random attributes are a pure function of the seed",
         random_attributes_are_a_pure_function_of_the_seed},
        {"graph: attribute access on a bare graph is refused", attribute_access_on_a_bare_graph_is_refused},
    };
    return run_cases(cases);
}
