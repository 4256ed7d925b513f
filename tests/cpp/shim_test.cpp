// Compiles against the header-only shim (include/walkforge_b200/engine.hpp)
// exactly as a reference caller would (WALKFORGE_B200_DROP_IN: namespace
// walkforge), runs the reference's own call pattern (test_engine.cpp:62-91,
// acceptance.cpp:178-200) and prints FNV-1a digests of the walk sets for
// tests/test_shim_gpu.py to compare with the golden fixtures.
#define WALKFORGE_B200_DROP_IN
#include "walkforge_b200/engine.hpp"
#include "walkforge_b200/output.hpp"

#include <cstdio>
#include <fstream>
#include <map>
#include <mutex>

using namespace walkforge;

// a user's device program, compiled separately (tests/programs/test_programs.cu)
extern "C" const wf_program_ops* wf_test_avoid_vertex_program(void);
extern "C" const wf_program_ops* wf_test_label_stop_program(void);
struct AvoidVertexObj {  // host mirror of AvoidVertexProgram's layout
    uint32_t banned;
    uint32_t length;
};
struct LabelStopObj {  // host mirror of LabelStopProgram's layout
    double stop;
    uint32_t stop_label;
};

static uint64_t fnv(const WalkSet& ws) {
    uint64_t h = 1469598103934665603ULL;
    auto mixin = [&](uint64_t x) {
        for (int i = 0; i < 8; ++i) { h ^= (x >> (8 * i)) & 0xFF; h *= 1099511628211ULL; }
    };
    for (const auto& r : ws) {
        mixin(r.query_id);
        mixin(static_cast<uint64_t>(r.status));
        mixin(r.path.size());
        for (auto v : r.path) mixin(v);
    }
    return h;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ifstream in(argv[1], std::ios::binary);
    uint32_t V;
    uint64_t E;
    in.read(reinterpret_cast<char*>(&V), 4);
    in.read(reinterpret_cast<char*>(&E), 8);
    std::vector<uint64_t> off(V + 1);
    std::vector<uint32_t> nbr(E);
    std::vector<float> w32(E);
    std::vector<uint32_t> lab(E);
    in.read(reinterpret_cast<char*>(off.data()), off.size() * 8);
    in.read(reinterpret_cast<char*>(nbr.data()), E * 4);
    in.read(reinterpret_cast<char*>(w32.data()), E * 4);
    in.read(reinterpret_cast<char*>(lab.data()), E * 4);
    std::vector<double> w(w32.begin(), w32.end());
    Graph g = Graph::from_csr(off, nbr, w, lab);

    ExecOptions eo;
    eo.seed = 7;
    eo.sampler = SamplerKind::Alias;
    RunResult a = run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 20, true), eo);
    std::printf("deepwalk_alias %016llx %llu\n", (unsigned long long)fnv(a.walks),
                (unsigned long long)a.metrics.total_steps);

    ExecOptions n2v;
    n2v.seed = 7;
    n2v.sampler = SamplerKind::ORej;
    RunResult b = run_interleaved(g, QuerySpec::one_per_vertex(),
                                  Node2VecProgram(g, {.a = 2.0, .b = 0.5, .target_length = 20}, true),
                                  64, 32, n2v);
    std::printf("node2vec_orej %016llx %llu\n", (unsigned long long)fnv(b.walks),
                (unsigned long long)b.metrics.total_steps);

    // streaming sink mode, as the CLI drives it (walkforge.cpp:157-175)
    ExecOptions mp;
    mp.seed = 7;
    mp.sampler = SamplerKind::Its;
    std::map<uint32_t, WalkSet> blocks;
    std::mutex mu;
    mp.sink = [&](uint32_t worker, WalkSet&& block) {
        std::lock_guard<std::mutex> lock(mu);
        blocks[worker] = std::move(block);
    };
    RunResult c = run_sequential(g, QuerySpec::one_per_vertex(), MetaPathProgram(g, {0, 1, 2, 3}), mp);
    WalkSet merged;
    for (auto& [k, blk] : blocks) for (auto& r : blk) merged.push_back(std::move(r));
    std::printf("metapath_its %016llx %llu sink_empty=%d\n", (unsigned long long)fnv(merged),
                (unsigned long long)c.metrics.total_steps, (int)c.walks.empty());

    try {
        ExecOptions bad;
        bad.sampler = SamplerKind::Naive;
        run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 5, false), bad);
        std::printf("naive_static no-error\n");
    } catch (const ConfigError&) {
        std::printf("naive_static ConfigError\n");
    }

    // Graph accessors (graph.hpp:27-71) against the CSR this program uploaded,
    // and the WFG1 round trip (graph.cpp:190-277)
    {
        bool ok = g.degree(5) == g.neighbors(5).size() && g.edge_begin(5) + g.degree(5) == g.edge_begin(6) &&
                  g.neighbor(g.edge_begin(5)) == g.neighbors(5)[0] && g.weights_data() != nullptr;
        const std::string wf = std::string(argv[1]) + ".wfg";
        g.write_binary(wf);
        Graph h = Graph::read_binary(wf);
        ok = ok && h.vertex_count() == g.vertex_count() && h.edge_count() == g.edge_count();
        for (uint64_t e = 0; ok && e < g.edge_count(); e += 7)
            ok = h.neighbor(e) == g.neighbor(e) && h.weight(e) == g.weight(e) && h.label(e) == g.label(e);
        std::remove(wf.c_str());
        try {
            g.degree(g.vertex_count());
            ok = false;
        } catch (const ConfigError&) {
        }
        std::printf("graph_accessors %s\n", ok ? "ok" : "mismatch");
    }

    // output.hpp: the reference CLI's writer pattern (BlockSink -> ordered
    // sink -> double-buffered writer), text and binary, from the DeepWalk run
    for (int fmt = 0; fmt < 2; ++fmt) {
        const std::string of = std::string(argv[1]) + (fmt ? ".walks.bin" : ".walks.txt");
        DoubleBufferedWriter w(of, fmt ? OutputFormat::Binary : OutputFormat::Text, kMinOutputBuffer);
        OrderedBlockSink sink(w, 2);
        ExecOptions wo = eo;
        wo.sink = [&](uint32_t, WalkSet&& ws) {
            // split into two worker blocks pushed out of order
            WalkSet first(ws.begin(), ws.begin() + ws.size() / 2), second(ws.begin() + ws.size() / 2, ws.end());
            sink.push(1, std::move(second));
            sink.push(0, std::move(first));
        };
        run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 20, true), wo);
        sink.finish();
        w.finish();
        std::printf("written_%s %s\n", fmt ? "bin" : "txt", of.c_str());
    }
    // the reference CLI's exact pattern with several workers (walkforge.cpp:
    // OrderedBlockSink(writer, threads), sink(w, block) once per worker range)
    {
        const std::string of = std::string(argv[1]) + ".walks4.txt";
        DoubleBufferedWriter w(of, OutputFormat::Text, kMinOutputBuffer);
        ExecOptions wo = eo;
        wo.threads = 5;
        OrderedBlockSink sink(w, wo.threads);
        std::vector<int> calls(wo.threads, 0);
        wo.sink = [&](uint32_t worker, WalkSet&& block) {
            calls.at(worker) += 1;
            sink.push(worker, std::move(block));
        };
        run_sequential(g, QuerySpec::one_per_vertex(), DeepWalkProgram(g, 20, true), wo);
        sink.finish();
        w.finish();
        bool once = true;
        for (int c : calls) once = once && c == 1;
        std::printf("written_txt_workers %s %s\n", of.c_str(), once ? "each_once" : "miscounted");
        // an empty query set still hands every worker its (empty) block
        std::vector<int> empty_calls(3, 0);
        ExecOptions eo3 = eo;
        eo3.threads = 3;
        eo3.sink = [&](uint32_t worker, WalkSet&& block) { empty_calls.at(worker) += block.empty() ? 1 : 100; };
        run_sequential(g, QuerySpec::from_source(0, 0), DeepWalkProgram(g, 20, true), eo3);
        std::printf("empty_workers %d %d %d\n", empty_calls[0], empty_calls[1], empty_calls[2]);
    }
    // PPR with a tiny stop probability: walks of ~10^4 vertices (no host
    // capacity guess; the blocks are sized after their walks ran)
    {
        ExecOptions pe;
        pe.seed = 3;
        RunResult p = run_sequential(g, QuerySpec::from_source(0, 3), PprProgram(1e-4), pe);
        std::printf("ppr_long %016llx %llu %zu\n", (unsigned long long)fnv(p.walks),
                    (unsigned long long)p.metrics.total_steps, p.walks.size());
        // threads -> worker blocks (each once, in order) for an unbounded program
        ExecOptions pt;
        pt.seed = 3;
        pt.threads = 3;
        std::vector<int> order;
        WalkSet merged;
        pt.sink = [&](uint32_t worker, WalkSet&& block) {
            order.push_back(static_cast<int>(worker));
            for (auto& r : block) merged.push_back(std::move(r));
        };
        std::vector<VertexId> src(200);
        for (size_t i = 0; i < src.size(); ++i) src[i] = static_cast<VertexId>((i * 37) % g.vertex_count());
        RunResult pb = run_sequential(g, QuerySpec::from_list(src), PprProgram(0.2), pt);
        std::printf("ppr_workers %016llx %llu order=%d%d%d n=%zu\n", (unsigned long long)fnv(merged),
                    (unsigned long long)pb.metrics.total_steps, order.size() > 0 ? order[0] : -1,
                    order.size() > 1 ? order[1] : -1, order.size() > 2 ? order[2] : -1, order.size());
    }
    // a user's device program through the drop-in entry points
    {
        const uint32_t hub = 0;
        ExecOptions ce;
        ce.seed = 3;
        DeviceProgram avoid(wf_test_avoid_vertex_program(), AvoidVertexObj{hub, 12});
        RunResult a2 = run_sequential(g, QuerySpec::one_per_vertex(), avoid, ce);
        std::printf("custom_avoid %016llx %llu\n", (unsigned long long)fnv(a2.walks),
                    (unsigned long long)a2.metrics.total_steps);
        ExecOptions ls;
        ls.seed = 5;
        DeviceProgram stop(wf_test_label_stop_program(), LabelStopObj{0.1, 4});
        RunResult b2 = run_interleaved(g, QuerySpec::one_per_vertex(), stop, 64, 32, ls);
        std::printf("custom_stop %016llx %llu\n", (unsigned long long)fnv(b2.walks),
                    (unsigned long long)b2.metrics.total_steps);
    }
    try {
        DoubleBufferedWriter bad("/nonexistent_dir/x.txt", OutputFormat::Text);
    } catch (const IoError&) {
        std::printf("writer_open IoError\n");
    }

    {
        TuneReport tr = tune_ring_sizes(g);
        std::printf("tune %u %u %d\n", tr.best_k, tr.best_k_prime,
                    tr.device_blocks_per_sm >= 1 && tr.task_ring.size() == 1 && tr.task_ring[0].steps_per_sec > 0);
    }

    // QuerySpec::from_file (walker.cpp:22-78) — the reference CLI test's file
    {
        const std::string qf = std::string(argv[1]) + ".queries.txt";
        { std::ofstream(qf) << "# sources\n3 2\n7\n"; }
        QuerySpec q = QuerySpec::from_file(qf);
        std::printf("query_file %zu %u %u %u\n", q.sources.size(), q.sources[0], q.sources[1], q.sources[2]);
        { std::ofstream(qf) << "1 2 3\n"; }
        try {
            QuerySpec::from_file(qf);
        } catch (const ParseError& e) {
            std::printf("query_file_error ParseError %s\n", e.what() + qf.size());
        }
        std::remove(qf.c_str());
    }
    return 0;
}
