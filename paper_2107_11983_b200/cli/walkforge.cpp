// walkforge_b200 — the reference CLI's front-end (proj/tools/walkforge.cpp)
// over the B200 engine.  Same subcommands, flags, defaults and stdout lines:
//
//   walkforge_b200 convert <edge-list> <out.wfg> [--undirected] [--weights none|file|random]
//                  [--labels none|file|random] [--label-count N] [--seed S]
//   walkforge_b200 run <graph> [-o out] [--algorithm ppr|deepwalk|node2vec|metapath|custom-uniform]
//                  [--sampler naive|its|alias|rej|orej] [--interleave on|off] [-k N] [--k-prime N]
//                  [--threads N] [--seed S] [--termination P] [--length L] [-a A] [-b B]
//                  [--schema l,l,..] [--weighted] [--queries one-per-vertex|source:<v>:<n>|file:<path>]
//                  [--prefetch l1|l2|l3|nta|off] [--binary-output] [--buffer-bytes N]
//                  [--no-static-tables]
//   walkforge_b200 tune <graph> [--threads N] [--budget S] [--seed S]
//
// `run` writes the same records (text or binary, qid order) as the reference's
// DoubleBufferedWriter; `--threads`, `-k`, `--k-prime` and `--prefetch` are
// accepted for compatibility (lanes replace worker threads and rings).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "walkforge_b200.h"

namespace {

struct CliError : std::runtime_error {
    int code;
    CliError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(int rc) {
    if (rc != WF_OK) throw CliError(rc, wf_last_error());
}

[[noreturn]] void usage_error(const std::string& m) { throw CliError(WF_ERR_CONFIG, m); }

bool parse_u64(const std::string& s, uint64_t& out) {
    if (s.empty()) return false;
    uint64_t v = 0;
    for (char c : s) {
        if (c < '0' || c > '9') return false;
        v = v * 10 + static_cast<uint64_t>(c - '0');
    }
    out = v;
    return true;
}

using GraphPtr = std::unique_ptr<wf_graph, void (*)(wf_graph*)>;

bool is_wfg_file(const std::string& path) {  // walkforge.cpp:20-28
    std::ifstream in(path, std::ios::binary);
    if (!in) throw CliError(WF_ERR_IO, "cannot open graph file " + path);
    char magic[4] = {};
    in.read(magic, 4);
    return in.gcount() == 4 && std::memcmp(magic, "WFG1", 4) == 0;
}

GraphPtr load_graph(const std::string& path) {  // walkforge.cpp:32-37
    wf_graph* g = nullptr;
    if (is_wfg_file(path)) {
        check(wf_graph_read_wfg1(path.c_str(), 0, &g));
    } else {
        wf_edge_list_options o{};
        check(wf_graph_load_edge_list(path.c_str(), &o, 0, &g));
    }
    return GraphPtr(g, wf_graph_destroy);
}

// QuerySpec::from_file (walker.cpp:22-78): `vertex [count]` lines, '#' comments
std::vector<uint32_t> read_query_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw CliError(WF_ERR_INVALID_ARG, "cannot open query file '" + path + "'");
    std::vector<uint32_t> out;
    std::string line;
    uint64_t line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        if (auto h = line.find('#'); h != std::string::npos) line.resize(h);
        std::vector<std::string> tok;
        size_t p = 0;
        while (p < line.size()) {
            while (p < line.size() && std::isspace(static_cast<unsigned char>(line[p]))) ++p;
            size_t s = p;
            while (p < line.size() && !std::isspace(static_cast<unsigned char>(line[p]))) ++p;
            if (p > s) tok.push_back(line.substr(s, p - s));
        }
        if (tok.empty()) continue;
        if (tok.size() > 2) throw CliError(WF_ERR_PARSE, path + ":" + std::to_string(line_no) + ": too many columns");
        uint64_t v = 0, c = 1;
        if (!parse_u64(tok[0], v) || (tok.size() == 2 && !parse_u64(tok[1], c)))
            throw CliError(WF_ERR_PARSE, path + ":" + std::to_string(line_no) + ": expected `vertex [count]`");
        if (v > UINT32_MAX) throw CliError(WF_ERR_PARSE, path + ":" + std::to_string(line_no) + ": vertex id out of range");
        for (uint64_t i = 0; i < c; ++i) out.push_back(static_cast<uint32_t>(v));
    }
    if (out.empty()) throw CliError(WF_ERR_PARSE, path + ": no queries");
    return out;
}

struct Args {
    std::vector<std::string> pos;
    std::vector<std::pair<std::string, std::string>> opt;
    std::vector<std::string> flags;
};

Args parse(int argc, char** argv, int start, const std::vector<std::string>& flag_names) {
    Args a;
    for (int i = start; i < argc; ++i) {
        std::string s = argv[i];
        if (s.size() > 1 && s[0] == '-' && !(s.size() > 1 && std::isdigit(static_cast<unsigned char>(s[1])))) {
            bool is_flag = false;
            for (const auto& f : flag_names) is_flag |= f == s;
            if (is_flag) {
                a.flags.push_back(s);
            } else {
                if (i + 1 >= argc) usage_error(s + " requires a value");
                a.opt.emplace_back(s, argv[++i]);
            }
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

std::string get(const Args& a, std::initializer_list<const char*> names, const std::string& def) {
    std::string v = def;
    for (const auto& [k, val] : a.opt)
        for (const char* n : names)
            if (k == n) v = val;
    return v;
}

bool has(const Args& a, const char* f) {
    for (const auto& x : a.flags)
        if (x == f) return true;
    return false;
}

uint64_t get_u64(const Args& a, std::initializer_list<const char*> names, uint64_t def) {
    std::string s = get(a, names, "");
    if (s.empty()) return def;
    uint64_t v;
    if (!parse_u64(s, v)) usage_error("bad integer '" + s + "'");
    return v;
}

double get_f64(const Args& a, std::initializer_list<const char*> names, double def) {
    std::string s = get(a, names, "");
    return s.empty() ? def : std::stod(s);
}

int attr_mode(const std::string& s) {
    if (s == "none") return WF_ATTR_NONE;
    if (s == "file") return WF_ATTR_FROM_FILE;
    if (s == "random") return WF_ATTR_RANDOM;
    usage_error("attribute mode must be none|file|random");
}

int cmd_convert(const Args& a) {  // walkforge.cpp:128-152
    if (a.pos.size() != 2) usage_error("convert needs <input> <output>");
    wf_edge_list_options o{};
    o.undirected = has(a, "--undirected");
    o.weights = attr_mode(get(a, {"--weights"}, "none"));
    o.labels = attr_mode(get(a, {"--labels"}, "none"));
    o.label_count = static_cast<uint32_t>(get_u64(a, {"--label-count"}, 5));
    o.seed = get_u64(a, {"--seed"}, 0);
    wf_graph* g = nullptr;
    check(wf_graph_load_edge_list(a.pos[0].c_str(), &o, 0, &g));
    GraphPtr gp(g, wf_graph_destroy);
    check(wf_graph_write_wfg1(g, a.pos[1].c_str()));
    wf_graph_info i{};
    check(wf_graph_info_get(g, &i));
    std::printf("V=%llu E=%llu d_avg=%.2f d_max=%llu\n", static_cast<unsigned long long>(i.vertex_count),
                static_cast<unsigned long long>(i.edge_count),
                static_cast<double>(i.edge_count) / i.vertex_count,
                static_cast<unsigned long long>(i.max_degree_lo));
    return 0;
}

int cmd_run(const Args& a) {  // walkforge.cpp:154-216
    if (a.pos.size() != 1) usage_error("run needs <graph>");
    GraphPtr g = load_graph(a.pos[0]);
    const std::string algo = get(a, {"--algorithm"}, "deepwalk");
    wf_program_desc d{};
    std::vector<uint32_t> schema;
    d.target_length = static_cast<uint32_t>(get_u64(a, {"--length"}, 80));
    d.weighted = has(a, "--weighted");
    if (algo == "ppr") {
        d.kind = WF_PROGRAM_PPR;
        d.termination = get_f64(a, {"--termination"}, 0.2);
    } else if (algo == "deepwalk") {
        d.kind = WF_PROGRAM_DEEPWALK;
    } else if (algo == "node2vec") {
        d.kind = WF_PROGRAM_NODE2VEC;
        d.a = get_f64(a, {"-a"}, 2.0);
        d.b = get_f64(a, {"-b"}, 0.5);
    } else if (algo == "metapath") {
        d.kind = WF_PROGRAM_METAPATH;
        std::string text = get(a, {"--schema"}, "");
        if (text.empty()) usage_error("--schema is required for metapath (comma-separated label ids)");
        size_t pos = 0;
        while (true) {
            size_t c = text.find(',', pos);
            uint64_t l;
            if (!parse_u64(text.substr(pos, c == std::string::npos ? std::string::npos : c - pos), l) || l > UINT32_MAX)
                usage_error("cannot parse schema label in '" + text + "'");
            schema.push_back(static_cast<uint32_t>(l));
            if (c == std::string::npos) break;
            pos = c + 1;
        }
        d.schema = schema.data();
        d.schema_len = static_cast<uint32_t>(schema.size());
    } else if (algo == "custom-uniform") {
        d.kind = WF_PROGRAM_UNIFORM;
    } else {
        usage_error("--algorithm must be ppr|deepwalk|node2vec|metapath|custom-uniform");
    }
    wf_exec_options o{};
    o.seed = get_u64(a, {"--seed"}, 0);
    const std::string smp = get(a, {"--sampler"}, "");
    o.sampler = smp.empty() ? WF_SAMPLER_DEFAULT
                : smp == "naive" ? WF_SAMPLER_NAIVE
                : smp == "its" ? WF_SAMPLER_ITS
                : smp == "alias" ? WF_SAMPLER_ALIAS
                : smp == "rej" ? WF_SAMPLER_REJ
                : smp == "orej" ? WF_SAMPLER_OREJ : -2;
    if (o.sampler == -2) usage_error("--sampler must be naive|its|alias|rej|orej");
    o.use_static_tables = !has(a, "--no-static-tables");
    o.threads = static_cast<uint32_t>(get_u64(a, {"--threads"}, 1));
    if (get(a, {"--interleave"}, "on") == "on") {
        o.k = static_cast<uint32_t>(get_u64(a, {"-k"}, 64));
        o.k_prime = static_cast<uint32_t>(get_u64(a, {"--k-prime"}, 32));
    }
    if (get_u64(a, {"--buffer-bytes"}, 4u << 20) < (1u << 20))
        usage_error("output buffer must be at least 1048576 bytes");
    // queries
    wf_query_spec q{};
    std::vector<uint32_t> sources;
    const std::string qs = get(a, {"--queries"}, "one-per-vertex");
    if (qs == "one-per-vertex") {
        q.mode = WF_QUERY_ONE_PER_VERTEX;
    } else if (qs.rfind("source:", 0) == 0) {
        std::string rest = qs.substr(7);
        size_t c = rest.find(':');
        uint64_t v, n;
        if (c == std::string::npos || !parse_u64(rest.substr(0, c), v) || !parse_u64(rest.substr(c + 1), n) ||
            v > UINT32_MAX)
            usage_error("cannot parse --queries value '" + qs + "'");
        q.mode = WF_QUERY_FROM_SOURCE;
        q.source = static_cast<uint32_t>(v);
        q.count = n;
    } else if (qs.rfind("file:", 0) == 0) {
        sources = read_query_file(qs.substr(5));
        q.mode = WF_QUERY_FROM_LIST;
        q.count = sources.size();
        q.sources = sources.data();
    } else {
        usage_error("--queries must be one-per-vertex, source:<v>:<n>, or file:<path>");
    }
    wf_walkset* ws = nullptr;
    wf_run_metrics m{};
    check(wf_run(g.get(), &d, &q, &o, &ws, &m));
    std::unique_ptr<wf_walkset, void (*)(wf_walkset*)> wsp(ws, wf_walkset_destroy);
    const std::string out = get(a, {"-o", "--output"}, "walks.out");
    check(wf_walkset_write(ws, out.c_str(), has(a, "--binary-output") ? WF_OUTPUT_BINARY : WF_OUTPUT_TEXT,
                           0, 0, nullptr));
    uint64_t n = 0;
    check(wf_walkset_info(ws, &n, nullptr, nullptr));
    double tp = m.exec_seconds > 0 ? static_cast<double>(m.total_steps) / m.exec_seconds : 0.0;
    std::printf("preprocess_seconds %.6f\n", m.preprocess_seconds);
    std::printf("exec_seconds %.6f\n", m.exec_seconds);
    std::printf("total_steps %llu\n", static_cast<unsigned long long>(m.total_steps));
    std::printf("queries %llu\n", static_cast<unsigned long long>(n));
    std::printf("mean_steps_per_query %.4f\n", n ? static_cast<double>(m.total_steps) / n : 0.0);
    std::printf("throughput_steps_per_sec %.1f\n", tp);
    return 0;
}

// tune: the reference sweeps its CPU rings (tune.cpp:46-111) and prints
// TuneReport::to_text (tune.cpp:92-111).  On the device k / k' are launch
// hints — resident walkers replace the rings — so the sweep runs the
// reference's probe (one uniform length-10 walk per vertex, tune.cpp:18-31)
// through the engine at every ring size the reference would try and prints
// the measured throughput in the reference's report format (a caller parsing
// `walkforge tune` keeps working); the flat curve is the finding.  The knob
// that does matter, resident walkers, is tuned by wf_session_tune and
// reported on the last line.
int cmd_tune(const Args& a) {
    if (a.pos.size() != 1) usage_error("tune needs <graph>");
    GraphPtr g = load_graph(a.pos[0]);
    wf_program_desc d{};
    d.kind = WF_PROGRAM_UNIFORM;
    d.target_length = 10;
    wf_exec_options o{};
    o.seed = get_u64(a, {"--seed"}, 0);
    o.sampler = WF_SAMPLER_DEFAULT;
    o.use_static_tables = 1;
    wf_query_spec q{};
    q.mode = WF_QUERY_ONE_PER_VERTEX;
    const double budget = static_cast<double>(get_u64(a, {"--budget"}, 120));
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    bool exhausted = false;
    uint32_t lanes = 0;
    auto probe = [&](uint32_t k, uint32_t k_prime) {
        wf_exec_options ok = o;
        ok.k = k;
        ok.k_prime = k_prime;
        wf_walkset* ws = nullptr;
        wf_run_metrics m{};
        check(wf_run(g.get(), &d, &q, &ok, &ws, &m));  // warm (tables, first launch)
        wf_walkset_destroy(ws);
        check(wf_run(g.get(), &d, &q, &ok, &ws, &m));
        wf_walkset_destroy(ws);
        lanes = m.max_in_flight;
        return m.exec_seconds > 0 ? static_cast<double>(m.total_steps) / m.exec_seconds : 0.0;
    };
    const uint32_t best_k = 64, best_k_prime = 32;  // the reference's defaults: k / k' do not move the device
    std::printf("task ring sweep (device: k is a launch hint, resident walkers replace the rings)\n");
    std::printf("k\tthroughput_steps_per_sec\n");
    for (uint32_t k = 1; k <= 1024 && !exhausted; k *= 2) {
        std::printf("%u\t%.1f\n", k, probe(k, 1));
        exhausted = elapsed() > budget;
    }
    std::printf("search ring sweep at k=%u (device: k' is a launch hint)\n", best_k);
    std::printf("k'\tthroughput_steps_per_sec\n");
    for (uint32_t kp = 1; kp <= best_k && !exhausted; kp *= 2) {
        std::printf("%u\t%.1f\n", kp, probe(best_k, kp));
        exhausted = elapsed() > budget;
    }
    std::printf("recommended k=%u k'=%u\n", best_k, best_k_prime);
    if (exhausted) std::printf("budget exhausted; recommendation is best-so-far\n");
    // the device knob the rings become: resident walkers (blocks/SM), timed
    // over whole launches of the probe (wf_session_tune)
    wf_session* s = nullptr;
    check(wf_session_create(g.get(), &d, &o, &s));
    int32_t blocks = 0;
    double ms = 0.0;
    const int rc = wf_session_tune(s, &q, 0, 0, &blocks, &ms);
    wf_session_destroy(s);
    check(rc);
    std::printf("device launch tuner: %d blocks/SM (%.3f ms per launch of the probe), %u lanes in flight\n", blocks,
                ms, lanes);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: walkforge_b200 convert|run|tune ...\n");
        return 2;
    }
    std::string cmd = argv[1];
    try {
        if (cmd == "convert") return cmd_convert(parse(argc, argv, 2, {"--undirected"}));
        if (cmd == "run")
            return cmd_run(parse(argc, argv, 2, {"--weighted", "--binary-output", "--no-static-tables"}));
        if (cmd == "tune") return cmd_tune(parse(argc, argv, 2, {}));
        std::fprintf(stderr, "unknown subcommand '%s'\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
