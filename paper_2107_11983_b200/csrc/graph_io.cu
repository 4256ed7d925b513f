// Graph ingest (SURVEY §8 f, row 2): WFG1 binary files (Graph::write_binary /
// read_binary, proj/src/graph.cpp:190-277) and the text edge-list loader
// (load_edge_list, graph.cpp:307-453) with the CSR assembled on the device:
// dense id remap by a device sort + unique, then a stable radix sort of
// (src, dst) keys carrying the input position, which is exactly
// assemble_csr's "bucket by source, sort by destination, input order breaks
// ties" (graph.cpp:37-102).
#include <cub/cub.cuh>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "runtime.hpp"

namespace wf {

namespace {

constexpr char kMagic[4] = {'W', 'F', 'G', '1'};
constexpr uint8_t kFlagWeights = 1;
constexpr uint8_t kFlagLabels = 2;
constexpr uint64_t kWeightSalt = 0x57464757454947ULL;  // graph.cpp:26
constexpr uint64_t kLabelSalt = 0x5746474C41424CULL;   // graph.cpp:27

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

__global__ void k_lower_bound(const uint64_t* __restrict__ ids, uint64_t nids,
                              const uint64_t* __restrict__ q, uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = q[i], lo = 0, hi = nids;
        while (lo < hi) {
            uint64_t mid = (lo + hi) >> 1;
            if (ids[mid] < x) lo = mid + 1; else hi = mid;
        }
        out[i] = static_cast<uint32_t>(lo);
    }
}

// edge j of the (possibly doubled) list: key = src << 32 | dst, value = j
__global__ void k_edge_keys(const uint32_t* __restrict__ ds, const uint32_t* __restrict__ dd,
                            uint64_t m, int undirected, uint64_t* __restrict__ key,
                            uint64_t* __restrict__ val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t s = ds[i], d = dd[i];
        if (undirected) {
            key[2 * i] = (s << 32) | d;
            val[2 * i] = 2 * i;
            key[2 * i + 1] = (d << 32) | s;
            val[2 * i + 1] = 2 * i + 1;
        } else {
            key[i] = (s << 32) | d;
            val[i] = i;
        }
    }
}

__global__ void k_csr_from_keys(const uint64_t* __restrict__ key, uint64_t E,
                                uint32_t* __restrict__ nbr, unsigned long long* __restrict__ deg) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[e];
        nbr[e] = static_cast<uint32_t>(k);
        atomicAdd(deg + (k >> 32), 1ULL);
    }
}

// attribute of input edge j (undirected: both directions share input line j/2)
template <typename T>
__global__ void k_gather_attr(const T* __restrict__ in, const uint64_t* __restrict__ perm, uint64_t E,
                              int undirected, T* __restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t j = perm[e];
        out[e] = in[undirected ? j / 2 : j];
    }
}

__global__ void k_synthetic_attrs(uint64_t E, uint64_t wmix, uint64_t lmix, double* __restrict__ w,
                                  uint8_t* __restrict__ lab, uint32_t label_count) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (w) {
            Rng r{stream_state(wmix, e)};
            w[e] = 1.0 + r.real(4.0);  // synthetic_weight (graph.cpp:279-283), f64 like the reference
        }
        if (lab) {
            Rng r{stream_state(lmix, e)};
            lab[e] = static_cast<uint8_t>(r.index(label_count));
        }
    }
}

inline int grid_for(uint64_t n, int dev) {
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, sm_count(dev) * 32ull)));
}

// std::from_chars-equivalent strict token parsers (graph.cpp:110-117)
bool parse_u64(const char* b, const char* e, uint64_t& out) {
    if (b == e) return false;
    uint64_t v = 0;
    for (const char* p = b; p < e; ++p) {
        if (*p < '0' || *p > '9') return false;
        uint64_t d = static_cast<uint64_t>(*p - '0');
        if (v > (UINT64_MAX - d) / 10) return false;
        v = v * 10 + d;
    }
    out = v;
    return true;
}

bool parse_f64(const char* b, const char* e, double& out) {
    // from_chars(double) accepts [-]digits[.digits][e[+-]digits] plus inf/nan,
    // no leading '+' or whitespace; strtod is correctly rounded like it.
    if (b == e || *b == '+' || std::isspace(static_cast<unsigned char>(*b))) return false;
    std::string tok(b, e);
    if (tok.size() > 1 && (tok[0] == '0' || (tok[0] == '-' && tok[1] == '0')) &&
        (tok.find('x') != std::string::npos || tok.find('X') != std::string::npos))
        return false;  // no hex floats in from_chars' general format
    char* end = nullptr;
    out = std::strtod(tok.c_str(), &end);
    return end == tok.c_str() + tok.size();
}

}  // namespace

GraphStore* graph_read_wfg1(const char* path, int device) {
    File f(path, "rb");
    if (!f.f) raise(WF_ERR_IO, std::string("cannot open '") + path + "'");
    std::fseek(f.f, 0, SEEK_END);
    const uint64_t file_size = static_cast<uint64_t>(std::ftell(f.f));
    std::fseek(f.f, 0, SEEK_SET);
    char magic[4] = {};
    uint64_t v = 0, e = 0;
    uint8_t flags = 0;
    bool ok = std::fread(magic, 1, 4, f.f) == 4 && std::fread(&v, 8, 1, f.f) == 1 &&
              std::fread(&e, 8, 1, f.f) == 1 && std::fread(&flags, 1, 1, f.f) == 1;
    const std::string p = std::string("'") + path + "'";
    if (!ok || std::memcmp(magic, kMagic, 4) != 0) raise(WF_ERR_FORMAT, p + " is not a WFG1 graph file");
    if (v == 0 || v > UINT32_MAX) raise(WF_ERR_FORMAT, p + " has an invalid vertex count");
    if (flags & ~(kFlagWeights | kFlagLabels)) raise(WF_ERR_FORMAT, p + " has unknown flag bits");
    uint64_t expected = 4 + 8 + 8 + 1 + (v + 1) * 8 + e * 4;
    if (flags & kFlagWeights) expected += e * 8;
    if (flags & kFlagLabels) expected += e * 4;
    if (file_size != expected)
        raise(WF_ERR_FORMAT, p + " is truncated or has trailing bytes (" + std::to_string(file_size) +
                                 " bytes, expected " + std::to_string(expected) + ")");
    std::vector<uint64_t> off(v + 1);
    std::vector<uint32_t> nbr(e);
    std::vector<double> w;
    std::vector<uint32_t> lab;
    ok = std::fread(off.data(), 8, v + 1, f.f) == v + 1 && std::fread(nbr.data(), 4, e, f.f) == e;
    if (ok && (flags & kFlagWeights)) {
        w.resize(e);
        ok = std::fread(w.data(), 8, e, f.f) == e;
    }
    if (ok && (flags & kFlagLabels)) {
        lab.resize(e);
        ok = std::fread(lab.data(), 4, e, f.f) == e;
    }
    if (!ok) raise(WF_ERR_FORMAT, p + " ended unexpectedly");
    try {
        // f64 weights as on disk (graph.cpp:206-208); a separate f64 array is
        // kept only when some weight is not float32-exact
        return graph_from_host_f64(off.data(), nbr.data(), w.empty() ? nullptr : w.data(),
                                   lab.empty() ? nullptr : lab.data(), static_cast<uint32_t>(v), e, device);
    } catch (const Error& err) {
        if (err.code == WF_ERR_CONFIG) raise(WF_ERR_FORMAT, p + " fails validation: " + err.what());
        throw;
    }
}

void graph_write_wfg1(const GraphStore& g, const char* path) {
    DeviceGuard guard(g.device);
    File f(path, "wb");
    if (!f.f) raise(WF_ERR_IO, std::string("cannot open '") + path + "' for writing");
    const uint64_t v = g.V, e = g.E;
    const uint8_t flags = (g.has_weights() ? kFlagWeights : 0) | (g.has_labels() ? kFlagLabels : 0);
    bool ok = std::fwrite(kMagic, 1, 4, f.f) == 4 && std::fwrite(&v, 8, 1, f.f) == 1 &&
              std::fwrite(&e, 8, 1, f.f) == 1 && std::fwrite(&flags, 1, 1, f.f) == 1;
    const uint64_t kChunk = 1ull << 24;
    std::vector<char> buf;
    auto dump = [&](const void* dev, uint64_t count, size_t elem) {
        for (uint64_t i = 0; ok && i < count; i += kChunk) {
            uint64_t c = std::min(kChunk, count - i);
            buf.resize(c * elem);
            WF_CUDA(cudaMemcpy(buf.data(), static_cast<const char*>(dev) + i * elem, c * elem,
                               cudaMemcpyDeviceToHost));
            ok = std::fwrite(buf.data(), 1, c * elem, f.f) == c * elem;
        }
    };
    dump(g.offsets.get(), v + 1, 8);
    dump(g.nbr.get(), e, 4);
    if (g.weights64.get()) {  // f64 on disk (graph.cpp:206-208)
        dump(g.weights64.get(), e, 8);
    } else if (g.has_weights()) {  // the f32 values widened exactly
        std::vector<float> w;
        std::vector<double> w64;
        for (uint64_t i = 0; ok && i < e; i += kChunk) {
            uint64_t c = std::min(kChunk, e - i);
            w.resize(c);
            w64.resize(c);
            WF_CUDA(cudaMemcpy(w.data(), g.weights.get() + i, c * 4, cudaMemcpyDeviceToHost));
            for (uint64_t j = 0; j < c; ++j) w64[j] = w[j];
            ok = std::fwrite(w64.data(), 8, c, f.f) == c;
        }
    }
    if (g.has_labels()) {  // u32 on disk
        std::vector<uint8_t> l;
        std::vector<uint32_t> l32;
        for (uint64_t i = 0; ok && i < e; i += kChunk) {
            uint64_t c = std::min(kChunk, e - i);
            l.resize(c);
            l32.resize(c);
            WF_CUDA(cudaMemcpy(l.data(), g.labels.get() + i, c, cudaMemcpyDeviceToHost));
            for (uint64_t j = 0; j < c; ++j) l32[j] = l[j];
            ok = std::fwrite(l32.data(), 4, c, f.f) == c;
        }
    }
    if (!ok || std::fflush(f.f) != 0) raise(WF_ERR_IO, std::string("write failed for '") + path + "'");
}

GraphStore* graph_load_edge_list(const char* path, const wf_edge_list_options& o, int device,
                                 std::vector<uint64_t>* original_ids) {
    File f(path, "rb");
    if (!f.f) raise(WF_ERR_IO, std::string("cannot open '") + path + "'");
    const bool want_w = o.weights == WF_ATTR_FROM_FILE;
    const bool want_l = o.labels == WF_ATTR_FROM_FILE;
    std::vector<uint64_t> src, dst;
    std::vector<double> fw;
    std::vector<uint32_t> fl;
    auto fail = [&](uint64_t line_no, const std::string& what) {
        raise(WF_ERR_PARSE, std::string(path) + ":" + std::to_string(line_no) + ": " + what);
    };
    // line-by-line parse, graph.cpp:319-378
    std::vector<char> chunk(1 << 22);
    std::string line;
    uint64_t line_no = 0;
    auto handle = [&](std::string& ln) {
        line_no += 1;
        size_t hash = ln.find('#');
        const size_t end = hash == std::string::npos ? ln.size() : hash;
        const char* tb[5];
        const char* te[5];
        int nt = 0;
        size_t pos = 0;
        while (pos < end) {
            while (pos < end && std::isspace(static_cast<unsigned char>(ln[pos]))) ++pos;
            size_t st = pos;
            while (pos < end && !std::isspace(static_cast<unsigned char>(ln[pos]))) ++pos;
            if (pos > st) {
                if (nt < 5) {
                    tb[nt] = ln.data() + st;
                    te[nt] = ln.data() + pos;
                }
                ++nt;
            }
        }
        if (nt == 0) return;
        if (nt < 2) fail(line_no, "expected `src dst [weight [label]]`");
        if (nt > 4) fail(line_no, "too many columns");
        uint64_t s = 0, d = 0;
        if (!parse_u64(tb[0], te[0], s) || !parse_u64(tb[1], te[1], d))
            fail(line_no, "vertex ids must be non-negative integers");
        if (want_w) {
            if (nt < 3) fail(line_no, "weight column missing");
            double w = 0.0;
            if (!parse_f64(tb[2], te[2], w)) fail(line_no, "malformed weight");
            if (!std::isfinite(w) || w < 0.0) fail(line_no, "weights must be finite and non-negative");
            fw.push_back(w);
        }
        if (want_l) {
            if (nt < 4) fail(line_no, "label column missing (format is `src dst weight label`)");
            uint64_t l = 0;
            if (!parse_u64(tb[3], te[3], l) || l > UINT32_MAX) fail(line_no, "malformed label");
            fl.push_back(static_cast<uint32_t>(l));
        }
        src.push_back(s);
        dst.push_back(d);
    };
    size_t got;
    while ((got = std::fread(chunk.data(), 1, chunk.size(), f.f)) > 0) {
        for (size_t i = 0; i < got; ++i) {
            if (chunk[i] == '\n') {
                handle(line);
                line.clear();
            } else {
                line.push_back(chunk[i]);
            }
        }
    }
    if (!line.empty()) handle(line);
    if (src.empty()) raise(WF_ERR_PARSE, std::string(path) + ": no edges");
    for (uint32_t l : fl)
        if (l > 255) config_error("edge labels must be < 256 on the device");

    DeviceGuard guard(device);
    cudaStream_t st = nullptr;
    const uint64_t m = src.size();
    const bool undirected = o.undirected != 0;
    // dense ids: sort + unique of all endpoints (graph.cpp:384-401)
    DeviceBuffer<uint64_t> ids(2 * m), ids_sorted(2 * m), d_src(m), d_dst(m);
    WF_CUDA(cudaMemcpy(d_src.get(), src.data(), m * 8, cudaMemcpyHostToDevice));
    WF_CUDA(cudaMemcpy(d_dst.get(), dst.data(), m * 8, cudaMemcpyHostToDevice));
    WF_CUDA(cudaMemcpy(ids.get(), src.data(), m * 8, cudaMemcpyHostToDevice));
    WF_CUDA(cudaMemcpy(ids.get() + m, dst.data(), m * 8, cudaMemcpyHostToDevice));
    DeviceBuffer<uint8_t> tmp;
    size_t tb = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tb, ids.get(), ids_sorted.get(), static_cast<int64_t>(2 * m), 0, 64, st);
    tmp.allocate(tb);
    WF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tb, ids.get(), ids_sorted.get(),
                                           static_cast<int64_t>(2 * m), 0, 64, st));
    count_launch();
    DeviceBuffer<unsigned long long> nuniq(1);
    tb = 0;
    cub::DeviceSelect::Unique(nullptr, tb, ids_sorted.get(), ids.get(), nuniq.get(), static_cast<int64_t>(2 * m), st);
    if (tmp.size() < tb) tmp.allocate(tb);
    WF_CUDA(cub::DeviceSelect::Unique(tmp.get(), tb, ids_sorted.get(), ids.get(), nuniq.get(),
                                      static_cast<int64_t>(2 * m), st));
    count_launch();
    unsigned long long nu = 0;
    WF_CUDA(cudaMemcpy(&nu, nuniq.get(), 8, cudaMemcpyDeviceToHost));
    if (nu > UINT32_MAX) raise(WF_ERR_PARSE, std::string(path) + ": more than 2^32 distinct vertex ids");
    const uint32_t V = static_cast<uint32_t>(nu);
    ids_sorted.release();
    DeviceBuffer<uint32_t> ds(m), dd(m);
    k_lower_bound<<<grid_for(m, device), 256, 0, st>>>(ids.get(), nu, d_src.get(), m, ds.get());
    WF_LAUNCHED();
    k_lower_bound<<<grid_for(m, device), 256, 0, st>>>(ids.get(), nu, d_dst.get(), m, dd.get());
    WF_LAUNCHED();
    if (original_ids) {
        original_ids->resize(V);
        WF_CUDA(cudaMemcpy(original_ids->data(), ids.get(), V * 8ull, cudaMemcpyDeviceToHost));
    }
    ids.release();
    d_src.release();
    d_dst.release();
    // assemble_csr: stable sort of (src, dst) keys, input order breaks ties
    const uint64_t E = undirected ? 2 * m : m;
    DeviceBuffer<uint64_t> key(E), val(E), key2(E), val2(E);
    k_edge_keys<<<grid_for(m, device), 256, 0, st>>>(ds.get(), dd.get(), m, undirected ? 1 : 0,
                                                     key.get(), val.get());
    WF_LAUNCHED();
    ds.release();
    dd.release();
    int hi_bit = 64;
    tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, key.get(), key2.get(), val.get(), val2.get(),
                                    static_cast<int64_t>(E), 0, hi_bit, st);
    if (tmp.size() < tb) tmp.allocate(tb);
    WF_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, key.get(), key2.get(), val.get(), val2.get(),
                                            static_cast<int64_t>(E), 0, hi_bit, st));
    count_launch();
    key.release();
    val.release();
    auto g = std::make_unique<GraphStore>();
    g->device = device;
    g->V = V;
    g->E = E;
    g->offsets.allocate(V + 1ull);
    g->nbr.allocate(E + kNbrPad);
    DeviceBuffer<unsigned long long> deg(V);
    WF_CUDA(cudaMemsetAsync(deg.get(), 0, V * 8ull, st));
    k_csr_from_keys<<<grid_for(E, device), 256, 0, st>>>(key2.get(), E, g->nbr.get(), deg.get());
    WF_LAUNCHED();
    WF_CUDA(cudaMemsetAsync(g->offsets.get(), 0, 8, st));
    tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, deg.get(), reinterpret_cast<unsigned long long*>(g->offsets.get()) + 1,
                                  static_cast<int64_t>(V), st);
    if (tmp.size() < tb) tmp.allocate(tb);
    WF_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, deg.get(),
                                          reinterpret_cast<unsigned long long*>(g->offsets.get()) + 1,
                                          static_cast<int64_t>(V), st));
    count_launch();
    key2.release();
    // attributes: from the file (permuted with the edges) or synthetic on the
    // final edge order (graph.cpp:430-446)
    // weights in f64, as the reference reads and synthesises them (graph.hpp:102)
    DeviceBuffer<double> w64;
    if (want_w || o.weights == WF_ATTR_RANDOM) w64.allocate(std::max<uint64_t>(E, 1));
    if (want_l || o.labels == WF_ATTR_RANDOM) g->labels.allocate(std::max<uint64_t>(E, 1));
    if (want_w) {
        DeviceBuffer<double> in(m);
        WF_CUDA(cudaMemcpy(in.get(), fw.data(), m * 8, cudaMemcpyHostToDevice));
        k_gather_attr<double><<<grid_for(E, device), 256, 0, st>>>(in.get(), val2.get(), E, undirected ? 1 : 0,
                                                                   w64.get());
        WF_LAUNCHED();
    }
    if (want_l) {
        std::vector<uint8_t> l8(fl.begin(), fl.end());
        DeviceBuffer<uint8_t> in(m);
        WF_CUDA(cudaMemcpy(in.get(), l8.data(), m, cudaMemcpyHostToDevice));
        k_gather_attr<uint8_t><<<grid_for(E, device), 256, 0, st>>>(in.get(), val2.get(), E, undirected ? 1 : 0,
                                                                    g->labels.get());
        WF_LAUNCHED();
    }
    if (o.labels == WF_ATTR_RANDOM && (o.label_count == 0 || o.label_count > 256))
        config_error("random labels need label_count in [1, 256]");
    if (o.weights == WF_ATTR_RANDOM || o.labels == WF_ATTR_RANDOM) {
        k_synthetic_attrs<<<grid_for(E, device), 256, 0, st>>>(
            E, seed_premix(o.seed ^ kWeightSalt), seed_premix(o.seed ^ kLabelSalt),
            o.weights == WF_ATTR_RANDOM ? w64.get() : nullptr,
            o.labels == WF_ATTR_RANDOM ? g->labels.get() : nullptr, o.label_count);
        WF_LAUNCHED();
    }
    WF_CUDA(cudaStreamSynchronize(st));
    if (w64.get()) g->adopt_weights64(std::move(w64), st);
    g->finalize(st);
    return g.release();
}

}  // namespace wf
