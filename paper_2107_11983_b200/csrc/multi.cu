// Multi-device execution: the reference's worker split over devices, and the
// path's one collective.
//
// The reference runs a query set as `threads` workers, each a contiguous qid
// block (worker_range, engine.hpp:296-298) on its own std::thread
// (parallel_workers, engine.hpp:302-328), each block handed to the BlockSink
// once, in worker order (engine.hpp:76-79), the first worker exception
// rethrown after the join (engine.hpp:323-327).  Here the workers' blocks are
// spread over devices in contiguous groups: the graph is replicated on every
// device (peer copies), the static tables are built once and peer-copied, one
// host thread per device walks its blocks, and the calling thread hands the
// blocks to the caller in worker order as they complete.  Walks depend only on
// (seed, qid), so the output is the single-device output.
//
// The only collective is the PPR visit-count reduction: one ncclAllReduce
// (sum) over the per-device count vectors.  NCCL is loaded at run time
// (dlopen "libnccl.so.2": the one a process already has loaded — torch's —
// or the system's), so the library carries no link-time NCCL dependency.  A
// device listed twice (several workers' shards on one GPU) cannot join an
// NCCL communicator; those runs sum the counts with a device kernel instead.
//
// wf_comm_* expose the same reduction to one-process-per-GPU jobs (torchrun):
// each rank runs its worker_range shard with the single-device API and
// all-reduces its counts through the library's own communicator.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "runtime.hpp"

namespace wf {

namespace {

// ---- NCCL, resolved at run time ------------------------------------------------------
struct NcclApi {
    bool ok = false;
    std::string error;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi load_nccl() {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        a.error = std::string("NCCL not available: ") + dlerror();
        return a;
    }
    auto sym = [&](auto& fn, const char* name) {
        fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        if (!fn && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.GetErrorString, "ncclGetErrorString");
    sym(a.GetVersion, "ncclGetVersion");
    a.ok = a.error.empty();
    return a;
}

const NcclApi& nccl() {
    static const NcclApi api = load_nccl();
    if (!api.ok) raise(WF_ERR_CUDA, api.error);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) raise(WF_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

__global__ void k_add_u32(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] += src[i];
}

void add_counts(uint32_t* dst, const uint32_t* src, uint64_t n, cudaStream_t st) {
    if (!n) return;
    const int blocks = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 4096));
    k_add_u32<<<blocks, 256, 0, st>>>(dst, src, n);
    WF_LAUNCHED();
}

// A replica of `src` on `device`: the CSR by peer copy, then the same
// finalisation (validation, statistics, vertex words) as any upload.
std::unique_ptr<GraphStore> replicate_graph(const GraphStore& src, int device) {
    DeviceGuard guard(device);
    auto g = std::make_unique<GraphStore>();
    g->device = device;
    g->V = src.V;
    g->E = src.E;
    auto peer = [&](auto& dst, const auto& from, size_t n) {
        if (!from.get()) return;
        dst.allocate(n);
        WF_CUDA(cudaMemcpyPeer(dst.get(), device, from.get(), src.device, n * sizeof(*from.get())));
    };
    peer(g->offsets, src.offsets, src.offsets.size());
    peer(g->nbr, src.nbr, src.nbr.size());
    peer(g->weights, src.weights, src.weights.size());
    peer(g->weights64, src.weights64, src.weights64.size());
    peer(g->labels, src.labels, src.labels.size());
    g->original_ids = src.original_ids;
    g->finalize(nullptr);
    return g;
}

}  // namespace

}  // namespace wf

using namespace wf;

struct wf_multi {
    std::vector<int> devices;
    std::vector<std::unique_ptr<GraphStore>> owned;
    std::vector<GraphStore*> graphs;  // per replica (replicas on one device share one)
    std::vector<std::unique_ptr<Session>> sessions;
    std::vector<DeviceBuffer<unsigned long long>> counters;
    std::vector<ncclComm_t> comms;  // one per replica when every device is distinct
    ~wf_multi() {
        for (size_t i = 0; i < comms.size(); ++i) {
            DeviceGuard guard(devices[i], std::nothrow);
            nccl().CommDestroy(comms[i]);
        }
    }
};

struct wf_comm {
    ncclComm_t comm = nullptr;
    int device = 0;
    int nranks = 1;
    int rank = 0;
    ~wf_comm() {
        if (comm) {
            DeviceGuard guard(device, std::nothrow);
            nccl().CommDestroy(comm);
        }
    }
};

namespace {

template <typename Fn>
int mguarded(Fn&& fn) {  // capi.cu's guarded: status code + wf_last_error()
    try {
        fn();
        return WF_OK;
    } catch (const wf::Error& e) {
        last_error_slot() = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        last_error_slot() = "host allocation failed";
        return WF_ERR_OOM;
    } catch (const std::exception& e) {
        last_error_slot() = e.what();
        return WF_ERR_INVALID_ARG;
    }
}

void mrequire(bool ok, const char* what) {
    if (!ok) raise(WF_ERR_INVALID_ARG, what);
}

// Replicas + one session per replica; `make` resolves the program on a session.
template <typename Make>
wf_multi* build_multi(const wf_graph* gh, const int32_t* devices, uint32_t n, const wf_exec_options* opts,
                      Make&& make) {
    mrequire(gh && devices && n > 0, "null argument");
    GraphStore& src = *graph_store(gh);
    int count = 0;
    WF_CUDA(cudaGetDeviceCount(&count));
    auto m = std::make_unique<wf_multi>();
    for (uint32_t i = 0; i < n; ++i) {
        mrequire(devices[i] >= 0 && devices[i] < count, "device id out of range");
        m->devices.push_back(devices[i]);
        GraphStore* g = nullptr;
        for (uint32_t j = 0; j < i && !g; ++j)
            if (m->devices[j] == devices[i]) g = m->graphs[j];
        if (!g && devices[i] == src.device) g = &src;
        if (!g) {
            if (devices[i] != src.device) {
                int can = 0;
                WF_CUDA(cudaDeviceCanAccessPeer(&can, devices[i], src.device));
                if (can) {
                    DeviceGuard guard(devices[i]);
                    cudaError_t e = cudaDeviceEnablePeerAccess(src.device, 0);
                    if (e != cudaErrorPeerAccessAlreadyEnabled && e != cudaSuccess) WF_CUDA(e);
                    cudaGetLastError();
                }
            }
            m->owned.push_back(replicate_graph(src, devices[i]));
            g = m->owned.back().get();
        }
        m->graphs.push_back(g);
    }
    for (uint32_t i = 0; i < n; ++i) {
        DeviceGuard guard(m->devices[i]);
        auto s = std::make_unique<Session>();
        s->g = m->graphs[i];
        make(*s);
        // the static tables (the Vose build) once, on the first replica
        setup_session(*s, opts, i == 0 ? nullptr : m->sessions[0].get());
        m->sessions.push_back(std::move(s));
        m->counters.emplace_back(2);
    }
    bool distinct = true;
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < i; ++j) distinct = distinct && m->devices[i] != m->devices[j];
    if (distinct && m->sessions[0]->desc.kind == WF_PROGRAM_PPR) {
        // the communicator for the visit-count all-reduce (the path's one collective)
        m->comms.resize(n);
        nccl_check(nccl().CommInitAll(m->comms.data(), static_cast<int>(n), m->devices.data()),
                   "ncclCommInitAll");
    }
    return m.release();
}

}  // namespace

extern "C" {

int wf_worker_range(uint64_t n, uint32_t workers, uint32_t w, uint64_t* begin, uint64_t* end) {
    return mguarded([&] {
        mrequire(begin && end && workers > 0 && w < workers, "bad worker range arguments");
        *begin = static_cast<uint64_t>((static_cast<unsigned __int128>(n) * w) / workers);  // engine.hpp:296-298
        *end = static_cast<uint64_t>((static_cast<unsigned __int128>(n) * (w + 1)) / workers);
    });
}

int wf_multi_create(const wf_graph* g, const int32_t* devices, uint32_t n_devices, const wf_program_desc* prog,
                    const wf_exec_options* opts, wf_multi** out) {
    return mguarded([&] {
        mrequire(prog && out, "null argument");
        *out = build_multi(g, devices, n_devices, opts, [&](Session& s) { resolve_program(s, *prog, opts); });
    });
}

int wf_multi_create_custom(const wf_graph* g, const int32_t* devices, uint32_t n_devices,
                           const wf_program_ops* ops, const void* program, const wf_exec_options* opts,
                           wf_multi** out) {
    return mguarded([&] {
        mrequire(ops && out, "null argument");
        *out = build_multi(g, devices, n_devices, opts,
                           [&](Session& s) { resolve_custom(s, *ops, program, opts); });
    });
}

int wf_multi_info(const wf_multi* m, uint32_t* n_devices, int32_t* collective) {
    return mguarded([&] {
        mrequire(m != nullptr, "null handle");
        if (n_devices) *n_devices = static_cast<uint32_t>(m->devices.size());
        if (collective) *collective = m->comms.empty() ? 0 : 1;
    });
}

int wf_multi_run(wf_multi* m, const wf_query_spec* spec, uint32_t workers, wf_shard_fn on_shard, void* user,
                 uint32_t* visit_counts, wf_run_metrics* metrics) {
    return mguarded([&] {
        mrequire(m && spec, "null argument");
        const uint32_t G = static_cast<uint32_t>(m->devices.size());
        const uint32_t W = workers ? workers : G;
        const GraphStore& g0 = *m->graphs[0];
        const uint64_t n = spec->mode == WF_QUERY_ONE_PER_VERTEX ? g0.V : spec->count;
        const bool counts = m->sessions[0]->desc.kind == WF_PROGRAM_PPR;

        // one slot per worker block, filled by its device's thread
        struct Slot {
            bool done = false;
            std::vector<uint32_t> records, vertices;
            uint64_t lo = 0, hi = 0;
        };
        std::vector<Slot> slots(W);
        std::mutex mu;
        std::condition_variable cv;
        bool cancel = false;
        std::vector<std::exception_ptr> errors(G);
        std::vector<DeviceBuffer<uint32_t>> acc(G);  // per-device visit counts
        std::vector<wf_run_metrics> dm(G);
        for (uint32_t w = 0; w < W; ++w) wf_worker_range(n, W, w, &slots[w].lo, &slots[w].hi);

        auto t0 = std::chrono::steady_clock::now();
        auto device_thread = [&](uint32_t d) {
            try {
                Session& s = *m->sessions[d];
                DeviceGuard guard(m->devices[d]);
                ResolvedSpec rs;
                resolve_spec(*s.g, spec, rs);  // QuerySpec::validate + sources on this device
                if (counts) {
                    acc[d].allocate(s.g->V);
                    WF_CUDA(cudaMemset(acc[d].get(), 0, s.g->V * 4ull));
                }
                for (uint32_t w = 0; w < W; ++w) {
                    if (static_cast<uint64_t>(w) * G / W != d) continue;  // contiguous worker groups
                    {
                        std::lock_guard<std::mutex> lk(mu);
                        if (cancel) return;
                    }
                    Slot& sl = slots[w];
                    auto ws = session_run(s, rs, sl.lo, sl.hi, m->counters[d].get());
                    const uint64_t nq = sl.hi - sl.lo;
                    std::vector<uint64_t> off(nq + 1);
                    std::vector<uint8_t> st(nq);
                    sl.vertices.resize(ws->total_vertices);
                    walkset_copy(*ws, 0, nq, off.data(), sl.vertices.data(), st.data());
                    sl.records.resize(nq);
                    for (uint64_t q = 0; q < nq; ++q)  // WalkRecord{length, status} (walker.hpp:47-55)
                        sl.records[q] = static_cast<uint32_t>(off[q + 1] - off[q]) | (st[q] ? 0x80000000u : 0u);
                    if (counts) add_counts(acc[d].get(), ws->visit_counts.get(), s.g->V, nullptr);
                    dm[d].total_steps += ws->metrics.total_steps;
                    dm[d].exec_seconds += ws->metrics.exec_seconds;
                    ws.reset();
                    std::lock_guard<std::mutex> lk(mu);
                    sl.done = true;
                    cv.notify_all();
                }
                WF_CUDA(cudaDeviceSynchronize());
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                errors[d] = std::current_exception();
                cancel = true;
                cv.notify_all();
            }
        };
        std::vector<std::thread> threads;
        for (uint32_t d = 0; d < G; ++d) threads.emplace_back(device_thread, d);
        // blocks reach the caller in worker order, as they complete
        int sink_rc = 0;
        for (uint32_t w = 0; w < W && !sink_rc; ++w) {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return slots[w].done || cancel; });
            if (!slots[w].done) break;
            lk.unlock();
            Slot& sl = slots[w];
            if (on_shard)
                sink_rc = on_shard(user, w, sl.lo, sl.hi, sl.records.data(), sl.vertices.data(), sl.vertices.size());
            std::vector<uint32_t>().swap(sl.records);
            std::vector<uint32_t>().swap(sl.vertices);
            if (sink_rc) {
                std::lock_guard<std::mutex> lk2(mu);
                cancel = true;
            }
        }
        for (auto& t : threads) t.join();
        for (uint32_t d = 0; d < G; ++d)
            if (errors[d]) std::rethrow_exception(errors[d]);  // parallel_workers, engine.hpp:323-327
        if (sink_rc) raise(WF_ERR_IO, "block sink stopped the run");
        if (counts) {
            if (!m->comms.empty()) {
                // the path's one collective: sum the per-device counts on every device
                nccl_check(nccl().GroupStart(), "ncclGroupStart");
                for (uint32_t d = 0; d < G; ++d) {
                    DeviceGuard guard(m->devices[d]);
                    nccl_check(nccl().AllReduce(acc[d].get(), acc[d].get(), g0.V, ncclUint32, ncclSum, m->comms[d],
                                                nullptr),
                               "ncclAllReduce");
                }
                nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
                for (uint32_t d = 0; d < G; ++d) {
                    DeviceGuard guard(m->devices[d]);
                    WF_CUDA(cudaDeviceSynchronize());
                }
            } else {
                // shards that shared a device (or a single device): sum into the first
                DeviceGuard guard(m->devices[0]);
                for (uint32_t d = 1; d < G; ++d) {
                    DeviceBuffer<uint32_t> tmp(g0.V);
                    WF_CUDA(cudaMemcpyPeer(tmp.get(), m->devices[0], acc[d].get(), m->devices[d], g0.V * 4ull));
                    add_counts(acc[0].get(), tmp.get(), g0.V, nullptr);
                    WF_CUDA(cudaDeviceSynchronize());
                }
            }
            if (visit_counts) {
                DeviceGuard guard(m->devices[0]);
                WF_CUDA(cudaMemcpy(visit_counts, acc[0].get(), g0.V * 4ull, cudaMemcpyDefault));
            }
        }
        if (metrics) {
            wf_run_metrics r{};
            for (uint32_t d = 0; d < G; ++d) {
                r.total_steps += dm[d].total_steps;
                r.preprocess_seconds = std::max(r.preprocess_seconds, m->sessions[d]->preprocess_seconds);
                r.max_in_flight += static_cast<uint32_t>(
                    std::min<uint64_t>(static_cast<uint64_t>(m->sessions[d]->grid) * kBlock, 0xFFFFFFFFull));
            }
            r.exec_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            *metrics = r;
        }
    });
}

void wf_multi_destroy(wf_multi* m) { delete m; }

int wf_comm_unique_id(uint8_t* id) {
    return mguarded([&] {
        mrequire(id != nullptr, "null argument");
        static_assert(sizeof(ncclUniqueId) == WF_COMM_ID_BYTES, "NCCL unique id size");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int wf_comm_create(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, wf_comm** out) {
    return mguarded([&] {
        mrequire(id && out && nranks > 0 && rank >= 0 && rank < nranks, "bad communicator arguments");
        DeviceGuard guard(device);
        auto c = std::make_unique<wf_comm>();
        c->device = device;
        c->nranks = nranks;
        c->rank = rank;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        nccl_check(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

int wf_comm_allreduce_u32(wf_comm* c, uint32_t* dev_counts, uint64_t count, void* stream) {
    return mguarded([&] {
        mrequire(c && (dev_counts || count == 0), "null argument");
        DeviceGuard guard(c->device);
        nccl_check(nccl().AllReduce(dev_counts, dev_counts, count, ncclUint32, ncclSum, c->comm,
                                    static_cast<cudaStream_t>(stream)),
                   "ncclAllReduce");
    });
}

void wf_comm_destroy(wf_comm* c) { delete c; }

int wf_nccl_version(int32_t* version) {
    return mguarded([&] {
        mrequire(version != nullptr, "null argument");
        int v = 0;
        nccl_check(nccl().GetVersion(&v), "ncclGetVersion");
        *version = v;
    });
}

}  // extern "C"
