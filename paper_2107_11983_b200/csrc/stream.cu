// Run + stream the walk set to host memory, overlapping the walk kernel of
// chunk k+1 with the compaction + device->host copy of chunk k (two streams,
// double-buffered staging).  This is the end-to-end path: the reference hands
// its walks back in host memory (RunResult::walks, engine.hpp:448-452) or
// through a BlockSink per worker block (engine.hpp:76-79, output.cpp:133-200).
// Streams, events and staging buffers are cached on the session (HostPipe) so
// repeated calls pay no allocation or synchronising cudaMalloc/cudaFree.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>

#include "runtime.hpp"

namespace wf {

namespace {

__global__ void k_compact_chunk(const uint32_t* __restrict__ rows, uint32_t stride,
                                const uint32_t* __restrict__ lengths,
                                const uint64_t* __restrict__ offs, uint64_t nrows,
                                uint32_t* __restrict__ out, uint64_t cap) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < nrows; r += nwarps) {
        uint32_t len = min(lengths[r], stride);
        const uint32_t* src = rows + r * stride;
        const uint64_t o = offs[r];
        // rows that outgrew `stride` leave gaps (patched on the host), so the
        // true chunk total may exceed the staging buffer: never write past it
        for (uint32_t j = lane; j < len; j += 32)
            if (o + j < cap) out[o + j] = src[j];
    }
}

// Packed record headers: length | status << 31 (wf_session_run_host_records).
__global__ void k_pack_records(const uint32_t* __restrict__ lens, const uint8_t* __restrict__ stat, uint64_t n,
                               uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = lens[i] | (static_cast<uint32_t>(stat[i]) << 31);
}

__global__ void k_add_base(uint64_t* __restrict__ offs, uint64_t n, uint64_t base) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        offs[i] += base;
}

}  // namespace

struct HostPipe {
    int device = 0;
    cudaStream_t a = nullptr, b = nullptr;
    cudaStream_t c = nullptr;            // host -> device source copies, per chunk
    std::vector<cudaEvent_t> ev_src;     // chunk k's sources resident
    cudaEvent_t ev_comp[2] = {nullptr, nullptr};
    cudaEvent_t ev_copy[2] = {nullptr, nullptr};
    uint64_t cap_rows = 0;     // chunk rows the buffers hold
    uint32_t cap_stride = 0;
    DeviceBuffer<uint32_t> rows[2], lens[2], stage[2];
    DeviceBuffer<uint8_t> stat[2];
    DeviceBuffer<uint32_t> packed[2];  // record headers (records mode)
    DeviceBuffer<uint64_t> offs[2];
    DeviceBuffer<uint8_t> scan_tmp;
    size_t scan_bytes = 0;
    DeviceBuffer<uint32_t> src;
    DeviceBuffer<unsigned long long> ctr;
    uint64_t* h_tot = nullptr;  // pinned chunk totals

    explicit HostPipe(int dev) : device(dev) {
        WF_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
        WF_CUDA(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking));
        WF_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            WF_CUDA(cudaEventCreateWithFlags(&ev_comp[i], cudaEventDisableTiming));
            WF_CUDA(cudaEventCreateWithFlags(&ev_copy[i], cudaEventDisableTiming));
        }
        WF_CUDA(cudaMallocHost(&h_tot, 2 * sizeof(uint64_t)));
        ctr.allocate(2);
    }
    ~HostPipe() {
        DeviceGuard guard(device);
        if (a) cudaStreamDestroy(a);
        if (b) cudaStreamDestroy(b);
        if (c) cudaStreamDestroy(c);
        for (cudaEvent_t e : ev_src) cudaEventDestroy(e);
        for (int i = 0; i < 2; ++i) {
            if (ev_comp[i]) cudaEventDestroy(ev_comp[i]);
            if (ev_copy[i]) cudaEventDestroy(ev_copy[i]);
        }
        if (h_tot) cudaFreeHost(h_tot);
    }
    void reserve_src_events(uint64_t nchunks) {
        while (ev_src.size() < nchunks) {
            cudaEvent_t e;
            WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev_src.push_back(e);
        }
    }
    void reserve(uint64_t chunk, uint32_t stride) {
        if (chunk <= cap_rows && stride <= cap_stride) return;
        cap_rows = std::max(cap_rows, chunk);
        cap_stride = std::max(cap_stride, stride);
        for (int i = 0; i < 2; ++i) {
            rows[i].allocate(cap_rows * cap_stride);
            stage[i].allocate(cap_rows * cap_stride);
            lens[i].allocate(cap_rows);
            stat[i].allocate(cap_rows);
            packed[i].allocate(cap_rows);
            offs[i].allocate(cap_rows + 1);
            WF_CUDA(cudaMemset(offs[i].get(), 0, 8));
        }
        cub::TransformInputIterator<uint64_t, WidenU64, const uint32_t*> in(nullptr, WidenU64{});
        scan_bytes = 0;
        cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, in, static_cast<uint64_t*>(nullptr),
                                      static_cast<int64_t>(cap_rows), a);
        scan_tmp.allocate(std::max<size_t>(scan_bytes, 1));
    }
};

void release_host_pipe(HostPipe* p) { delete p; }

void raise_device_error(const Session& s, int code) {
    if (code == WF_ERR_REJECTION_CAP)
        raise(code, "rejection sampling exceeded " + std::to_string(s.trial_cap) +
                        " trials; asserted bound does not match the weights");
    if (code == WF_ERR_CONFIG) raise(code, "query source is not a vertex");
    raise(code, "device-side contract violation");
}

void run_to_host(Session& s, const wf_query_spec& spec, const uint32_t* host_sources, uint64_t qb,
                 uint64_t qe, uint64_t* offsets, uint32_t* vertices, uint64_t capacity, uint8_t* status,
                 uint64_t chunk, wf_run_metrics* metrics, uint32_t* records) {
    GraphStore& g = *s.g;
    DeviceGuard guard(g.device);
    auto t0 = std::chrono::steady_clock::now();
    // WF_TRACE_HOST=1: host-side timeline of the pipeline on stderr (diagnostics)
    static const bool trace_on = getenv("WF_TRACE_HOST") != nullptr;
    auto trace = [&](const char* what, long long k) {
        if (trace_on)
            std::fprintf(stderr, "[run_host %8.1f us] %s %lld\n",
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(),
                         what, k);
    };
    const uint32_t stride = s.default_stride;
    const uint64_t n = qe - qb;
    if (chunk == 0) {
        // ~8 chunks for overlap, each at least 64 Ki queries, staging <= 256 MiB
        chunk = std::max<uint64_t>(n / 8, 1ull << 19);  // tools/e2e_sweep.py
        chunk = std::min<uint64_t>(chunk, std::max<uint64_t>(1, (256ull << 20) / (4ull * stride)));
    }
    chunk = std::max<uint64_t>(1, std::min<uint64_t>(chunk, std::max<uint64_t>(n, 1)));
    if (!s.pipe) s.pipe.reset(new HostPipe(g.device));
    HostPipe& P = *s.pipe;
    P.reserve(chunk, stride);
    cudaStream_t A = P.a, B = P.b;

    // Chunk boundaries.  (A geometric ramp of small first chunks, to start the
    // first device->host copy earlier, measured slower on C2: each PPR launch
    // pays its own tail of long walks.)
    std::vector<uint64_t> bounds{0};
    while (bounds.back() < n) bounds.push_back(std::min(n, bounds.back() + chunk));
    const uint64_t nchunks = bounds.size() - 1;
    // the shard's slice of the source list, addressed by absolute qid in the
    // kernel; copied chunk by chunk on stream C so chunk k+1's sources move
    // while chunk k computes
    const uint32_t* src_by_qid = nullptr;
    const bool list = spec.mode == WF_QUERY_FROM_LIST && n;
    if (list) {
        if (P.src.size() < n) P.src.allocate(n);
        src_by_qid = P.src.get() - qb;
        P.reserve_src_events(nchunks);
        for (uint64_t k = 0; k < nchunks; ++k) {
            const uint64_t r0 = bounds[k], r1 = bounds[k + 1];
            WF_CUDA(cudaMemcpyAsync(P.src.get() + r0, host_sources + qb + r0, (r1 - r0) * 4,
                                    cudaMemcpyHostToDevice, P.c));
            WF_CUDA(cudaEventRecord(P.ev_src[k], P.c));
        }
    }
    WF_CUDA(cudaMemsetAsync(P.ctr.get(), 0, 16, A));

    bool copy_pending[2] = {false, false};
    std::vector<uint64_t> chunk_base(nchunks + 1, 0);

    auto enqueue_compute = [&](uint64_t k) {
        const int b = static_cast<int>(k & 1);
        const uint64_t r0 = bounds[k], r1 = bounds[k + 1], nr = r1 - r0;
        if (list) WF_CUDA(cudaStreamWaitEvent(A, P.ev_src[k], 0));
        // buffer b (status / offsets / staging) is free once chunk k-2's copy drained
        if (copy_pending[b]) WF_CUDA(cudaStreamWaitEvent(A, P.ev_copy[b], 0));
        // offs[b][0] = 0 (the previous user of this buffer rebased it in place)
        WF_CUDA(cudaMemsetAsync(P.offs[b].get(), 0, 8, A));
        launch_walk(s, spec, src_by_qid, qb + r0, qb + r1, nullptr, P.rows[b].get(), stride,
                    P.lens[b].get(), P.stat[b].get(), nullptr, P.ctr.get(), P.ctr.get() + 1,
                    s.cursor.get(), A);
        cub::TransformInputIterator<uint64_t, WidenU64, const uint32_t*> in(P.lens[b].get(), WidenU64{});
        size_t sb = P.scan_bytes;
        WF_CUDA(cub::DeviceScan::InclusiveSum(P.scan_tmp.get(), sb, in, P.offs[b].get() + 1,
                                              static_cast<int64_t>(nr), A));
        count_launch();
        int blocks = static_cast<int>(std::min<uint64_t>((nr * 32 + 255) / 256, 65535));
        k_compact_chunk<<<std::max(blocks, 1), 256, 0, A>>>(P.rows[b].get(), stride, P.lens[b].get(),
                                                            P.offs[b].get(), nr, P.stage[b].get(),
                                                            P.stage[b].size());
        WF_LAUNCHED();
        if (records) {
            k_pack_records<<<std::max(1, static_cast<int>(std::min<uint64_t>((nr + 255) / 256, 4096))), 256, 0, A>>>(
                P.lens[b].get(), P.stat[b].get(), nr, P.packed[b].get());
            WF_LAUNCHED();
        }
        WF_CUDA(cudaMemcpyAsync(P.h_tot + b, P.offs[b].get() + nr, 8, cudaMemcpyDeviceToHost, A));
        WF_CUDA(cudaEventRecord(P.ev_comp[b], A));
    };

    if (nchunks) enqueue_compute(0);
    for (uint64_t k = 0; k < nchunks; ++k) {
        const int b = static_cast<int>(k & 1);
        const uint64_t r0 = bounds[k], r1 = bounds[k + 1], nr = r1 - r0;
        // chunk k+1's walk is queued behind chunk k's before the host waits for
        // chunk k's vertex count, so the compute stream never idles on the host
        if (k + 1 < nchunks) enqueue_compute(k + 1);
        trace("queued compute", static_cast<long long>(k + 1));
        WF_CUDA(cudaEventSynchronize(P.ev_comp[b]));
        trace("chunk computed", static_cast<long long>(k));
        uint64_t cnt = P.h_tot[b];
        chunk_base[k + 1] = chunk_base[k] + cnt;
        if (chunk_base[k + 1] > capacity) {
            // drain what is in flight into the caller's buffers before unwinding
            cudaStreamSynchronize(A);
            cudaStreamSynchronize(B);
            cudaStreamSynchronize(P.c);
            raise(WF_ERR_INVALID_ARG, "vertices_capacity too small for the walk set");
        }
        if (cnt > P.stage[b].size()) {
            // rare (walks outgrew their rows): stage this chunk in a larger buffer
            WF_CUDA(cudaStreamSynchronize(B));
            DeviceBuffer<uint32_t> big(cnt);
            int blocks = static_cast<int>(std::min<uint64_t>((nr * 32 + 255) / 256, 65535));
            k_compact_chunk<<<std::max(blocks, 1), 256, 0, A>>>(P.rows[b].get(), stride,
                                                                P.lens[b].get(), P.offs[b].get(), nr,
                                                                big.get(), cnt);
            WF_LAUNCHED();
            WF_CUDA(cudaStreamSynchronize(A));
            WF_CUDA(cudaMemcpy(vertices + chunk_base[k], big.get(), cnt * 4, cudaMemcpyDeviceToHost));
            P.stage[b].allocate(cnt);  // grown for the next user (nothing pending on it)
            WF_CUDA(cudaMemsetAsync(P.stage[b].get(), 0, 4, A));
            WF_CUDA(cudaStreamSynchronize(A));
            cnt = 0;  // already copied
        }
        WF_CUDA(cudaStreamWaitEvent(B, P.ev_comp[b], 0));
        if (cnt)
            WF_CUDA(cudaMemcpyAsync(vertices + chunk_base[k], P.stage[b].get(), cnt * 4,
                                    cudaMemcpyDeviceToHost, B));
        if (offsets) {
            if (chunk_base[k]) {  // chunk-relative -> absolute, on the copy stream
                int blocks = static_cast<int>(std::min<uint64_t>((nr + 255) / 256, 4096));
                k_add_base<<<std::max(blocks, 1), 256, 0, B>>>(P.offs[b].get(), nr, chunk_base[k]);
                WF_LAUNCHED();
            }
            WF_CUDA(cudaMemcpyAsync(offsets + r0, P.offs[b].get(), nr * 8, cudaMemcpyDeviceToHost, B));
        }
        if (status)
            WF_CUDA(cudaMemcpyAsync(status + r0, P.stat[b].get(), nr, cudaMemcpyDeviceToHost, B));
        if (records)
            WF_CUDA(cudaMemcpyAsync(records + r0, P.packed[b].get(), nr * 4, cudaMemcpyDeviceToHost, B));
        WF_CUDA(cudaEventRecord(P.ev_copy[b], B));
        copy_pending[b] = true;
        trace("copies queued", static_cast<long long>(k));
    }
    WF_CUDA(cudaStreamSynchronize(B));
    trace("copies done", -1);
    WF_CUDA(cudaStreamSynchronize(A));
    int err = 0;
    WF_CUDA(cudaMemcpy(&err, s.error_word.get(), 4, cudaMemcpyDeviceToHost));
    if (err) {
        WF_CUDA(cudaMemset(s.error_word.get(), 0, 4));
        if (err == WF_ERR_CONFIG && spec.mode == WF_QUERY_FROM_LIST) {
            // the kernel flagged a source outside [0, V): name it as the host check would
            for (uint64_t i = qb; i < qe; ++i)
                if (host_sources[i] >= g.V)
                    config_error("query source " + std::to_string(host_sources[i]) +
                                 " is not a vertex (V=" + std::to_string(g.V) + ")");
        }
        raise_device_error(s, err);
    }
    if (offsets) offsets[n] = chunk_base[nchunks];
    unsigned long long hc[2] = {0, 0};
    WF_CUDA(cudaMemcpy(hc, P.ctr.get(), 16, cudaMemcpyDeviceToHost));
    std::vector<uint64_t> rec_offs;  // records mode: offsets rebuilt on the host when needed
    if (hc[1] > 0 && !offsets && records) {
        rec_offs.resize(n + 1);
        rec_offs[0] = 0;
        for (uint64_t r = 0; r < n; ++r) rec_offs[r + 1] = rec_offs[r] + (records[r] & 0x7FFFFFFFu);
        offsets = rec_offs.data();
    }
    if (hc[1] > 0) {
        // walks longer than a row: re-run them whole and patch their paths
        if (!offsets) raise(WF_ERR_INVALID_ARG, "offsets are required to place overflowing walks");
        std::vector<uint64_t> qids;
        uint32_t mx = 0;
        for (uint64_t r = 0; r < n; ++r) {
            uint64_t len = offsets[r + 1] - offsets[r];
            if (len > stride) {
                qids.push_back(qb + r);
                mx = std::max<uint32_t>(mx, static_cast<uint32_t>(len));
            }
        }
        DeviceBuffer<uint64_t> dq(qids.size());
        WF_CUDA(cudaMemcpy(dq.get(), qids.data(), qids.size() * 8, cudaMemcpyHostToDevice));
        DeviceBuffer<uint32_t> p(qids.size() * static_cast<uint64_t>(mx)), l(qids.size());
        DeviceBuffer<uint8_t> sst(qids.size());
        DeviceBuffer<unsigned long long> c2(2);
        WF_CUDA(cudaMemset(c2.get(), 0, 16));
        launch_walk(s, spec, src_by_qid, 0, qids.size(), dq.get(), p.get(), mx, l.get(), sst.get(),
                    nullptr, c2.get(), c2.get() + 1, s.cursor.get(), nullptr);
        std::vector<uint32_t> hp(qids.size() * static_cast<uint64_t>(mx));
        WF_CUDA(cudaMemcpy(hp.data(), p.get(), hp.size() * 4, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < qids.size(); ++i) {
            uint64_t r = qids[i] - qb;
            std::copy(hp.begin() + i * mx, hp.begin() + i * mx + (offsets[r + 1] - offsets[r]),
                      vertices + offsets[r]);
        }
    }
    trace("done", -1);
    if (metrics) {
        metrics->preprocess_seconds = s.preprocess_seconds;
        metrics->exec_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        metrics->total_steps = hc[0];
        metrics->max_in_flight = static_cast<uint32_t>(static_cast<uint64_t>(s.grid) * kBlock);
    }
}

}  // namespace wf
