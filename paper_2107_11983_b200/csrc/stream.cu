// Run + stream the walk set to host memory.  This is the end-to-end path: the
// reference hands its walks back in host memory (RunResult::walks,
// engine.hpp:448-452) or through a BlockSink per worker block
// (engine.hpp:76-79, output.cpp:133-200).  DESIGN.md 5.2.
//
// Rows are grouped in chunks; each chunk's vertex total is published to
// host-mapped memory as soon as all its walks are done, and this thread,
// polling those flags, queues the compaction of every published chunk (a
// batch) on a side stream and its device->host copies on the copy stream
// while the walks go on:
//   * fixed-length walks (chunks mode): one persistent launch whose streaming
//     instantiation (walk_kernel<..., true>) reports finished rows per tile
//     and publishes each chunk itself (stream_report);
//   * short geometric walks (whole mode, PPR): they end all at once near the
//     end of any launch, so the batch runs as two launches (5/16, then
//     the rest), each followed by k_tile_sums + k_publish.
// A pinned source list is copied in a few pieces on a third stream and the
// kernel waits (src_ready) only where its claims get ahead of them.  Large
// runs are split into segments that fit a 4 GiB staging budget.  Streams,
// events, mapped flags and staging buffers are cached on the session
// (HostPipe): repeated calls pay no allocation.
#include <cub/cub.cuh>
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <vector>

#include "runtime.hpp"

namespace wf {

namespace {

constexpr uint32_t kTileShift = 8;  // rows per tile (one compaction block)
// Small compaction blocks at <= 32 registers: they must fit beside the walk
// kernel's blocks on every SM (launch_walk leaves 8192 registers for two),
// or the chunks would only compact once the whole walk kernel has ended.
constexpr int kCompactThreads = 128;
constexpr int kRowsPerThread = (1 << kTileShift) / kCompactThreads;
constexpr uint64_t kStageBudget = 4ull << 30;  // bytes of rows (and of staging) per segment
constexpr uint64_t kSrcFirstPiece = 1ull << 16;  // rows of the first source-list copy
constexpr uint64_t kBatchRows = 1ull << 20;      // rows one compaction + copy batch may cover

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Compaction of one completed chunk: a block per tile.  The tile's first
// vertex comes from the walk kernel's per-tile vertex sums, the rows' from a
// block scan of their lengths (-> records, length | status << 31, or absolute
// offsets); then the tile's vertices are packed (min(len, stride) per walk;
// walks longer than a row leave a gap the host patches).
// Reads go through L2 only: the walk kernel is still running on other rows.
__global__ void __launch_bounds__(kCompactThreads, 16) k_stream_compact(
    const uint32_t* __restrict__ rows, uint32_t stride, const uint32_t* __restrict__ lens,
    const uint8_t* __restrict__ stat, const unsigned long long* __restrict__ tile_word,
    const unsigned long long* __restrict__ chunk_word, uint32_t tile_shift, uint32_t chunk_tiles_shift,
    uint64_t row0, uint64_t nrows, uint32_t* __restrict__ out, uint64_t cap, uint32_t* __restrict__ records,
    uint64_t* __restrict__ offs, uint64_t off_base, volatile unsigned int* over_flag) {
    using Scan = cub::BlockScan<unsigned long long, kCompactThreads>;
    using Reduce = cub::BlockReduce<unsigned long long, kCompactThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Reduce::TempStorage reduce;
    } tmp;
    __shared__ unsigned long long s_base;
    __shared__ unsigned long long s_start[1 << kTileShift];  // rows' tile-relative starts
    // the tile's first vertex, relative to the batch (whole chunks from row0):
    // the earlier chunks' totals plus the earlier tiles of its own chunk
    const uint64_t tile = (row0 >> tile_shift) + blockIdx.x;
    const uint64_t chunk = tile >> chunk_tiles_shift, chunk0 = row0 >> (tile_shift + chunk_tiles_shift);
    const uint64_t ctile0 = chunk << chunk_tiles_shift;
    unsigned long long acc = 0;
    for (uint64_t c = chunk0 + threadIdx.x; c < chunk; c += kCompactThreads) {
        unsigned long long w;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(w) : "l"(chunk_word + c) : "memory");
        acc += w & kSumMask;
    }
    for (uint64_t t = ctile0 + threadIdx.x; t < tile; t += kCompactThreads) {
        unsigned long long w;
        asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(w) : "l"(tile_word + t) : "memory");
        acc += w & kSumMask;
    }
    const unsigned long long before = Reduce(tmp.reduce).Sum(acc);
    if (threadIdx.x == 0) s_base = before;
    __syncthreads();
    const uint64_t base = s_base;
    const uint64_t r_first = static_cast<uint64_t>(blockIdx.x) << tile_shift;  // batch-relative
    const uint64_t r_mine = r_first + static_cast<uint64_t>(threadIdx.x) * kRowsPerThread;
    const uint64_t r_end = nrows - r_first < (1ull << tile_shift) ? nrows : r_first + (1ull << tile_shift);
    uint32_t len[kRowsPerThread];
    unsigned long long sum = 0;
#pragma unroll
    for (int i = 0; i < kRowsPerThread; ++i) {
        len[i] = r_mine + i < r_end ? ldcg(lens + row0 + r_mine + i) : 0;
        sum += len[i];
    }
    __syncthreads();  // tmp is reused
    unsigned long long pos, tile_total;
    Scan(tmp.scan).ExclusiveSum(sum, pos, tile_total);
    // records / offsets, and each row's tile-relative start for the copy
#pragma unroll
    for (int i = 0; i < kRowsPerThread; ++i) {
        const uint64_t r = r_mine + i;
        if (r < r_end) {
            const uint64_t row = row0 + r;
            if (records) records[row] = len[i] | (static_cast<uint32_t>(stat[row]) << 31);
            if (offs) offs[row] = off_base + base + pos;
            if (over_flag && len[i] > stride) *over_flag = 1u;  // host-mapped: patched after the run
            s_start[r - r_first] = pos;
        }
        pos += len[i];
    }
    __syncthreads();
    // The copy runs over the tile's OUTPUT words: thread t moves words t,
    // t + 256, ... (coalesced stores; reads coalesced within each row), the
    // source row found by a binary search over the row starts.  Words of a
    // walk past its row (len > stride) are left for the host to patch.
    const int tile_rows = static_cast<int>(r_end - r_first);
    const uint32_t* tile_src = rows + (row0 + r_first) * stride;
    uint32_t* tile_dst = out + base;
    const uint64_t room = cap > base ? cap - base : 0;
    const uint64_t limit = tile_total < room ? tile_total : room;
    constexpr int kBatch = 4;
    for (uint64_t p0 = threadIdx.x; p0 < limit; p0 += kBatch * kCompactThreads) {
        uint32_t v[kBatch];
        bool ok[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const uint64_t p = p0 + static_cast<uint64_t>(u) * kCompactThreads;
            ok[u] = false;
            v[u] = 0;
            if (p < limit) {
                int lo = 0, hi = tile_rows - 1;  // last row starting at or before p
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_start[mid] <= p) lo = mid;
                    else hi = mid - 1;
                }
                const uint64_t j = p - s_start[lo];
                if (j < stride) {
                    v[u] = ldcg(tile_src + static_cast<uint64_t>(lo) * stride + j);
                    ok[u] = true;
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u)
            if (ok[u]) tile_dst[p0 + static_cast<uint64_t>(u) * kCompactThreads] = v[u];
    }
}

// Whole-launch mode (short walks, which finish all at once near the end of
// the launch): the walk kernel does not report; after it, per-tile vertex
// sums (the tile words the compaction reads) and per-chunk totals ...
__global__ void __launch_bounds__(kCompactThreads) k_tile_sums(const uint32_t* __restrict__ lens, uint64_t n,
                                                               uint32_t tile_shift, uint32_t chunk_tiles_shift,
                                                               unsigned long long* __restrict__ tile_word,
                                                               unsigned long long* __restrict__ chunk_word) {
    using Reduce = cub::BlockReduce<unsigned long long, kCompactThreads>;
    __shared__ typename Reduce::TempStorage tmp;
    const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) << tile_shift;
    const uint64_t r1 = n - r0 < (1ull << tile_shift) ? n : r0 + (1ull << tile_shift);
    unsigned long long sum = 0;
    for (uint64_t r = r0 + threadIdx.x; r < r1; r += kCompactThreads) sum += lens[r];
    sum = Reduce(tmp).Sum(sum);
    if (threadIdx.x == 0) {
        tile_word[blockIdx.x] = ((r1 - r0) << kCountShift) | sum;
        atomicAdd(chunk_word + (blockIdx.x >> chunk_tiles_shift), (1ull << kCountShift) | sum);
    }
}

// ... published to the host-mapped flags in one go.
__global__ void k_publish(const unsigned long long* __restrict__ chunk_word, uint64_t nch,
                          unsigned long long* flags) {
    for (uint64_t c = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; c < nch;
         c += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags + c), "l"((chunk_word[c] & kSumMask) + 1)
                     : "memory");
}

uint32_t log2_ceil(uint64_t x) {
    uint32_t b = 0;
    while ((1ull << b) < x && b < 63) ++b;
    return b;
}

}  // namespace

struct HostPipe {
    int device = 0;
    cudaStream_t a = nullptr;  // walk kernel
    cudaStream_t b = nullptr;  // device -> host copies
    cudaStream_t c = nullptr;  // host -> device source copies
    cudaStream_t d = nullptr;  // chunk compaction
    std::vector<cudaEvent_t> ev_chunk;  // chunk k compacted
    cudaEvent_t ev_src0 = nullptr, ev_walk = nullptr, ev_copy = nullptr, ev_last_copy = nullptr;
    cudaEvent_t ev_trace_src = nullptr;  // WF_TRACE_HOST: sources resident
    uint64_t cap_rows = 0;  // segment rows the buffers hold
    uint32_t cap_stride = 0;
    DeviceBuffer<uint32_t> rows, lens, stage, packed;
    DeviceBuffer<uint8_t> stat;
    DeviceBuffer<uint64_t> offs;
    DeviceBuffer<unsigned long long> tile_word, chunk_word;
    DeviceBuffer<unsigned int> src_ready;
    DeviceBuffer<uint32_t> src;
    DeviceBuffer<unsigned long long> ctr;
    unsigned long long* flags = nullptr;  // host-mapped chunk flags
    unsigned long long* h_end = nullptr;  // pinned: steps, overflow, error word
    unsigned int* h_over = nullptr;       // host-mapped, per block: a walk outgrew its row
    uint64_t cap_over = 0;
    std::vector<cudaEvent_t> ev_block;    // block k's copies landed (wf_session_run_host_blocks)
    uint64_t cap_flags = 0;
    using WriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    WriteValue32 write_value32 = nullptr;

    explicit HostPipe(int dev) : device(dev) {
        for (cudaStream_t* s : {&a, &b, &c, &d}) WF_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&ev_src0, &ev_walk, &ev_copy, &ev_last_copy})
            WF_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        ctr.allocate(2);
        src_ready.allocate(1);
        WF_CUDA(cudaMallocHost(&h_end, 4 * sizeof(unsigned long long)));
        // cuStreamWriteValue32 (the copy stream's "sources resident" marks) from
        // the driver, without linking libcuda
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &fn, 12000, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            write_value32 = reinterpret_cast<WriteValue32>(fn);
        else
            cudaGetLastError();
    }
    ~HostPipe() {
        DeviceGuard guard(device, std::nothrow);
        for (cudaStream_t s : {a, b, c, d})
            if (s) cudaStreamDestroy(s);
        for (cudaEvent_t e : ev_chunk) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_src0, ev_walk, ev_copy, ev_last_copy})
            if (e) cudaEventDestroy(e);
        if (flags) cudaFreeHost(flags);
        if (h_end) cudaFreeHost(h_end);
        if (h_over) cudaFreeHost(h_over);
        for (cudaEvent_t e : ev_block) cudaEventDestroy(e);
    }
    // per-block state of a wf_session_run_host_blocks call with up to `blocks` blocks
    void reserve_blocks(uint64_t blocks) {
        while (ev_block.size() < blocks) {
            cudaEvent_t e;
            WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev_block.push_back(e);
        }
        if (blocks > cap_over) {
            if (h_over) WF_CUDA(cudaFreeHost(h_over));
            h_over = nullptr;
            WF_CUDA(cudaHostAlloc(&h_over, blocks * sizeof(unsigned int), cudaHostAllocMapped));
            cap_over = blocks;
        }
        std::fill(h_over, h_over + blocks, 0u);
    }
    void reserve(uint64_t seg_rows, uint32_t stride, uint64_t nchunks) {
        while (ev_chunk.size() < nchunks) {
            cudaEvent_t e;
            WF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ev_chunk.push_back(e);
        }
        if (nchunks > cap_flags) {
            if (flags) WF_CUDA(cudaFreeHost(flags));
            flags = nullptr;
            WF_CUDA(cudaHostAlloc(&flags, nchunks * sizeof(unsigned long long), cudaHostAllocMapped));
            cap_flags = nchunks;
        }
        if (seg_rows <= cap_rows && stride <= cap_stride) return;
        cap_rows = std::max(cap_rows, seg_rows);
        cap_stride = std::max(cap_stride, stride);
        rows.allocate(cap_rows * cap_stride);
        stage.allocate(cap_rows * cap_stride);
        lens.allocate(cap_rows);
        stat.allocate(cap_rows);
        packed.allocate(cap_rows);
        offs.allocate(cap_rows);
        tile_word.allocate((cap_rows >> 5) + 1);  // tiles are >= 32 rows (tiny chunks: a tile each)
        chunk_word.allocate((cap_rows >> 5) + 1);  // chunks are >= 32 rows
    }
};

void release_host_pipe(HostPipe* p) { delete p; }

void raise_device_error(const Session& s, int code) {
    if (code == WF_ERR_REJECTION_CAP)
        raise(code, "rejection sampling exceeded " + std::to_string(s.trial_cap) +
                        " trials; asserted bound does not match the weights");
    if (code == WF_ERR_CONFIG) raise(code, "query source is not a vertex");
    if (code == WF_ERR_CUDA) raise(code, "walk kernel timed out waiting for its source list");
    if (code == WF_ERR_CONTRACT)  // check_program_weight, engine.hpp:97-101
        raise(code, "program emitted a weight that is negative or not finite");
    raise(code, "device-side contract violation");
}

// A device-side error word after a run: the reference's exception, naming a
// non-vertex source as QuerySpec::validate would (walker.cpp:8-109).
[[noreturn]] void raise_run_error(const Session& s, const wf_query_spec& spec, const uint32_t* host_sources,
                                  uint64_t qb, uint64_t qe, int err) {
    WF_CUDA(cudaMemset(s.error_word.get(), 0, 4));
    if (err == WF_ERR_CONFIG && spec.mode == WF_QUERY_FROM_LIST) {
        for (uint64_t i = qb; i < qe; ++i)
            if (host_sources[i] >= s.g->V)
                config_error("query source " + std::to_string(host_sources[i]) + " is not a vertex (V=" +
                             std::to_string(s.g->V) + ")");
    }
    raise_device_error(s, err);
}

// Walks longer than a row (rare: PPR beyond the row capacity) left gaps in
// the streamed vertices: re-run exactly those queries with rows long enough
// and patch their paths in place.  `offsets` are relative to qb.
void patch_long_walks(Session& s, const wf_query_spec& spec, const uint32_t* host_sources, uint64_t qb,
                      uint64_t n, uint32_t stride, const uint64_t* offsets, uint32_t* vertices) {
    std::vector<uint64_t> qids;
    uint32_t mx = 0;
    for (uint64_t r = 0; r < n; ++r) {
        const uint64_t len = offsets[r + 1] - offsets[r];
        if (len > stride) {
            qids.push_back(qb + r);
            mx = std::max<uint32_t>(mx, static_cast<uint32_t>(len));
        }
    }
    if (qids.empty()) return;
    DeviceBuffer<uint64_t> dq(qids.size());
    WF_CUDA(cudaMemcpy(dq.get(), qids.data(), qids.size() * 8, cudaMemcpyHostToDevice));
    DeviceBuffer<uint32_t> p(qids.size() * static_cast<uint64_t>(mx)), l(qids.size());
    DeviceBuffer<uint8_t> sst(qids.size());
    DeviceBuffer<unsigned long long> c2(2);
    WF_CUDA(cudaMemset(c2.get(), 0, 16));
    DeviceBuffer<uint32_t> all_src;  // the shard's sources, addressed by qid
    const uint32_t* src_by_qid = nullptr;
    if (host_sources) {
        all_src.allocate(n);
        WF_CUDA(cudaMemcpy(all_src.get(), host_sources + qb, n * 4, cudaMemcpyHostToDevice));
        src_by_qid = all_src.get() - qb;
    }
    launch_walk(s, spec, src_by_qid, 0, qids.size(), dq.get(), p.get(), mx, l.get(), sst.get(), nullptr,
                c2.get(), c2.get() + 1, s.cursor.get(), nullptr);
    // a device error of the re-run (e.g. the rejection cap) is the run's error
    WF_CUDA(cudaDeviceSynchronize());
    int err = 0;
    WF_CUDA(cudaMemcpy(&err, s.error_word.get(), 4, cudaMemcpyDeviceToHost));
    if (err) raise_run_error(s, spec, host_sources, qb, qb + n, err);
    std::vector<uint32_t> hp(qids.size() * static_cast<uint64_t>(mx));
    WF_CUDA(cudaMemcpy(hp.data(), p.get(), hp.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < qids.size(); ++i) {
        const uint64_t r = qids[i] - qb;
        std::copy(hp.begin() + i * mx, hp.begin() + i * mx + (offsets[r + 1] - offsets[r]), vertices + offsets[r]);
    }
}

// WF_TRACE_HOST: the device timeline of one segment relative to its first
// kernel's start (tev: kernel start / end, copies end; cev: per batch
// compaction end, copy start, copy end); destroys the events.
void print_segment_timeline(uint64_t s0, cudaEvent_t (&tev)[3], std::vector<cudaEvent_t>& cev, uint64_t nch,
                            cudaEvent_t& ev_src) {
    WF_CUDA(cudaEventSynchronize(tev[2]));
    float kms = 0, cms = 0;
    WF_CUDA(cudaEventElapsedTime(&kms, tev[0], tev[1]));
    WF_CUDA(cudaEventElapsedTime(&cms, tev[0], tev[2]));
    std::fprintf(stderr, "[run_host] segment %llu: kernel %.1f us, copies end %.1f us after kernel start\n",
                 static_cast<unsigned long long>(s0), kms * 1e3, cms * 1e3);
    if (ev_src) {
        float sms = 0;
        if (cudaEventElapsedTime(&sms, tev[0], ev_src) == cudaSuccess)
            std::fprintf(stderr, "[run_host] sources resident %.1f us after kernel start\n", sms * 1e3);
        cudaEventDestroy(ev_src);
        ev_src = nullptr;
    }
    for (uint64_t k = 0; k < nch; ++k) {  // batches start at the chunks with events
        float t[3] = {0, 0, 0};
        bool any = false;
        for (int i = 0; i < 3; ++i)
            if (cudaEventElapsedTime(&t[i], tev[0], cev[3 * k + i]) == cudaSuccess) any = true;
        if (!any) continue;
        std::fprintf(stderr, "[run_host]   batch at chunk %llu: compacted %.1f us, copy %.1f -> %.1f us\n",
                     static_cast<unsigned long long>(k), t[0] * 1e3, t[1] * 1e3, t[2] * 1e3);
    }
    cudaGetLastError();
    for (cudaEvent_t e : cev) cudaEventDestroy(e);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
}

void run_to_host(Session& s, const wf_query_spec& spec, const uint32_t* host_sources, uint64_t qb,
                 uint64_t qe, uint64_t* offsets, uint32_t* vertices, uint64_t capacity, uint8_t* status,
                 uint64_t chunk, wf_run_metrics* metrics, uint32_t* records, wf_block_fn on_block,
                 void* user) {
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
    if (!s.pipe) s.pipe.reset(new HostPipe(g.device));
    HostPipe& P = *s.pipe;
    const bool list = spec.mode == WF_QUERY_FROM_LIST && n;
    // Short geometric walks (PPR) finish all at once near the end of a launch,
    // so in-kernel chunk reports would only slow the walk kernel (C2: 0.16 ->
    // 0.23 ms): whole-launch mode publishes every chunk after it instead.
    // Fixed-length walks finish chunk by chunk and stream.
    const char* mode_env = getenv("WF_STREAM_MODE");  // tests / experiments: "whole" / "chunks"
    const bool whole = mode_env ? std::string(mode_env) == "whole" : s.unbounded;

    // segment: rows one launch covers; chunk: rows one flag / copy covers
    const char* budget_env = getenv("WF_STREAM_STAGE_BYTES");  // tests: force several segments
    const uint64_t budget = budget_env ? std::strtoull(budget_env, nullptr, 10) : kStageBudget;
    const uint64_t seg_max = std::max<uint64_t>(1ull << kTileShift, budget / (4ull * std::max(stride, 1u)));
    const uint64_t seg_rows = std::max<uint64_t>(1, std::min(n, seg_max));
    // 64 Ki rows: long walks publish a chunk every few hundred us (C3: the
    // first copy starts ~0.5 ms in); short ones are batched (kBatchRows)
    if (chunk == 0) chunk = 1ull << 16;
    const uint32_t chunk_shift = std::max<uint32_t>(5, log2_ceil(std::max<uint64_t>(chunk, 1)));
    const uint32_t tile_shift = std::min(kTileShift, chunk_shift);
    const uint64_t chunk_rows = 1ull << chunk_shift;
    const uint64_t seg_chunks = (seg_rows + chunk_rows - 1) >> chunk_shift;
    P.reserve(seg_rows, stride, seg_chunks);
    if (list && P.src.size() < seg_rows) P.src.allocate(seg_rows);
    cudaStream_t A = P.a, B = P.b, C = P.c, D = P.d;

    // wf_session_run_host_blocks: blocks (batches) are handed to the caller in
    // qid order as their copies land; one holding a walk longer than its row
    // (patched after the run) holds back itself and everything after it
    struct Block {
        uint64_t q0, q1, v0, slot;
    };
    std::vector<Block> pending;
    size_t next_block = 0;
    uint64_t nblocks = 0;
    bool patched = false;
    auto drain = [&] {
        for (cudaStream_t st : {P.a, P.b, P.c, P.d}) cudaStreamSynchronize(st);
    };
    if (on_block) P.reserve_blocks(((n + chunk_rows - 1) >> chunk_shift) + (n + seg_rows - 1) / seg_rows);
    auto deliver = [&](bool wait) {
        while (next_block < pending.size()) {
            const Block& b = pending[next_block];
            cudaEvent_t ev = P.ev_block[b.slot];
            if (!wait) {
                const cudaError_t e = cudaEventQuery(ev);
                if (e == cudaErrorNotReady) return;
                WF_CUDA(e);
            } else {
                WF_CUDA(cudaEventSynchronize(ev));
            }
            if (!patched && P.h_over[b.slot]) return;
            if (on_block(user, next_block, b.q0, b.q1, b.v0) != 0) {
                drain();
                raise(WF_ERR_IO, "the block callback stopped the run at block " + std::to_string(next_block));
            }
            ++next_block;
        }
    };
    WF_CUDA(cudaMemsetAsync(P.ctr.get(), 0, 16, A));
    uint64_t total = 0;  // vertices written before the current chunk
    bool first_seg = true;
    for (uint64_t s0 = 0; s0 < n; s0 += seg_rows) {
        const uint64_t s1 = std::min(n, s0 + seg_rows), sn = s1 - s0;
        const uint64_t nch = (sn + chunk_rows - 1) >> chunk_shift;
        const uint64_t ntiles = (sn + (1ull << tile_shift) - 1) >> tile_shift;
        if (!first_seg) {
            // the previous segment's kernel, compactions and copies are done
            // with the buffers this one overwrites
            WF_CUDA(cudaStreamWaitEvent(A, P.ev_copy, 0));
            WF_CUDA(cudaStreamWaitEvent(C, P.ev_walk, 0));
        }
        std::fill(P.flags, P.flags + nch, 0ull);
        StreamLaunch SL;
        SL.tile_word = whole ? nullptr : P.tile_word.get();
        SL.chunk_word = P.chunk_word.get();
        SL.chunk_flag = P.flags;
        SL.tile_shift = tile_shift;
        SL.chunk_tiles_shift = chunk_shift - tile_shift;
        // whole mode: the first launch covers 5/16 of the chunks (C2 e2e: 3/16
        // 0.636, 4/16 0.615, 5/16 0.606, 6/16 0.616 ms) — long enough that
        // its copies cover the second launch, short enough to start them early
        const uint64_t split = whole && nch >= 4 ? ((nch * 5 + 15) / 16) << chunk_shift : sn;
        uint64_t src_rest = sn;  // source rows still to queue (before the launch that needs them)
        auto copy_src = [&](uint64_t r0, uint64_t r1) {
            if (r1 <= r0) return;
            WF_CUDA(cudaMemcpyAsync(P.src.get() + r0, host_sources + qb + s0 + r0, (r1 - r0) * 4,
                                    cudaMemcpyHostToDevice, C));
            // resident 1024-row blocks: a piece ending inside a block leaves
            // that block unpublished until the piece that completes it (or the
            // list's end) lands; the claims past it wait for that copy
            const uint64_t blocks = r1 == sn ? (r1 + 1023) >> 10 : r1 >> 10;
            CUresult cr = P.write_value32(reinterpret_cast<CUstream>(C), reinterpret_cast<CUdeviceptr>(P.src_ready.get()),
                                          static_cast<cuuint32_t>(blocks), 0);
            if (cr != CUDA_SUCCESS) raise(WF_ERR_CUDA, "cuStreamWriteValue32 failed");
        };
        const uint32_t* src_by_qid = nullptr;
        if (list) {
            src_by_qid = P.src.get() - (qb + s0);
            // The kernel may only wait on copies that cannot wait on it: a
            // pageable list is staged by the driver with the host blocked, so it
            // is copied whole before the launch instead.
            cudaPointerAttributes pa{};
            const bool pinned = cudaPointerGetAttributes(&pa, host_sources) == cudaSuccess &&
                                pa.type == cudaMemoryTypeHost;
            cudaGetLastError();
            if (P.write_value32 && pinned) {
                // the kernel starts once the first piece of the list has
                // landed and waits for the rest only where it gets ahead of the
                // copies (src_ready, in 1024-row units).  Every piece is
                // queued before the first launch that may wait on it: a copy
                // queued behind a spinning kernel can be held up by it
                // (streams may share a hardware queue), which would deadlock.
                // Few pieces: each costs the host a few us before the launch.
                WF_CUDA(cudaMemsetAsync(P.src_ready.get(), 0, 4, C));
                WF_CUDA(cudaEventRecord(P.ev_src0, C));
                copy_src(0, std::min<uint64_t>(sn, kSrcFirstPiece));
                if (whole) {
                    copy_src(std::min<uint64_t>(sn, kSrcFirstPiece), split);  // the first launch's rows
                    src_rest = split;  // queued before the second launch
                } else {
                    for (uint64_t r0 = kSrcFirstPiece, piece = kSrcFirstPiece; r0 < sn; r0 += piece, piece *= 2)
                        copy_src(r0, std::min<uint64_t>(sn, r0 + piece));
                }
                if (trace_on) {
                    WF_CUDA(cudaEventCreate(&P.ev_trace_src));
                    WF_CUDA(cudaEventRecord(P.ev_trace_src, C));
                }
                SL.src_ready = P.src_ready.get();
                SL.src_shift = 10;
            } else {
                WF_CUDA(cudaMemcpyAsync(P.src.get(), host_sources + qb + s0, sn * 4, cudaMemcpyHostToDevice, C));
                WF_CUDA(cudaEventRecord(P.ev_src0, C));
            }
            WF_CUDA(cudaStreamWaitEvent(A, P.ev_src0, 0));
        }
        WF_CUDA(cudaMemsetAsync(P.tile_word.get(), 0, ntiles * 8, A));
        WF_CUDA(cudaMemsetAsync(P.chunk_word.get(), 0, nch * 8, A));
        cudaEvent_t tev[3] = {nullptr, nullptr, nullptr};  // trace: kernel start / end, copies end
        if (trace_on) {
            for (cudaEvent_t& e : tev) WF_CUDA(cudaEventCreate(&e));
            WF_CUDA(cudaEventRecord(tev[0], A));
        }
        if (!whole) {
            launch_walk(s, spec, src_by_qid, qb + s0, qb + s1, nullptr, P.rows.get(), stride, P.lens.get(),
                        P.stat.get(), nullptr, P.ctr.get(), P.ctr.get() + 1, s.cursor.get(), A, &SL);
        } else {
            // Two launches, the first over ~5/16 of the rows: its chunks
            // are published (and their copies start) while the second runs.
            // One launch would publish everything only at its end; halves
            // would make the first copy wait longer.
            for (uint64_t a = 0; a < sn;) {
                const uint64_t b = a == 0 ? split : sn;
                if (a == src_rest) {
                    copy_src(src_rest, sn);
                    src_rest = sn;
                }
                SL.src_row0 = a;
                launch_walk(s, spec, src_by_qid, qb + s0 + a, qb + s0 + b, nullptr, P.rows.get() + a * stride,
                            stride, P.lens.get() + a, P.stat.get() + a, nullptr, P.ctr.get(), P.ctr.get() + 1,
                            s.cursor.get(), A, &SL);
                trace("launch queued, first row", static_cast<long long>(s0 + a));
                const uint64_t t0 = a >> tile_shift, c0 = a >> chunk_shift;
                const uint64_t nt = ((b - a) + (1ull << tile_shift) - 1) >> tile_shift;
                const uint64_t nc = ((b - a) + chunk_rows - 1) >> chunk_shift;
                k_tile_sums<<<static_cast<unsigned>(nt), kCompactThreads, 0, A>>>(
                    P.lens.get() + a, b - a, tile_shift, chunk_shift - tile_shift, P.tile_word.get() + t0,
                    P.chunk_word.get() + c0);
                WF_LAUNCHED();
                k_publish<<<static_cast<unsigned>(std::min<uint64_t>((nc + 255) / 256, 1024)), 256, 0, A>>>(
                    P.chunk_word.get() + c0, nc, P.flags + c0);
                WF_LAUNCHED();
                a = b;
            }
        }
        WF_CUDA(cudaEventRecord(P.ev_walk, A));
        if (trace_on) WF_CUDA(cudaEventRecord(tev[1], A));
        if (!first_seg) WF_CUDA(cudaStreamWaitEvent(D, P.ev_copy, 0));  // staging drained
        trace("segment launched", static_cast<long long>(s0));

        std::vector<cudaEvent_t> cev;  // trace: per chunk compaction end, copy start, copy end
        if (trace_on) {
            cev.resize(3 * nch);
            for (cudaEvent_t& e : cev) WF_CUDA(cudaEventCreate(&e));
        }
        // Chunks are taken in order; chunks already published when chunk k is
        // picked up may join its batch (one compaction, one copy per output
        // array): short walks finish all at once near the kernel's end, long
        // ones chunk by chunk.
        // Batch size adapts to the copy engine: one chunk when it is idle (the
        // copy starts as soon as that chunk is compacted), everything published
        // up to kBatchRows when it is busy (fewer, larger copies; each costs a
        // few us of setup).  C2 0.64 -> 0.615 ms, C3 16.3 -> 15.3 ms.
        const uint64_t big_batch = std::max<uint64_t>(1, kBatchRows >> chunk_shift);
        bool copies_queued = false;
        for (uint64_t k = 0; k < nch;) {
            // wait for the kernel to publish chunk k (bounded by the kernel's
            // own life: a launch that ends or faults without it is an error)
            volatile unsigned long long* flags = P.flags;
            uint64_t spins = 0;
            while (flags[k] == 0) {
                if ((++spins & 255) == 0) {
                    if (on_block) deliver(false);
                    cudaError_t e = cudaStreamQuery(A);
                    if (e == cudaSuccess) {
                        if (flags[k] != 0) break;
                        raise(WF_ERR_CUDA, "walk kernel ended without publishing chunk " + std::to_string(k));
                    }
                    if (e != cudaErrorNotReady) WF_CUDA(e);
                }
            }
            const cudaError_t q_last = copies_queued ? cudaEventQuery(P.ev_last_copy) : cudaSuccess;
            cudaGetLastError();  // (cudaErrorNotReady is not an error)
            // the first chunk of a launch (whole mode) is taken alone too: the
            // copy engine has drained during that launch's tail
            const bool idle = q_last == cudaSuccess || (whole && (k << chunk_shift) == split);
            const uint64_t cap_batch = idle ? 1 : big_batch;
            uint64_t k1 = k, cnt = 0;
            do {
                cnt += flags[k1] - 1;
                ++k1;
            } while (k1 < nch && k1 - k < cap_batch && flags[k1] != 0);
            const uint64_t r0 = k << chunk_shift, r1 = std::min(sn, k1 << chunk_shift), nr = r1 - r0;
            trace(idle ? "chunks published (copy engine idle), batch up to"
                       : "chunks published (copy engine busy), batch up to",
                  static_cast<long long>(k1 - 1));
            if (total + cnt > capacity) {
                // drain what is in flight into the caller's buffers before unwinding
                drain();
                raise(WF_ERR_INVALID_ARG, "vertices_capacity too small for the walk set");
            }
            const uint64_t slot_cap = nr * stride;
            uint32_t* slot = P.stage.get() + r0 * stride;
            // one block per tile (a chunk below a tile, for a tiny explicit
            // chunk_queries, is a tile of its own)
            const unsigned tiles = static_cast<unsigned>((nr + (1ull << tile_shift) - 1) >> tile_shift);
            auto compact = [&](uint32_t* out, uint64_t cap, cudaStream_t st) {
                k_stream_compact<<<tiles, kCompactThreads, 0, st>>>(
                    P.rows.get(), stride, P.lens.get(), P.stat.get(), P.tile_word.get(), P.chunk_word.get(),
                    tile_shift, chunk_shift - tile_shift, r0, nr, out, cap, records ? P.packed.get() : nullptr,
                    offsets ? P.offs.get() : nullptr, total, on_block ? P.h_over + nblocks : nullptr);
                WF_LAUNCHED();
            };
            if (cnt <= slot_cap) {
                compact(slot, slot_cap, D);
                WF_CUDA(cudaEventRecord(P.ev_chunk[k], D));
                WF_CUDA(cudaStreamWaitEvent(B, P.ev_chunk[k], 0));
                if (trace_on) {
                    WF_CUDA(cudaEventRecord(cev[3 * k], D));
                    WF_CUDA(cudaEventRecord(cev[3 * k + 1], B));
                }
                if (cnt)
                    WF_CUDA(cudaMemcpyAsync(vertices + total, slot, cnt * 4, cudaMemcpyDeviceToHost, B));
            } else {
                // rare (walks outgrew their rows): this batch through its own buffer
                DeviceBuffer<uint32_t> big(cnt);
                compact(big.get(), cnt, D);
                WF_CUDA(cudaStreamSynchronize(D));
                WF_CUDA(cudaMemcpy(vertices + total, big.get(), cnt * 4, cudaMemcpyDeviceToHost));
                WF_CUDA(cudaEventRecord(P.ev_chunk[k], D));
                WF_CUDA(cudaStreamWaitEvent(B, P.ev_chunk[k], 0));
            }
            if (offsets)
                WF_CUDA(cudaMemcpyAsync(offsets + s0 + r0, P.offs.get() + r0, nr * 8, cudaMemcpyDeviceToHost, B));
            if (status)
                WF_CUDA(cudaMemcpyAsync(status + s0 + r0, P.stat.get() + r0, nr, cudaMemcpyDeviceToHost, B));
            if (records)
                WF_CUDA(cudaMemcpyAsync(records + s0 + r0, P.packed.get() + r0, nr * 4, cudaMemcpyDeviceToHost, B));
            WF_CUDA(cudaEventRecord(P.ev_last_copy, B));
            copies_queued = true;
            if (on_block) {
                WF_CUDA(cudaEventRecord(P.ev_block[nblocks], B));
                pending.push_back({s0 + r0, s0 + r1, total, nblocks});
                ++nblocks;
            }
            total += cnt;
            if (trace_on) WF_CUDA(cudaEventRecord(cev[3 * k + 2], B));
            trace("copies queued", static_cast<long long>(k1 - 1));
            k = k1;
            if (on_block) deliver(false);
        }
        WF_CUDA(cudaEventRecord(P.ev_copy, B));
        if (trace_on) {
            WF_CUDA(cudaEventRecord(tev[2], B));
            print_segment_timeline(s0, tev, cev, nch, P.ev_trace_src);
        }
        first_seg = false;
    }
    // the step / overflow counters and the error word ride behind the last
    // kernel into pinned memory (no synchronous round trips at the end)
    WF_CUDA(cudaMemcpyAsync(P.h_end, P.ctr.get(), 16, cudaMemcpyDeviceToHost, A));
    WF_CUDA(cudaMemcpyAsync(P.h_end + 2, s.error_word.get(), 4, cudaMemcpyDeviceToHost, A));
    WF_CUDA(cudaStreamSynchronize(B));
    trace("copies done", -1);
    WF_CUDA(cudaStreamSynchronize(A));
    WF_CUDA(cudaStreamSynchronize(D));
    const int err = static_cast<int>(P.h_end[2] & 0xFFFFFFFFu);
    if (err) raise_run_error(s, spec, host_sources, qb, qe, err);
    if (offsets) offsets[n] = total;
    const unsigned long long hc[2] = {P.h_end[0], P.h_end[1]};
    std::vector<uint64_t> rec_offs;  // records mode: offsets rebuilt on the host when needed
    if (hc[1] > 0 && !offsets && records) {
        rec_offs.resize(n + 1);
        rec_offs[0] = 0;
        for (uint64_t r = 0; r < n; ++r) rec_offs[r + 1] = rec_offs[r] + (records[r] & 0x7FFFFFFFu);
        offsets = rec_offs.data();
    }
    if (hc[1] > 0) {
        if (!offsets) raise(WF_ERR_INVALID_ARG, "offsets are required to place overflowing walks");
        patch_long_walks(s, spec, list ? host_sources : nullptr, qb, n, stride, offsets, vertices);
    }
    if (on_block) {
        patched = true;
        deliver(true);
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
