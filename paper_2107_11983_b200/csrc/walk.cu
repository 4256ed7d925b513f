// Kernel instantiation + launch for every legal (program, sampler, flow)
// pairing (resolve_flow, engine.hpp:255-272), and the walk-set copy-out.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "kernel_table.cuh"
#include "runtime.hpp"

namespace wf {

namespace {

// Every program x sampler x flow the reference accepts; the host-streaming
// instantiations live in walk_stream.cu (compiled in parallel).
KernelFn select_kernel(int prog, int sampler, int flow) {
#define WF_CASE(P, S, F) \
    if (prog == P && sampler == S && flow == F) return &walk_kernel<Program<P>, S, F, false>;
    WF_FOR_EACH_COMBO(WF_CASE)
#undef WF_CASE
    config_error("no kernel for this program/sampler/flow combination");
}

}  // namespace

int row_bucket(uint64_t n_rows) {
    int b = 0;
    while ((1ull << b) < n_rows && b < 63) ++b;
    return b;
}

// A custom program's kernels live in the user's translation unit: their
// occupancy and launches go through its wf_program_ops table.
void custom_occupancy(const Session& s, int streaming, int* per_sm, int* regs) {
    int32_t b = 0, r = 0;
    const int rc = s.custom->occupancy(s.kind, s.flow, streaming, &b, &r);
    if (rc != 0) raise(WF_ERR_CUDA, std::string("custom program occupancy: ") +
                                        cudaGetErrorString(static_cast<cudaError_t>(rc)));
    if (per_sm) *per_sm = b;
    if (regs) *regs = r;
}

int occupancy_grid(const Session& s) {
    int per_sm = 0;
    if (s.custom) {
        custom_occupancy(s, 0, &per_sm, nullptr);
    } else {
        KernelFn fn = select_kernel(s.desc.kind, s.kind, s.flow);
        WF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, 0));
    }
    return std::max(1, per_sm) * sm_count(s.g->device);
}

void launch_walk(Session& s, const wf_query_spec& spec, const uint32_t* dev_sources,
                 uint64_t qid_begin, uint64_t qid_end, const uint64_t* qid_map, uint32_t* paths,
                 uint32_t stride, uint32_t* lengths, uint8_t* status, uint32_t* visit_counts,
                 unsigned long long* steps_out, unsigned long long* overflow_out,
                 unsigned long long* cursor, cudaStream_t st, const StreamLaunch* stream) {
    GraphStore& g = *s.g;
    if (qid_end <= qid_begin) return;
    if (stride == 0) config_error("path stride must be >= 1");
    KernelFn fn = s.custom ? nullptr
                  : stream ? select_stream_kernel(s.desc.kind, s.kind, s.flow)
                           : select_kernel(s.desc.kind, s.kind, s.flow);
    WalkLaunch L{};
    L.g = g.view();
    if (!s.use_edge_hash) L.g.ehash = nullptr;  // per-session choice (B-tree opt-in)
    if (!s.use_edge_filter) L.g.efilter = nullptr;
    L.sview = s.any_exhausted ? s.sview.get() : g.vword.get();
    L.alias = s.alias.get();
    L.its = s.its.get();
    L.rej_pstar = s.rej.get();
    L.prog = s.params;
    L.qmode = spec.mode;
    L.qsource = spec.source;
    L.qsources = dev_sources;
    L.qid_begin = qid_begin;
    L.qid_map = qid_map;
    L.n_rows = qid_end - qid_begin;
    L.seed_mixed = seed_premix(s.seed);
    L.trial_cap = s.trial_cap;
    L.stride = stride;
    L.paths = paths;
    L.lengths = lengths;
    L.status = status;
    L.visit_counts = visit_counts;
    L.steps_out = steps_out;
    L.overflow_out = overflow_out;
    L.cursor = cursor;
    L.error_word = s.error_word.get();
    L.use_label_index = g.label_index_built ? 1 : 0;
    L.g.stats = s.collect_stats ? s.stats.get() : nullptr;
    L.staged = (stride % 8 == 0 && reinterpret_cast<uintptr_t>(paths) % 32 == 0) ? 1 : 0;
    L.alias_wide = s.alias_wide ? 1 : 0;
    L.alias_idx = s.alias_idx ? 1 : 0;
    L.adj = s.adj.get();
    L.adj8 = s.adj8.get();
    L.adj8_vbits = s.adj8_vbits;
    L.adj8_dbits = s.adj8_dbits;
    L.mp_adj = s.mp_adj.get();
    if (stream) {
        L.tile_word = stream->tile_word;
        L.chunk_word = stream->chunk_word;
        L.chunk_flag = stream->chunk_flag;
        L.tile_shift = stream->tile_shift;
        L.chunk_tiles_shift = stream->chunk_tiles_shift;
        L.src_ready = stream->src_ready;
        L.src_shift = stream->src_shift;
        L.src_row0 = stream->src_row0;
    }
    int grid = s.grid > 0 ? s.grid : occupancy_grid(s);
    if (!s.tuned_blocks.empty()) {
        // wf_session_tune's pick for the nearest tuned launch size (row buckets
        // are powers of two: a chunked run of a tuned batch lands one or two
        // buckets below it)
        const int b = row_bucket(L.n_rows);
        int best = -1, dist = 1 << 30;
        for (const auto& kv : s.tuned_blocks) {
            const int d = kv.first > b ? kv.first - b : b - kv.first;
            if (d < dist) {
                dist = d;
                best = kv.second;
            }
        }
        if (best > 0 && dist <= 3) grid = best * sm_count(g.device);
    }
    if (stream && stream->tile_word) {
        // host streaming: leave two compaction blocks' registers (128 threads
        // x 32 each) free on every SM, so the chunk compactions run beside the
        // walk kernel instead of after it
        static std::mutex mu;
        static std::map<KernelFn, int> regs;  // cudaFuncGetAttributes costs the host a few us
        int nregs;
        if (s.custom) {
            custom_occupancy(s, 1, nullptr, &nregs);
        } else {
            std::lock_guard<std::mutex> lock(mu);
            auto it = regs.find(fn);
            if (it == regs.end()) {
                cudaFuncAttributes fa{};
                WF_CUDA(cudaFuncGetAttributes(&fa, fn));
                it = regs.emplace(fn, fa.numRegs).first;
            }
            nregs = it->second;
        }
        const int per_block = ((nregs + 7) / 8 * 8) * kBlock;
        const int fit = std::max(1, (65536 - 8192) / std::max(per_block, 1));
        grid = std::min(grid, fit * sm_count(g.device));
    }
    uint64_t lanes_needed = (L.n_rows + 31) / 32 * 32;
    int grid_needed = static_cast<int>(std::min<uint64_t>((lanes_needed + kBlock - 1) / kBlock, 1u << 30));
    grid = std::max(1, std::min(grid, grid_needed));
    if (s.kind == WF_SAMPLER_ALIAS && s.flow == kGathered && g.max_degree >= kCoopDegree) {
        // a row per warp for the cooperative hub steps (coop_step): the hub's
        // weights, then the compacted scaled weights Vose's replay runs over
        // (vose_bucket_staged); lanes below kCoopDegree park in local memory
        const uint64_t per_warp = 2ull * g.max_degree;
        const uint64_t budget = 16ull << 30;
        const uint64_t warps = std::max<uint64_t>(kBlock / 32, budget / (per_warp * 8));
        grid = std::max(1, std::min<int>(grid, static_cast<int>(warps / (kBlock / 32))));
        const uint64_t need = static_cast<uint64_t>(grid) * (kBlock / 32) * per_warp;
        if (s.scratch.size() < need) s.scratch.allocate(need);
        L.scratch = s.scratch.get();
        L.scratch_stride = g.max_degree;
    } else if (s.kind == WF_SAMPLER_ITS && s.flow == kGathered && g.max_degree >= kCoopDegree &&
               !(s.desc.kind == WF_PROGRAM_METAPATH && g.label_index_built)) {
        // a row per warp keeps a hub's weights from the sum pass for the pick
        // pass (coop_step), so each is evaluated once
        const uint64_t half = (static_cast<uint64_t>(g.max_degree) + 1) / 2;  // warp rows stride 2 x scratch_stride
        const uint64_t per_warp = 2 * half;
        const uint64_t budget = 8ull << 30;
        const uint64_t warps = std::max<uint64_t>(kBlock / 32, budget / (per_warp * 8));
        grid = std::max(1, std::min<int>(grid, static_cast<int>(warps / (kBlock / 32))));
        const uint64_t need = static_cast<uint64_t>(grid) * (kBlock / 32) * per_warp;
        if (s.scratch.size() < need) s.scratch.allocate(need);
        L.scratch = s.scratch.get();
        L.scratch_stride = half;
    }
    {
        // PPR's short geometric walks refill a lane every few moves: half of
        // the rows are dealt statically in blocks, the rest claimed through the
        // cursor (walk_kernel).  C2: 0.228 -> 0.200 ms.  Fixed-length walks
        // refill rarely and measured slower with any static share (C3-C5).
        const uint64_t warps = static_cast<uint64_t>(grid) * (kBlock / 32);
        const uint64_t pct = s.unbounded ? 50 : 0;
        L.static_blocks = static_cast<uint32_t>(std::min<uint64_t>(L.n_rows * pct / 100 / (warps * kClaim), 1u << 30));
        L.dyn_base = warps * L.static_blocks * kClaim;
    }
    WF_CUDA(cudaMemsetAsync(cursor, 0, sizeof(unsigned long long), st));
    if (s.custom) {
        const int rc = s.custom->launch(&L, s.kind, s.flow, stream ? 1 : 0, grid, st);
        if (rc != 0) raise(WF_ERR_CUDA, std::string("custom program launch: ") +
                                            cudaGetErrorString(static_cast<cudaError_t>(rc)));
        count_launch();
        return;
    }
    fn<<<grid, kBlock, 0, st>>>(L);
    WF_LAUNCHED();
}

// ---- walk-set copy-out -------------------------------------------------------------

namespace {

__global__ void k_compact_rows(const uint32_t* __restrict__ paths, uint32_t stride,
                               const uint32_t* __restrict__ lengths,
                               const uint64_t* __restrict__ offs, uint64_t r0, uint64_t nrows,
                               uint64_t out_base, uint32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = warp; i < nrows; i += nwarps) {
        uint64_t r = r0 + i;
        uint32_t len = min(lengths[r], stride);
        const uint32_t* src = paths + r * stride;
        uint32_t* dst = out + (offs[r] - out_base);
        for (uint32_t j = lane; j < len; j += 32) dst[j] = src[j];
    }
}

__global__ void k_count_visits(const uint32_t* __restrict__ paths, uint32_t stride,
                               const uint32_t* __restrict__ lengths, uint64_t n,
                               uint32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < n; r += nwarps) {
        uint32_t len = min(lengths[r], stride);
        for (uint32_t j = lane; j < len; j += 32) atomicAdd(counts + paths[r * stride + j], 1u);
    }
}

}  // namespace

// Occurrences of each vertex over all stored rows (sources included).  Walks
// that outgrew their row are counted from their re-run rows.
void walkset_visit_counts(const WalkSetStore& w, uint32_t* counts, cudaStream_t st) {
    WF_CUDA(cudaMemsetAsync(counts, 0, w.V * 4ull, st));
    if (w.n) {
        int blocks = static_cast<int>(std::min<uint64_t>((w.n * 32 + 255) / 256, 65535));
        k_count_visits<<<blocks, 256, 0, st>>>(w.paths.get(), w.stride, w.lengths.get(), w.n, counts);
        WF_LAUNCHED();
    }
    if (!w.over_rows.empty()) {
        // full paths of the overflowed walks replace their truncated rows
        std::vector<uint32_t> lens(w.over_rows.size());
        for (size_t i = 0; i < w.over_rows.size(); ++i)
            WF_CUDA(cudaMemcpy(&lens[i], w.lengths.get() + w.over_rows[i], 4, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> hp(w.over_rows.size() * static_cast<size_t>(w.over_stride));
        WF_CUDA(cudaMemcpy(hp.data(), w.over_paths.get(), hp.size() * 4, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> hc(w.V);
        WF_CUDA(cudaMemcpyAsync(hc.data(), counts, w.V * 4ull, cudaMemcpyDeviceToHost, st));
        WF_CUDA(cudaStreamSynchronize(st));
        for (size_t i = 0; i < w.over_rows.size(); ++i)
            for (uint32_t j = w.stride; j < lens[i]; ++j) hc[hp[i * w.over_stride + j]] += 1;
        WF_CUDA(cudaMemcpy(counts, hc.data(), w.V * 4ull, cudaMemcpyHostToDevice));
    }
}

void walkset_copy(const WalkSetStore& w, uint64_t qb, uint64_t qe, uint64_t* offsets,
                  uint32_t* vertices, uint8_t* status) {
    DeviceGuard guard(w.device);
    if (qe > w.n || qb > qe) raise(WF_ERR_INVALID_ARG, "query range out of bounds");
    const uint64_t n = qe - qb;
    cudaStream_t st = nullptr;
    // offsets over [qb, qe) relative to qb
    DeviceBuffer<uint64_t> d_off(n + 1);
    WF_CUDA(cudaMemsetAsync(d_off.get(), 0, 8, st));
    if (n) {
        size_t tb = 0;
        cub::TransformInputIterator<uint64_t, WidenU64, const uint32_t*> in(w.lengths.get() + qb, WidenU64{});
        cub::DeviceScan::InclusiveSum(nullptr, tb, in, d_off.get() + 1, static_cast<int64_t>(n), st);
        DeviceBuffer<uint8_t> tmp(tb);
        WF_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tb, in, d_off.get() + 1, static_cast<int64_t>(n), st));
        count_launch();
    }
    std::vector<uint64_t> h_off(n + 1);
    WF_CUDA(cudaMemcpyAsync(h_off.data(), d_off.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    if (offsets) {
        if (is_device_pointer(offsets)) WF_CUDA(cudaMemcpy(offsets, d_off.get(), (n + 1) * 8, cudaMemcpyDeviceToDevice));
        else std::copy(h_off.begin(), h_off.end(), offsets);
    }
    if (status && n) {
        WF_CUDA(cudaMemcpy(status, w.status.get() + qb, n, cudaMemcpyDefault));
    }
    if (!vertices || n == 0) return;
    const bool dev_out = is_device_pointer(vertices);
    const uint64_t total = h_off[n];
    // offsets for the compaction kernel are absolute per row: shift by qb
    const uint64_t* row_offs = d_off.get();
    auto compact = [&](uint64_t r0, uint64_t r1, uint32_t* out, uint64_t out_base) {
        uint64_t rows = r1 - r0;
        if (!rows) return;
        int blocks = static_cast<int>(std::min<uint64_t>((rows * 32 + 255) / 256, 65535));
        k_compact_rows<<<blocks, 256, 0, st>>>(w.paths.get() + qb * w.stride, w.stride,
                                               w.lengths.get() + qb, row_offs, r0, rows, out_base, out);
        WF_LAUNCHED();
    };
    if (dev_out) {
        compact(0, n, vertices, 0);
    } else {
        // bounded staging: rows in chunks of <= 64 Mi vertices
        const uint64_t kStage = 64ull << 20;
        DeviceBuffer<uint32_t> stage(std::min<uint64_t>(std::max<uint64_t>(total, 1), kStage));
        uint64_t r0 = 0;
        while (r0 < n) {
            uint64_t r1 = r0;
            uint64_t lo = h_off[r0];
            while (r1 < n && (h_off[r1 + 1] - lo <= kStage || r1 == r0)) ++r1;
            uint64_t cnt = h_off[r1] - lo;
            if (cnt > stage.size()) stage.allocate(cnt);
            compact(r0, r1, stage.get(), lo);
            WF_CUDA(cudaMemcpyAsync(vertices + lo, stage.get(), cnt * 4, cudaMemcpyDeviceToHost, st));
            WF_CUDA(cudaStreamSynchronize(st));
            r0 = r1;
        }
    }
    WF_CUDA(cudaStreamSynchronize(st));
    // walks that outgrew the row capacity: their full paths from the re-run
    for (size_t i = 0; i < w.over_rows.size(); ++i) {
        uint64_t r = w.over_rows[i];
        if (r < qb || r >= qe) continue;
        uint64_t len = h_off[r - qb + 1] - h_off[r - qb];
        WF_CUDA(cudaMemcpy(vertices + h_off[r - qb], w.over_paths.get() + i * w.over_stride,
                           len * 4, cudaMemcpyDefault));
    }
}

}  // namespace wf
