// Device graph residency: upload + validation (Graph::from_csr, graph.cpp:118-159),
// statistics (finalize_stats, graph.cpp:161-180), packed vertex words, the
// MetaPath label index, batched has_edge, and the synthetic R-MAT generator
// with an on-device CSR build (symmetrise, drop self-loops, dedup, sort).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>

#include "runtime.hpp"

namespace wf {

std::atomic<uint64_t> g_kernel_launches{0};

namespace {

enum : unsigned {
    kBadOffsets = 1u,
    kBadDegree = 2u,
    kBadNeighbor = 4u,
    kBadWeight = 8u,
    kBadLabel = 16u,
    kUnsorted = 32u,
};

inline int blocks_for(uint64_t n, int threads, int dev) {
    uint64_t b = (n + threads - 1) / threads;
    uint64_t cap = static_cast<uint64_t>(sm_count(dev)) * 32;
    return static_cast<int>(std::max<uint64_t>(1, std::min(b, cap)));
}

__global__ void k_check_offsets(const uint64_t* __restrict__ off, uint32_t V, unsigned* flags) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t a = off[v], b = off[v + 1];
        if (b < a) atomicOr(flags, kBadOffsets);
        else if (b - a > 0xFFFFFFFFull) atomicOr(flags, kBadDegree);
    }
}

__global__ void k_check_neighbors(const uint32_t* __restrict__ nbr, uint64_t E, uint32_t V,
                                  unsigned* flags) {
    bool bad = false;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x)
        bad |= nbr[e] >= V;
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kBadNeighbor);
}

// finite, non-negative; max weight as the max over the float bit patterns
// (monotone for non-negative IEEE floats).
__global__ void k_check_weights(const float* __restrict__ w, uint64_t E, unsigned* flags,
                                unsigned* max_bits) {
    bool bad = false;
    unsigned mx = 0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        float x = w[e];
        if (!isfinite(x) || x < 0.0f) bad = true;
        else mx = max(mx, __float_as_uint(x));
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kBadWeight);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_bits, mx);
}

// The reference's f64 weights (graph.hpp:102): validated (finite,
// non-negative), their maximum, whether any is not float32-exact, and the
// f32 mirror the hot-path layouts read (saturated, never inf).
__global__ void k_weights_f64(const double* __restrict__ w64, uint64_t E, float* __restrict__ w32,
                              unsigned* flags, unsigned long long* max_bits) {
    bool bad = false, inexact = false;
    unsigned long long mx = 0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const double x = w64[e];
        if (!(x >= 0.0 && x <= 1.7976931348623157e308)) {
            bad = true;
            w32[e] = 0.0f;
            continue;
        }
        const float f = static_cast<float>(fmin(x, 3.4028234663852886e38));
        w32[e] = f;
        inexact = inexact || static_cast<double>(f) != x;
        mx = max(mx, static_cast<unsigned long long>(__double_as_longlong(x)));  // x >= 0: bits order as values
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kBadWeight);
    if (__any_sync(kFull, inexact) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u << 30);
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_bits, mx);
}

__global__ void k_narrow_labels(const uint32_t* __restrict__ in, uint8_t* __restrict__ out,
                                uint64_t E, unsigned* flags) {
    bool bad = false;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t l = in[e];
        bad |= l > 255;
        out[e] = static_cast<uint8_t>(l);
    }
    if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, kBadLabel);
}

__global__ void k_label_presence(const uint8_t* __restrict__ lab, uint64_t E, unsigned* present) {
    __shared__ unsigned local[8];
    if (threadIdx.x < 8) local[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint8_t l = lab[e];
        atomicOr(&local[l >> 5], 1u << (l & 31));
    }
    __syncthreads();
    if (threadIdx.x < 8 && local[threadIdx.x]) atomicOr(present + threadIdx.x, local[threadIdx.x]);
}

// Warp per vertex: sortedness, max degree, packed vertex word.
__global__ void k_vertex_stats(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                               uint32_t V, uint64_t* __restrict__ vword, unsigned* flags,
                               unsigned* max_deg, int pack) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    bool unsorted = false;
    unsigned md = 0;
    for (uint64_t v = warp; v < V; v += nwarps) {
        uint64_t a = off[v], b = off[v + 1];
        uint64_t d = b - a;
        for (uint64_t e = a + 1 + lane; e < b; e += 32) unsorted |= nbr[e - 1] > nbr[e];
        if (lane == 0) {
            md = max(md, static_cast<unsigned>(d));
            uint64_t dd = d >= kDegEscape || !pack ? kDegEscape : d;
            vword[v] = (pack ? (a << kDegBits) : 0) | dd;
        }
    }
    if (__any_sync(kFull, unsorted) && lane == 0) atomicOr(flags, kUnsorted);
    if (lane == 0) atomicMax(max_deg, md);
}

// Label index: per vertex, counts per label (warp per vertex), written as the
// 32 B record {base, end[0..5]} with end[l] = #edges with label <= l; then the
// neighbours are stably partitioned by label into lab_nbr.
__global__ void k_label_index(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                              const uint8_t* __restrict__ lab, uint32_t V, uint4* __restrict__ rec,
                              uint32_t* __restrict__ lab_nbr) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        uint64_t a = off[v], b = off[v + 1];
        uint32_t cnt[kMaxIndexedLabels] = {0, 0, 0, 0, 0, 0};
        for (uint64_t e0 = a; e0 < b; e0 += 32) {
            uint64_t e = e0 + lane;
            uint32_t l = e < b ? lab[e] : 0xFF;
#pragma unroll
            for (int i = 0; i < kMaxIndexedLabels; ++i) cnt[i] += __popc(__ballot_sync(kFull, l == (uint32_t)i));
        }
        uint32_t ends[kMaxIndexedLabels];
        uint32_t run = 0;
#pragma unroll
        for (int i = 0; i < kMaxIndexedLabels; ++i) { run += cnt[i]; ends[i] = run; }
        if (lane == 0) {
            rec[2 * v] = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32), ends[0], ends[1]);
            rec[2 * v + 1] = make_uint4(ends[2], ends[3], ends[4], ends[5]);
        }
        // stable partition: position = start(label) + #earlier same-label edges
        uint32_t seen[kMaxIndexedLabels] = {0, 0, 0, 0, 0, 0};
        for (uint64_t e0 = a; e0 < b; e0 += 32) {
            uint64_t e = e0 + lane;
            uint32_t l = e < b ? lab[e] : 0xFF;
            unsigned lower = (1u << lane) - 1;
#pragma unroll
            for (int i = 0; i < kMaxIndexedLabels; ++i) {
                unsigned m = __ballot_sync(kFull, l == (uint32_t)i);
                if (l == (uint32_t)i) {
                    uint32_t start = i == 0 ? 0 : ends[i - 1];
                    lab_nbr[a + start + seen[i] + __popc(m & lower)] = nbr[e];
                }
                seen[i] += __popc(m);
            }
        }
    }
}

__global__ void k_has_edge(GraphView g, const uint32_t* __restrict__ src,
                           const uint32_t* __restrict__ dst, uint64_t n, uint8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = src[i];
        uint64_t a = g.offsets[s];
        uint32_t d = static_cast<uint32_t>(g.offsets[s + 1] - a);
        out[i] = has_edge(g, a, d, dst[i]) ? 1 : 0;
    }
}

// ---- R-MAT ---------------------------------------------------------------------
// Edge draw i: a SplitMix64 stream RngStream(seed ^ kRmatSalt, i); each 64-bit
// draw decides two recursion levels (high then low 32 bits) against the
// cumulative quadrant thresholds floor(a 2^32), floor((a+b) 2^32),
// floor((a+b+c) 2^32).  Source bits are filled MSB first.

constexpr uint64_t kRmatSalt = 0x524D4154454447ULL;  // "RMATEDG"

struct RmatGen {
    uint64_t premixed;
    uint32_t scale;
    uint32_t t1, t2, t3;
    __device__ __forceinline__ void edge(uint64_t i, uint32_t& s, uint32_t& d) const {
        Rng r{stream_state(premixed, i)};
        s = 0;
        d = 0;
        for (uint32_t lvl = 0; lvl < scale; lvl += 2) {
            uint64_t x = r.next();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t l = lvl + h;
                if (l >= scale) break;
                uint32_t u = h == 0 ? static_cast<uint32_t>(x >> 32) : static_cast<uint32_t>(x);
                uint32_t bit = 1u << (scale - 1 - l);
                if (u >= t1) {
                    if (u < t2) d |= bit;
                    else if (u < t3) s |= bit;
                    else { s |= bit; d |= bit; }
                }
            }
        }
    }
};

__global__ void k_rmat_count(RmatGen gen, uint64_t n_draws, unsigned* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_draws;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s, d;
        gen.edge(i, s, d);
        if (s != d) {
            atomicAdd(deg + s, 1u);
            atomicAdd(deg + d, 1u);
        }
    }
}

__global__ void k_rmat_fill(RmatGen gen, uint64_t n_draws, unsigned long long* __restrict__ cursor,
                            uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_draws;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s, d;
        gen.edge(i, s, d);
        if (s != d) {
            out[atomicAdd(cursor + s, 1ULL)] = d;
            out[atomicAdd(cursor + d, 1ULL)] = s;
        }
    }
}

// Warp per vertex over its sorted segment: count distinct values (pass 0) or
// copy them to their final position (pass 1).
__global__ void k_dedup(const uint64_t* __restrict__ off0, const uint32_t* __restrict__ sorted_in,
                        uint32_t V, uint32_t* __restrict__ ndeg, const uint64_t* __restrict__ off1,
                        uint32_t* __restrict__ out, int pass) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        uint64_t a = off0[v], b = off0[v + 1];
        uint64_t w = pass ? off1[v] : 0;
        uint32_t cnt = 0;
        for (uint64_t e0 = a; e0 < b; e0 += 32) {
            uint64_t e = e0 + lane;
            bool keep = e < b && (e == a || sorted_in[e] != sorted_in[e - 1]);
            unsigned m = __ballot_sync(kFull, keep);
            if (pass && keep) out[w + cnt + __popc(m & ((1u << lane) - 1))] = sorted_in[e];
            cnt += __popc(m);
        }
        if (!pass && lane == 0) ndeg[v] = cnt;
    }
}

// Synthetic attributes keyed on the final CSR edge index: synthetic_weight /
// synthetic_label (graph.cpp:279-287) — weight = 1 + uniform_real(4) of
// RngStream(seed ^ kWeightSalt, e), rounded to f32; label = uniform_index(L)
// of RngStream(seed ^ kLabelSalt, e).
constexpr uint64_t kWeightSalt = 0x57464757454947ULL;  // graph.cpp:26
constexpr uint64_t kLabelSalt = 0x5746474C41424CULL;   // graph.cpp:27

__global__ void k_attributes(uint64_t E, uint64_t wmix, uint64_t lmix, float* __restrict__ w,
                             uint8_t* __restrict__ lab, uint32_t label_count) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        if (w) {
            Rng r{stream_state(wmix, e)};
            w[e] = static_cast<float>(1.0 + r.real(4.0));
        }
        if (lab) {
            Rng r{stream_state(lmix, e)};
            lab[e] = static_cast<uint8_t>(r.index(label_count));
        }
    }
}

struct FlagBlock {
    unsigned flags;
    unsigned max_weight_bits;
    unsigned max_degree;
    unsigned present[8];
};

}  // namespace

void GraphStore::adopt_weights64(DeviceBuffer<double>&& w64, cudaStream_t st) {
    DeviceGuard guard(device);
    weights.allocate(std::max<uint64_t>(E, 1));
    DeviceBuffer<unsigned> flags(1);
    DeviceBuffer<unsigned long long> mx(1);
    WF_CUDA(cudaMemsetAsync(flags.get(), 0, 4, st));
    WF_CUDA(cudaMemsetAsync(mx.get(), 0, 8, st));
    if (E) {
        k_weights_f64<<<blocks_for(E, 256, device), 256, 0, st>>>(w64.get(), E, weights.get(), flags.get(), mx.get());
        WF_LAUNCHED();
    }
    unsigned hf = 0;
    unsigned long long hm = 0;
    WF_CUDA(cudaMemcpyAsync(&hf, flags.get(), 4, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaMemcpyAsync(&hm, mx.get(), 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    if (hf & kBadWeight) config_error("edge weights must be finite and non-negative");
    if (hf & (1u << 30)) {
        // some weight is not float32-exact: the f64 array is what samplers,
        // tables and programs read (edge_weight); the f32 one mirrors it
        weights64 = std::move(w64);
        std::memcpy(&max_weight64, &hm, 8);
    } else {
        weights64.release();
    }
}

void GraphStore::finalize(cudaStream_t st) {
    DeviceGuard guard(device);
    if (E >= (1ULL << 40)) config_error("edge count exceeds the 40-bit packed vertex word range");
    DeviceBuffer<FlagBlock> fb(1);
    WF_CUDA(cudaMemsetAsync(fb.get(), 0, sizeof(FlagBlock), st));
    FlagBlock* f = fb.get();
    // offsets frame [0, E]
    uint64_t ends[2] = {0, 0};
    WF_CUDA(cudaMemcpyAsync(&ends[0], offsets.get(), 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaMemcpyAsync(&ends[1], offsets.get() + V, 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    if (ends[0] != 0 || ends[1] != E) config_error("CSR offsets do not frame the neighbor array");
    k_check_offsets<<<blocks_for(V, 256, device), 256, 0, st>>>(offsets.get(), V, &f->flags);
    WF_LAUNCHED();
    if (E) {
        k_check_neighbors<<<blocks_for(E, 256, device), 256, 0, st>>>(nbr.get(), E, V, &f->flags);
        WF_LAUNCHED();
    }
    if (weights.get() && E) {
        k_check_weights<<<blocks_for(E, 256, device), 256, 0, st>>>(weights.get(), E, &f->flags,
                                                                    &f->max_weight_bits);
        WF_LAUNCHED();
    }
    if (labels.get() && E) {
        k_label_presence<<<blocks_for(E, 256, device), 256, 0, st>>>(labels.get(), E, f->present);
        WF_LAUNCHED();
    }
    vword.allocate(V);
    k_vertex_stats<<<blocks_for((uint64_t)V * 32, 256, device), 256, 0, st>>>(
        offsets.get(), nbr.get(), V, vword.get(), &f->flags, &f->max_degree, 1);
    WF_LAUNCHED();
    FlagBlock h{};
    WF_CUDA(cudaMemcpyAsync(&h, f, sizeof(h), cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    if (h.flags & kBadOffsets) config_error("CSR offsets must be non-decreasing");
    if (h.flags & kBadDegree) config_error("vertex degree exceeds 32-bit range");
    if (h.flags & kBadNeighbor) config_error("neighbor id out of range");
    if (h.flags & kBadWeight) config_error("edge weights must be finite and non-negative");
    sorted = !(h.flags & kUnsorted);
    max_degree = h.max_degree;
    float mw;
    std::memcpy(&mw, &h.max_weight_bits, 4);
    max_weight = weights.get() ? static_cast<double>(mw) : 0.0;
    if (weights64.get()) max_weight = max_weight64;  // graph.hpp:56 over the f64 weights
    label_present.assign(256, 0);
    label_count = 0;
    if (labels.get()) {
        for (int l = 0; l < 256; ++l) {
            if (h.present[l >> 5] & (1u << (l & 31))) {
                label_present[l] = 1;
                label_count = l + 1;
            }
        }
    }
}

void GraphStore::ensure_label_index(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    if (label_index_built || !labels.get() || label_count > kMaxIndexedLabels) return;
    DeviceGuard guard(device);
    lab_rec.allocate(2 * static_cast<size_t>(V));
    lab_nbr.allocate(std::max<uint64_t>(E, 1));
    k_label_index<<<blocks_for((uint64_t)V * 32, 256, device), 256, 0, st>>>(
        offsets.get(), nbr.get(), labels.get(), V, lab_rec.get(), lab_nbr.get());
    WF_LAUNCHED();
    WF_CUDA(cudaStreamSynchronize(st));
    label_index_built = true;
}

namespace {
__global__ void k_search_index(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                               uint32_t V, int shift, uint32_t* __restrict__ level) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        uint64_t a = off[v], d = off[v + 1] - a;
        if (d <= kSidxBlock) continue;
        uint64_t n = (d + (1ull << shift) - 1) >> shift;
        uint32_t* ix = level + sidx_base(a, v, shift);
        for (uint64_t k = lane; k < n; k += 32) ix[k] = nbr[a + (k << shift)];
    }
}
}  // namespace

// Sector B-tree over every adjacency list for has_edge_indexed (Node2Vec's
// distance test); only for sorted adjacency, where std::binary_search
// semantics apply.  Level l has stride 16 * 8^l; levels are added until the
// largest list has <= 8 heads at the top.
void GraphStore::ensure_search_index(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    if (search_index_built || !sorted || E == 0) return;
    DeviceGuard guard(device);
    int levels = 0;
    if (max_degree > kSidxBlock) {
        while (levels < kSidxMaxLevels) {
            const int sh = sidx_shift(levels);
            ++levels;
            if (((static_cast<uint64_t>(max_degree) + (1ull << sh) - 1) >> sh) <= 8) break;
        }
    }
    for (int l = 0; l < levels; ++l) {
        const int sh = sidx_shift(l);
        sidx[l].allocate(sidx_base(E, V, sh) + 16);  // +16: two-sector reads at the end
        k_search_index<<<blocks_for((uint64_t)V * 32, 256, device), 256, 0, st>>>(
            offsets.get(), nbr.get(), V, sh, sidx[l].get());
        WF_LAUNCHED();
    }
    WF_CUDA(cudaStreamSynchronize(st));
    sidx_levels = levels;
    search_index_built = true;
}

namespace {
// Warp per vertex: insert every (v, nbr) key with atomicCAS into the first
// empty slot of its bucket chain (open addressing, 4 slots per 32 B bucket).
__global__ void k_edge_hash(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                            uint32_t V, unsigned long long* __restrict__ table, uint64_t nb) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        const uint64_t a = off[v], b = off[v + 1];
        for (uint64_t e = a + lane; e < b; e += 32) {
            const unsigned long long key = (static_cast<unsigned long long>(v) << 32) | nbr[e];
            uint64_t bk = ehash_bucket(key, nb);
            for (bool done = false; !done;) {
                for (int s = 0; s < 4 && !done; ++s) {
                    unsigned long long old = atomicCAS(table + 4 * bk + s, kHashEmpty, key);
                    done = old == kHashEmpty || old == key;  // duplicates (multigraphs) stored once
                }
                bk = bk + 1 == nb ? 0 : bk + 1;
            }
        }
    }
}
}  // namespace

namespace {
// Warp per vertex: set each edge's kFilterBits bits in its pair's sector.
__global__ void k_edge_filter(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                              uint32_t V, uint32_t* __restrict__ words, uint64_t sectors) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        const uint64_t a = off[v], b = off[v + 1];
        for (uint64_t e = a + lane; e < b; e += 32) {
            const uint64_t h = efilter_hash(static_cast<uint32_t>(v), nbr[e]);
            uint32_t* sec = words + 8 * (h & (sectors - 1));
            for (int i = 0; i < kFilterBits; ++i) {
                const uint32_t bit = static_cast<uint32_t>(h >> (32 + 8 * i)) & 255u;
                atomicOr(sec + (bit >> 5), 1u << (bit & 31));
            }
        }
    }
}
}  // namespace

// Pre-filter for Node2Vec's distance test: ~8 bits per stored pair (a
// power-of-two number of 32 B sectors, at most 64 MiB so it can stay in L2).
// Only ~5 % of the distance tests on R-MAT find an edge, so most are answered
// by one L2-resident sector instead of a DRAM bucket of the exact set.
void GraphStore::ensure_edge_filter(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    if (edge_filter_built || E == 0) return;
    DeviceGuard guard(device);
    uint64_t sectors = 1;
#ifndef WF_FILTER_MAX_LOG2
#define WF_FILTER_MAX_LOG2 21
#endif
    while (sectors * 256 < 8 * E && sectors < (1ull << WF_FILTER_MAX_LOG2)) sectors <<= 1;
    efilter.allocate(2 * sectors);
    WF_CUDA(cudaMemsetAsync(efilter.get(), 0, efilter.bytes(), st));
    k_edge_filter<<<blocks_for((uint64_t)V * 32, 256, device), 256, 0, st>>>(
        offsets.get(), nbr.get(), V, reinterpret_cast<uint32_t*>(efilter.get()), sectors);
    WF_LAUNCHED();
    WF_CUDA(cudaStreamSynchronize(st));
    efilter_sectors = sectors;
    edge_filter_built = true;
}

// Exact edge set for Node2Vec's distance test (has_edge_hashed), 2 slots per
// edge (load factor 1/2): one random 32 B bucket per membership query.
void GraphStore::ensure_edge_hash(cudaStream_t st) {
    std::lock_guard<std::mutex> lock(mu);
    if (edge_hash_built || E == 0) return;
    DeviceGuard guard(device);
    const uint64_t nb = std::max<uint64_t>(1, (2 * E + 3) / 4);
    ehash.allocate(4 * nb);
    WF_CUDA(cudaMemsetAsync(ehash.get(), 0xFF, ehash.bytes(), st));
    k_edge_hash<<<blocks_for((uint64_t)V * 32, 256, device), 256, 0, st>>>(offsets.get(), nbr.get(), V,
                                                                           ehash.get(), nb);
    WF_LAUNCHED();
    WF_CUDA(cudaStreamSynchronize(st));
    ehash_buckets = nb;
    edge_hash_built = true;
}

static std::unique_ptr<GraphStore> alloc_graph(uint32_t V, uint64_t E, bool w, bool l, int device) {
    if (V == 0) config_error("graph must have at least one vertex");
    auto g = std::make_unique<GraphStore>();
    g->device = device;
    g->V = V;
    g->E = E;
    g->offsets.allocate(static_cast<size_t>(V) + 1);
    g->nbr.allocate(E + kNbrPad);  // padded: search reads whole 32 B sectors
    if (w) g->weights.allocate(std::max<uint64_t>(E, 1));
    if (l) g->labels.allocate(std::max<uint64_t>(E, 1));
    return g;
}

GraphStore* graph_from_host(const uint64_t* offsets, const uint32_t* neighbors, const float* weights,
                            const uint32_t* labels, uint32_t V, uint64_t E, int device, bool finalize) {
    DeviceGuard guard(device);
    auto g = alloc_graph(V, E, weights != nullptr, labels != nullptr, device);
    cudaStream_t st = nullptr;
    WF_CUDA(cudaMemcpy(g->offsets.get(), offsets, (static_cast<size_t>(V) + 1) * 8, cudaMemcpyHostToDevice));
    if (E) WF_CUDA(cudaMemcpy(g->nbr.get(), neighbors, E * 4, cudaMemcpyHostToDevice));
    if (weights && E) WF_CUDA(cudaMemcpy(g->weights.get(), weights, E * 4, cudaMemcpyHostToDevice));
    if (labels && E) {
        DeviceBuffer<uint32_t> tmp(E);
        DeviceBuffer<unsigned> flag(1);
        WF_CUDA(cudaMemset(flag.get(), 0, 4));
        WF_CUDA(cudaMemcpy(tmp.get(), labels, E * 4, cudaMemcpyHostToDevice));
        k_narrow_labels<<<blocks_for(E, 256, device), 256>>>(tmp.get(), g->labels.get(), E, flag.get());
        WF_LAUNCHED();
        unsigned h = 0;
        WF_CUDA(cudaMemcpy(&h, flag.get(), 4, cudaMemcpyDeviceToHost));
        if (h) config_error("edge labels must be < 256 on the device");
    }
    if (finalize) g->finalize(st);
    return g.release();
}

GraphStore* graph_from_host_f64(const uint64_t* offsets, const uint32_t* neighbors, const double* weights,
                                const uint32_t* labels, uint32_t V, uint64_t E, int device) {
    if (!weights) return graph_from_host(offsets, neighbors, nullptr, labels, V, E, device);
    DeviceGuard guard(device);
    std::unique_ptr<GraphStore> g(graph_from_host(offsets, neighbors, nullptr, labels, V, E, device, false));
    DeviceBuffer<double> w64(std::max<uint64_t>(E, 1));
    if (E) WF_CUDA(cudaMemcpy(w64.get(), weights, E * 8, cudaMemcpyHostToDevice));
    g->adopt_weights64(std::move(w64), nullptr);
    g->finalize(nullptr);
    return g.release();
}

GraphStore* graph_from_device(const uint64_t* offsets, const uint32_t* neighbors,
                              const float* weights, const uint8_t* labels, uint32_t V, uint64_t E,
                              int device) {
    DeviceGuard guard(device);
    auto g = alloc_graph(V, E, weights != nullptr, labels != nullptr, device);
    WF_CUDA(cudaMemcpy(g->offsets.get(), offsets, (static_cast<size_t>(V) + 1) * 8, cudaMemcpyDeviceToDevice));
    if (E) WF_CUDA(cudaMemcpy(g->nbr.get(), neighbors, E * 4, cudaMemcpyDeviceToDevice));
    if (weights && E) WF_CUDA(cudaMemcpy(g->weights.get(), weights, E * 4, cudaMemcpyDeviceToDevice));
    if (labels && E) WF_CUDA(cudaMemcpy(g->labels.get(), labels, E, cudaMemcpyDeviceToDevice));
    g->finalize(nullptr);
    return g.release();
}

GraphStore* graph_generate_rmat(const wf_rmat_params& p, int device) {
    DeviceGuard guard(device);
    if (p.scale < 1 || p.scale > 31) config_error("R-MAT scale must be in [1, 31]");
    if (p.edge_factor < 1) config_error("R-MAT edge factor must be >= 1");
    double d = 1.0 - p.a - p.b - p.c;
    if (!(p.a >= 0 && p.b >= 0 && p.c >= 0 && d >= -1e-12))
        config_error("R-MAT probabilities must be non-negative and sum to <= 1");
    if (p.label_count > 256) config_error("label count must be <= 256");
    const uint32_t V = 1u << p.scale;
    const uint64_t n_draws = static_cast<uint64_t>(p.edge_factor) << p.scale;
    auto thr = [](double x) -> uint32_t {
        double t = std::floor(x * 4294967296.0);
        return t >= 4294967295.0 ? 0xFFFFFFFFu : static_cast<uint32_t>(t);
    };
    RmatGen gen{seed_premix(p.seed ^ kRmatSalt), p.scale, thr(p.a), thr(p.a + p.b),
                thr(p.a + p.b + p.c)};
    cudaStream_t st = nullptr;
    const int sms = sm_count(device);
    const int gblocks = sms * 8;

    // 1. degrees of the symmetrised multigraph (self-loops dropped)
    DeviceBuffer<unsigned> deg(V);
    WF_CUDA(cudaMemsetAsync(deg.get(), 0, V * 4ull, st));
    k_rmat_count<<<gblocks, 256, 0, st>>>(gen, n_draws, deg.get());
    WF_LAUNCHED();
    // 2. offsets (u64)
    DeviceBuffer<uint64_t> off0(static_cast<size_t>(V) + 1);
    {
        size_t tmp_bytes = 0;
        cub::TransformInputIterator<uint64_t, WidenU64, const unsigned*> degw(deg.get(), WidenU64{});
        WF_CUDA(cudaMemsetAsync(off0.get(), 0, 8, st));
        cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, degw, off0.get() + 1, static_cast<int>(V), st);
        DeviceBuffer<uint8_t> tmp(tmp_bytes);
        WF_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tmp_bytes, degw, off0.get() + 1, static_cast<int>(V), st));
    }
    uint64_t E0 = 0;
    WF_CUDA(cudaMemcpyAsync(&E0, off0.get() + V, 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    deg.release();
    // 3. scatter both directions
    DeviceBuffer<uint32_t> raw(std::max<uint64_t>(E0, 1));
    {
        DeviceBuffer<unsigned long long> cursor(V);
        WF_CUDA(cudaMemcpyAsync(cursor.get(), off0.get(), V * 8ull, cudaMemcpyDeviceToDevice, st));
        k_rmat_fill<<<gblocks, 256, 0, st>>>(gen, n_draws, cursor.get(), raw.get());
        WF_LAUNCHED();
    }
    // 4. sort each adjacency list (segmented, chunked below 2^31 items)
    DeviceBuffer<uint32_t> sorted_buf(std::max<uint64_t>(E0, 1));
    {
        std::vector<uint64_t> h_off(static_cast<size_t>(V) + 1);
        WF_CUDA(cudaMemcpyAsync(h_off.data(), off0.get(), (V + 1ull) * 8, cudaMemcpyDeviceToHost, st));
        WF_CUDA(cudaStreamSynchronize(st));
        const uint64_t kChunk = 1ull << 30;
        uint32_t v0 = 0;
        DeviceBuffer<uint8_t> tmp;
        DeviceBuffer<int> seg_off;
        while (v0 < V) {
            uint32_t v1 = v0;
            // at least one vertex per chunk; a single vertex never exceeds 2^31 here
            while (v1 < V && (h_off[v1 + 1] - h_off[v0] <= kChunk || v1 == v0)) ++v1;
            uint64_t base = h_off[v0];
            uint64_t items = h_off[v1] - base;
            int nseg = static_cast<int>(v1 - v0);
            std::vector<int> so(static_cast<size_t>(nseg) + 1);
            for (int i = 0; i <= nseg; ++i) so[i] = static_cast<int>(h_off[v0 + i] - base);
            seg_off.allocate(so.size());
            WF_CUDA(cudaMemcpyAsync(seg_off.get(), so.data(), so.size() * 4, cudaMemcpyHostToDevice, st));
            if (items > 0) {
                size_t tb = 0;
                cub::DeviceSegmentedSort::SortKeys(nullptr, tb, raw.get() + base, sorted_buf.get() + base,
                                                   static_cast<int>(items), nseg, seg_off.get(),
                                                   seg_off.get() + 1, st);
                if (tb > tmp.size()) tmp.allocate(tb);
                WF_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp.get(), tb, raw.get() + base,
                                                           sorted_buf.get() + base,
                                                           static_cast<int>(items), nseg,
                                                           seg_off.get(), seg_off.get() + 1, st));
                count_launch();
            }
            WF_CUDA(cudaStreamSynchronize(st));
            v0 = v1;
        }
    }
    raw.release();
    // 5. dedup: distinct counts -> final offsets -> compaction
    DeviceBuffer<uint32_t> ndeg(V);
    const int wblocks = blocks_for(static_cast<uint64_t>(V) * 32, 256, device);
    k_dedup<<<wblocks, 256, 0, st>>>(off0.get(), sorted_buf.get(), V, ndeg.get(), nullptr, nullptr, 0);
    WF_LAUNCHED();
    auto g = std::make_unique<GraphStore>();
    g->device = device;
    g->V = V;
    g->offsets.allocate(static_cast<size_t>(V) + 1);
    {
        size_t tmp_bytes = 0;
        cub::TransformInputIterator<uint64_t, WidenU64, const uint32_t*> ndegw(ndeg.get(), WidenU64{});
        WF_CUDA(cudaMemsetAsync(g->offsets.get(), 0, 8, st));
        cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, ndegw, g->offsets.get() + 1, static_cast<int>(V), st);
        DeviceBuffer<uint8_t> tmp(tmp_bytes);
        WF_CUDA(cub::DeviceScan::InclusiveSum(tmp.get(), tmp_bytes, ndegw, g->offsets.get() + 1, static_cast<int>(V), st));
    }
    WF_CUDA(cudaMemcpyAsync(&g->E, g->offsets.get() + V, 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    g->nbr.allocate(g->E + kNbrPad);
    k_dedup<<<wblocks, 256, 0, st>>>(off0.get(), sorted_buf.get(), V, nullptr, g->offsets.get(),
                                     g->nbr.get(), 1);
    WF_LAUNCHED();
    sorted_buf.release();
    off0.release();
    // 6. attributes
    if (p.weighted) g->weights.allocate(std::max<uint64_t>(g->E, 1));
    if (p.label_count > 0) g->labels.allocate(std::max<uint64_t>(g->E, 1));
    if ((p.weighted || p.label_count) && g->E) {
        k_attributes<<<gblocks, 256, 0, st>>>(g->E, seed_premix(p.seed ^ kWeightSalt),
                                              seed_premix(p.seed ^ kLabelSalt), g->weights.get(),
                                              g->labels.get(), p.label_count);
        WF_LAUNCHED();
    }
    WF_CUDA(cudaStreamSynchronize(st));
    g->finalize(st);
    return g.release();
}

void graph_has_edge(const GraphStore& g, const uint32_t* src, const uint32_t* dst, uint64_t n,
                    uint8_t* out) {
    DeviceGuard guard(g.device);
    for (uint64_t i = 0; i < n; ++i)
        if (src[i] >= g.V) config_error("vertex id " + std::to_string(src[i]) + " out of range");
    DeviceBuffer<uint32_t> s(n), d(n);
    DeviceBuffer<uint8_t> o(n);
    WF_CUDA(cudaMemcpy(s.get(), src, n * 4, cudaMemcpyHostToDevice));
    WF_CUDA(cudaMemcpy(d.get(), dst, n * 4, cudaMemcpyHostToDevice));
    k_has_edge<<<blocks_for(n, 256, g.device), 256>>>(g.view(), s.get(), d.get(), n, o.get());
    WF_LAUNCHED();
    WF_CUDA(cudaMemcpy(out, o.get(), n, cudaMemcpyDeviceToHost));
}

}  // namespace wf
