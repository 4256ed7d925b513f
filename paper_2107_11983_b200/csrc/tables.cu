// Static-Gather preprocessing on the device: preprocess_static
// (engine.hpp:190-251) for ALIAS, ITS and REJ, one thread per vertex.
//
// Per vertex the reference sums the weights sequentially (engine.hpp:218-226),
// marks the vertex exhausted when the sum is not positive, and builds
//   ALIAS  Vose's table with FIFO worklists (sampler.hpp:89-120), decorated with
//          destinations (engine.hpp:118-127);
//   ITS    the running-sum cumulative table (engine.hpp:232-238);
//   REJ    p* = max weight (engine.hpp:244-246).
// Everything runs in fp64 in the reference's operation order, so the tables are
// bit-identical (checked against the reference's own preprocess_static output
// in tests/test_engine_gpu.py).  The ALIAS build replays the FIFO worklists with
// three ascending cursors and parks demoted larges' values in their own
// output bucket, so it needs no E-sized scratch (SURVEY §7 hard part 1).
//
// Device bucket (16 B): {u64 thr = ceil(split * 2^53), u32 first_dst,
// u32 second_dst}; `y < split` with y = uniform_real(1.0) is exactly
// `(r >> 11) < thr` (rng.cuh unit_threshold).
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "runtime.hpp"

namespace wf {

namespace {

struct UnitWeight {
    __device__ __forceinline__ double operator()(uint64_t) const { return 1.0; }
};
struct EdgeWeight {  // the graph's weights (f64 when they are not all float32-exact)
    const float* __restrict__ w;
    const double* __restrict__ w64;
    __device__ __forceinline__ double operator()(uint64_t e) const {
        return w64 ? __ldg(w64 + e) : static_cast<double>(__ldg(w + e));
    }
};
struct F64Weight {  // a custom program's weight(nullptr, e), materialised once
    const double* __restrict__ w;
    __device__ __forceinline__ double operator()(uint64_t e) const { return __ldg(w + e); }
};

__device__ __forceinline__ void store_bucket(uint4* b, double split, uint32_t first_dst,
                                             uint32_t second_dst) {
    uint64_t thr = unit_threshold(split);
    *b = make_uint4(static_cast<uint32_t>(thr), static_cast<uint32_t>(thr >> 32), first_dst, second_dst);
}

__device__ __forceinline__ void park(uint4* b, double v) {
    uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
    b->x = static_cast<uint32_t>(bits);
    b->y = static_cast<uint32_t>(bits >> 32);
}

__device__ __forceinline__ double unpark(const uint4* b) {
    uint64_t bits = (static_cast<uint64_t>(b->y) << 32) | b->x;
    return __longlong_as_double(static_cast<long long>(bits));
}

// IDX: buckets carry the positions {first, second} in E_v (EngineAliasSlot,
// engine.hpp:22-28) instead of their destinations.
// ITS and REJ: vertices with at least kHubDeg edges are built by a warp
// (k_*_warp below), the rest one thread per vertex.  ALIAS stays one thread
// per vertex: Vose's pairing loop is an order-dependent fp64 chain, and a
// warp replaying it for a hub (cursor scans by ballot over a row of scaled
// weights) measured far slower at C5 — 11.3 s against 0.12 s for the whole
// per-thread build: the chain serialises on L2 round trips, and a row per
// warp left too few warps for the ~10^5 vertices of 1000+ edges.
constexpr uint32_t kHubDeg = 64;

// Vose's construction for one vertex of n edges (sampler.hpp:89-120) with the
// scaled weights given by `scaled(i)` (w_i * n / sum, sampler.hpp:97), three
// ascending cursors replaying the FIFO worklists, demoted larges parked in
// their own output bucket.
template <bool IDX, typename Scaled>
__device__ void vose_vertex(uint32_t n, Scaled scaled, const uint32_t* __restrict__ nb, uint4* __restrict__ out,
                            uint32_t bs) {
    auto dst = [&](uint32_t i) { return IDX ? i : nb[i]; };
    {
        auto next_large = [&](uint32_t from) {
            while (from < n && !(scaled(from) >= 1.0)) ++from;
            return from;
        };
        auto next_small = [&](uint32_t from) {
            while (from < n && !(scaled(from) < 1.0)) ++from;
            return from;
        };
        uint32_t lcur = next_large(0);
        double lval = lcur < n ? scaled(lcur) : 0.0;
        uint32_t a = next_small(0);
        uint32_t c = 0, demoted = 0, consumed = 0;
        while (lcur < n) {  // sampler.hpp:103-111
            uint32_t s;
            double sval;
            if (a < n) {
                s = a;
                sval = scaled(a);
                a = next_small(a + 1);
            } else if (consumed < demoted) {
                c = next_large(c);
                s = c;
                sval = unpark(out + c * bs);
                ++c;
                ++consumed;
            } else {
                break;
            }
            store_bucket(out + s * bs, sval, dst(s), dst(lcur));
            lval -= 1.0 - sval;
            if (lval < 1.0) {
                park(out + lcur * bs, lval);
                ++demoted;
                lcur = next_large(lcur + 1);
                if (lcur < n) lval = scaled(lcur);
            }
        }
        // leftovers at probability exactly 1 (sampler.hpp:112-119)
        for (uint32_t s = a; s < n; s = next_small(s + 1)) store_bucket(out + s * bs, 1.0, dst(s), dst(s));
        while (consumed < demoted) {
            c = next_large(c);
            store_bucket(out + c * bs, 1.0, dst(c), dst(c));
            ++c;
            ++consumed;
        }
        for (uint32_t l = lcur; l < n; l = next_large(l + 1)) store_bucket(out + l * bs, 1.0, dst(l), dst(l));
    }
}

template <typename WF, bool IDX>
__global__ void k_static_alias(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr,
                               uint32_t V, WF wf, uint4* __restrict__ bucket, uint32_t bs,
                               uint8_t* __restrict__ exhausted, unsigned* any_exhausted) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a0 = off[v];
        const uint32_t n = static_cast<uint32_t>(off[v + 1] - a0);
        if (n == 0) continue;
        double sum = 0.0;
        for (uint32_t i = 0; i < n; ++i) sum += wf(a0 + i);  // engine.hpp:218-226
        if (!(sum > 0.0)) {
            exhausted[v] = 1;
            atomicOr(any_exhausted, 1u);
            continue;
        }
        vose_vertex<IDX>(n, [&](uint32_t i) { return wf(a0 + i) * n / sum; }, nbr + a0, bucket + a0 * bs, bs);
    }
}

// ---- hubs: a warp per vertex ---------------------------------------------------------
// The reference sums a vertex's weights in edge order (engine.hpp:218-226).  A
// warp's reordered sum is the same number when every partial sum is exact:
// all weights multiples of 2^q and the total below 2^(52+q) (f32 weights in
// [1,5) qualify with room to spare; SURVEY 8(a) verified the reordered ITS
// scan on 32 M entries).  Otherwise lane 0 sums in edge order.
__device__ __forceinline__ int quantum_of(double w) {  // exponent of the lowest set bit of w > 0
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(w));
    const int e = static_cast<int>((b >> 52) & 0x7FF);
    const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (e ? (1ull << 52) : 0ull);
    return (e ? e : 1) - 1075 + __ffsll(static_cast<long long>(m)) - 1;
}

// Sum and max of a vertex's weights as the reference computes them; every
// lane returns the same values.
template <typename WF>
__device__ __forceinline__ void warp_sum_max(WF wf, uint64_t a0, uint32_t n, double& sum, double& mx, bool& exact) {
    const int lane = threadIdx.x & 31;
    double ls = 0.0, lm = 0.0;
    int q = 0x7FFFFFFF;
    for (uint32_t i = lane; i < n; i += 32) {
        const double w = wf(a0 + i);
        ls += w;
        lm = w > lm ? w : lm;
        if (w > 0.0) q = min(q, quantum_of(w));
    }
    for (int o = 16; o > 0; o >>= 1) {
        ls += __shfl_xor_sync(0xFFFFFFFFu, ls, o);
        const double m2 = __shfl_xor_sync(0xFFFFFFFFu, lm, o);
        lm = m2 > lm ? m2 : lm;
        q = min(q, __shfl_xor_sync(0xFFFFFFFFu, q, o));
    }
    exact = ls < ldexp(1.0, 52 + max(q, -1000));
    if (!exact) {  // the edge-order sum, by lane 0
        double seq = 0.0;
        if (lane == 0)
            for (uint32_t i = 0; i < n; ++i) seq += wf(a0 + i);
        ls = __shfl_sync(0xFFFFFFFFu, seq, 0);
    }
    sum = ls;
    mx = lm;
}

template <typename WF>
__global__ void k_static_its(const uint64_t* __restrict__ off, uint32_t V, WF wf,
                             double* __restrict__ cum, uint8_t* __restrict__ exhausted,
                             unsigned* any_exhausted) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a0 = off[v];
        const uint32_t n = static_cast<uint32_t>(off[v + 1] - a0);
        if (n == 0 || n >= kHubDeg) continue;
        double run = 0.0;
        for (uint32_t i = 0; i < n; ++i) {
            run += wf(a0 + i);
            cum[a0 + i] = run;
        }
        if (!(run > 0.0)) {
            exhausted[v] = 1;
            atomicOr(any_exhausted, 1u);
        }
    }
}

// ITS for hubs: the running sums (engine.hpp:232-238) as a segmented scan, 32
// edges per round, when the reordering is exact; else lane 0 in edge order.
template <typename WF>
__global__ void k_static_its_warp(const uint64_t* __restrict__ off, uint32_t V, WF wf,
                                  double* __restrict__ cum, uint8_t* __restrict__ exhausted,
                                  unsigned* any_exhausted) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        const uint64_t a0 = off[v];
        const uint32_t n = static_cast<uint32_t>(off[v + 1] - a0);
        if (n < kHubDeg) continue;
        double sum, mx;
        bool exact;
        warp_sum_max(wf, a0, n, sum, mx, exact);
        if (exact) {
            double running = 0.0;
            for (uint32_t c = 0; c < n; c += 32) {
                const uint32_t i = c + lane;
                double x = i < n ? wf(a0 + i) : 0.0;
                for (int o = 1; o < 32; o <<= 1) {
                    const double u = __shfl_up_sync(0xFFFFFFFFu, x, o);
                    if (lane >= o) x += u;
                }
                if (i < n) cum[a0 + i] = running + x;
                running += __shfl_sync(0xFFFFFFFFu, x, 31);
            }
        } else if (lane == 0) {
            double run = 0.0;
            for (uint32_t i = 0; i < n; ++i) {
                run += wf(a0 + i);
                cum[a0 + i] = run;
            }
        }
        if (!(sum > 0.0) && lane == 0) {
            exhausted[v] = 1;
            atomicOr(any_exhausted, 1u);
        }
    }
}

template <typename WF>
__global__ void k_static_rej(const uint64_t* __restrict__ off, uint32_t V, WF wf,
                             double* __restrict__ pstar, uint8_t* __restrict__ exhausted,
                             unsigned* any_exhausted) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a0 = off[v];
        const uint32_t n = static_cast<uint32_t>(off[v + 1] - a0);
        if (n == 0 || n >= kHubDeg) continue;
        double sum = 0.0, mx = 0.0;
        for (uint32_t i = 0; i < n; ++i) {
            double w = wf(a0 + i);
            sum += w;
            mx = w > mx ? w : mx;
        }
        if (!(sum > 0.0)) {
            exhausted[v] = 1;
            atomicOr(any_exhausted, 1u);
        } else {
            pstar[v] = mx;
        }
    }
}

// REJ for hubs: p* = max weight (engine.hpp:244-246), exact in any order;
// exhausted iff no weight is positive.
template <typename WF>
__global__ void k_static_rej_warp(const uint64_t* __restrict__ off, uint32_t V, WF wf,
                                  double* __restrict__ pstar, uint8_t* __restrict__ exhausted,
                                  unsigned* any_exhausted) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t v = warp; v < V; v += nwarps) {
        const uint64_t a0 = off[v];
        const uint32_t n = static_cast<uint32_t>(off[v + 1] - a0);
        if (n < kHubDeg) continue;
        double mx = 0.0;
        for (uint32_t i = lane; i < n; i += 32) {
            const double w = wf(a0 + i);
            mx = w > mx ? w : mx;
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double m2 = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
            mx = m2 > mx ? m2 : mx;
        }
        if (lane == 0) {
            if (!(mx > 0.0)) {
                exhausted[v] = 1;
                atomicOr(any_exhausted, 1u);
            } else {
                pstar[v] = mx;
            }
        }
    }
}

__global__ void k_sampling_view(const uint64_t* __restrict__ vword, const uint8_t* __restrict__ ex,
                                uint32_t V, uint64_t* __restrict__ out) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < V;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t w = vword[v];
        // exhausted: degree 0 (dead end, no draws).  Escaped words keep their
        // escape only when live.
        out[v] = ex[v] ? (w & ~static_cast<uint64_t>(kDegEscape)) : w;
    }
}

// Second half of each wide bucket: the sampling-view vertex words of its two
// destinations, so a move lands with the next vertex's (base, degree) in hand.
__global__ void k_decorate_alias(uint4* __restrict__ bucket, uint64_t E,
                                 const uint64_t* __restrict__ sview) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint4 b = bucket[2 * e];
        uint64_t w1 = sview[b.z], w2 = sview[b.w];
        bucket[2 * e + 1] = make_uint4(static_cast<uint32_t>(w1), static_cast<uint32_t>(w1 >> 32),
                                       static_cast<uint32_t>(w2), static_cast<uint32_t>(w2 >> 32));
    }
}

// Packed decorated adjacency: dst | deg << vbits | base << (vbits + dbits).
__global__ void k_decorate_adj8(const uint32_t* __restrict__ nbr, uint64_t E, const uint64_t* __restrict__ vword,
                                const uint64_t* __restrict__ off, uint32_t vbits, uint32_t dbits,
                                unsigned long long* __restrict__ adj8) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = nbr[e];
        const uint64_t base = off[d];
        const uint64_t deg = off[d + 1] - base;
        adj8[e] = d | (deg << vbits) | (base << (vbits + dbits));
    }
}

// Decorated adjacency for Direct flows (NAIVE / O-REJ): {dst, 0, word(dst)}.
__global__ void k_decorate_adj(const uint32_t* __restrict__ nbr, uint64_t E,
                               const uint64_t* __restrict__ vword, uint4* __restrict__ adj) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E;
         e += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t d = nbr[e];
        uint64_t w = vword[d];
        adj[e] = make_uint4(d, 0u, static_cast<uint32_t>(w), static_cast<uint32_t>(w >> 32));
    }
}

template <typename WF>
void launch_tables(Session& s, WF wf, unsigned* any, cudaStream_t st) {
    GraphStore& g = *s.g;
    const int threads = 128;
    uint64_t blocks = (g.V + threads - 1) / threads;
    blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, static_cast<uint64_t>(sm_count(g.device)) * 64));
    // hubs (>= kHubDeg edges): a warp each, on a second stream beside the
    // per-thread kernel (the two touch disjoint vertices)
    const bool hubs = s.kind != WF_SAMPLER_ALIAS && g.max_degree >= kHubDeg;
    const int wblocks = sm_count(g.device) * 16;  // 8 warps per block
    cudaStream_t hs = st;
    cudaEvent_t ev = nullptr;
    if (hubs) {
        WF_CUDA(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
        WF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    auto fork = [&] {  // the hub stream starts after the buffers are ready
        if (!hubs) return;
        WF_CUDA(cudaEventRecord(ev, st));
        WF_CUDA(cudaStreamWaitEvent(hs, ev, 0));
    };
    if (s.kind == WF_SAMPLER_ALIAS) {
        const uint32_t bs = s.alias_wide ? 2 : 1;
        s.alias.allocate((g.E + 2) * bs);  // +2: 32 B reads of the last 16 B entry stay in bounds
        // buckets of exhausted vertices are never built; zero them so the
        // decoration pass reads valid vertex ids there
        WF_CUDA(cudaMemsetAsync(s.alias.get(), 0, s.alias.bytes(), st));
        fork();
        if (s.alias_idx)
            k_static_alias<WF, true><<<blocks, threads, 0, st>>>(g.offsets.get(), g.nbr.get(), g.V, wf,
                                                                 s.alias.get(), bs, s.exhausted.get(), any);
        else
            k_static_alias<WF, false><<<blocks, threads, 0, st>>>(g.offsets.get(), g.nbr.get(), g.V, wf,
                                                                  s.alias.get(), bs, s.exhausted.get(), any);
        WF_LAUNCHED();
    } else if (s.kind == WF_SAMPLER_ITS) {
        s.its.allocate(std::max<uint64_t>(g.E, 1));
        fork();
        k_static_its<<<blocks, threads, 0, st>>>(g.offsets.get(), g.V, wf, s.its.get(), s.exhausted.get(), any);
        WF_LAUNCHED();
        if (hubs) {
            k_static_its_warp<<<wblocks, 256, 0, hs>>>(g.offsets.get(), g.V, wf, s.its.get(), s.exhausted.get(), any);
            WF_LAUNCHED();
        }
    } else {
        s.rej.allocate(g.V);
        WF_CUDA(cudaMemsetAsync(s.rej.get(), 0, g.V * sizeof(double), st));
        fork();
        k_static_rej<<<blocks, threads, 0, st>>>(g.offsets.get(), g.V, wf, s.rej.get(), s.exhausted.get(), any);
        WF_LAUNCHED();
        if (hubs) {
            k_static_rej_warp<<<wblocks, 256, 0, hs>>>(g.offsets.get(), g.V, wf, s.rej.get(), s.exhausted.get(), any);
            WF_LAUNCHED();
        }
    }
    if (hubs) {  // join: the caller's stream continues after both
        WF_CUDA(cudaEventRecord(ev, hs));
        WF_CUDA(cudaStreamWaitEvent(st, ev, 0));
        WF_CUDA(cudaStreamSynchronize(hs));
        cudaEventDestroy(ev);
        cudaStreamDestroy(hs);
    }
}

}  // namespace

void Session::build_tables(cudaStream_t st) {
    GraphStore& gs = *g;
    DeviceGuard guard(gs.device);
    auto t0 = std::chrono::steady_clock::now();
    exhausted.allocate(gs.V);
    WF_CUDA(cudaMemsetAsync(exhausted.get(), 0, gs.V, st));
    DeviceBuffer<unsigned> any(1);
    WF_CUDA(cudaMemsetAsync(any.get(), 0, 4, st));
    bool edge_weight = desc.kind == WF_PROGRAM_DEEPWALK && desc.weighted;
    DeviceBuffer<double> custom_w;
    if (custom) {
        // weight(nullptr, e) over every edge by the program's own kernel, with
        // check_program_weight (engine.hpp:97-101) on each
        custom_w.allocate(std::max<uint64_t>(gs.E, 1));
        DeviceBuffer<int> bad(1);
        WF_CUDA(cudaMemsetAsync(bad.get(), 0, 4, st));
        const GraphView gv = gs.view();
        const int rc = custom->static_weights(&gv, params.user, custom_w.get(), bad.get(), st);
        if (rc != 0) raise(WF_ERR_CUDA, std::string("custom program static weights: ") +
                                            cudaGetErrorString(static_cast<cudaError_t>(rc)));
        count_launch();
        int h_bad = 0;
        WF_CUDA(cudaMemcpyAsync(&h_bad, bad.get(), 4, cudaMemcpyDeviceToHost, st));
        WF_CUDA(cudaStreamSynchronize(st));
        if (h_bad) raise(WF_ERR_CONTRACT, "program emitted a weight that is negative or not finite");
        launch_tables(*this, F64Weight{custom_w.get()}, any.get(), st);
    } else if (edge_weight) {
        launch_tables(*this, EdgeWeight{gs.weights.get(), gs.weights64.get()}, any.get(), st);
    } else {
        launch_tables(*this, UnitWeight{}, any.get(), st);
    }
    unsigned h = 0;
    WF_CUDA(cudaMemcpyAsync(&h, any.get(), 4, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    const bool trace = getenv("WF_TRACE_PRE") != nullptr;  // diagnostics: phase times
    auto phase = [&](const char* what) {
        if (trace)
            std::fprintf(stderr, "[pre] %s %.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    };
    phase("tables");
    any_exhausted = h != 0;
    if (any_exhausted) {
        sview.allocate(gs.V);
        uint64_t blocks = std::min<uint64_t>((gs.V + 255) / 256, 65535);
        k_sampling_view<<<std::max<uint64_t>(blocks, 1), 256, 0, st>>>(gs.vword.get(), exhausted.get(), gs.V,
                                                                     sview.get());
        WF_LAUNCHED();
        WF_CUDA(cudaStreamSynchronize(st));
    }
    if (kind == WF_SAMPLER_ALIAS && alias_wide && gs.E) {
        const uint64_t* sv = any_exhausted ? sview.get() : gs.vword.get();
        int blocks = std::max(1, std::min<int>(static_cast<int>((gs.E + 255) / 256), sm_count(gs.device) * 32));
        k_decorate_alias<<<blocks, 256, 0, st>>>(alias.get(), gs.E, sv);
        WF_LAUNCHED();
        WF_CUDA(cudaStreamSynchronize(st));
        phase("decorate");
    }
    preprocess_seconds =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

namespace {
// Warp per vertex u over its label-partitioned edges: edge p of group l
// (label l) gets {dst, 0, word} with word = (base_g << 24 | count) of dst's
// group for label next[l]; ~0 when there is no successor label or the group
// does not fit the packed word (the kernel then reads dst's label record).
__global__ void k_metapath_successors(const uint4* __restrict__ rec, const uint32_t* __restrict__ lab_nbr,
                                      uint32_t V, const int* __restrict__ next,
                                      uint4* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t u = warp; u < V; u += nwarps) {
        uint4 r0 = rec[2 * u], r1 = rec[2 * u + 1];
        uint64_t base = (static_cast<uint64_t>(r0.y) << 32) | r0.x;
        uint32_t ends[kMaxIndexedLabels] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        uint32_t deg = ends[kMaxIndexedLabels - 1];
        for (uint32_t p = lane; p < deg; p += 32) {
            int l = 0;
            while (l < kMaxIndexedLabels - 1 && p >= ends[l]) ++l;
            uint32_t d = lab_nbr[base + p];
            uint64_t word = ~0ull;
            int nl = next[l];
            if (nl >= 0 && nl < kMaxIndexedLabels) {
                uint4 s0 = rec[2 * (uint64_t)d], s1 = rec[2 * (uint64_t)d + 1];
                uint64_t db = (static_cast<uint64_t>(s0.y) << 32) | s0.x;
                uint32_t de[kMaxIndexedLabels] = {s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
                uint32_t lo = nl == 0 ? 0 : de[nl - 1], hi = de[nl];
                uint64_t gb = db + lo;
                uint32_t cnt = hi - lo;
                if (cnt < kDegEscape && gb < (1ull << 40)) word = (gb << kDegBits) | cnt;
            }
            out[base + p] = make_uint4(d, 0u, static_cast<uint32_t>(word), static_cast<uint32_t>(word >> 32));
        }
    }
}
}  // namespace

bool Session::build_metapath_successors(cudaStream_t st) {
    GraphStore& gs = *g;
    if (!gs.label_index_built || schema.size() < 2) return false;
    int next[kMaxIndexedLabels];
    for (int i = 0; i < kMaxIndexedLabels; ++i) next[i] = -1;
    for (size_t i = 0; i + 1 < schema.size(); ++i) {
        uint32_t l = schema[i], n = schema[i + 1];
        if (l >= static_cast<uint32_t>(kMaxIndexedLabels)) return false;
        if (next[l] >= 0 && next[l] != static_cast<int>(n)) return false;  // not a function of l
        next[l] = static_cast<int>(n);
    }
    DeviceGuard guard(gs.device);
    auto t0 = std::chrono::steady_clock::now();
    DeviceBuffer<int> dnext(kMaxIndexedLabels);
    WF_CUDA(cudaMemcpy(dnext.get(), next, sizeof(next), cudaMemcpyHostToDevice));
    mp_adj.allocate(gs.E + 2);
    int blocks = std::max(1, std::min<int>(static_cast<int>((gs.V * 32ull + 255) / 256), sm_count(gs.device) * 32));
    k_metapath_successors<<<blocks, 256, 0, st>>>(gs.lab_rec.get(), gs.lab_nbr.get(), gs.V, dnext.get(),
                                                  mp_adj.get());
    WF_LAUNCHED();
    WF_CUDA(cudaStreamSynchronize(st));
    preprocess_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
}

bool Session::build_adjacency8(cudaStream_t st) {
    GraphStore& gs = *g;
    auto bits = [](uint64_t x) {  // bits to hold values 0..x
        uint32_t b = 1;
        while (b < 64 && (x >> b) != 0) ++b;
        return b;
    };
    const uint32_t vb = bits(gs.V - 1), db = bits(gs.max_degree), bb = bits(gs.E);
    if (vb + db + bb > 64 || gs.max_degree >= kDegEscape || gs.E >= (1ull << 40)) return false;
    DeviceGuard guard(gs.device);
    auto t0 = std::chrono::steady_clock::now();
    adj8.allocate(gs.E + 4);
    if (gs.E) {
        int blocks = std::max(1, std::min<int>(static_cast<int>((gs.E + 255) / 256), sm_count(gs.device) * 32));
        k_decorate_adj8<<<blocks, 256, 0, st>>>(gs.nbr.get(), gs.E, gs.vword.get(), gs.offsets.get(), vb, db,
                                                adj8.get());
        WF_LAUNCHED();
    }
    WF_CUDA(cudaStreamSynchronize(st));
    adj8_vbits = vb;
    adj8_dbits = db;
    preprocess_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
}

void Session::build_adjacency(cudaStream_t st) {
    GraphStore& gs = *g;
    DeviceGuard guard(gs.device);
    auto t0 = std::chrono::steady_clock::now();
    adj.allocate(gs.E + 2);
    if (gs.E) {
        int blocks = std::max(1, std::min<int>(static_cast<int>((gs.E + 255) / 256), sm_count(gs.device) * 32));
        k_decorate_adj<<<blocks, 256, 0, st>>>(gs.nbr.get(), gs.E, gs.vword.get(), adj.get());
        WF_LAUNCHED();
    }
    WF_CUDA(cudaStreamSynchronize(st));
    preprocess_seconds +=
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace wf

namespace wf {

void Session::copy_tables_from(const Session& src, cudaStream_t st) {
    DeviceGuard guard(g->device);
    auto t0 = std::chrono::steady_clock::now();
    auto peer = [&](auto& dst, const auto& from) {
        if (!from.get()) return;
        dst.allocate(from.size());
        WF_CUDA(cudaMemcpyPeerAsync(dst.get(), g->device, from.get(), src.g->device, from.bytes(), st));
    };
    peer(alias, src.alias);
    peer(its, src.its);
    peer(rej, src.rej);
    peer(exhausted, src.exhausted);
    peer(sview, src.sview);
    any_exhausted = src.any_exhausted;
    alias_wide = src.alias_wide;
    alias_idx = src.alias_idx;
    WF_CUDA(cudaStreamSynchronize(st));
    preprocess_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace wf
