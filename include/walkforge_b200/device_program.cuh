// walkforge_b200/device_program.cuh — write your own walk program for the
// device engine: the reference's WalkProgram concept (program.hpp:49-93) as a
// C++ type with __device__ members, compiled in YOUR .cu translation unit.
//
//   #include <walkforge_b200/device_program.cuh>
//   namespace wfd = walkforge_b200::device;
//
//   struct AvoidVertex {                       // tests/test_engine.cpp:29-40
//       uint32_t banned, length;
//       static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Static;
//       __device__ double weight(const wfd::WalkerView*, const wfd::EdgeRef& e) const {
//           return e.dst() == banned ? 0.0 : 1.0;
//       }
//       __device__ bool update(wfd::WalkerView& q, const wfd::EdgeRef&) const {
//           return q.path_size() >= length;
//       }
//       __host__ __device__ double max_weight() const { return 1.0; }
//   };
//   WF_DEVICE_PROGRAM(AvoidVertex, avoid_vertex_ops)   // extern "C" const wf_program_ops* avoid_vertex_ops()
//
// then wf_session_create_custom(graph, avoid_vertex_ops(), &prog, &opts, &session)
// and every run / launch / streaming entry point of walkforge_b200.h, or the
// C++ shim's run_sequential / run_interleaved (walkforge_b200/engine.hpp),
// which accept such a program directly.
//
// The concept, member by member (reference → here):
//   walker_type()                 static constexpr WalkerType walker_type
//   weight(const Walker* q, e)    __device__ double weight(const WalkerView* q, const EdgeRef& e) const
//                                 (q null in static contexts: preprocessing, table REJ)
//   update(Walker& q, e)          __device__ bool update(WalkerView& q, const EdgeRef& e) const
//                                 (once per completed move, path already extended; the
//                                 only place that may draw: q.rng().uniform_real(...))
//   max_weight()   [optional]     __host__ __device__ double max_weight() const
//   preferred_sampler() [opt.]    static constexpr wf_sampler preferred_sampler
//   finished(q)    [optional]     __device__ bool finished(const WalkerView& q) const
//   (device only)  [optional]     __host__ __device__ uint32_t max_path_vertices() const: a
//                                 bound on a walk's vertices (fixed-length programs); without
//                                 it rows are path_stride long and longer walks are re-run
//                                 into bigger rows (update() then runs again for them)
//
// WalkerView: id(), cur(), prev() (after one move), path_size(), moves(),
// rng() — the walker's own RngStream(seed, qid).  EdgeRef: src(), index()
// (global edge index), dst(), weight() (f64, as the reference), label().
// The program object must be trivially copyable and at most 256 bytes: it
// travels in the kernel's parameter space.  Walks are bit-identical to the
// reference engine running the same program with the same seed.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <type_traits>

#include "../walkforge_b200.h"
#include "device/engine.cuh"

namespace walkforge_b200 {
namespace device {

enum class WalkerType : int { Unbiased = wf::kUnbiased, Static = wf::kStatic, Dynamic = wf::kDynamic };

using wf::EdgeRef;
using wf::WalkerRng;
using wf::WalkerView;

namespace detail {

template <class U, class = void>
struct preferred_of {
    static constexpr int value = WF_SAMPLER_DEFAULT;
};
template <class U>
struct preferred_of<U, std::void_t<decltype(U::preferred_sampler)>> {
    static constexpr int value = static_cast<int>(U::preferred_sampler);
};
template <class U, class = void>
struct has_max_path : std::false_type {};
template <class U>
struct has_max_path<U, std::void_t<decltype(std::declval<const U&>().max_path_vertices())>> : std::true_type {};

using Kernel = void (*)(const wf::WalkLaunch);

// The legal (sampler, flow) pairings for U (resolve_flow, engine.hpp:255-272):
// NAIVE only for unbiased programs, O-REJ only with max_weight(), tables only
// for non-dynamic programs; gathered ITS / ALIAS / REJ always.
template <class U, bool ST>
Kernel select(int sampler, int flow) {
    using P = wf::Custom<U>;
    if constexpr (P::type == wf::kUnbiased)
        if (sampler == WF_SAMPLER_NAIVE && flow == wf::kDirect)
            return &wf::walk_kernel<P, WF_SAMPLER_NAIVE, wf::kDirect, ST>;
    if constexpr (P::has_max_weight)
        if (sampler == WF_SAMPLER_OREJ && flow == wf::kDirect)
            return &wf::walk_kernel<P, WF_SAMPLER_OREJ, wf::kDirect, ST>;
    if constexpr (P::type != wf::kDynamic) {
        if (flow == wf::kTables) {
            if (sampler == WF_SAMPLER_ITS) return &wf::walk_kernel<P, WF_SAMPLER_ITS, wf::kTables, ST>;
            if (sampler == WF_SAMPLER_ALIAS) return &wf::walk_kernel<P, WF_SAMPLER_ALIAS, wf::kTables, ST>;
            if (sampler == WF_SAMPLER_REJ) return &wf::walk_kernel<P, WF_SAMPLER_REJ, wf::kTables, ST>;
        }
    }
    if (flow == wf::kGathered) {
        if (sampler == WF_SAMPLER_ITS) return &wf::walk_kernel<P, WF_SAMPLER_ITS, wf::kGathered, ST>;
        if (sampler == WF_SAMPLER_ALIAS) return &wf::walk_kernel<P, WF_SAMPLER_ALIAS, wf::kGathered, ST>;
        if (sampler == WF_SAMPLER_REJ) return &wf::walk_kernel<P, WF_SAMPLER_REJ, wf::kGathered, ST>;
    }
    return nullptr;
}

template <class U>
Kernel select(int sampler, int flow, int streaming) {
    return streaming ? select<U, true>(sampler, flow) : select<U, false>(sampler, flow);
}

template <class U>
int launch(const void* walk_launch, int32_t sampler, int32_t flow, int32_t streaming, int32_t grid,
           void* stream) {
    Kernel k = select<U>(sampler, flow, streaming);
    if (!k) return static_cast<int>(cudaErrorInvalidValue);
    k<<<grid, wf::kBlock, 0, static_cast<cudaStream_t>(stream)>>>(
        *static_cast<const wf::WalkLaunch*>(walk_launch));
    return static_cast<int>(cudaGetLastError());
}

template <class U>
int occupancy(int32_t sampler, int32_t flow, int32_t streaming, int32_t* blocks_per_sm, int32_t* regs) {
    Kernel k = select<U>(sampler, flow, streaming);
    if (!k) return static_cast<int>(cudaErrorInvalidValue);
    int b = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, wf::kBlock, 0);
    if (e != cudaSuccess) return static_cast<int>(e);
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) return static_cast<int>(e);
    if (blocks_per_sm) *blocks_per_sm = b;
    if (regs) *regs = fa.numRegs;
    return 0;
}

// weight(nullptr, e) for every edge, a warp per vertex (EdgeRef needs the
// source), with check_program_weight (engine.hpp:97-101).
template <class U>
__global__ void k_static_weights(const wf::GraphView g, const U prog, double* __restrict__ out,
                                 int32_t* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
    const uint64_t warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t v = warp; v < g.V; v += warps) {
        const uint64_t a = g.offsets[v], b = g.offsets[v + 1];
        for (uint64_t e = a + lane; e < b; e += 32) {
            const double w = prog.weight(static_cast<const WalkerView*>(nullptr),
                                         EdgeRef(g, static_cast<uint32_t>(v), e));
            if (!(w >= 0.0 && w <= 1.7976931348623157e308)) atomicExch(bad, 1);
            out[e] = w;
        }
    }
}

template <class U>
int static_weights(const void* graph_view, const void* program, double* out, int32_t* bad, void* stream) {
    const wf::GraphView& g = *static_cast<const wf::GraphView*>(graph_view);
    U prog;
    memcpy(static_cast<void*>(&prog), program, sizeof(U));
    int sms = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t want = (static_cast<uint64_t>(g.V) * 32 + 255) / 256;
    const int blocks = static_cast<int>(want < static_cast<uint64_t>(sms) * 16 ? (want ? want : 1) : sms * 16);
    k_static_weights<U><<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(g, prog, out, bad);
    return static_cast<int>(cudaGetLastError());
}

template <class U>
double max_weight(const void* program) {
    if constexpr (wf::Custom<U>::has_max_weight) {
        U prog;
        memcpy(static_cast<void*>(&prog), program, sizeof(U));
        return prog.max_weight();
    } else {
        return 0.0;
    }
}

template <class U>
uint32_t max_path(const void* program) {
    if constexpr (has_max_path<U>::value) {
        U prog;
        memcpy(static_cast<void*>(&prog), program, sizeof(U));
        return prog.max_path_vertices();
    } else {
        return 0;
    }
}

template <class U>
const wf_program_ops* ops_for(const char* name) {
    using P = wf::Custom<U>;
    static const wf_program_ops ops = {
        WF_ABI_VERSION,
        static_cast<uint32_t>(sizeof(wf::WalkLaunch)),
        name,
        P::type,
        preferred_of<U>::value,
        P::has_max_weight ? 1 : 0,
        P::prechecked ? 1 : 0,
        static_cast<uint32_t>(sizeof(U)),
        wf::kEngineAbi,
        &launch<U>,
        &occupancy<U>,
        &static_weights<U>,
        &max_weight<U>,
        &max_path<U>,
    };
    return &ops;
}

}  // namespace detail
}  // namespace device
}  // namespace walkforge_b200

// Instantiates the walk kernel for `Type` and exports its operations table as
// `extern "C" const wf_program_ops* symbol(void)`.
#define WF_DEVICE_PROGRAM(Type, symbol)                                                 \
    extern "C" const wf_program_ops* symbol(void) {                                   \
        return ::walkforge_b200::device::detail::ops_for<Type>(#Type);                 \
    }
