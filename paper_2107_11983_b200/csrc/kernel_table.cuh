// The walk kernel instantiations: every program x sampler x flow pairing the
// reference accepts (resolve_flow, engine.hpp:255-272; the 30 legal
// combinations of acceptance.cpp:234-283 plus UniformProgram).
#pragma once

#include "common.cuh"
#include "walkforge_b200/device/engine.cuh"

namespace wf {

using KernelFn = void (*)(const WalkLaunch);

#define WF_UNBIASED_COMBOS(X, P)   \
    X(P, WF_SAMPLER_NAIVE, kDirect) \
    X(P, WF_SAMPLER_OREJ, kDirect)  \
    X(P, WF_SAMPLER_ITS, kTables)   \
    X(P, WF_SAMPLER_ALIAS, kTables) \
    X(P, WF_SAMPLER_REJ, kTables)   \
    X(P, WF_SAMPLER_ITS, kGathered) \
    X(P, WF_SAMPLER_ALIAS, kGathered) \
    X(P, WF_SAMPLER_REJ, kGathered)

#define WF_FOR_EACH_COMBO(X)                               \
    WF_UNBIASED_COMBOS(X, WF_PROGRAM_PPR)                  \
    WF_UNBIASED_COMBOS(X, WF_PROGRAM_UNIFORM)              \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_OREJ, kDirect)       \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_ITS, kTables)        \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_ALIAS, kTables)      \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_REJ, kTables)        \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_ITS, kGathered)      \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_ALIAS, kGathered)    \
    X(WF_PROGRAM_DEEPWALK, WF_SAMPLER_REJ, kGathered)      \
    X(WF_PROGRAM_NODE2VEC, WF_SAMPLER_OREJ, kDirect)       \
    X(WF_PROGRAM_NODE2VEC, WF_SAMPLER_ITS, kGathered)      \
    X(WF_PROGRAM_NODE2VEC, WF_SAMPLER_ALIAS, kGathered)    \
    X(WF_PROGRAM_NODE2VEC, WF_SAMPLER_REJ, kGathered)      \
    X(WF_PROGRAM_METAPATH, WF_SAMPLER_ITS, kGathered)      \
    X(WF_PROGRAM_METAPATH, WF_SAMPLER_ALIAS, kGathered)    \
    X(WF_PROGRAM_METAPATH, WF_SAMPLER_REJ, kGathered)

// walk_stream.cu: the host-streaming instantiation for a combination
KernelFn select_stream_kernel(int prog, int sampler, int flow);

}  // namespace wf
