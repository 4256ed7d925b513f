// Host-streaming instantiations of the walk kernel (walk_kernel<..., true>),
// used by run_to_host (stream.cu); a TU of their own so they compile beside
// walk.cu's.
#include "common.cuh"
#include "kernel_table.cuh"

namespace wf {

KernelFn select_stream_kernel(int prog, int sampler, int flow) {
#define WF_CASE(P, S, F) \
    if (prog == P && sampler == S && flow == F) return &walk_kernel<Program<P>, S, F, true>;
    WF_FOR_EACH_COMBO(WF_CASE)
#undef WF_CASE
    config_error("no kernel for this program/sampler/flow combination");
}

}  // namespace wf
