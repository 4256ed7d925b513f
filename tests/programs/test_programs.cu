// User-written device programs (TEST CODE): the custom programs of the
// reference's own engine tests, re-expressed against the device program API
// (include/walkforge_b200/device_program.cuh) exactly as a user of the engine
// would write them, plus two that exercise the rest of the concept.  The same
// programs written against the reference API live in oracle/ref_harness.cpp
// (wfref_run_test_program); tests/test_custom_programs_gpu.py checks the two
// bit for bit.
//
//   CountingProgram       /root/reference/proj/tests/test_engine.cpp:17-27
//   AvoidVertexProgram    /root/reference/proj/tests/test_engine.cpp:29-40
//   NegativeWeightProgram /root/reference/proj/tests/test_engine.cpp:42-46
//   LabelWeightProgram    SURVEY §8 A7: weighted MetaPath (weight = label match ? w_e : 0),
//                         a dynamic program with no reference built-in
//   LabelStopProgram      unbiased, unbounded: update() draws a stop coin and reads the
//                         traversed edge's label (EdgeRef in update, rng in update)
//
// Built by __graft_entry__.build() into tests/programs/libwf_test_programs.so.
#include <walkforge_b200/device_program.cuh>

namespace wfd = walkforge_b200::device;

struct CountingProgram {
    uint32_t length;
    unsigned long long* updates;  // device counter: update() calls

    static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Unbiased;
    __device__ double weight(const wfd::WalkerView*, const wfd::EdgeRef&) const { return 1.0; }
    __device__ bool update(wfd::WalkerView& q, const wfd::EdgeRef&) const {
        atomicAdd(updates, 1ull);
        return q.path_size() >= length;
    }
    // no finished(): a walk always makes one move, so length 1 still emits two vertices
    __host__ __device__ uint32_t max_path_vertices() const { return length < 2 ? 2 : length; }
};

struct AvoidVertexProgram {
    uint32_t banned;
    uint32_t length;

    static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Static;
    __device__ double weight(const wfd::WalkerView*, const wfd::EdgeRef& e) const {
        return e.dst() == banned ? 0.0 : 1.0;
    }
    __device__ bool update(wfd::WalkerView& q, const wfd::EdgeRef&) const { return q.path_size() >= length; }
    __host__ __device__ double max_weight() const { return 1.0; }
    // no finished(): a walk always makes one move, so length 1 still emits two vertices
    __host__ __device__ uint32_t max_path_vertices() const { return length < 2 ? 2 : length; }
};

struct NegativeWeightProgram {
    uint32_t unused;

    static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Static;
    __device__ double weight(const wfd::WalkerView*, const wfd::EdgeRef&) const { return -1.0; }
    __device__ bool update(wfd::WalkerView&, const wfd::EdgeRef&) const { return true; }
};

struct LabelWeightProgram {
    uint32_t schema_len;
    uint32_t schema[48];

    static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Dynamic;
    __device__ double weight(const wfd::WalkerView* q, const wfd::EdgeRef& e) const {
        if (q == nullptr) return 0.0;
        return e.label() == schema[q->moves()] ? e.weight() : 0.0;
    }
    __device__ bool update(wfd::WalkerView& q, const wfd::EdgeRef&) const { return q.moves() >= schema_len; }
    __device__ bool finished(const wfd::WalkerView& q) const { return q.moves() >= schema_len; }
    __host__ __device__ uint32_t max_path_vertices() const { return schema_len + 1; }
};

struct LabelStopProgram {
    double stop;
    uint32_t stop_label;

    static constexpr wfd::WalkerType walker_type = wfd::WalkerType::Unbiased;
    __device__ double weight(const wfd::WalkerView*, const wfd::EdgeRef&) const { return 1.0; }
    __device__ bool update(wfd::WalkerView& q, const wfd::EdgeRef& e) const {
        const bool coin = q.rng().uniform_real(1.0) < stop;
        return coin || e.label() == stop_label;
    }
    __host__ __device__ double max_weight() const { return 1.0; }
};

WF_DEVICE_PROGRAM(CountingProgram, wf_test_counting_program)
WF_DEVICE_PROGRAM(AvoidVertexProgram, wf_test_avoid_vertex_program)
WF_DEVICE_PROGRAM(NegativeWeightProgram, wf_test_negative_weight_program)
WF_DEVICE_PROGRAM(LabelWeightProgram, wf_test_label_weight_program)
WF_DEVICE_PROGRAM(LabelStopProgram, wf_test_label_stop_program)

// A counting program owns device memory of its own: these let a plain C++
// caller (tests/cpp/ref_suite.cpp, compiled with g++) create and read the
// counter CountingProgram::updates points at.
extern "C" unsigned long long* wf_test_counter_new(void) {
    unsigned long long* p = nullptr;
    if (cudaMalloc(&p, sizeof(*p)) != cudaSuccess) return nullptr;
    cudaMemset(p, 0, sizeof(*p));
    return p;
}
extern "C" unsigned long long wf_test_counter_read(const unsigned long long* p) {
    unsigned long long v = 0;
    cudaMemcpy(&v, p, sizeof(v), cudaMemcpyDeviceToHost);
    return v;
}
extern "C" void wf_test_counter_free(unsigned long long* p) { cudaFree(p); }
