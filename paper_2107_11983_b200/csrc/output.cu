// Walk-record encoding on the device (SURVEY §8 f, row 1): the reference's
// text and binary record formats (append_text_record / append_binary_record,
// proj/src/output.cpp:26-47), byte for byte, and a double-buffered file writer
// (DoubleBufferedWriter + OrderedBlockSink, output.cpp:49-200): block k is
// encoded on the device and copied to pinned memory while a host thread
// writes block k-1.
#include <cub/cub.cuh>

#include <cstdio>
#include <cstring>
#include <future>
#include <memory>
#include <vector>

#include "runtime.hpp"

namespace wf {

namespace {

__device__ __forceinline__ uint32_t ndigits(uint64_t x) {
    uint32_t d = 1;
    while (x >= 10000) { x /= 10000; d += 4; }
    while (x >= 10) { x /= 10; ++d; }
    return d;
}

__device__ __forceinline__ void put_dec(char* p, uint64_t x, uint32_t nd) {
    for (int i = static_cast<int>(nd) - 1; i >= 0; --i) {
        p[i] = static_cast<char>('0' + x % 10);
        x /= 10;
    }
}

__device__ __forceinline__ void put_le(char* p, uint64_t x, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = static_cast<char>((x >> (8 * i)) & 0xFF);
}

constexpr uint32_t kStatusChars = 8;  // "complete" / "dead_end" (walker.hpp:14-16)

// Warp per record: encoded byte size.
__global__ void k_record_size(const uint64_t* __restrict__ off, const uint32_t* __restrict__ verts,
                              uint64_t n, uint64_t qid_base, int fmt, uint64_t* __restrict__ size) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < n; r += nwarps) {
        const uint64_t a = off[r], len = off[r + 1] - a;
        if (fmt == WF_OUTPUT_BINARY) {
            if (lane == 0) size[r] = 8 + 1 + 4 + 4 * len;
            continue;
        }
        uint64_t s = 0;
        for (uint64_t j = lane; j < len; j += 32) s += ndigits(verts[a + j]);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
        if (lane == 0)
            size[r] = ndigits(qid_base + r) + 1 + kStatusChars + 1 + s + (len ? len - 1 : 0) + 1;
    }
}

__global__ void k_encode(const uint64_t* __restrict__ off, const uint32_t* __restrict__ verts,
                         const uint8_t* __restrict__ st, uint64_t n, uint64_t qid_base, int fmt,
                         const uint64_t* __restrict__ pos, char* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t r = warp; r < n; r += nwarps) {
        const uint64_t a = off[r], len = off[r + 1] - a;
        char* p = out + pos[r];
        const uint64_t qid = qid_base + r;
        if (fmt == WF_OUTPUT_BINARY) {  // output.cpp:40-47
            if (lane == 0) {
                put_le(p, qid, 8);
                p[8] = st[r] == WF_WALK_COMPLETE ? '\0' : '\1';
                put_le(p + 9, len, 4);
            }
            for (uint64_t j = lane; j < len; j += 32) put_le(p + 13 + 4 * j, verts[a + j], 4);
            continue;
        }
        // text, output.cpp:26-38
        uint32_t hq = ndigits(qid);
        if (lane == 0) {
            put_dec(p, qid, hq);
            p[hq] = '\t';
            const char* s = st[r] == WF_WALK_COMPLETE ? "complete" : "dead_end";
            for (uint32_t i = 0; i < kStatusChars; ++i) p[hq + 1 + i] = s[i];
            p[hq + 1 + kStatusChars] = '\t';
        }
        uint64_t cur = hq + 1 + kStatusChars + 1;
        for (uint64_t j0 = 0; j0 < len; j0 += 32) {
            const uint64_t j = j0 + lane;
            const uint32_t v = j < len ? verts[a + j] : 0;
            const uint32_t nd = j < len ? ndigits(v) : 0;
            uint32_t incl = j < len ? nd + 1 : 0;  // digits + separator
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(kFull, incl, o);
                if (lane >= o) incl += t;
            }
            const uint32_t excl = incl - (j < len ? nd + 1 : 0);
            if (j < len) {
                put_dec(p + cur + excl, v, nd);
                p[cur + excl + nd] = (j + 1 == len) ? '\n' : ' ';
            }
            cur += __shfl_sync(kFull, incl, 31);
        }
        if (len == 0 && lane == 0) p[cur] = '\n';
    }
}

struct Scratch {
    DeviceBuffer<uint64_t> off;
    DeviceBuffer<uint32_t> verts;
    DeviceBuffer<uint8_t> st;
    DeviceBuffer<uint64_t> size, pos;
    DeviceBuffer<uint8_t> tmp;
    DeviceBuffer<char> out;
};

// Encodes device-resident ragged records into s.out (grown as needed); returns bytes.
uint64_t encode_device(const uint64_t* d_off, const uint32_t* d_verts, const uint8_t* d_st,
                       uint64_t n, uint64_t qid_base, int fmt, Scratch& s, cudaStream_t st) {
    if (n == 0) return 0;
    if (s.size.size() < n) s.size.allocate(n);
    if (s.pos.size() < n + 1) s.pos.allocate(n + 1);
    const int blocks = static_cast<int>(std::min<uint64_t>((n * 32 + 255) / 256, 65535));
    k_record_size<<<blocks, 256, 0, st>>>(d_off, d_verts, n, qid_base, fmt, s.size.get());
    WF_LAUNCHED();
    WF_CUDA(cudaMemsetAsync(s.pos.get(), 0, 8, st));
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, s.size.get(), s.pos.get() + 1, static_cast<int64_t>(n), st);
    if (s.tmp.size() < tb) s.tmp.allocate(tb);
    WF_CUDA(cub::DeviceScan::InclusiveSum(s.tmp.get(), tb, s.size.get(), s.pos.get() + 1,
                                          static_cast<int64_t>(n), st));
    count_launch();
    uint64_t total = 0;
    WF_CUDA(cudaMemcpyAsync(&total, s.pos.get() + n, 8, cudaMemcpyDeviceToHost, st));
    WF_CUDA(cudaStreamSynchronize(st));
    if (s.out.size() < total) s.out.allocate(total);
    k_encode<<<blocks, 256, 0, st>>>(d_off, d_verts, d_st, n, qid_base, fmt, s.pos.get(), s.out.get());
    WF_LAUNCHED();
    return total;
}

template <typename T>
const T* to_device(const T* p, uint64_t count, DeviceBuffer<T>& buf) {
    if (p == nullptr || is_device_pointer(p)) return p;
    if (buf.size() < count) buf.allocate(std::max<uint64_t>(count, 1));
    WF_CUDA(cudaMemcpy(buf.get(), p, count * sizeof(T), cudaMemcpyHostToDevice));
    return buf.get();
}

}  // namespace

uint64_t encode_walks(const uint64_t* offsets, const uint32_t* vertices, const uint8_t* status,
                      uint64_t n, uint64_t qid_base, int fmt, char* out, uint64_t capacity) {
    if (fmt != WF_OUTPUT_TEXT && fmt != WF_OUTPUT_BINARY) config_error("unknown output format");
    Scratch s;
    uint64_t last = 0;
    if (n) {
        if (is_device_pointer(offsets)) WF_CUDA(cudaMemcpy(&last, offsets + n, 8, cudaMemcpyDeviceToHost));
        else last = offsets[n];
    }
    const uint64_t* d_off = to_device(offsets, n + 1, s.off);
    const uint32_t* d_v = to_device(vertices, last, s.verts);
    const uint8_t* d_s = to_device(status, n, s.st);
    const uint64_t total = encode_device(d_off, d_v, d_s, n, qid_base, fmt, s, nullptr);
    if (out) {
        if (total > capacity) raise(WF_ERR_INVALID_ARG, "output buffer too small for the encoded records");
        if (total) WF_CUDA(cudaMemcpy(out, s.out.get(), total, cudaMemcpyDefault));
    }
    WF_CUDA(cudaDeviceSynchronize());
    return total;
}

uint64_t write_walkset(const WalkSetStore& w, const char* path, int fmt, uint64_t qb, uint64_t qe) {
    if (fmt != WF_OUTPUT_TEXT && fmt != WF_OUTPUT_BINARY) config_error("unknown output format");
    DeviceGuard guard(w.device);
    if (qe == 0) qe = w.n;
    if (qb > qe || qe > w.n) raise(WF_ERR_INVALID_ARG, "query range out of bounds");
    FILE* f = std::fopen(path, "wb");
    if (!f) raise(WF_ERR_IO, std::string("cannot open output file ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard_f(f, std::fclose);
    const uint64_t kBlock = 1ull << 20;  // records per block
    Scratch s;
    DeviceBuffer<uint64_t> d_off(kBlock + 1);
    char* host[2] = {nullptr, nullptr};
    uint64_t host_cap[2] = {0, 0};
    std::future<size_t> pending;  // at most one write in flight: file order = qid order
    uint64_t pending_bytes = 0;
    uint64_t written = 0;
    auto release = [&] {
        for (int i = 0; i < 2; ++i)
            if (host[i]) cudaFreeHost(host[i]);
    };
    auto settle = [&] {
        if (!pending.valid()) return;
        if (pending.get() != pending_bytes) raise(WF_ERR_IO, std::string("write failed for ") + path);
        written += pending_bytes;
    };
    try {
        int b = 0;
        for (uint64_t r0 = qb; r0 < qe; r0 += kBlock, b ^= 1) {
            const uint64_t r1 = std::min(qe, r0 + kBlock), n = r1 - r0;
            // block k: ragged records + encoding on the device, while the host
            // thread is still writing block k-1 from the other pinned buffer
            std::vector<uint64_t> hoff(n + 1);
            walkset_copy(w, r0, r1, hoff.data(), nullptr, nullptr);
            const uint64_t nv = hoff[n];
            if (s.verts.size() < nv) s.verts.allocate(std::max<uint64_t>(nv, 1));
            if (s.st.size() < n) s.st.allocate(n);
            walkset_copy(w, r0, r1, d_off.get(), s.verts.get(), s.st.get());
            const uint64_t bytes = encode_device(d_off.get(), s.verts.get(), s.st.get(), n, r0, fmt, s, nullptr);
            settle();  // block k-1 written; buffer b (block k-2) long free
            if (host_cap[b] < bytes) {
                if (host[b]) cudaFreeHost(host[b]);
                WF_CUDA(cudaMallocHost(&host[b], bytes));
                host_cap[b] = bytes;
            }
            if (bytes) WF_CUDA(cudaMemcpy(host[b], s.out.get(), bytes, cudaMemcpyDeviceToHost));
            char* buf = host[b];
            pending_bytes = bytes;
            pending = std::async(std::launch::async, [f, buf, bytes] { return std::fwrite(buf, 1, bytes, f); });
        }
        settle();
    } catch (...) {
        if (pending.valid()) pending.wait();
        release();
        throw;
    }
    release();
    if (std::fflush(f) != 0) raise(WF_ERR_IO, std::string("write failed for ") + path);
    return written;
}

}  // namespace wf
