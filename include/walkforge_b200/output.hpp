// Walk-record output for callers of the C++ shim: the reference's output.hpp
// interface (proj/include/walkforge/output.hpp:17-96, src/output.cpp:26-200)
// with the same record bytes, error classes and ordering guarantees.
//
//   append_text_record    `qid<TAB>complete|dead_end<TAB>v0 v1 ...` + LF
//   append_binary_record  u64 qid | u8 status | u32 length | u32 path[length], LE
//   DoubleBufferedWriter  one buffer fills while a flusher thread writes the other
//   OrderedBlockSink      per-worker blocks written in worker order
//
// Bulk device-resident walk sets are better written with wf_walkset_write
// (records encoded on the device, walkforge_b200.h); this header serves the
// reference's host-side call pattern (BlockSink -> writer).
#pragma once

#include <charconv>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace walkforge_b200 {

enum class OutputFormat : uint8_t { Text, Binary };
constexpr size_t kMinOutputBuffer = 1u << 20;

namespace detail {
template <typename T>
inline void put_decimal(std::string& buf, T v) {
    char tmp[24];
    auto res = std::to_chars(tmp, tmp + sizeof(tmp), v);
    buf.append(tmp, res.ptr);
}
template <typename T>
inline void put_le(std::string& buf, T v) {  // the host is little-endian (x86-64 / aarch64)
    char tmp[sizeof(T)];
    std::memcpy(tmp, &v, sizeof(T));
    buf.append(tmp, sizeof(T));
}
}  // namespace detail

inline void append_text_record(std::string& buf, const WalkRecord& r) {
    detail::put_decimal(buf, r.query_id);
    buf += r.status == WalkStatus::Complete ? "\tcomplete\t" : "\tdead_end\t";
    for (size_t i = 0; i < r.path.size(); ++i) {
        if (i) buf += ' ';
        detail::put_decimal(buf, r.path[i]);
    }
    buf += '\n';
}

inline void append_binary_record(std::string& buf, const WalkRecord& r) {
    detail::put_le<uint64_t>(buf, r.query_id);
    buf += static_cast<char>(r.status == WalkStatus::Complete ? 0 : 1);
    detail::put_le<uint32_t>(buf, static_cast<uint32_t>(r.path.size()));
    for (VertexId v : r.path) detail::put_le<uint32_t>(buf, v);
}

// Two buffers: records are formatted into the active one; a full buffer is
// handed to a flusher thread and the other becomes active.  A failed write is
// reported at the next hand-off or at finish().
class DoubleBufferedWriter {
public:
    DoubleBufferedWriter(const std::string& path, OutputFormat format, size_t buffer_bytes = 4 * kMinOutputBuffer)
        : path_(path), format_(format), capacity_(buffer_bytes) {
        if (buffer_bytes < kMinOutputBuffer)
            throw ConfigError("output buffer must be at least " + std::to_string(kMinOutputBuffer) +
                              " bytes, got " + std::to_string(buffer_bytes));
        file_ = std::fopen(path.c_str(), "wb");
        if (!file_) throw IoError("cannot open output file " + path);
        active_.reserve(capacity_);
        flusher_ = std::thread([this] { flush_loop(); });
    }
    ~DoubleBufferedWriter() {
        try {
            finish();
        } catch (...) {
        }
    }
    DoubleBufferedWriter(const DoubleBufferedWriter&) = delete;
    DoubleBufferedWriter& operator=(const DoubleBufferedWriter&) = delete;

    void write(const WalkRecord& r) {
        const bool was_empty = active_.empty();
        if (format_ == OutputFormat::Text) append_text_record(active_, r);
        else append_binary_record(active_, r);
        if (was_empty && active_.size() > capacity_ && !warned_) {
            std::fprintf(stderr,
                         "walkforge: warning: a single record (%zu bytes) exceeds the output buffer (%zu bytes); "
                         "buffer grown\n",
                         active_.size(), capacity_);
            warned_ = true;
        }
        if (active_.size() >= capacity_) hand_off();
    }
    void write_all(const WalkSet& walks) {
        for (const WalkRecord& r : walks) write(r);
    }
    // Writes what is buffered and closes the file; idempotent.  Call it to
    // observe write errors (the destructor swallows them).
    void finish() {
        if (finished_) return;
        finished_ = true;
        std::exception_ptr err;
        try {
            hand_off();
        } catch (...) {
            err = std::current_exception();
        }
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        flusher_.join();
        const bool close_ok = std::fclose(file_) == 0;
        file_ = nullptr;
        if (err) std::rethrow_exception(err);
        if (error_) std::rethrow_exception(error_);
        if (!close_ok) throw IoError("write to " + path_ + " failed");
    }

private:
    void hand_off() {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !pending_ || error_; });  // the flusher took the previous buffer
        if (error_) {  // a failed flush surfaces at the next hand-off
            std::exception_ptr e = error_;
            error_ = nullptr;
            std::rethrow_exception(e);
        }
        if (active_.empty()) return;
        std::swap(active_, spare_);
        pending_ = true;
        active_.clear();
        active_.reserve(capacity_);
        cv_.notify_all();
    }
    void flush_loop() {
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return pending_ || stop_; });
            if (!pending_) return;
            std::string buf = std::move(spare_);
            spare_.clear();
            lk.unlock();
            const bool ok = std::fwrite(buf.data(), 1, buf.size(), file_) == buf.size();
            lk.lock();
            if (!ok && !error_) error_ = std::make_exception_ptr(IoError("write to " + path_ + " failed"));
            pending_ = false;
            cv_.notify_all();
        }
    }

    std::string path_;
    OutputFormat format_;
    size_t capacity_;
    std::FILE* file_ = nullptr;
    std::string active_, spare_;
    std::mutex mu_;
    std::condition_variable cv_;
    bool pending_ = false, stop_ = false, finished_ = false, warned_ = false;
    std::exception_ptr error_;
    std::thread flusher_;
};

// Blocks from `workers` producers (one each) reach the writer in worker
// order.  A producer whose block is not the next one waits while `max_pending`
// blocks are already parked, so memory stays bounded and the writer always
// makes progress.
class OrderedBlockSink {
public:
    OrderedBlockSink(DoubleBufferedWriter& writer, uint32_t workers, uint32_t max_pending = 2)
        : writer_(writer), slots_(workers), max_pending_(max_pending < 1 ? 1 : max_pending) {
        writer_thread_ = std::thread([this] { run(); });
    }
    ~OrderedBlockSink() {
        if (writer_thread_.joinable()) writer_thread_.join();
    }
    OrderedBlockSink(const OrderedBlockSink&) = delete;
    OrderedBlockSink& operator=(const OrderedBlockSink&) = delete;

    void push(uint32_t worker, WalkSet&& block) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return failed_ || cancelled_ || worker == next_ || parked_ < max_pending_; });
        if (failed_ || cancelled_) return;  // finish() reports a writer failure
        slots_[worker] = std::move(block);
        ++parked_;
        cv_.notify_all();
    }
    // Waits until every block is written; rethrows a writer failure.
    void finish() {
        if (writer_thread_.joinable()) writer_thread_.join();
        if (error_) std::rethrow_exception(error_);
    }
    // For failed runs: releases the writer thread; the file is left partial.
    void cancel() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            cancelled_ = true;
        }
        cv_.notify_all();
        if (writer_thread_.joinable()) writer_thread_.join();
    }

private:
    void run() {
        try {
            for (uint32_t w = 0; w < slots_.size(); ++w) {
                WalkSet block;
                {
                    std::unique_lock<std::mutex> lk(mu_);
                    cv_.wait(lk, [&] { return cancelled_ || slots_[w].has_value(); });
                    if (cancelled_) return;
                    block = std::move(*slots_[w]);
                    slots_[w].reset();
                    --parked_;
                    next_ = w + 1;
                    cv_.notify_all();
                }
                writer_.write_all(block);
            }
        } catch (...) {
            std::lock_guard<std::mutex> lk(mu_);
            error_ = std::current_exception();
            failed_ = true;
            cv_.notify_all();
        }
    }

    DoubleBufferedWriter& writer_;
    std::vector<std::optional<WalkSet>> slots_;
    uint32_t max_pending_;
    uint32_t parked_ = 0, next_ = 0;
    bool cancelled_ = false, failed_ = false;
    std::exception_ptr error_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::thread writer_thread_;
};

}  // namespace walkforge_b200
