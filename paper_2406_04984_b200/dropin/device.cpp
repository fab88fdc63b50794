// Drop-in shim plumbing (see device.hpp).
#include "device.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace meft::dropin {

std::recursive_mutex& api_mutex() {
    static std::recursive_mutex m;
    return m;
}

meft_ctx* ctx() {
    static meft_ctx* c = [] {
        meft_ctx* p = nullptr;
        const meft_status st = meft_ctx_create(0, MEFT_OWN_STREAM, &p);
        if (st != MEFT_OK) throw std::runtime_error(std::string("meft: cannot create device context: ") +
                                                    meft_last_error(nullptr));
        return p;
    }();
    return c;
}

void check(meft_status st) {
    if (st == MEFT_OK) return;
    const std::string msg = meft_last_error(ctx());
    switch (st) {
        case MEFT_E_SHAPE: throw ShapeError(msg);
        case MEFT_E_INVALID: throw std::invalid_argument(msg);
        case MEFT_E_RANGE: throw std::out_of_range(msg);
        case MEFT_E_LOGIC: throw std::logic_error(msg);
        case MEFT_E_NONFINITE: throw std::runtime_error(msg);
        default: throw std::runtime_error("meft device error: " + msg);
    }
}

// Device buffers are recycled through a size-class cache: the API calls allocate and release the same few shapes
// over and over, and cudaFree synchronises the whole device. Every use is enqueued on the one context stream, so a
// recycled block is only touched after the work of its previous owner (stream order).
namespace {
struct Pool {
    std::mutex mu;
    std::multimap<size_t, void*> free;  // size class -> blocks
    size_t cached = 0;
    static constexpr size_t kLimit = size_t(8) << 30;  // keep at most 8 GB of idle blocks
};
Pool& pool() {
    static Pool* p = new Pool();  // never destroyed: blocks outlive static destruction order
    return *p;
}
size_t size_class(size_t bytes) {
    if (bytes <= 256) return 256;
    if (bytes <= (size_t(64) << 20)) {
        size_t c = 256;
        while (c < bytes) c <<= 1;
        return c;
    }
    const size_t g = size_t(64) << 20;
    return (bytes + g - 1) / g * g;
}
void* pool_get(size_t cls) {
    Pool& P = pool();
    {
        std::lock_guard<std::mutex> lk(P.mu);
        auto it = P.free.find(cls);
        if (it != P.free.end()) {
            void* p = it->second;
            P.free.erase(it);
            P.cached -= cls;
            return p;
        }
    }
    void* p = nullptr;
    meft_status st = meft_device_alloc(ctx(), cls, &p);
    if (st == MEFT_E_OOM) {  // give the idle blocks back and retry once
        std::lock_guard<std::mutex> lk(P.mu);
        for (auto& kv : P.free) meft_device_free(ctx(), kv.second);
        P.free.clear();
        P.cached = 0;
        st = meft_device_alloc(ctx(), cls, &p);
    }
    check(st);
    return p;
}
void pool_put(void* p, size_t cls) {
    Pool& P = pool();
    std::lock_guard<std::mutex> lk(P.mu);
    if (P.cached + cls > Pool::kLimit) {
        meft_device_free(ctx(), p);
        return;
    }
    P.free.emplace(cls, p);
    P.cached += cls;
}
}  // namespace

DevBuf::DevBuf(size_t bytes) : n_(bytes) {
    if (bytes) p_ = pool_get(size_class(bytes));
}

DevBuf::~DevBuf() {
    if (p_) pool_put(p_, size_class(n_));
}

DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        if (p_) pool_put(p_, size_class(n_));
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
    }
    return *this;
}

DevBuf upload(const double* host, size_t count) {
    DevBuf b(count * sizeof(double));
    if (count) check(meft_copy_to_device(ctx(), b.get(), host, count * sizeof(double)));
    return b;
}

// Large pageable sources (whole host tables: ke_select's keys, gather_adapter's tables) go through two page-locked
// chunks: the host's threads copy chunk i into one while the DMA of chunk i-1 drains the other (the driver's own
// pageable path copies on one thread).
DevBuf upload(const Matrix& m) {
    const size_t count = m.data.size();
    constexpr size_t kChunk = size_t(4) << 20;  // doubles (32 MB)
    if (count < 2 * kChunk) return upload(m.data.data(), count);
    DevBuf b(count * sizeof(double));
    double* buf[2] = {staging(kStagingSlots - 2, kChunk), staging(kStagingSlots - 1, kChunk)};
    const unsigned workers = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    size_t i = 0;
    for (size_t off = 0; off < count; off += kChunk, ++i) {
        const size_t n = std::min(kChunk, count - off);
        double* dst = buf[i & 1];
        const double* src = m.data.data() + off;
        std::vector<std::thread> pool;
        const size_t per = (n + workers - 1) / workers;
        for (size_t lo = 0; lo < n; lo += per)
            pool.emplace_back([=] { std::memcpy(dst + lo, src + lo, std::min(per, n - lo) * sizeof(double)); });
        for (auto& t : pool) t.join();
        check(meft_synchronize(ctx()));  // chunk i-1's DMA is done: its buffer is free for chunk i+1
        check(meft_copy_to_device(ctx(), static_cast<double*>(b.get()) + off, dst, n * sizeof(double)));
    }
    check(meft_synchronize(ctx()));  // the chunks are reused by the next call
    return b;
}

DevBuf upload_indices(const std::vector<index_t>& idx) {
    std::vector<int32_t> tmp(idx.begin(), idx.end());
    DevBuf b(tmp.size() * sizeof(int32_t));
    if (!tmp.empty()) check(meft_copy_to_device(ctx(), b.get(), tmp.data(), tmp.size() * sizeof(int32_t)));
    check(meft_synchronize(ctx()));  // tmp is released on return
    return b;
}

void upload_bytes(DevBuf& dst, const void* host, size_t bytes) {
    if (bytes) check(meft_copy_to_device(ctx(), dst.get(), host, bytes));
    check(meft_synchronize(ctx()));  // the host buffer may be released on return
}

void download(double* host, const DevBuf& b, size_t count) {
    if (count) check(meft_copy_to_host(ctx(), host, b.get(), count * sizeof(double)));
}

// Large results come back through the same two page-locked chunks: the DMA of chunk i+1 runs while the host's
// threads copy chunk i out (the driver's pageable path copies on one thread).
Matrix download_matrix(const DevBuf& b, index_t rows, index_t cols) {
    Matrix m(rows, cols);
    const size_t count = m.data.size();
    constexpr size_t kChunk = size_t(4) << 20;  // doubles (32 MB)
    if (count < 2 * kChunk) {
        download(m.data.data(), b, count);
        return m;
    }
    double* buf[2] = {staging(kStagingSlots - 2, kChunk), staging(kStagingSlots - 1, kChunk)};
    const unsigned workers = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    size_t i = 0;
    for (size_t off = 0; off < count; off += kChunk, ++i) {
        const size_t n = std::min(kChunk, count - off);
        double* src = buf[i & 1];
        // chunk i-1's copy-out still reads the other buffer; this DMA fills `src` (synchronous)
        check(meft_copy_to_host(ctx(), src, static_cast<const double*>(b.get()) + off, n * sizeof(double)));
        for (auto& t : pool) t.join();  // chunk i-1 copied out: its buffer is free for chunk i+1
        pool.clear();
        double* dst = m.data.data() + off;
        const size_t per = (n + workers - 1) / workers;
        for (size_t lo = 0; lo < n; lo += per)
            pool.emplace_back([=] { std::memcpy(dst + lo, src + lo, std::min(per, n - lo) * sizeof(double)); });
    }
    for (auto& t : pool) t.join();
    return m;
}

void download_i32(std::vector<int32_t>& host, const DevBuf& b, size_t count) {
    host.resize(count);
    if (count) check(meft_copy_to_host(ctx(), host.data(), b.get(), count * sizeof(int32_t)));
}

DevBuf transposed(const DevBuf& src, index_t rows, index_t cols) {
    DevBuf out(size_t(rows * cols) * sizeof(double));
    if (rows * cols > 0) check(meft_transpose_f64(ctx(), src.as<double>(), out.as<double>(), rows, cols));
    return out;
}

double* staging(int slot, size_t count) {
    struct Slot {
        void* p = nullptr;
        size_t bytes = 0;
    };
    static Slot slots[kStagingSlots];
    if (slot < 0 || slot >= kStagingSlots) throw std::logic_error("staging: slot out of range");
    Slot& s = slots[slot];
    const size_t want = std::max<size_t>(count, 1) * sizeof(double);
    if (s.bytes < want) {
        if (s.p) check(meft_host_free(ctx(), s.p));
        s.p = nullptr;
        s.bytes = 0;
        check(meft_host_alloc(ctx(), want, &s.p));
        s.bytes = want;
    }
    return static_cast<double*>(s.p);
}

void require_finite(const Matrix& m, const char* where) {
    for (double x : m.data)
        if (!std::isfinite(x)) throw std::runtime_error(std::string(where) + ": non-finite entry");
}

}  // namespace meft::dropin
