// Internal plumbing of the drop-in shim: one process-wide meft_ctx, RAII device buffers, status -> exception
// translation with the reference's exception types. No numerics here.
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "meft/matrix.hpp"
#include "meft_cuda.h"

namespace meft::dropin {

meft_ctx* ctx();
std::recursive_mutex& api_mutex();

// meft_status -> ShapeError / invalid_argument / out_of_range / logic_error / runtime_error.
void check(meft_status st);

class DevBuf {
  public:
    DevBuf() = default;
    explicit DevBuf(size_t bytes);
    ~DevBuf();
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept;

    void* get() const { return p_; }
    template <class T>
    T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return n_; }

  private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

DevBuf upload(const double* host, size_t count);
DevBuf upload(const Matrix& m);
DevBuf upload_indices(const std::vector<index_t>& idx);  // int32 on device
void upload_bytes(DevBuf& dst, const void* host, size_t bytes);
void download(double* host, const DevBuf& b, size_t count);
Matrix download_matrix(const DevBuf& b, index_t rows, index_t cols);
void download_i32(std::vector<int32_t>& host, const DevBuf& b, size_t count);

// Device transpose of a row-major [rows x cols] float64 buffer.
DevBuf transposed(const DevBuf& src, index_t rows, index_t cols);

// Reusable page-locked host staging for the row-mirroring transfers: slot `slot` holds at least `count` doubles
// (grown on demand, never shrunk), so repeated calls neither re-fault fresh pages nor copy through the driver's
// pageable bounce buffers. Callers hold api_mutex.
double* staging(int slot, size_t count);
constexpr int kStagingSlots = 10;  // 0-7: callers' transfer blocks; 8-9: upload(const Matrix&) chunks

// Throws runtime_error("<where>: non-finite entry") like check_finite (kernels.cpp:7-13).
void require_finite(const Matrix& m, const char* where);

}  // namespace meft::dropin
