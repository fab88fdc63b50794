// Drop-in implementation of kernels.hpp / matrix.hpp / diag.hpp / grad_check.hpp.
// matmul, relu and silu execute on the B200 (meft_matmul_f64 reproduces the compiled reference's ascending-k fma
// chain bit for bit); the element-wise helpers below are single IEEE operations per entry.
#include <atomic>
#include <cmath>
#include <cstdio>

#include "device.hpp"
#include "meft/diag.hpp"
#include "meft/grad_check.hpp"
#include "meft/kernels.hpp"

namespace meft {

namespace {
std::atomic<long> g_warns{0};

Matrix device_activation(const Matrix& x, int act) {
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    if (x.size() == 0) return Matrix(x.rows, x.cols);
    dropin::DevBuf in = dropin::upload(x);
    dropin::DevBuf out(in.bytes());
    dropin::check(meft_activation_f64(dropin::ctx(), act, in.as<double>(), out.as<double>(), x.size()));
    return dropin::download_matrix(out, x.rows, x.cols);
}

void same_shape_or_throw(const Matrix& a, const Matrix& b, const char* op) {
    if (!a.same_shape(b)) throw ShapeError(std::string(op) + ": shape mismatch: " + shape_str(a) + " vs " + shape_str(b));
}
}  // namespace

void warn(const std::string& msg) {
    g_warns.fetch_add(1);
    std::fprintf(stderr, "[meft] warning: %s\n", msg.c_str());
}

long warn_count() { return g_warns.load(); }

void check_finite(const Matrix& m, const char* where) { dropin::require_finite(m, where); }

double sigmoid(double x) { return 1.0 / (1.0 + std::exp(-x)); }
double silu_scalar(double x) { return x * sigmoid(x); }
double silu_grad_scalar(double x) {
    const double s = sigmoid(x);
    return s * (1.0 + x * (1.0 - s));
}

Matrix matmul(const Matrix& a, const Matrix& b) {
    if (a.cols != b.rows)
        throw ShapeError("matmul: inner dimensions disagree: " + shape_str(a) + " * " + shape_str(b));
    if (a.rows == 0 || b.cols == 0) return Matrix(a.rows, b.cols);
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf da = dropin::upload(a), db = dropin::upload(b);
    dropin::DevBuf dc(size_t(a.rows * b.cols) * sizeof(double));
    dropin::check(meft_matmul_f64(dropin::ctx(), da.as<double>(), db.as<double>(), a.rows, a.cols, b.cols,
                                  dc.as<double>()));
    return dropin::download_matrix(dc, a.rows, b.cols);
}

Matrix relu(const Matrix& x) { return device_activation(x, 1); }
Matrix silu(const Matrix& x) { return device_activation(x, 0); }

namespace ref {
// The device GEMM is deterministic and thread-count independent, so the serial twins are the same functions.
Matrix matmul(const Matrix& a, const Matrix& b) { return meft::matmul(a, b); }
Matrix relu(const Matrix& x) { return meft::relu(x); }
Matrix silu(const Matrix& x) { return meft::silu(x); }
}  // namespace ref

Matrix transpose(const Matrix& a) {
    Matrix out(a.cols, a.rows);
    for (index_t i = 0; i < a.rows; ++i)
        for (index_t j = 0; j < a.cols; ++j) out.at(j, i) = a.at(i, j);
    return out;
}

Matrix add(const Matrix& a, const Matrix& b) {
    same_shape_or_throw(a, b, "add");
    Matrix out(a.rows, a.cols);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] + b.data[i];
    return out;
}

Matrix sub(const Matrix& a, const Matrix& b) {
    same_shape_or_throw(a, b, "sub");
    Matrix out(a.rows, a.cols);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] - b.data[i];
    return out;
}

Matrix hadamard(const Matrix& a, const Matrix& b) {
    same_shape_or_throw(a, b, "hadamard");
    Matrix out(a.rows, a.cols);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] * b.data[i];
    return out;
}

Matrix scale(const Matrix& a, double s) {
    Matrix out(a.rows, a.cols);
    for (size_t i = 0; i < out.data.size(); ++i) out.data[i] = a.data[i] * s;
    return out;
}

void add_inplace(Matrix& a, const Matrix& b) {
    same_shape_or_throw(a, b, "add_inplace");
    for (size_t i = 0; i < a.data.size(); ++i) a.data[i] += b.data[i];
}

Matrix finite_diff_grad(const std::function<double(const Matrix&)>& f, const Matrix& theta, double eps) {
    if (!(eps > 0.0)) throw std::invalid_argument("finite_diff_grad: eps must be > 0");
    Matrix grad(theta.rows, theta.cols);
    Matrix probe = theta;
    for (size_t i = 0; i < probe.data.size(); ++i) {
        const double keep = probe.data[i];
        probe.data[i] = keep + eps;
        const double up = f(probe);
        probe.data[i] = keep - eps;
        const double down = f(probe);
        probe.data[i] = keep;
        if (!std::isfinite(up) || !std::isfinite(down))
            throw std::runtime_error("finite_diff_grad: non-finite function value");
        grad.data[i] = (up - down) / (2.0 * eps);
    }
    return grad;
}

}  // namespace meft
