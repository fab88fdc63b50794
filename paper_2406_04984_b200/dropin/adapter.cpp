// Drop-in implementation of adapter.hpp over the C ABI: selection, gather and the sparse FFN run on the B200
// in float64 (the API path keeps the reference's precision; indices bit-exact, FFN chains bitwise equal to the
// compiled reference). Argument validation mirrors adapter.cpp line by line (same exception types, messages).
#include <algorithm>
#include <chrono>
#include <functional>
#include <numeric>

#include "device.hpp"
#include "meft/adapter.hpp"
#include "meft/diag.hpp"
#include "meft/kernels.hpp"

namespace meft {

namespace {

using Clock = std::chrono::steady_clock;

SelectionSet selection_from_device(const dropin::DevBuf& per, const dropin::DevBuf& uni, const dropin::DevBuf& usz,
                                   index_t tokens, index_t take, index_t budget) {
    std::vector<int32_t> p, u, n;
    dropin::download_i32(n, usz, 1);
    dropin::download_i32(p, per, size_t(tokens * take));
    dropin::download_i32(u, uni, size_t(n[0]));
    SelectionSet sel;
    sel.budget = budget;
    sel.per_token.resize(size_t(tokens));
    for (index_t t = 0; t < tokens; ++t)
        sel.per_token[size_t(t)].assign(p.begin() + t * take, p.begin() + (t + 1) * take);
    sel.unioned.assign(u.begin(), u.end());
    return sel;
}

// Device-resident pieces of one sparse FFN call.
struct FfnDevice {
    dropin::DevBuf h, keys_s, values_s;
};

int act_code(Activation a) { return a == Activation::ReLU ? 1 : 0; }

}  // namespace

SelectionSet topk_select(const HiddenBatch& h, const Matrix& w_a, index_t k) {
    if (k < 1) throw std::invalid_argument("topk_select: K must be >= 1");
    if (h.dim() != w_a.rows) throw ShapeError("topk_select: dim mismatch");
    const index_t r = w_a.cols, tokens = h.tokens(), d = h.dim();
    if (k > r) warn("topk_select: K=" + std::to_string(k) + " > r=" + std::to_string(r) + ", clamped");
    const index_t take = std::min(k, r);
    if (r == 0 || tokens == 0) {
        SelectionSet sel;
        sel.budget = k;
        sel.per_token.assign(size_t(tokens), {});
        return sel;
    }
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf dh = dropin::upload(h.values);
    dropin::DevBuf keys = dropin::transposed(dropin::upload(w_a), d, r);  // neuron-major [r x d]
    dropin::DevBuf per(size_t(tokens * take) * 4), uni(size_t(r) * 4), usz(4);
    dropin::check(meft_topk_select(dropin::ctx(), MEFT_F64, dh.get(), keys.get(), tokens, d, r, k, per.as<int32_t>(),
                                   uni.as<int32_t>(), usz.as<int32_t>()));
    return selection_from_device(per, uni, usz, tokens, take, k);
}

GatheredAdapter gather_adapter(const AdapterWeights& adapter, const std::vector<index_t>& s) {
    const index_t d = adapter.dim(), r = adapter.pairs();
    for (size_t i = 0; i < s.size(); ++i) {  // adapter.cpp:89-98, first violation in order wins
        if (s[i] < 0 || s[i] >= r)
            throw std::out_of_range("gather_adapter: index " + std::to_string(s[i]) + " out of range [0," +
                                    std::to_string(r) + ")");
        if (i > 0 && s[i] <= s[i - 1]) throw std::invalid_argument("gather_adapter: indices not sorted ascending");
    }
    const index_t m = static_cast<index_t>(s.size());
    GatheredAdapter g{Matrix(d, m), Matrix(m, d)};
    if (m == 0 || d == 0) return g;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf keys = dropin::transposed(dropin::upload(adapter.w_a), d, r);
    dropin::DevBuf vals = dropin::upload(adapter.w_b);
    dropin::DevBuf idx = dropin::upload_indices(s);
    dropin::DevBuf ks(size_t(m * d) * 8), vs(size_t(m * d) * 8);
    dropin::check(meft_gather_adapter(dropin::ctx(), MEFT_F64, keys.get(), vals.get(), r, d, idx.as<int32_t>(), m,
                                      ks.get(), vs.get()));
    dropin::DevBuf kt = dropin::transposed(ks, m, d);  // back to the reference's d x |S| columns
    g.w_a_k = dropin::download_matrix(kt, d, m);
    g.w_b_k = dropin::download_matrix(vs, m, d);
    return g;
}

HiddenBatch sparse_ffn_pa(const HiddenBatch& h, const BaseFfn& base, const Matrix& w_a_k, const Matrix& w_b_k,
                          FfnCache* cache, FfnPhaseTimes* phases) {
    if (h.dim() != base.w_in.rows) throw ShapeError("sparse_ffn_pa: base dim mismatch");
    if (w_a_k.cols != w_b_k.rows || (w_a_k.cols > 0 && w_a_k.rows != h.dim()))
        throw ShapeError("sparse_ffn_pa: gathered shapes inconsistent");
    if (base.w_out.rows != base.w_in.cols || base.w_out.cols != h.dim())
        throw ShapeError("matmul: inner dimensions disagree: " + shape_str(base.w_in) + " * " + shape_str(base.w_out));
    const index_t tokens = h.tokens(), d = h.dim(), n = base.w_in.cols, s = w_a_k.cols;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    meft_ctx* c = dropin::ctx();
    const auto t0 = Clock::now();
    dropin::DevBuf dh = dropin::upload(h.values);
    dropin::DevBuf win = dropin::upload(base.w_in), wout = dropin::upload(base.w_out);
    dropin::DevBuf pre(size_t(std::max<index_t>(tokens * n, 1)) * 8), out(size_t(std::max<index_t>(tokens * d, 1)) * 8);
    dropin::check(meft_base_ffn_forward(c, dh.as<double>(), win.as<double>(), wout.as<double>(), tokens, d, n,
                                        act_code(base.act), pre.as<double>(), out.as<double>()));
    dropin::check(meft_synchronize(c));
    const auto t1 = Clock::now();
    Matrix z(tokens, s);
    dropin::DevBuf dz(size_t(std::max<index_t>(tokens * s, 1)) * 8);
    if (s > 0 && tokens > 0) {
        dropin::DevBuf keys = dropin::transposed(dropin::upload(w_a_k), d, s);
        dropin::DevBuf vals = dropin::upload(w_b_k);
        dropin::check(meft_ffn_forward(c, MEFT_F64, dh.get(), keys.get(), vals.get(), tokens, d, s, s, dz.get(),
                                       out.get(), 1));
        z = dropin::download_matrix(dz, tokens, s);
    }
    Matrix result = dropin::download_matrix(out, tokens, d);
    const auto t2 = Clock::now();
    Matrix base_pre = dropin::download_matrix(pre, tokens, n);
    // the reference checks every matmul output (kernels.cpp:51,74)
    dropin::require_finite(base_pre, "matmul");
    dropin::require_finite(z, "matmul");
    dropin::require_finite(result, "matmul");
    if (phases) {
        phases->base_s += std::chrono::duration<double>(t1 - t0).count();
        phases->adapter_s += std::chrono::duration<double>(t2 - t1).count();
    }
    if (cache) {
        cache->h = h.values;
        cache->z = std::move(z);
        cache->base_pre = std::move(base_pre);
    }
    return HiddenBatch(h.batch, h.seq, std::move(result));
}

HiddenBatch dense_ffn_pa(const HiddenBatch& h, const BaseFfn& base, const AdapterWeights& adapter) {
    if (h.dim() != base.w_in.rows || h.dim() != adapter.w_a.rows) throw ShapeError("dense_ffn_pa: model dim mismatch");
    // identical device chains to sparse_ffn_pa over the full adapter (bitwise equal, test_adapter.cpp:178-185)
    return sparse_ffn_pa(h, base, adapter.w_a, adapter.w_b, nullptr);
}

SparseFfnGrads sparse_backward(const Matrix& grad_out, const FfnCache& cache, const Matrix& w_a_k,
                               const Matrix& w_b_k, const BaseFfn& base) {
    if (grad_out.rows != cache.h.rows || grad_out.cols != cache.h.cols)
        throw ShapeError("sparse_backward: grad_out shape mismatch");
    if (cache.z.cols != w_a_k.cols || w_a_k.cols != w_b_k.rows)
        throw ShapeError("sparse_backward: cache/selection mismatch");
    const index_t tokens = cache.h.rows, d = cache.h.cols, n = base.w_in.cols, s = w_a_k.cols;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    meft_ctx* c = dropin::ctx();
    dropin::DevBuf g = dropin::upload(grad_out);
    dropin::DevBuf win = dropin::upload(base.w_in), wout = dropin::upload(base.w_out), pre = dropin::upload(cache.base_pre);
    dropin::DevBuf gh(size_t(std::max<index_t>(tokens * d, 1)) * 8);
    dropin::check(meft_base_ffn_backward(c, g.as<double>(), pre.as<double>(), win.as<double>(), wout.as<double>(),
                                         tokens, d, n, act_code(base.act), gh.as<double>()));
    SparseFfnGrads out;
    if (s > 0 && tokens > 0) {
        dropin::DevBuf dh = dropin::upload(cache.h), dz = dropin::upload(cache.z);
        dropin::DevBuf keys = dropin::transposed(dropin::upload(w_a_k), d, s);
        dropin::DevBuf vals = dropin::upload(w_b_k);
        dropin::DevBuf masked(size_t(tokens * s) * 8), gk(size_t(s * d) * 8), gv(size_t(s * d) * 8);
        dropin::check(meft_ffn_backward(c, MEFT_F64, g.get(), dh.get(), dz.get(), keys.get(), vals.get(), tokens, d, s,
                                        s, masked.get(), gk.get(), gv.get(), gh.get(), 1));
        out.grad_w_a_k = dropin::download_matrix(dropin::transposed(gk, s, d), d, s);
        out.grad_w_b_k = dropin::download_matrix(gv, s, d);
    } else {
        out.grad_w_a_k = Matrix(d, s);
        out.grad_w_b_k = Matrix(s, d);
    }
    out.grad_h = dropin::download_matrix(gh, tokens, d);
    dropin::require_finite(out.grad_h, "matmul");
    dropin::require_finite(out.grad_w_a_k, "matmul");
    dropin::require_finite(out.grad_w_b_k, "matmul");
    return out;
}

ActivationProfile activation_profile(const AdapterWeights& adapter, const std::vector<Matrix>& corpus) {
    const index_t r = adapter.pairs(), d = adapter.dim();
    index_t tokens = 0;
    std::vector<double> sums(size_t(r), 0.0);
    {
        // On the device: per batch, act = ReLU(h w_a) (meft_matmul_f64 + meft_activation_f64), then the running
        // column sums as ONE ascending fp64 chain over [sums; act] (a 1 x (rows+1) ones vector times that stack):
        // acc = sums[j], then acc + act[0][j], acc + act[1][j], ... -- the reference's sequential loop
        // (adapter.cpp:190-193) bit for bit, fma(1, x, acc) being the exact add.
        std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
        dropin::DevBuf dsums(size_t(std::max<index_t>(r, 1)) * sizeof(double));
        dropin::DevBuf wa = r > 0 ? dropin::upload(adapter.w_a) : dropin::DevBuf();
        for (const Matrix& h : corpus) {
            if (h.rows == 0) continue;
            if (h.cols != d) throw ShapeError("activation_profile: dim mismatch");
            if (r == 0) {
                tokens += h.rows;
                continue;
            }
            const index_t T = h.rows;
            dropin::DevBuf dh = dropin::upload(h);
            dropin::DevBuf stack(size_t((T + 1) * r) * sizeof(double));  // row 0: the running sums, rows 1..T: act
            dropin::check(meft_copy_to_device(dropin::ctx(), stack.get(), sums.data(), size_t(r) * sizeof(double)));
            dropin::check(meft_matmul_f64(dropin::ctx(), dh.as<double>(), wa.as<double>(), T, d, r,
                                          stack.as<double>() + r));
            dropin::check(meft_activation_f64(dropin::ctx(), 1, stack.as<double>() + r, stack.as<double>() + r,
                                              T * r));
            std::vector<double> ones(size_t(T + 1), 1.0);
            dropin::DevBuf dones = dropin::upload(ones.data(), ones.size());
            dropin::check(meft_matmul_f64(dropin::ctx(), dones.as<double>(), stack.as<double>(), 1, T + 1, r,
                                          dsums.as<double>()));
            dropin::download(sums.data(), dsums, sums.size());  // synchronous: `ones` may go on return
            tokens += T;
        }
    }
    if (tokens == 0) throw std::invalid_argument("activation_profile: empty corpus");
    std::vector<double> means(sums);
    for (double& x : means) x /= static_cast<double>(tokens);
    std::sort(means.begin(), means.end(), std::greater<double>());
    ActivationProfile p;
    p.sorted_means.resize(means.size());
    p.cumulative.resize(means.size());
    const double total = std::accumulate(means.begin(), means.end(), 0.0);
    const double lo = means.empty() ? 0.0 : means.back(), hi = means.empty() ? 0.0 : means.front();
    double run = 0.0;
    for (size_t i = 0; i < means.size(); ++i) {
        p.sorted_means[i] = hi > lo ? (means[i] - lo) / (hi - lo) : 0.0;
        run += means[i];
        p.cumulative[i] = total > 0.0 ? run / total : 0.0;
    }
    return p;
}

}  // namespace meft
