// Drop-in implementation of model.hpp: the reference's frozen toy trunk. Parameter initialisation is host RNG work
// (the reference's per-tensor streams, model.cpp:23-48); embedding, attention forward / backward, the tied LM loss
// and greedy argmax run on the B200 through the fp64 trunk entry points of include/meft_cuda.h. Argument errors
// are raised here, on the host, with the reference's exception types and messages.
#include <cmath>
#include <stdexcept>
#include <string>

#include "device.hpp"
#include "meft/model.hpp"

namespace meft {

namespace {

std::vector<index_t> as_index(const std::vector<char>& v) { return std::vector<index_t>(v.begin(), v.end()); }

void require_inner(const Matrix& a, const Matrix& b, const char* what) {
    if (a.cols != b.rows)
        throw ShapeError(std::string(what) + ": inner dimensions disagree: " + shape_str(a) + " * " + shape_str(b));
}

void require_square(const AttnWeights& w, index_t d) {
    for (const Matrix* m : {&w.wq, &w.wk, &w.wv, &w.wo})
        if (m->rows != d || m->cols != d) throw ShapeError("attention: weights must be d x d, got " + shape_str(*m));
}

void require_rows(const Batch& batch, index_t rows, const char* what) {
    if (rows != batch.total()) throw ShapeError(std::string(what) + ": rows != batch * seq");
    if (static_cast<index_t>(batch.segments.size()) < rows)
        throw std::invalid_argument(std::string(what) + ": segments shorter than the batch");
}

}  // namespace

void ToyConfig::validate() const {
    if (vocab < 2) throw std::invalid_argument("config: vocab must be >= 2");
    if (dim < 1 || layers < 1 || ffn_width < 1 || pairs < 1 || max_seq < 1)
        throw std::invalid_argument("config: dimensions must be >= 1");
    if (experts < 1 || experts_per_token < 1 || budget < 1)
        throw std::invalid_argument("config: experts, experts_per_token and budget must be >= 1");
    if (pairs % experts != 0) throw std::invalid_argument("config: experts must divide pairs (N | r)");
}

FrozenBase init_frozen_base(const ToyConfig& cfg, std::uint64_t seed) {
    // one RNG stream per tensor (ids 1, 2, then 0x100 + 8*layer + {0..5}) so no geometry change reshuffles another
    auto draw = [seed](std::uint64_t id, index_t rows, index_t cols, double stddev) {
        return SeededRng(mix_seed(seed, id)).normal_matrix(rows, cols, stddev);
    };
    const double attn_std = 1.0 / std::sqrt(static_cast<double>(cfg.dim));
    constexpr double kResidual = 0.5;
    FrozenBase base;
    base.embedding = draw(1, cfg.vocab, cfg.dim, 1.0);
    base.pos = draw(2, cfg.max_seq, cfg.dim, 0.3);
    for (index_t layer = 0; layer < cfg.layers; ++layer) {
        const std::uint64_t id = 0x100 + 8 * static_cast<std::uint64_t>(layer);
        AttnWeights a;
        a.wq = draw(id + 0, cfg.dim, cfg.dim, attn_std);
        a.wk = draw(id + 1, cfg.dim, cfg.dim, attn_std);
        a.wv = draw(id + 2, cfg.dim, cfg.dim, attn_std);
        a.wo = draw(id + 3, cfg.dim, cfg.dim, kResidual * attn_std);
        base.attn.push_back(std::move(a));
        BaseFfn f;
        f.w_in = draw(id + 4, cfg.dim, cfg.ffn_width, attn_std);
        f.w_out = draw(id + 5, cfg.ffn_width, cfg.dim, kResidual / std::sqrt(static_cast<double>(cfg.ffn_width)));
        f.act = cfg.base_act;
        base.ffn.push_back(std::move(f));
    }
    return base;
}

Matrix embed(const FrozenBase& base, const Batch& batch) {
    const index_t d = base.embedding.cols, rows = batch.total();
    for (index_t b = 0; b < batch.batch; ++b)  // the reference's checks, in its visiting order
        for (index_t i = 0; i < batch.seq; ++i) {
            const index_t tok = batch.tokens[static_cast<size_t>(b * batch.seq + i)];
            if (tok < 0 || tok >= base.embedding.rows) throw std::out_of_range("embed: token id out of vocab");
            if (i >= base.pos.rows) throw std::out_of_range("embed: sequence longer than max_seq");
        }
    if (rows == 0 || d == 0) return Matrix(rows, d);
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf e = dropin::upload(base.embedding), p = dropin::upload(base.pos);
    dropin::DevBuf tok = dropin::upload_indices(batch.tokens);
    dropin::DevBuf h(size_t(rows * d) * sizeof(double));
    dropin::check(meft_embed_f64(dropin::ctx(), e.as<double>(), base.embedding.rows, p.as<double>(), base.pos.rows,
                                 d, tok.as<int32_t>(), batch.batch, batch.seq, h.as<double>()));
    return dropin::download_matrix(h, rows, d);
}

Matrix attention_forward(const AttnWeights& w, const Batch& batch, const Matrix& h, AttnCache* cache) {
    const index_t d = h.cols, rows = h.rows, l = batch.seq;
    require_inner(h, w.wq, "matmul");
    require_square(w, d);
    require_rows(batch, rows, "attention_forward");
    Matrix out(rows, d), q(rows, d), k(rows, d), v(rows, d), probs(rows, l);
    if (rows > 0 && d > 0) {
        std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
        dropin::DevBuf dh = dropin::upload(h), wq = dropin::upload(w.wq), wk = dropin::upload(w.wk),
                       wv = dropin::upload(w.wv), wo = dropin::upload(w.wo);
        dropin::DevBuf seg = dropin::upload_indices(batch.segments);
        const size_t n = size_t(rows * d) * sizeof(double);
        dropin::DevBuf o(n), dq(n), dk(n), dv(n), dp(size_t(rows * l) * sizeof(double));
        dropin::check(meft_attention_forward_f64(dropin::ctx(), dh.as<double>(), wq.as<double>(), wk.as<double>(),
                                                 wv.as<double>(), wo.as<double>(), seg.as<int32_t>(), batch.batch, l,
                                                 d, o.as<double>(), dq.as<double>(), dk.as<double>(), dv.as<double>(),
                                                 dp.as<double>()));
        out = dropin::download_matrix(o, rows, d);
        if (cache) {
            q = dropin::download_matrix(dq, rows, d);
            k = dropin::download_matrix(dk, rows, d);
            v = dropin::download_matrix(dv, rows, d);
            probs = dropin::download_matrix(dp, rows, l);
        }
    }
    if (cache) {
        cache->h_in = h;
        cache->q = std::move(q);
        cache->k = std::move(k);
        cache->v = std::move(v);
        cache->probs = std::move(probs);
    }
    return out;
}

Matrix attention_backward(const AttnWeights& w, const Batch& batch, const AttnCache& cache, const Matrix& dh_out) {
    const index_t d = dh_out.cols, rows = dh_out.rows, l = batch.seq;
    require_square(w, d);
    require_rows(batch, rows, "attention_backward");
    if (!cache.q.same_shape(dh_out) || !cache.k.same_shape(dh_out) || !cache.v.same_shape(dh_out) ||
        cache.probs.rows != rows || cache.probs.cols != l)
        throw ShapeError("attention_backward: cache does not match the gradient");
    if (rows == 0 || d == 0) return dh_out;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf wq = dropin::upload(w.wq), wk = dropin::upload(w.wk), wv = dropin::upload(w.wv),
                   wo = dropin::upload(w.wo);
    dropin::DevBuf seg = dropin::upload_indices(batch.segments);
    dropin::DevBuf q = dropin::upload(cache.q), k = dropin::upload(cache.k), v = dropin::upload(cache.v),
                   p = dropin::upload(cache.probs), g = dropin::upload(dh_out);
    dropin::DevBuf dh(size_t(rows * d) * sizeof(double));
    dropin::check(meft_attention_backward_f64(dropin::ctx(), wq.as<double>(), wk.as<double>(), wv.as<double>(),
                                              wo.as<double>(), seg.as<int32_t>(), batch.batch, l, d, q.as<double>(),
                                              k.as<double>(), v.as<double>(), p.as<double>(), g.as<double>(),
                                              dh.as<double>()));
    return dropin::download_matrix(dh, rows, d);
}

LossResult lm_loss_and_grad(const FrozenBase& base, const Batch& batch, const Matrix& h_final, double loss_scale) {
    const index_t V = base.embedding.rows, d = base.embedding.cols, rows = h_final.rows;
    if (h_final.cols != d)
        throw ShapeError("matmul: inner dimensions disagree: " + shape_str(h_final) + " * E^T " +
                         shape_str(base.embedding));
    if (static_cast<index_t>(batch.targets.size()) < rows || static_cast<index_t>(batch.loss_mask.size()) < rows)
        throw std::invalid_argument("lm_loss_and_grad: targets / loss_mask shorter than the batch");
    for (index_t t = 0; t < rows; ++t)
        if (batch.loss_mask[size_t(t)] && (batch.targets[size_t(t)] < 0 || batch.targets[size_t(t)] >= V))
            throw std::out_of_range("lm_loss_and_grad: target id out of vocab");
    LossResult res;
    res.dh = Matrix(rows, d);
    if (rows == 0 || d == 0) return res;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf e = dropin::upload(base.embedding), h = dropin::upload(h_final);
    dropin::DevBuf tgt = dropin::upload_indices(batch.targets);
    std::vector<index_t> mask = as_index(batch.loss_mask);
    std::vector<uint8_t> m8(mask.size());
    for (size_t i = 0; i < mask.size(); ++i) m8[i] = mask[i] != 0;
    dropin::DevBuf dm(m8.size());
    dropin::upload_bytes(dm, m8.data(), m8.size());
    dropin::DevBuf dh(size_t(rows * d) * sizeof(double));
    dropin::check(meft_lm_loss_f64(dropin::ctx(), e.as<double>(), V, d, h.as<double>(), rows, tgt.as<int32_t>(),
                                   dm.as<uint8_t>(), loss_scale, &res.loss_sum, dh.as<double>()));
    res.dh = dropin::download_matrix(dh, rows, d);
    return res;
}

index_t argmax_logits(const FrozenBase& base, const double* h_row) {
    const index_t V = base.embedding.rows, d = base.embedding.cols;
    if (V == 0 || d == 0) return 0;
    std::lock_guard<std::recursive_mutex> lk(dropin::api_mutex());
    dropin::DevBuf e = dropin::upload(base.embedding), h = dropin::upload(h_row, size_t(d));
    int64_t tok = 0;
    dropin::check(meft_argmax_logits_f64(dropin::ctx(), e.as<double>(), V, d, h.as<double>(), &tok));
    return static_cast<index_t>(tok);
}

}  // namespace meft
