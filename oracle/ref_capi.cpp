// ORACLE / TEST INFRASTRUCTURE ONLY. Never linked into the product library.
//
// Plain C entry points over the UNMODIFIED reference implementation, compiled
// from the sources where they lie under /root/reference/proj (recipe:
// oracle/Makefile, output: oracle/_ref/libmeft_ref.so). Tests use it to pin
// the C restatement (oracle/meft_oracle.c) and to generate golden fixtures;
// bench.py --impl reference times ref_layer_step on the host cores.
//
// Each wrapper calls exactly one reference public entry point:
//   ref_ke_select        -> meft::ke_select          proj/include/meft/experts.hpp:55-57
//   ref_topk_select      -> meft::topk_select        proj/include/meft/adapter.hpp:73
//   ref_route_scores     -> meft::route_scores       proj/include/meft/experts.hpp:45
//   ref_select_experts   -> meft::select_experts     proj/include/meft/experts.hpp:49
//   ref_gather_adapter   -> meft::gather_adapter     proj/include/meft/adapter.hpp:80
//   ref_ffn_forward      -> meft::sparse_ffn_pa      proj/include/meft/adapter.hpp:90-91
//   ref_ffn_backward     -> meft::sparse_backward    proj/include/meft/adapter.hpp:97-98
//   ref_scatter_grads    -> meft::scatter_grads      proj/include/meft/memtier.hpp:149-151
//   ref_sparse_adam      -> meft::sparse_adam_update proj/include/meft/memtier.hpp:161
//   ref_layer_step       -> meft_ffn -> sparse_backward -> scatter_grads -> sparse_adam_update
//                           (the trainer's per-layer sequence, proj/src/trainer.cpp:220,270,283,525)
//   ref_step_begin / ref_step_rows / ref_step_finish
//                        -> the same sequence split into its phases for bench.py's bounded CPU sample:
//                           meft_ffn's push_hidden + ke_select + fetch on the whole batch
//                           (meft_ffn.cpp:18-28), sparse_ffn_pa + sparse_backward on a slice of the batch's
//                           token rows against that union (every row of both is independent of the others,
//                           adapter.cpp:112-180), then scatter_grads + sparse_adam_update of the union.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include <omp.h>

#include "meft/adapter.hpp"
#include "meft/diag.hpp"
#include "meft/experts.hpp"
#include "meft/kernels.hpp"
#include "meft/meft_ffn.hpp"
#include "meft/memtier.hpp"
#include "meft/rng.hpp"

using namespace meft;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 5;
    } catch (...) {
        g_err = "unknown exception";
        return 9;
    }
}

Matrix to_matrix(const double* p, int64_t rows, int64_t cols) {
    Matrix m(rows, cols);
    if (rows * cols > 0) std::memcpy(m.data.data(), p, sizeof(double) * rows * cols);
    return m;
}

void from_matrix(const Matrix& m, double* out) {
    if (m.size() > 0) std::memcpy(out, m.data.data(), sizeof(double) * m.size());
}

BaseFfn make_base(const double* w_in, const double* w_out, int64_t d, int64_t n, int act) {
    BaseFfn b;
    b.w_in = (n > 0) ? to_matrix(w_in, d, n) : Matrix(d, 0);
    b.w_out = (n > 0) ? to_matrix(w_out, n, d) : Matrix(0, d);
    b.act = act == 1 ? Activation::ReLU : Activation::SiLU;
    return b;
}

Matrix* store_tensor(HostLayer& hl, int id) {
    switch (id) {
        case 0: return &hl.adapter.w_a;
        case 1: return &hl.adapter.w_b;
        case 2: return &hl.router.w_g;
        case 3: return &hl.m_a;
        case 4: return &hl.v_a;
        case 5: return &hl.m_b;
        case 6: return &hl.v_b;
        case 7: return &hl.stage_a;
        case 8: return &hl.stage_b;
        default: throw std::invalid_argument("bad tensor id");
    }
}

void write_selection(const SelectionSet& sel, int64_t take, int64_t* per_token, int64_t* union_out,
                     int64_t* union_size) {
    for (size_t t = 0; t < sel.per_token.size(); ++t) {
        const auto& pt = sel.per_token[t];
        if (static_cast<int64_t>(pt.size()) != take) throw std::logic_error("take mismatch");
        for (int64_t i = 0; i < take; ++i) per_token[t * take + i] = pt[i];
    }
    for (size_t i = 0; i < sel.unioned.size(); ++i) union_out[i] = sel.unioned[i];
    *union_size = static_cast<int64_t>(sel.unioned.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
long ref_warn_count() { return warn_count(); }
void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

uint64_t ref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void ref_uniform_matrix(uint64_t seed, int64_t rows, int64_t cols, double lo, double hi, double* out) {
    SeededRng rng(seed);
    from_matrix(rng.uniform_matrix(rows, cols, lo, hi), out);
}

int ref_route_scores(const double* h_token, int64_t d, const double* w_g, int64_t n, double* p) {
    return guard([&] {
        Router r{to_matrix(w_g, n, d)};
        const auto v = route_scores(h_token, d, r);
        std::memcpy(p, v.data(), sizeof(double) * v.size());
    });
}

int ref_select_experts(const double* p, int64_t n, int64_t kk, int64_t* out, int64_t* out_n) {
    return guard([&] {
        const auto v = select_experts(std::vector<double>(p, p + n), kk);
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
        *out_n = static_cast<int64_t>(v.size());
    });
}

// w_a in the reference layout d x r (keys are columns).
int ref_ke_select(const double* h, int64_t tokens, int64_t d, const double* w_g, int64_t n_experts,
                  const double* w_a, int64_t r, int64_t kk, int64_t k, int64_t* per_token,
                  int64_t* tau, int64_t* union_out, int64_t* union_size, int64_t* take_out) {
    return guard([&] {
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        Router router{to_matrix(w_g, n_experts, d)};
        const ExpertPartition part = ExpertPartition::make(r, n_experts);
        AdapterWeights ad;
        ad.w_a = to_matrix(w_a, d, r);
        ad.w_b = Matrix(r, 0);
        ExpertSelection taus;
        const SelectionSet sel = ke_select(hb, router, part, ad, kk, k, &taus);
        const int64_t kk_eff = std::min<int64_t>(kk, n_experts);
        const int64_t take = std::min<int64_t>(k, kk_eff * part.expert_size);
        *take_out = take;
        write_selection(sel, take, per_token, union_out, union_size);
        if (tau) {
            for (int64_t t = 0; t < tokens; ++t)
                for (int64_t i = 0; i < kk_eff; ++i) tau[t * kk_eff + i] = taus.per_token_tau[t][i];
        }
    });
}

int ref_topk_select(const double* h, int64_t tokens, int64_t d, const double* w_a, int64_t r, int64_t k,
                    int64_t* per_token, int64_t* union_out, int64_t* union_size, int64_t* take_out) {
    return guard([&] {
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        const SelectionSet sel = topk_select(hb, to_matrix(w_a, d, r), k);
        const int64_t take = std::min<int64_t>(k, r);
        *take_out = take;
        write_selection(sel, take, per_token, union_out, union_size);
    });
}

int ref_gather_adapter(const double* w_a, const double* w_b, int64_t d, int64_t r, const int64_t* s,
                       int64_t ns, double* w_a_k, double* w_b_k) {
    return guard([&] {
        AdapterWeights ad{to_matrix(w_a, d, r), to_matrix(w_b, r, d)};
        const GatheredAdapter g = gather_adapter(ad, std::vector<index_t>(s, s + ns));
        from_matrix(g.w_a_k, w_a_k);
        from_matrix(g.w_b_k, w_b_k);
    });
}

// out = f(h w_in) w_out + ReLU(h w_a_k) w_b_k; z (T x s) and base_pre (T x n) are the cache.
int ref_ffn_forward(const double* h, int64_t tokens, int64_t d, const double* w_in, const double* w_out,
                    int64_t n, int act, const double* w_a_k, const double* w_b_k, int64_t s, double* out,
                    double* z, double* base_pre) {
    return guard([&] {
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        const BaseFfn base = make_base(w_in, w_out, d, n, act);
        FfnCache cache;
        const HiddenBatch o = sparse_ffn_pa(hb, base, to_matrix(w_a_k, d, s), to_matrix(w_b_k, s, d), &cache);
        from_matrix(o.values, out);
        if (z) from_matrix(cache.z, z);
        if (base_pre) from_matrix(cache.base_pre, base_pre);
    });
}

// Runs sparse_ffn_pa (to build the cache) then sparse_backward.
int ref_ffn_backward(const double* h, int64_t tokens, int64_t d, const double* w_in, const double* w_out,
                     int64_t n, int act, const double* w_a_k, const double* w_b_k, int64_t s,
                     const double* grad_out, double* grad_w_a_k, double* grad_w_b_k, double* grad_h) {
    return guard([&] {
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        const BaseFfn base = make_base(w_in, w_out, d, n, act);
        const Matrix wak = to_matrix(w_a_k, d, s);
        const Matrix wbk = to_matrix(w_b_k, s, d);
        FfnCache cache;
        sparse_ffn_pa(hb, base, wak, wbk, &cache);
        const SparseFfnGrads g = sparse_backward(to_matrix(grad_out, tokens, d), cache, wak, wbk, base);
        from_matrix(g.grad_w_a_k, grad_w_a_k);
        from_matrix(g.grad_w_b_k, grad_w_b_k);
        from_matrix(g.grad_h, grad_h);
    });
}

void* ref_store_init(int64_t layers, int64_t d, int64_t r, int64_t n, int train_router, uint64_t seed) {
    HostStore* s = nullptr;
    guard([&] { s = new HostStore(HostStore::init(layers, d, r, n, train_router != 0, seed)); });
    return s;
}

void ref_store_free(void* s) { delete static_cast<HostStore*>(s); }

// stage_router_grads (memtier.cpp:157-172): stage_g[rows[j]] += grad_rows[j], staged_g = 1.
int ref_stage_router_grads(void* sp, int64_t layer, const int64_t* rows, int64_t n, const double* grad_rows) {
    return guard([&] {
        HostStore& st = *static_cast<HostStore*>(sp);
        stage_router_grads(st, layer, std::vector<index_t>(rows, rows + n), to_matrix(grad_rows, n, st.dim()));
    });
}

// router rows of the layer (memtier.cpp:211-227 state): w_g, m_g, v_g [N x d] and router_step [N]
int ref_store_router(void* sp, int64_t layer, double* w_g, double* m_g, double* v_g, int64_t* step) {
    return guard([&] {
        const HostLayer& hl = static_cast<HostStore*>(sp)->layer(layer);
        if (w_g) from_matrix(hl.router.w_g, w_g);
        if (m_g) from_matrix(hl.m_g, m_g);
        if (v_g) from_matrix(hl.v_g, v_g);
        if (step)
            for (size_t i = 0; i < hl.router_step.size(); ++i) step[i] = hl.router_step[i];
    });
}

// save_checkpoint (memtier.cpp:288-326) of the reference store, global_step set first.
int ref_store_save(void* sp, const char* path, const char* extra_json, int64_t step) {
    return guard([&] {
        HostStore& st = *static_cast<HostStore*>(sp);
        st.global_step = step;
        save_checkpoint(st, path, extra_json);
    });
}

int ref_store_get(void* sp, int64_t layer, int id, double* out) {
    return guard([&] { from_matrix(*store_tensor(static_cast<HostStore*>(sp)->layer(layer), id), out); });
}

int ref_store_set(void* sp, int64_t layer, int id, const double* in) {
    return guard([&] {
        Matrix* m = store_tensor(static_cast<HostStore*>(sp)->layer(layer), id);
        *m = to_matrix(in, m->rows, m->cols);
    });
}

int ref_store_pair_step(void* sp, int64_t layer, int64_t* out) {
    return guard([&] {
        const auto& v = static_cast<HostStore*>(sp)->layer(layer).pair_step;
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}

int ref_store_staged(void* sp, int64_t layer, int8_t* out) {
    return guard([&] {
        const auto& v = static_cast<HostStore*>(sp)->layer(layer).staged;
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}

int ref_scatter_grads(void* sp, int64_t layer, const int64_t* s, int64_t ns, const double* gwa,
                      const double* gwb, int64_t* meter_d2h) {
    return guard([&] {
        HostStore& st = *static_cast<HostStore*>(sp);
        CommMeter meter;
        scatter_grads(st, meter, layer, std::vector<index_t>(s, s + ns), to_matrix(gwa, st.dim(), ns),
                      to_matrix(gwb, ns, st.dim()));
        if (meter_d2h) *meter_d2h = meter.total_device_to_host();
    });
}

int ref_sparse_adam(void* sp, int64_t layer, double beta1, double beta2, double eps, double lr) {
    return guard([&] {
        AdamHyper hy;
        hy.beta1 = beta1;
        hy.beta2 = beta2;
        hy.eps = eps;
        sparse_adam_update(*static_cast<HostStore*>(sp), layer, hy, lr);
    });
}

// One MEFT layer step exactly as trainer.cpp drives it (base FFN width 0):
// meft_ffn -> sparse_backward -> scatter_grads -> sparse_adam_update.
// phase_s[0..5] = selection, fetch, forward, backward, scatter, adam seconds.
int ref_layer_step(void* sp, int64_t layer, const double* h, int64_t tokens, const double* grad_out,
                   int64_t kk, int64_t k, double lr, double* out, double* grad_h, int64_t* union_size,
                   double* phase_s) {
    return guard([&] {
        using clk = std::chrono::steady_clock;
        HostStore& st = *static_cast<HostStore*>(sp);
        const int64_t d = st.dim();
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        BaseFfn base;
        base.w_in = Matrix(d, 0);
        base.w_out = Matrix(0, d);
        const ExpertPartition part = ExpertPartition::make(st.pairs(), st.experts());
        CommMeter meter;
        MeftFfnCache cache;
        MeftFfnTimers tm;
        auto t0 = clk::now();
        const HiddenBatch o = meft_ffn(hb, base, st.layer(layer).router, part, kk, k, st, meter, layer,
                                       &cache, &tm);
        auto t1 = clk::now();
        const SparseFfnGrads g =
            sparse_backward(to_matrix(grad_out, tokens, d), cache.ffn, cache.slice.w_a_k, cache.slice.w_b_k, base);
        auto t2 = clk::now();
        scatter_grads(st, meter, layer, cache.sel.unioned, g.grad_w_a_k, g.grad_w_b_k, &cache.slice);
        auto t3 = clk::now();
        sparse_adam_update(st, layer, AdamHyper{}, lr);
        auto t4 = clk::now();
        if (out) from_matrix(o.values, out);
        if (grad_h) from_matrix(g.grad_h, grad_h);
        if (union_size) *union_size = static_cast<int64_t>(cache.sel.unioned.size());
        if (phase_s) {
            phase_s[0] = tm.selection_s;
            phase_s[1] = tm.fetch_s;
            phase_s[2] = tm.base_s + tm.adapter_s;
            phase_s[3] = std::chrono::duration<double>(t2 - t1).count();
            phase_s[4] = std::chrono::duration<double>(t3 - t2).count();
            phase_s[5] = std::chrono::duration<double>(t4 - t3).count();
            (void)t0;
        }
    });
}

// ---- the layer step in phases (bench.py's reference arm; see the header comment)
struct RefStep {
    int64_t layer = 0;
    BaseFfn base;
    CommMeter meter;
    MeftFfnCache cache;  // sel + taus + slice of the whole batch (meft_ffn.cpp:22-28)
    SparseFfnGrads grads;  // of the last row slice (scatter_grads' cost does not depend on the values)
};

// push_hidden + ke_select + fetch of the whole T-token batch, timed; returns the step state (nullptr on error).
void* ref_step_begin(void* sp, int64_t layer, const double* h, int64_t tokens, int64_t kk, int64_t k,
                     double* select_s, double* fetch_s, int64_t* union_size) {
    RefStep* rs = nullptr;
    const int rc = guard([&] {
        using clk = std::chrono::steady_clock;
        HostStore& st = *static_cast<HostStore*>(sp);
        const int64_t d = st.dim();
        auto state = std::make_unique<RefStep>();
        state->layer = layer;
        state->base.w_in = Matrix(d, 0);
        state->base.w_out = Matrix(0, d);
        HiddenBatch hb(1, tokens, to_matrix(h, tokens, d));
        state->meter.set_layer(layer);
        push_hidden(state->meter, hb.batch, hb.seq, hb.dim());
        const ExpertPartition part = ExpertPartition::make(st.pairs(), st.experts());
        auto t0 = clk::now();
        state->cache.sel = ke_select(hb, st.layer(layer).router, part, st.layer(layer).adapter, kk, k,
                                     &state->cache.taus);
        auto t1 = clk::now();
        state->cache.slice = fetch(st, state->meter, layer, state->cache.sel.unioned);
        auto t2 = clk::now();
        *select_s = std::chrono::duration<double>(t1 - t0).count();
        *fetch_s = std::chrono::duration<double>(t2 - t1).count();
        *union_size = static_cast<int64_t>(state->cache.sel.unioned.size());
        rs = state.release();
    });
    return rc == 0 ? rs : nullptr;
}

// sparse_ffn_pa + sparse_backward of `rows` token rows of the batch against the whole batch's union, timed.
int ref_step_rows(void* state, const double* h_rows, const double* g_rows, int64_t rows, double* forward_s,
                  double* backward_s) {
    return guard([&] {
        using clk = std::chrono::steady_clock;
        RefStep& rs = *static_cast<RefStep*>(state);
        const int64_t d = rs.cache.slice.w_b_k.cols;
        HiddenBatch hb(1, rows, to_matrix(h_rows, rows, d));
        FfnCache fc;
        auto t0 = clk::now();
        const HiddenBatch o = sparse_ffn_pa(hb, rs.base, rs.cache.slice.w_a_k, rs.cache.slice.w_b_k, &fc);
        auto t1 = clk::now();
        rs.grads = sparse_backward(to_matrix(g_rows, rows, d), fc, rs.cache.slice.w_a_k, rs.cache.slice.w_b_k,
                                   rs.base);
        auto t2 = clk::now();
        (void)o;
        *forward_s = std::chrono::duration<double>(t1 - t0).count();
        *backward_s = std::chrono::duration<double>(t2 - t1).count();
    });
}

// scatter_grads of the union + sparse_adam_update, timed; frees the step state.
int ref_step_finish(void* state, void* sp, double lr, double* scatter_s, double* adam_s) {
    std::unique_ptr<RefStep> rs(static_cast<RefStep*>(state));
    return guard([&] {
        using clk = std::chrono::steady_clock;
        HostStore& st = *static_cast<HostStore*>(sp);
        auto t0 = clk::now();
        scatter_grads(st, rs->meter, rs->layer, rs->cache.sel.unioned, rs->grads.grad_w_a_k, rs->grads.grad_w_b_k,
                      &rs->cache.slice);
        auto t1 = clk::now();
        sparse_adam_update(st, rs->layer, AdamHyper{}, lr);
        auto t2 = clk::now();
        *scatter_s = std::chrono::duration<double>(t1 - t0).count();
        *adam_s = std::chrono::duration<double>(t2 - t1).count();
    });
}

}  // extern "C"
