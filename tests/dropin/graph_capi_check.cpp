// A C++ caller of the C ABI alone (no Python, no torch): the enqueue-only layer step (meft_ctx_set_host_sync(ctx,
// 0)) of a two-layer store captured into a CUDA graph (meft_graph_*) and replayed, against the synchronising (host sync on)
// meft_layer_step on a twin store, bit for bit -- out, grad_h, the selection and every table -- over three
// iterations with fresh inputs copied into the captured buffers. The sequence INTEGRATION.md §2 shows for a trainer
// that launches a whole iteration's adapter layers as one graph (trainer.cpp:523-526's per-layer loop). Built by
// paper_2406_04984_b200/build.py:build_capi_checks; run by tests/test_gpu_enqueue_only.py.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "meft_cuda.h"

namespace {

void ck(meft_status st, meft_ctx* ctx, const char* what) {
    if (st != MEFT_OK) {
        std::printf("%s failed (%d): %s\n", what, int(st), meft_last_error(ctx));
        std::exit(1);
    }
}

std::vector<uint16_t> bf16_bits(const std::vector<double>& x) {  // values are bf16-exact (round_bf16 = 1)
    std::vector<uint16_t> out(x.size());
    for (size_t i = 0; i < x.size(); ++i) {
        const float f = float(x[i]);
        uint32_t u;
        std::memcpy(&u, &f, 4);
        out[i] = uint16_t(u >> 16);
    }
    return out;
}

template <class T>
std::vector<T> host_copy(meft_ctx* ctx, const void* dev, size_t n) {
    std::vector<T> v(n);
    ck(meft_copy_to_host(ctx, v.data(), dev, n * sizeof(T)), ctx, "copy_to_host");
    return v;
}

void* dev_alloc(meft_ctx* ctx, size_t bytes) {
    void* p = nullptr;
    ck(meft_device_alloc(ctx, bytes, &p), ctx, "device_alloc");
    return p;
}

}  // namespace

int main() {
    const int64_t d = 1024, M = 16384, N = 64, K = 32, kk = 4, T = 300, L = 2;  // a sparse union: kernel gather
    const double lr = 1e-3, b1 = 0.9, b2 = 0.999, eps = 1e-8;
    meft_ctx* ref = nullptr;  // host sync on, legacy default stream
    meft_ctx* ctx = nullptr;  // host sync off, its own (capturable) stream
    ck(meft_ctx_create(0, nullptr, &ref), nullptr, "ctx_create");
    ck(meft_ctx_create(0, MEFT_OWN_STREAM, &ctx), nullptr, "ctx_create");
    ck(meft_ctx_set_host_sync(ref, 1), ref, "set_host_sync");  // the synchronising reference step
    ck(meft_ctx_set_host_sync(ctx, 0), ctx, "set_host_sync");
    meft_store* st[2] = {nullptr, nullptr};  // [0] reference steps on `ref`, [1] the graph's store on `ctx`
    meft_ctx* owner[2] = {ref, ctx};
    for (int i = 0; i < 2; ++i) {
        ck(meft_store_create(owner[i], L, d, M, N, MEFT_STORE_MIXED, &st[i]), owner[i], "store_create");
        ck(meft_store_init_reference(owner[i], st[i], 7), owner[i], "init_reference");
    }
    const size_t td = size_t(T * d);
    uint16_t* h = static_cast<uint16_t*>(dev_alloc(ctx, td * 2));  // the captured input buffers
    uint16_t* g = static_cast<uint16_t*>(dev_alloc(ctx, td * 2));
    float* out[2][2];
    float* gh[2][2];
    int32_t* per[2][2];
    for (int i = 0; i < 2; ++i)
        for (int l = 0; l < L; ++l) {
            out[i][l] = static_cast<float*>(dev_alloc(ctx, td * 4));
            gh[i][l] = static_cast<float*>(dev_alloc(ctx, td * 4));
            per[i][l] = static_cast<int32_t*>(dev_alloc(ctx, size_t(T * K) * 4));
        }
    auto load_inputs = [&](int step) {
        std::vector<double> hd(td), gd(td);
        ck(meft_reference_uniform(9, 0x7002 + step, int64_t(td), -1.0, 1.0, 1, hd.data()), ctx, "h");
        ck(meft_reference_uniform(9, 0x7003 + step, int64_t(td), -1.0, 1.0, 1, gd.data()), ctx, "g");
        const auto hb = bf16_bits(hd), gb = bf16_bits(gd);
        ck(meft_copy_to_device(ctx, h, hb.data(), td * 2), ctx, "copy h");
        ck(meft_copy_to_device(ctx, g, gb.data(), td * 2), ctx, "copy g");
        ck(meft_synchronize(ctx), ctx, "synchronize");  // h, g also feed the reference context's stream
    };
    auto step_of = [&](int i, meft_ctx* c) {
        for (int64_t l = 0; l < L; ++l)
            ck(meft_layer_step(c, st[i], l, h, g, T, kk, K, b1, b2, eps, lr, out[i][l], gh[i][l], per[i][l], nullptr,
                               nullptr),
               c, "layer_step");
    };
    int failures = 0;
    auto compare = [&](int it) {
        ck(meft_synchronize(ctx), ctx, "synchronize");
        ck(meft_synchronize(ref), ref, "synchronize");
        bool same = true;
        for (int64_t l = 0; l < L; ++l) {
            same = same && host_copy<float>(ctx, out[0][l], td) == host_copy<float>(ctx, out[1][l], td);
            same = same && host_copy<float>(ctx, gh[0][l], td) == host_copy<float>(ctx, gh[1][l], td);
            same = same && host_copy<int32_t>(ctx, per[0][l], size_t(T * K)) ==
                               host_copy<int32_t>(ctx, per[1][l], size_t(T * K));
            for (meft_tensor t : {MEFT_T_W_A, MEFT_T_W_B, MEFT_T_M_A, MEFT_T_V_A, MEFT_T_M_B, MEFT_T_V_B,
                                  MEFT_T_PAIR_STEP, MEFT_T_W_A_COMPUTE}) {
                void* p[2];
                int64_t r_, c_;
                meft_dtype dt_;
                for (int i = 0; i < 2; ++i) ck(meft_store_tensor(st[i], l, t, &p[i], &dt_, &r_, &c_), ctx, "tensor");
                const size_t words = (t == MEFT_T_PAIR_STEP || t == MEFT_T_W_A_COMPUTE)
                                         ? size_t(r_ * c_) / (t == MEFT_T_W_A_COMPUTE ? 2 : 1)
                                         : size_t(r_ * c_);
                same = same && host_copy<uint32_t>(ctx, p[0], words) == host_copy<uint32_t>(ctx, p[1], words);
            }
        }
        std::printf("iteration %d: graph replay %s the synchronising steps\n", it, same ? "equals" : "DIFFERS from");
        failures += !same;
    };

    load_inputs(0);  // one eager iteration on both (allocates the graph context's scratch), then capture one
    step_of(0, ref);
    step_of(1, ctx);
    compare(0);
    meft_graph* graph = nullptr;
    ck(meft_graph_begin(ctx), ctx, "graph_begin");
    step_of(1, ctx);
    ck(meft_graph_end(ctx, &graph), ctx, "graph_end");
    for (int it = 1; it <= 3; ++it) {
        load_inputs(it);
        ck(meft_graph_launch(ctx, graph), ctx, "graph_launch");
        step_of(0, ref);
        compare(it);
    }
    meft_graph_destroy(graph);
    for (int i = 0; i < 2; ++i)
        for (int l = 0; l < L; ++l) {
            meft_device_free(ctx, out[i][l]);
            meft_device_free(ctx, gh[i][l]);
            meft_device_free(ctx, per[i][l]);
        }
    meft_device_free(ctx, h);
    meft_device_free(ctx, g);
    meft_store_destroy(st[0]);
    meft_store_destroy(st[1]);
    meft_ctx_destroy(ctx);
    meft_ctx_destroy(ref);
    std::printf("graph_capi_check: %s\n", failures ? "FAILED" : "OK");
    return failures ? 1 : 0;
}
