// TEST / MEASUREMENT INFRASTRUCTURE: the MEFT layer step through the reference's public C++ API -- exactly the
// trainer's per-layer calls (trainer.cpp:220, 270, 283, 525): meft_ffn -> sparse_backward -> scatter_grads ->
// sparse_adam_update -- timed per phase with steady_clock. The same file is compiled twice:
//   * against the reference library (proj/src, CPU, OpenMP)           -> oracle/_ref/tests/layer_bench
//   * against the drop-in (include/meft/*.hpp + libmeft_dropin.so)      -> build/dropin_tests/layer_bench
// so a C++ user of the reference sees what switching the library buys on the API path (host tables in, host tables
// out; tools/dropin_bench.py runs both). Inputs: HostStore::init(seed 1), W_B ~ U(+-1/sqrt d) from mix_seed(1,
// 0x7001), h / grad_out ~ U(-1, 1) from 0x7002 / 0x7003.
// Usage: layer_bench d M N K kk T steps   -> one JSON line per timed step
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "meft/adapter.hpp"
#include "meft/experts.hpp"
#include "meft/meft_ffn.hpp"
#include "meft/memtier.hpp"
#include "meft/rng.hpp"

using namespace meft;

int main(int argc, char** argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: layer_bench d M N K kk T steps\n");
        return 2;
    }
    const index_t d = std::atol(argv[1]), M = std::atol(argv[2]), N = std::atol(argv[3]), K = std::atol(argv[4]),
                  kk = std::atol(argv[5]), T = std::atol(argv[6]);
    const int steps = std::atoi(argv[7]);
    HostStore store = HostStore::init(1, d, M, N, false, 1);
    const double b = 1.0 / std::sqrt(double(d));
    store.layer(0).adapter.w_b = SeededRng(mix_seed(1, 0x7001)).uniform_matrix(M, d, -b, b);
    const HiddenBatch h(1, T, SeededRng(mix_seed(1, 0x7002)).uniform_matrix(T, d, -1.0, 1.0));
    const Matrix g = SeededRng(mix_seed(1, 0x7003)).uniform_matrix(T, d, -1.0, 1.0);
    BaseFfn base;
    base.w_in = Matrix(d, 0);
    base.w_out = Matrix(0, d);
    const ExpertPartition part = ExpertPartition::make(M, N);
    using clk = std::chrono::steady_clock;
    auto sec = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); };
    for (int s = 0; s <= steps; ++s) {  // step 0: warm-up (first-touch allocations, device context)
        CommMeter meter;
        MeftFfnCache cache;
        MeftFfnTimers tm;
        const auto t0 = clk::now();
        const HiddenBatch out = meft_ffn(h, base, store.layer(0).router, part, kk, K, store, meter, 0, &cache, &tm);
        const auto t1 = clk::now();
        const SparseFfnGrads gr = sparse_backward(g, cache.ffn, cache.slice.w_a_k, cache.slice.w_b_k, base);
        const auto t2 = clk::now();
        scatter_grads(store, meter, 0, cache.sel.unioned, gr.grad_w_a_k, gr.grad_w_b_k, &cache.slice);
        const auto t3 = clk::now();
        sparse_adam_update(store, 0, AdamHyper{}, 1e-4);
        const auto t4 = clk::now();
        if (s == 0) continue;
        const double total = sec(t0, t4);
        std::printf("{\"step\": %d, \"tokens\": %lld, \"union\": %zu, \"select_s\": %.6f, \"fetch_s\": %.6f, "
                    "\"forward_s\": %.6f, \"backward_s\": %.6f, \"scatter_s\": %.6f, \"adam_s\": %.6f, "
                    "\"step_s\": %.6f, \"tokens_per_s\": %.3f, \"check\": %.17g}\n",
                    s, static_cast<long long>(T), cache.sel.unioned.size(), tm.selection_s, tm.fetch_s,
                    sec(t0, t1) - tm.selection_s - tm.fetch_s, sec(t1, t2), sec(t2, t3), sec(t3, t4), total,
                    double(T) / total, out.values.at(0, 0) + gr.grad_h.at(T - 1, d - 1));
        std::fflush(stdout);
    }
    return 0;
}
