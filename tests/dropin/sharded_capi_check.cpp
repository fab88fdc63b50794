// A C++ caller of the C ABI alone (no Python, no torch): runs the expert-sharded layer step over the library's own
// NCCL communicator at world 1 and checks it against the single-GPU meft_layer_step bit for bit -- the sequence a
// C++ trainer would issue for a sharded layer (trainer.cpp:220, 270, 283, 525). Built by
// paper_2406_04984_b200/build.py:build_capi_checks; run by tests/test_gpu_sharded_capi.py.
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

void* dev_copy(meft_ctx* ctx, const void* host, size_t bytes) {
    void* p = nullptr;
    ck(meft_device_alloc(ctx, bytes, &p), ctx, "device_alloc");
    if (host) ck(meft_copy_to_device(ctx, p, host, bytes), ctx, "copy_to_device");
    return p;
}

template <class T>
std::vector<T> host_copy(meft_ctx* ctx, const void* dev, size_t n) {
    std::vector<T> v(n);
    ck(meft_copy_to_host(ctx, v.data(), dev, n * sizeof(T)), ctx, "copy_to_host");
    return v;
}

}  // namespace

int main() {
    const int64_t d = 512, M = 4096, N = 64, K = 32, kk = 4, T = 256;
    const double lr = 1e-3, b1 = 0.9, b2 = 0.999, eps = 1e-8;
    meft_ctx* ctx = nullptr;
    ck(meft_ctx_create(0, nullptr, &ctx), nullptr, "ctx_create");
    meft_store* st[2] = {nullptr, nullptr};  // [0] reference single-GPU step, [1] the world-1 shard
    std::vector<double> w_b(size_t(M * d));
    ck(meft_reference_uniform(1, 0x7001, M * d, -0.044, 0.044, 1, w_b.data()), ctx, "reference_uniform");
    for (auto& s : st) {
        ck(meft_store_create(ctx, 1, d, M, N, MEFT_STORE_MIXED, &s), ctx, "store_create");
        ck(meft_store_init_reference(ctx, s, 1), ctx, "init_reference");
        ck(meft_store_upload_host(ctx, s, 0, MEFT_T_W_B, w_b.data(), M, d), ctx, "upload w_b");
    }
    void* w_g = nullptr;  // the replicated router: the store's bf16 compute copy
    meft_dtype dt;
    int64_t rows, cols;
    ck(meft_store_tensor(st[1], 0, MEFT_T_W_G_COMPUTE, &w_g, &dt, &rows, &cols), ctx, "store_tensor");

    unsigned char id[128];
    ck(meft_nccl_unique_id(id), ctx, "nccl_unique_id");
    ck(meft_ctx_comm_init(ctx, id, 0, 1), ctx, "ctx_comm_init");

    const size_t td = size_t(T * d);
    float* out[2] = {static_cast<float*>(dev_copy(ctx, nullptr, td * 4)), static_cast<float*>(dev_copy(ctx, nullptr, td * 4))};
    float* gh[2] = {static_cast<float*>(dev_copy(ctx, nullptr, td * 4)), static_cast<float*>(dev_copy(ctx, nullptr, td * 4))};
    int32_t* per[2] = {static_cast<int32_t*>(dev_copy(ctx, nullptr, size_t(T * K) * 4)),
                       static_cast<int32_t*>(dev_copy(ctx, nullptr, size_t(T * K) * 4))};
    int failures = 0;
    for (int step = 0; step < 2; ++step) {
        std::vector<double> hd(td), gd(td);
        ck(meft_reference_uniform(5, 0x7002 + step, int64_t(td), -1.0, 1.0, 1, hd.data()), ctx, "h");
        ck(meft_reference_uniform(5, 0x7003 + step, int64_t(td), -1.0, 1.0, 1, gd.data()), ctx, "g");
        const auto hb = bf16_bits(hd), gb = bf16_bits(gd);
        const uint16_t* h = static_cast<const uint16_t*>(dev_copy(ctx, hb.data(), td * 2));
        const uint16_t* g = static_cast<const uint16_t*>(dev_copy(ctx, gb.data(), td * 2));
        meft_step_info info[2];
        int32_t* uni = static_cast<int32_t*>(dev_copy(ctx, nullptr, size_t(M) * 4));
        ck(meft_layer_step(ctx, st[0], 0, h, g, T, kk, K, b1, b2, eps, lr, out[0], gh[0], per[0], uni, &info[0]), ctx,
           "layer_step");
        ck(meft_layer_step_sharded(ctx, st[1], 0, static_cast<const uint16_t*>(w_g), h, g, T, kk, K, b1, b2, eps, lr,
                                   out[1], gh[1], per[1], &info[1]),
           ctx, "layer_step_sharded");
        ck(meft_synchronize(ctx), ctx, "synchronize");
        const bool same_out = host_copy<float>(ctx, out[0], td) == host_copy<float>(ctx, out[1], td);
        const bool same_gh = host_copy<float>(ctx, gh[0], td) == host_copy<float>(ctx, gh[1], td);
        const bool same_sel = host_copy<int32_t>(ctx, per[0], size_t(T * K)) == host_copy<int32_t>(ctx, per[1], size_t(T * K));
        const bool same_s = info[0].union_size == info[1].union_size;
        bool same_tables = true;
        for (meft_tensor t : {MEFT_T_W_A, MEFT_T_W_B, MEFT_T_M_A, MEFT_T_V_B, MEFT_T_PAIR_STEP}) {
            void* p[2];
            int64_t r_, c_;
            meft_dtype dt_;
            for (int i = 0; i < 2; ++i) ck(meft_store_tensor(st[i], 0, t, &p[i], &dt_, &r_, &c_), ctx, "store_tensor");
            same_tables = same_tables && host_copy<uint32_t>(ctx, p[0], size_t(r_ * c_)) ==
                                             host_copy<uint32_t>(ctx, p[1], size_t(r_ * c_));
        }
        int peer = -1, overlap = -1;
        ck(meft_ctx_sharded_paths(ctx, &peer, &overlap), ctx, "sharded_paths");
        std::printf("step %d: |S| %lld, selection %s, out %s, grad_h %s, tables %s, peer path %d, overlap %d\n", step,
                    (long long)info[1].union_size, same_sel ? "equal" : "DIFFER", same_out ? "equal" : "DIFFER",
                    same_gh ? "equal" : "DIFFER", same_tables ? "equal" : "DIFFER", peer, overlap);
        failures += !(same_out && same_gh && same_sel && same_s && same_tables);
        meft_device_free(ctx, const_cast<uint16_t*>(h));
        meft_device_free(ctx, const_cast<uint16_t*>(g));
        meft_device_free(ctx, uni);
    }
    ck(meft_ctx_clear_comm(ctx), ctx, "ctx_clear_comm");
    for (int i = 0; i < 2; ++i) {
        meft_device_free(ctx, out[i]);
        meft_device_free(ctx, gh[i]);
        meft_device_free(ctx, per[i]);
        meft_store_destroy(st[i]);
    }
    meft_ctx_destroy(ctx);
    std::printf("sharded_capi_check: %s\n", failures ? "FAILED" : "OK");
    return failures ? 1 : 0;
}
