// Trainable router on the fused layer step (train_router): the straight-through gradient of trainer.cpp:140-181
// (stage_router_ste) built from tensors the step already holds, then staged + Adam'd like memtier.cpp:157-172 and
// 211-227.
//
//   dL/dp[t, e] = <grad_out_t, y_e,t>,  y_e,t = sum_{c in S, c in expert e, z[t,c] > 0} z[t,c] * w_b[c]
//               = sum_{c in S cap e} act[t,c] * (grad_out_t . w_b[c])  =  sum_{c in S cap e} act[t,c] * masked[t,c]
// because act = ReLU(z) and masked = (grad_out . w_b^T) where z > 0: a segmented row-sum over the union columns of
// expert e of the two [T x |S|] bf16 matrices the FFN forward/backward already produced. Then
//   grad_g[e] = sum over (t, slot) routed to e (and with some z > 0 there) of dL/dp[t, e] * h_t.
#include <cstdint>

#include "common.cuh"
#include "stream_ops.h"

namespace meft_dev {
namespace {

// lo[e] = first union position of expert e (S ascending, experts are contiguous id ranges), lo[N] = |S|.
__global__ void k_expert_ranges(const int32_t* __restrict__ uni, int su, int E, int N, int32_t* __restrict__ lo) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e > N) return;
    const int key = e * E;
    int a = 0, b = su;  // first position with uni[p] >= key
    while (a < b) {
        const int m = (a + b) >> 1;
        if (uni[m] < key) a = m + 1; else b = m;
    }
    lo[e] = a;
}

// Warp per (token, routed slot): dldp = sum_{c in [lo[e], lo[e+1])} act[t,c] * masked[t,c] (fp32 products of bf16,
// fp64 accumulation); live = any act[t,c] > 0 there (the reference skips the pair otherwise).
__global__ void k_router_dldp(const uint16_t* __restrict__ act, const uint16_t* __restrict__ masked, int64_t ld,
                              const int32_t* __restrict__ tau, int T, int kk, const int32_t* __restrict__ lo,
                              float* __restrict__ dldp, uint8_t* __restrict__ live) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= T * kk) return;
    const int t = w / kk, e = tau[w];
    const int c0 = lo[e], c1 = lo[e + 1];
    const uint16_t* a = act + int64_t(t) * ld;
    const uint16_t* m = masked + int64_t(t) * ld;
    double s = 0.0;
    int any = 0;
    for (int c = c0 + lane; c < c1; c += 32) {
        const float av = bf16_bits_to_f32(a[c]);
        any |= av > 0.0f;
        s += double(av) * double(bf16_bits_to_f32(m[c]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        any |= __shfl_xor_sync(0xffffffffu, any, o);
    }
    if (lane == 0) {
        dldp[w] = float(s);
        live[w] = uint8_t(any);
    }
}

// CTA per expert: grad_g[e] = sum over live (t, slot) routed to e, in (t, slot) order (deterministic), of
// dldp * h_t; touched[e] = any such pair. Each thread owns d / blockDim columns in fp32.
constexpr int RG_THREADS = 256;
constexpr int RG_CHUNK = 1024;
__global__ void __launch_bounds__(RG_THREADS) k_router_grad(const int32_t* __restrict__ tau, int TK, int kk,
                                                            const float* __restrict__ dldp,
                                                            const uint8_t* __restrict__ live,
                                                            const uint16_t* __restrict__ h, int d,
                                                            float* __restrict__ grad_g, uint8_t* __restrict__ touched) {
    const int e = blockIdx.x, tid = threadIdx.x;
    __shared__ int s_idx[RG_CHUNK];
    __shared__ int s_cnt[RG_THREADS / 32];
    __shared__ int s_n;
    constexpr int MAXC = 32;  // columns per thread (d <= 8192)
    float acc[MAXC];
#pragma unroll
    for (int j = 0; j < MAXC; ++j) acc[j] = 0.f;
    int total = 0;
    for (int base = 0; base < TK; base += RG_CHUNK) {
        // ordered compaction of this chunk's matches: 4 entries per thread, warp + block prefix
        int flags[RG_CHUNK / RG_THREADS];
        int mine = 0;
#pragma unroll
        for (int q = 0; q < RG_CHUNK / RG_THREADS; ++q) {
            const int i = base + tid * (RG_CHUNK / RG_THREADS) + q;
            flags[q] = (i < TK && tau[i] == e && live[i]) ? 1 : 0;
            mine += flags[q];
        }
        const int lane = tid & 31, wid = tid >> 5;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) s_cnt[wid] = incl;
        __syncthreads();
        int before = incl - mine;
        for (int w = 0; w < wid; ++w) before += s_cnt[w];
        if (tid == RG_THREADS - 1) s_n = before + mine;
#pragma unroll
        for (int q = 0; q < RG_CHUNK / RG_THREADS; ++q)
            if (flags[q]) s_idx[before++] = base + tid * (RG_CHUNK / RG_THREADS) + q;
        __syncthreads();
        const int n = s_n;
        for (int k = 0; k < n; ++k) {
            const int i = s_idx[k];
            const float g = dldp[i];
            const uint16_t* hr = h + int64_t(i / kk) * d;
#pragma unroll
            for (int j = 0; j < MAXC; ++j) {
                const int x = tid + j * RG_THREADS;
                if (x < d) acc[j] = fmaf(g, bf16_bits_to_f32(hr[x]), acc[j]);
            }
        }
        total += n;
        __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < MAXC; ++j) {
        const int x = tid + j * RG_THREADS;
        if (x < d) grad_g[int64_t(e) * d + x] = acc[j];
    }
    if (tid == 0) touched[e] = total > 0 ? 1 : 0;
}

}  // namespace

void router_ste_grads(cudaStream_t st, const int32_t* uni, int64_t su, int64_t E, int64_t N, const uint16_t* act,
                      const uint16_t* masked, int64_t ld, const int32_t* tau, int64_t T, int64_t kk,
                      const uint16_t* h, int64_t d, int32_t* lo_ws, float* dldp_ws, uint8_t* live_ws, float* grad_g,
                      uint8_t* touched) {
    if (d > 32 * RG_THREADS) throw MeftError(2, "router training: d must be <= 8192");
    k_expert_ranges<<<int((N + 1 + 255) / 256), 256, 0, st>>>(uni, int(su), int(E), int(N), lo_ws);
    check_launch("k_expert_ranges");
    const int64_t TK = T * kk;
    k_router_dldp<<<int((TK * 32 + 255) / 256), 256, 0, st>>>(act, masked, ld, tau, int(T), int(kk), lo_ws, dldp_ws,
                                                              live_ws);
    check_launch("k_router_dldp");
    k_router_grad<<<int(N), RG_THREADS, 0, st>>>(tau, int(TK), int(kk), dldp_ws, live_ws, h, int(d), grad_g, touched);
    check_launch("k_router_grad");
}

}  // namespace meft_dev
