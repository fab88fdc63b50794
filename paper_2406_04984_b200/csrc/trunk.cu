// The reference's frozen toy trunk (model.cpp:50-218) on the device, fp64, for the end-to-end trainer over the
// drop-in: token + positional embedding, single-head causal segment-local attention forward / backward, the tied
// LM loss and greedy argmax. Every reduction runs in the reference's order (dot: ascending unfused multiply-add,
// kernels.hpp:37-41; the contracted `+= a * b` loops as fma chains), so results are deterministic and independent
// of launch geometry. The matrix products go through dgemm (the reference matmul's ascending-k fma chain).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "stream_ops.h"
#include "trunk.h"

namespace meft_dev {
namespace {

__device__ __forceinline__ double dot_seq(const double* __restrict__ a, const double* __restrict__ b, int d) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc = __dadd_rn(acc, __dmul_rn(a[k], b[k]));
    return acc;
}

// model.cpp:50-68: h[t] = E[tok[t]] + pos[i], t = b*l + i
__global__ void k_embed(const double* __restrict__ emb, const double* __restrict__ pos,
                        const int32_t* __restrict__ tok, int64_t T, int l, int d, double* __restrict__ h) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < T * d; e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t t = e / d;
        const int x = int(e - t * d);
        const int i = int(t % l);
        h[e] = emb[int64_t(tok[t]) * d + x] + pos[int64_t(i) * d + x];
    }
}

// model.cpp:82-111, warp per query row t: scores over the same-segment causal sources (lanes over sources), the
// max / denominator chains in source order (lane 0), probabilities, then ctx[t] = sum_j p_j v_j (lanes over x,
// sources ascending). probs[t] holds the probabilities (0 where masked).
__global__ void k_attn_forward_rows(const double* __restrict__ q, const double* __restrict__ k,
                                    const double* __restrict__ v, const int32_t* __restrict__ seg, int64_t T, int l,
                                    int d, double inv_sqrt_d, double* __restrict__ probs, double* __restrict__ ctx) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    if (t >= T) return;
    const int i = int(t % l);
    const int64_t base = t - i;
    double* p = probs + t * l;
    for (int j = lane; j < l; j += 32) {
        const bool live = j <= i && seg[base + j] == seg[t];
        p[j] = live ? __dmul_rn(dot_seq(q + t * d, k + (base + j) * d, d), inv_sqrt_d) : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
        double mx = -1e300;
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t] && p[j] > mx) mx = p[j];
        double den = 0.0;
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) den += exp(p[j] - mx);
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) p[j] = exp(p[j] - mx) / den;
    }
    __syncwarp();
    for (int x = lane; x < d; x += 32) {
        double c = 0.0;
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) c = fma(p[j], v[(base + j) * d + x], c);
        ctx[t * d + x] = c;
    }
}

// model.cpp:135-160, warp per row t: dprobs_j = dot(dctx_t, v_j), common = sum_j p_j dprobs_j (source order),
// ds[t][j] = p_j (dprobs_j - common) / sqrt(d), dq[t] = sum_j ds_j k_j (lanes over x, sources ascending).
__global__ void k_attn_backward_rows(const double* __restrict__ k, const double* __restrict__ v,
                                     const double* __restrict__ probs, const double* __restrict__ dctx,
                                     const int32_t* __restrict__ seg, int64_t T, int l, int d, double inv_sqrt_d,
                                     double* __restrict__ ds, double* __restrict__ dq) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    if (t >= T) return;
    const int i = int(t % l);
    const int64_t base = t - i;
    const double* p = probs + t * l;
    double* s = ds + t * l;
    for (int j = lane; j < l; j += 32)
        s[j] = (j <= i && seg[base + j] == seg[t]) ? dot_seq(dctx + t * d, v + (base + j) * d, d) : 0.0;
    __syncwarp();
    if (lane == 0) {
        double common = 0.0;
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) common = fma(p[j], s[j], common);
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) s[j] = __dmul_rn(__dmul_rn(p[j], s[j] - common), inv_sqrt_d);
    }
    __syncwarp();
    for (int x = lane; x < d; x += 32) {
        double a = 0.0;
        for (int j = 0; j <= i; ++j)
            if (seg[base + j] == seg[t]) a = fma(s[j], k[(base + j) * d + x], a);
        dq[t * d + x] = a;
    }
}

// dk[j] = sum_{i >= j} ds[i][j] q_i and dv[j] = sum_{i >= j} p[i][j] dctx_i over the same segment, i ascending --
// the order in which the reference's outer query loop accumulates them (model.cpp:148-157). Warp per source row.
__global__ void k_attn_backward_cols(const double* __restrict__ q, const double* __restrict__ probs,
                                     const double* __restrict__ dctx, const double* __restrict__ ds,
                                     const int32_t* __restrict__ seg, int64_t T, int l, int d,
                                     double* __restrict__ dk, double* __restrict__ dv) {
    const int lane = threadIdx.x & 31;
    const int64_t tj = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    if (tj >= T) return;
    const int j = int(tj % l);
    const int64_t base = tj - j;
    for (int x = lane; x < d; x += 32) {
        double ak = 0.0, av = 0.0;
        for (int i = j; i < l; ++i) {
            const int64_t ti = base + i;
            if (seg[ti] != seg[tj]) continue;
            ak = fma(ds[ti * l + j], q[ti * d + x], ak);
            av = fma(probs[ti * l + j], dctx[ti * d + x], av);
        }
        dk[tj * d + x] = ak;
        dv[tj * d + x] = av;
    }
}

// model.cpp:175-203 per masked row (warp): max, denominator (vocabulary order, lane 0), the row's -log p
// (log_denom - logit[target], accumulated by the caller as loss = fma(term, scale, loss) in row order like the
// compiled reference), and dlogits = softmax * scale - scale at the target. Unmasked rows: zero gradient, no term.
__global__ void k_lm_loss_rows(const double* __restrict__ logits, int64_t T, int V,
                               const int32_t* __restrict__ target, const uint8_t* __restrict__ mask, double scale,
                               double* __restrict__ dlogits, double* __restrict__ term) {
    const int lane = threadIdx.x & 31;
    const int64_t t = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    if (t >= T) return;
    const double* lr = logits + t * V;
    double* dr = dlogits + t * V;
    if (!mask[t]) {
        for (int j = lane; j < V; j += 32) dr[j] = 0.0;
        if (lane == 0) term[t] = 0.0;
        return;
    }
    double log_den = 0.0;
    if (lane == 0) {
        double mx = lr[0];
        for (int j = 1; j < V; ++j) mx = mx < lr[j] ? lr[j] : mx;  // std::max
        double den = 0.0;
        for (int j = 0; j < V; ++j) den += exp(lr[j] - mx);
        log_den = log(den) + mx;
        term[t] = log_den - lr[target[t]];
    }
    log_den = __shfl_sync(0xffffffffu, log_den, 0);
    for (int j = lane; j < V; j += 32) dr[j] = exp(lr[j] - log_den) * scale;
    __syncwarp();
    if (lane == 0) dr[target[t]] -= scale;
}

// model.cpp:205-218: argmax_tok dot(h, E[tok]); ties toward the lowest token id. One warp.
__global__ void k_argmax_logits(const double* __restrict__ emb, int V, int d, const double* __restrict__ h,
                                int64_t* __restrict__ out) {
    const int lane = threadIdx.x;
    double best = -1e300;
    int bi = 0;
    for (int tok = lane; tok < V; tok += 32) {
        const double s = dot_seq(h, emb + int64_t(tok) * d, d);
        if (s > best) {
            best = s;
            bi = tok;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if (lane == 0) *out = bi;
}

int warps_grid(int64_t rows) { return int((rows * 32 + 255) / 256); }

}  // namespace

void embed_f64(cudaStream_t st, const double* emb, const double* pos, const int32_t* tok, int64_t T, int64_t l,
               int64_t d, double* h) {
    if (T <= 0 || d <= 0) return;
    k_embed<<<int(std::min<int64_t>((T * d + 255) / 256, 65535)), 256, 0, st>>>(emb, pos, tok, T, int(l), int(d), h);
    check_launch("k_embed");
}

void attention_forward_f64(cudaStream_t st, const double* h, const double* wq, const double* wk, const double* wv,
                           const double* wo, const int32_t* seg, int64_t T, int64_t l, int64_t d, double* q,
                           double* k, double* v, double* probs, double* ctx, double* out) {
    if (T <= 0) return;
    const DOperand H{h, d, 1};
    dgemm(st, T, d, d, H, DOperand{wq, d, 1}, q, d, DEPI_STORE, nullptr);
    dgemm(st, T, d, d, H, DOperand{wk, d, 1}, k, d, DEPI_STORE, nullptr);
    dgemm(st, T, d, d, H, DOperand{wv, d, 1}, v, d, DEPI_STORE, nullptr);
    k_attn_forward_rows<<<warps_grid(T), 256, 0, st>>>(q, k, v, seg, T, int(l), int(d), 1.0 / sqrt(double(d)), probs,
                                                       ctx);
    check_launch("k_attn_forward_rows");
    // out = h + ctx wo  (model.cpp:113: add(h, matmul(ctx, wo)))
    dgemm(st, T, d, d, DOperand{ctx, d, 1}, DOperand{wo, d, 1}, out, d, DEPI_STORE, nullptr);
    add_f64(st, out, h, T * d);
}

void attention_backward_f64(cudaStream_t st, const double* wq, const double* wk, const double* wv, const double* wo,
                            const int32_t* seg, int64_t T, int64_t l, int64_t d, const double* q, const double* k,
                            const double* v, const double* probs, const double* dh_out, double* dctx, double* ds,
                            double* dq, double* dk, double* dv, double* dh) {
    if (T <= 0) return;
    // dctx = dh_out wo^T
    dgemm(st, T, d, d, DOperand{dh_out, d, 1}, DOperand{wo, 1, d}, dctx, d, DEPI_STORE, nullptr);
    const double inv = 1.0 / sqrt(double(d));
    k_attn_backward_rows<<<warps_grid(T), 256, 0, st>>>(k, v, probs, dctx, seg, T, int(l), int(d), inv, ds, dq);
    check_launch("k_attn_backward_rows");
    k_attn_backward_cols<<<warps_grid(T), 256, 0, st>>>(q, probs, dctx, ds, seg, T, int(l), int(d), dk, dv);
    check_launch("k_attn_backward_cols");
    // dh = dh_out; dh += dq wq^T; dh += dk wk^T; dh += dv wv^T  (model.cpp:166-170, one add per product)
    MEFT_CUDA_CHECK(cudaMemcpyAsync(dh, dh_out, size_t(T * d) * 8, cudaMemcpyDeviceToDevice, st));
    const double* g[3] = {dq, dk, dv};
    const double* w[3] = {wq, wk, wv};
    for (int a = 0; a < 3; ++a) {
        dgemm(st, T, d, d, DOperand{g[a], d, 1}, DOperand{w[a], 1, d}, dctx, d, DEPI_STORE, nullptr);
        add_f64(st, dh, dctx, T * d);
    }
}

void lm_loss_rows_f64(cudaStream_t st, const double* logits, int64_t T, int64_t V, const int32_t* target,
                      const uint8_t* mask, double scale, double* dlogits, double* term) {
    if (T <= 0) return;
    k_lm_loss_rows<<<warps_grid(T), 256, 0, st>>>(logits, T, int(V), target, mask, scale, dlogits, term);
    check_launch("k_lm_loss_rows");
}

void argmax_logits_f64(cudaStream_t st, const double* emb, int64_t V, int64_t d, const double* h, int64_t* out) {
    k_argmax_logits<<<1, 32, 0, st>>>(emb, int(V), int(d), h, out);
    check_launch("k_argmax_logits");
}

}  // namespace meft_dev
