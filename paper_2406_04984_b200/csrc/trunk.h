// Internal launch API of the toy-trunk kernels (trunk.cu): fp64 device buffers, row-major, T = batch * l rows.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace meft_dev {

void embed_f64(cudaStream_t st, const double* emb, const double* pos, const int32_t* tok, int64_t T, int64_t l,
               int64_t d, double* h);
// q, k, v, ctx, out: [T x d]; probs: [T x l]
void attention_forward_f64(cudaStream_t st, const double* h, const double* wq, const double* wk, const double* wv,
                           const double* wo, const int32_t* seg, int64_t T, int64_t l, int64_t d, double* q,
                           double* k, double* v, double* probs, double* ctx, double* out);
// scratch: dctx, dq, dk, dv [T x d], ds [T x l]
void attention_backward_f64(cudaStream_t st, const double* wq, const double* wk, const double* wv, const double* wo,
                            const int32_t* seg, int64_t T, int64_t l, int64_t d, const double* q, const double* k,
                            const double* v, const double* probs, const double* dh_out, double* dctx, double* ds,
                            double* dq, double* dk, double* dv, double* dh);
void lm_loss_rows_f64(cudaStream_t st, const double* logits, int64_t T, int64_t V, const int32_t* target,
                      const uint8_t* mask, double scale, double* dlogits, double* term);
void argmax_logits_f64(cudaStream_t st, const double* emb, int64_t V, int64_t d, const double* h, int64_t* out);

}  // namespace meft_dev
