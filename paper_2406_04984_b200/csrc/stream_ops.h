// Internal launch API of the HBM-streaming kernels (see stream_ops.cu). dtype codes: 0 f64, 1 f32, 2 bf16.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace meft_dev {

void gather_rows1(cudaStream_t st, const void* src, int64_t row_bytes, const int32_t* idx, int64_t n, void* dst);
// count_dev (optional): the row count is *count_dev (at most count when count > 0); pad64 (with count_dev and the
// capacity as count): rows up to the next multiple of 64 after the count are written as zeros
void gather_rows2(cudaStream_t st, const void* a, const void* b, int64_t row_bytes, const int32_t* idx,
                  const int32_t* count_dev, int64_t count, void* oa, void* ob, bool pad64 = false);
void check_sorted_unique(cudaStream_t st, const int32_t* idx, int64_t n, int64_t limit, int32_t* err_dev);
void stage_add(cudaStream_t st, int stage_dtype, void* stage, int64_t d, const int32_t* idx, int64_t n, int g_dtype,
               const void* g, uint8_t* staged);
// scatter_grads with repeated ids (scatter_seg.cu): stable sort by id, one CTA per run of equal ids adding its rows
// in position order -- atomic-free and bit-identical to the sequential per-entry loop.
size_t stage_add_segmented_ws(int64_t n);
void stage_add_segmented(cudaStream_t st, int stage_dtype, void* stage, int64_t d, const int32_t* idx, int64_t n,
                         int g_dtype, const void* g, uint8_t* staged, void* ws, size_t ws_bytes);
void mark_rows(cudaStream_t st, uint8_t* staged, const int32_t* idx, const int32_t* count_dev, int64_t count);
void union_holes(cudaStream_t st, const int32_t* idx, const int32_t* n_dev, int32_t* out);
void slot_sum(cudaStream_t st, const float* recv, int world, int64_t n, float* out);  // sum of `world` slots of n
void histogram_add(cudaStream_t st, const int32_t* idx, int64_t n, int64_t* hist);  // hist[idx[i]] += 1
// router.cu: straight-through router gradient of the fused step (trainer.cpp:140-181). grad_g [N x d] fp32 is
// fully written; touched[e] = some token routed to e had a positive activation in e's union columns.
void router_ste_grads(cudaStream_t st, const int32_t* uni, int64_t su, int64_t E, int64_t N, const uint16_t* act,
                      const uint16_t* masked, int64_t ld, const int32_t* tau, int64_t T, int64_t kk,
                      const uint16_t* h, int64_t d, int32_t* lo_ws, float* dldp_ws, uint8_t* live_ws, float* grad_g,
                      uint8_t* touched);
void union_holes_n(cudaStream_t st, const int32_t* idx, int64_t n, int32_t* out);
void adam_mixed(cudaStream_t st, const int32_t* rows, const int32_t* count_dev, int64_t count, int64_t d, float* wa,
                void* ma, void* va, float* sa, uint16_t* ca, float* wb, void* mb, void* vb, float* sb,
                uint16_t* cb, int32_t* step, uint8_t* staged, double b1, double b2, double eps, double lr,
                int tables = 3, bool bump = true,  // tables: bit 0 keys, bit 1 values
                bool grads_by_position = false,    // sa/sb = [count x d] gradients of rows[0..count), kept as is
                float* key_norms = nullptr, int32_t* key_lsb = nullptr,  // refresh updated keys' select stats
                bool moments_bf16 = false);  // m/v tables are bf16 (COMPACT store), else fp32
// Adam fused into the weight-gradient GEMMs (EPI_ADAM_F32): advance step[rows[r]] and tabulate its
// (lr / (1 - b1^t), 1 / (1 - b2^t)) by position; then fold the epilogue's key statistics partials.
// n_dev (optional): the row count is min(n, *n_dev) -- a device-resident union size with n its capacity
void adam_coef_bump(cudaStream_t st, const int32_t* rows, int64_t n, int32_t* step, float2* coef, double b1,
                    double b2, double lr, const int32_t* n_dev = nullptr);
void adam_stats_finalize(cudaStream_t st, const int32_t* rows, int64_t n, const double* ss, const int32_t* lsb,
                         int64_t parts, float* kn, int32_t* kl, const int32_t* n_dev = nullptr);
void adam_f64(cudaStream_t st, const int32_t* rows, const int32_t* count_dev, int64_t count, int64_t d, double* wa,
              double* ma, double* va, double* sa, double* wb, double* mb, double* vb, double* sb, int32_t* step,
              uint8_t* staged, double b1, double b2, double eps, double lr);
void adam_rows_f64(cudaStream_t st, double* w, double* m, double* v, double* stage, int64_t* step, uint8_t* staged,
                   const int32_t* rows, int64_t n, int64_t d, double b1, double b2, double eps, double lr);
void convert(cudaStream_t st, int ddt, void* dst, int sdt, const void* src, int64_t n);
void convert_index(cudaStream_t st, bool to64, void* dst, const void* src, int64_t n);
void act_forward(cudaStream_t st, const double* x, double* y, int64_t n, int act);   // 0 SiLU, 1 ReLU
void act_backward(cudaStream_t st, double* g, const double* pre, int64_t n, int act);  // g *= act'(pre)
void flag_nonfinite(cudaStream_t st, const double* x, int64_t n, int32_t* flag_dev);
void flag_nonfinite_f32(cudaStream_t st, const float* x, int64_t n, int32_t* flag_dev);
void add_f64(cudaStream_t st, double* a, const double* b, int64_t n);                  // a += b (add_inplace)
void transpose8(cudaStream_t st, const void* src, void* dst, int64_t rows, int64_t cols);
void transpose2(cudaStream_t st, const void* src, void* dst, int64_t rows, int64_t cols);  // bf16 rows x cols

}  // namespace meft_dev
