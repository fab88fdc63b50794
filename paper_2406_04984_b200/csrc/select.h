// Internal selection launch API (see select.cu / select_tc.cuh).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace meft_dev {

size_t select_workspace_bytes(int64_t T, int64_t d, int64_t M, int64_t N, int64_t kk_eff);

// Key-Experts selection for T tokens against N experts of E = M/N keys each.
// dtype 0: h/w_g/keys are f64 (exact fp64 SIMT scoring); 2: bf16 bits (certified tensor-core scoring with exact
// fp64 re-scoring of ambiguous candidates when allow_certified and the shape qualifies, else exact SIMT).
// keys is neuron-major [M x d]. per_token [T x take] ascending rows; tau_out [T x kk_eff] (nullable); union_idx
// [M] ascending with the device-side count in *union_size; stats (nullable, device int32[2]) receives the number
// of re-scored candidates and of sequential fallbacks. N == 1 is the flat topk_select of adapter.cpp:42-84.
void ke_select_device(cudaStream_t st, int dtype, const void* h, const void* w_g, const void* keys, int64_t T,
                      int64_t d, int64_t M, int64_t N, int64_t kk_eff, int64_t take, void* ws, size_t ws_bytes,
                      int32_t* per_token, int32_t* tau_out, int32_t* union_idx, int32_t* union_size,
                      int32_t* stats = nullptr, bool allow_certified = true,
                      const float* key_norms = nullptr, const int32_t* key_lsb = nullptr);  // cached key stats

// select_experts (experts.cpp:30-45) over precomputed router scores [T x N].
void route_topk_device(cudaStream_t st, const double* scores, int64_t T, int64_t N, int64_t kk, int32_t* tau);

// Ordered compaction: out_idx = ascending indices with flags[i] != 0, *count_dev = their number.
// block_ws needs ceil(M/1024) int32.
void compact_flags(cudaStream_t st, const uint8_t* flags, int64_t M, int32_t* out_idx, int32_t* count_dev,
                   int32_t* block_ws);

}  // namespace meft_dev

// ---- building blocks of the expert-sharded selection (tokens live on their home rank, keys on their owner)
namespace meft_dev {
// norms (rounded up) and minimum LSB exponents of bf16 rows
void row_stats(cudaStream_t st, const uint16_t* x, int64_t rows, int64_t d, float* norms, int32_t* minlsb);
// certified router: tau [T x kk_eff] ascending (exact), counts may be null. ws >= route_workspace_bytes.
size_t route_workspace_bytes(int64_t T, int64_t d, int64_t N);
void route_certified(cudaStream_t st, const uint16_t* h, const uint16_t* w_g, int64_t T, int64_t d, int64_t N,
                     int64_t kk_eff, void* ws, int32_t* tau, int32_t* stats);
// approximate scores of R token rows against the E keys of their (local) expert: cand [R x E] fp32.
size_t score_workspace_bytes(int64_t R, int64_t d, int64_t n_experts, int64_t E);
void score_candidates(cudaStream_t st, const uint16_t* rows, const int32_t* expert, int64_t R, int64_t d,
                      const uint16_t* keys, int64_t n_experts, int64_t E, void* ws, float* cand);
// exact reference scores of Q (row, key) pairs
void exact_pair_scores(cudaStream_t st, const uint16_t* rows, const float* rn, const int32_t* rl,
                       const uint16_t* keys, const float* kn, const int32_t* kl, const int32_t* pair_row,
                       const int32_t* pair_key, int64_t Q, int64_t d, double* out, int32_t* stats);
// certified top-K classification / finalisation (see select_tc.cuh)
void topk_classify(cudaStream_t st, const float* cand, const int32_t* tau, int64_t T, int64_t kk, int64_t E,
                   int64_t take, int64_t d, const float* hn, const float* kn, int32_t* sure, int32_t* n_sure,
                   int32_t* amb, int32_t* n_amb, int32_t* amb_count_per_expert);
void topk_finalize(cudaStream_t st, const int32_t* sure, const int32_t* n_sure, const int32_t* amb,
                   const int32_t* n_amb, const double* x, int64_t T, int64_t C, int64_t take, int32_t* per_token,
                   uint8_t* flags);
}  // namespace meft_dev
