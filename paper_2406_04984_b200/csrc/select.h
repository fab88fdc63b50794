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
                      int32_t* stats = nullptr, bool allow_certified = true);

// select_experts (experts.cpp:30-45) over precomputed router scores [T x N].
void route_topk_device(cudaStream_t st, const double* scores, int64_t T, int64_t N, int64_t kk, int32_t* tau);

// Ordered compaction: out_idx = ascending indices with flags[i] != 0, *count_dev = their number.
// block_ws needs ceil(M/1024) int32.
void compact_flags(cudaStream_t st, const uint8_t* flags, int64_t M, int32_t* out_idx, int32_t* count_dev,
                   int32_t* block_ws);

}  // namespace meft_dev
