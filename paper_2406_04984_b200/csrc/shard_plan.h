// Internal launch API of the sharded-selection bookkeeping kernels (shard_plan.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace meft_dev {

// Dispatch plan: (token, slot) i = t*kk + s goes to owner tau[i] / n_loc; stable bucket order by owner.
// pos_ws: T*kk ints; send_rows [T*kk x d] bf16 = h[t]; send_exp: owner-local expert; order[p] = i; inv[i] = p;
// counts[P] (device) rows per owner. send_rows may be null (no row copy: owners gather rows by token id).
void shard_dispatch(cudaStream_t st, const int32_t* tau, int64_t T, int64_t kk, int64_t n_loc, int P,
                    const uint16_t* h, int64_t d, int32_t* pos_ws, uint16_t* send_rows, int32_t* send_exp,
                    int32_t* order, int32_t* inv, int32_t* counts);
// dst[order[p]] = src[p], rows of `cols` fp32
void shard_unpermute_rows(cudaStream_t st, const float* src, const int32_t* order, int64_t n, int64_t cols, float* dst);
// Request plan, two steps around the host read of the total (ws[T]): fill one entry per ambiguous (t, a) --
// owner, the owner's receive row inv[t*kk + slot] + row_base[owner], owner-local key, back index t*C + a -- then
// bucket the n entries by owner (stable) into row / key / back with counts[P].
void shard_requests_fill(cudaStream_t st, const int32_t* amb, const int32_t* n_amb, const int32_t* tau,
                         const int32_t* inv, int64_t T, int64_t C, int64_t kk, int64_t E, int64_t M_loc,
                         const int32_t* row_base, int32_t* ws);
void shard_requests_sort(cudaStream_t st, int64_t T, int64_t C, int64_t M_loc, int P, int64_t n, int32_t* ws,
                         int32_t* row, int32_t* key, int32_t* back, int32_t* counts);
size_t shard_requests_ws_ints(int64_t T, int64_t C);
// dst[back[i]] = x[i]
void shard_scatter_f64(cudaStream_t st, const double* x, const int32_t* back, int64_t n, double* dst);

}  // namespace meft_dev
