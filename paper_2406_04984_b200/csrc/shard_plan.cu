// Index bookkeeping of the expert-sharded selection protocol (sharded.py) as device kernels: the
// dispatch plan (which (token, slot) rows go to which expert owner, in a stable order), the exact-rescoring request
// plan, and the scatters that put returned candidate scores / exact scores back in token order. Replaces chains of
// small framework ops whose launch latency dominated the sharded selection; all orders are deterministic.
#include "common.cuh"
#include "shard_plan.h"

namespace meft_dev {
namespace {

constexpr int kPlanThreads = 1024;

// Block-wide exclusive scan of one int per thread (kPlanThreads threads); returns the block total.
__device__ int block_exclusive_scan(int v, int* s_warp, int& excl) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = s_warp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        s_warp[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    excl = x - v + (w > 0 ? s_warp[w - 1] : 0);
    const int total = s_warp[31];
    __syncthreads();
    return total;
}

// Stable counting sort by a small key in [0, P): pos[i] = start[key(i)] + #{j < i : key(j) == key(i)}.
// key(i) = src[i] / div. One block; thread t owns the contiguous range [t*chunk, (t+1)*chunk).
__global__ void __launch_bounds__(kPlanThreads) k_stable_bucket(const int32_t* __restrict__ src, int n, int div, int P,
                                                                int32_t* __restrict__ pos, int32_t* __restrict__ counts) {
    __shared__ int s_warp[32];
    const int chunk = (n + kPlanThreads - 1) / kPlanThreads;
    const int lo = min(n, int(threadIdx.x) * chunk), hi = min(n, lo + chunk);
    int base = 0;
    for (int o = 0; o < P; ++o) {
        int c = 0;
        for (int i = lo; i < hi; ++i) c += (src[i] / div) == o;
        int excl;
        const int total = block_exclusive_scan(c, s_warp, excl);
        int p = base + excl;
        for (int i = lo; i < hi; ++i)
            if ((src[i] / div) == o) pos[i] = p++;
        if (threadIdx.x == 0) counts[o] = total;
        base += total;
    }
}

// Dispatch rows in bucket order: order[pos] = i, send_exp[pos] = local expert of tau[i], inv[i] = pos.
__global__ void k_dispatch_fill(const int32_t* __restrict__ tau, int n, int n_loc, const int32_t* __restrict__ pos,
                                int32_t* __restrict__ order, int32_t* __restrict__ inv, int32_t* __restrict__ send_exp) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int p = pos[i], e = tau[i];
    order[p] = i;
    inv[i] = p;
    send_exp[p] = e - (e / n_loc) * n_loc;
}

// send_rows[p] = h[order[p] / kk] (bf16 rows, 16-byte vectors, warp per row)
__global__ void k_gather_dispatch_rows(const uint16_t* __restrict__ h, int d, const int32_t* __restrict__ order, int n,
                                       int kk, uint16_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int nv = d / 8;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        const uint4* s = reinterpret_cast<const uint4*>(h + int64_t(order[r] / kk) * d);
        uint4* o = reinterpret_cast<uint4*>(out + int64_t(r) * d);
        for (int v = lane; v < nv; v += 32) o[v] = __ldg(s + v);
    }
}

// dst[order[p]] = src[p] for rows of `cols` fp32
__global__ void k_unpermute_rows(const float* __restrict__ src, const int32_t* __restrict__ order, int n, int cols,
                                 float* __restrict__ dst) {
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < int64_t(n) * cols;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = e / cols;
        dst[int64_t(order[p]) * cols + (e - p * cols)] = src[e];
    }
}

// Exclusive scan of the per-token ambiguous counts (one block): aoff[t] = sum_{u < t} n_amb[u], aoff[T] = total.
__global__ void __launch_bounds__(kPlanThreads) k_scan_counts(const int32_t* __restrict__ n_amb, int T,
                                                              int32_t* __restrict__ aoff) {
    __shared__ int s_warp[32];
    const int chunk = (T + kPlanThreads - 1) / kPlanThreads;
    const int lo = min(T, int(threadIdx.x) * chunk), hi = min(T, lo + chunk);
    int c = 0;
    for (int t = lo; t < hi; ++t) c += n_amb[t];
    int excl;
    const int total = block_exclusive_scan(c, s_warp, excl);
    for (int t = lo; t < hi; ++t) {
        aoff[t] = excl;
        excl += n_amb[t];
    }
    if (threadIdx.x == 0) aoff[T] = total;
}

// One entry per ambiguous (token, position): the owner's receive row of the token's dispatched (token, slot) row,
// the owner-local key, and where the exact score goes back (t*C + a). Flat order: token-major, position ascending.
__global__ void k_request_fill(const int32_t* __restrict__ amb, const int32_t* __restrict__ n_amb,
                               const int32_t* __restrict__ aoff, const int32_t* __restrict__ tau,
                               const int32_t* __restrict__ inv, int T, int C, int kk, int E, int M_loc,
                               const int32_t* __restrict__ row_base, int32_t* __restrict__ f_owner,
                               int32_t* __restrict__ f_row, int32_t* __restrict__ f_key, int32_t* __restrict__ f_back) {
    const int t = blockIdx.x;
    if (t >= T) return;
    const int na = n_amb[t], o0 = aoff[t];
    for (int a = threadIdx.x; a < na; a += blockDim.x) {
        const int idx = amb[int64_t(t) * C + a];
        const int e = idx / E;
        int slot = 0;
        for (int s = 0; s < kk; ++s)
            if (tau[int64_t(t) * kk + s] == e) slot = s;
        const int owner = idx / M_loc;
        const int f = o0 + a;
        f_owner[f] = owner;
        f_row[f] = inv[int64_t(t) * kk + slot] + row_base[owner];
        f_key[f] = idx - owner * M_loc;
        f_back[f] = t * C + a;
    }
}

__global__ void k_request_sort(const int32_t* __restrict__ pos, const int32_t* __restrict__ n_dev,
                               const int32_t* __restrict__ f_row, const int32_t* __restrict__ f_key,
                               const int32_t* __restrict__ f_back, int32_t* __restrict__ row, int32_t* __restrict__ key,
                               int32_t* __restrict__ back) {
    const int n = *n_dev;
    for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < n; f += gridDim.x * blockDim.x) {
        const int p = pos[f];
        row[p] = f_row[f];
        key[p] = f_key[f];
        back[p] = f_back[f];
    }
}

__global__ void k_scatter_f64(const double* __restrict__ x, const int32_t* __restrict__ back, int n,
                              double* __restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[back[i]] = x[i];
}

int grid_of(int64_t n, int per = 256) { return int(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 65535))); }

}  // namespace

void shard_dispatch(cudaStream_t st, const int32_t* tau, int64_t T, int64_t kk, int64_t n_loc, int P,
                    const uint16_t* h, int64_t d, int32_t* pos_ws, uint16_t* send_rows, int32_t* send_exp,
                    int32_t* order, int32_t* inv, int32_t* counts) {
    const int n = int(T * kk);
    if (n <= 0) return;
    k_stable_bucket<<<1, kPlanThreads, 0, st>>>(tau, n, int(n_loc), P, pos_ws, counts);
    check_launch("k_stable_bucket");
    k_dispatch_fill<<<grid_of(n), 256, 0, st>>>(tau, n, int(n_loc), pos_ws, order, inv, send_exp);
    check_launch("k_dispatch_fill");
    if (!send_rows) return;  // the owners gather the rows themselves (from the all-gathered hidden states)
    k_gather_dispatch_rows<<<std::max(1, std::min(n / 8 + 1, num_sms() * 16)), 256, 0, st>>>(h, int(d), order, n,
                                                                                               int(kk), send_rows);
    check_launch("k_gather_dispatch_rows");
}

void shard_unpermute_rows(cudaStream_t st, const float* src, const int32_t* order, int64_t n, int64_t cols, float* dst) {
    if (n <= 0) return;
    k_unpermute_rows<<<grid_of(n * cols), 256, 0, st>>>(src, order, int(n), int(cols), dst);
    check_launch("k_unpermute_rows");
}

void shard_requests_fill(cudaStream_t st, const int32_t* amb, const int32_t* n_amb, const int32_t* tau,
                         const int32_t* inv, int64_t T, int64_t C, int64_t kk, int64_t E, int64_t M_loc,
                         const int32_t* row_base, int32_t* ws) {
    if (T <= 0) return;
    const int64_t cap = T * C;
    int32_t* aoff = ws;
    int32_t* f_owner = aoff + (T + 1);
    int32_t* f_row = f_owner + cap;
    int32_t* f_key = f_row + cap;
    int32_t* f_back = f_key + cap;
    k_scan_counts<<<1, kPlanThreads, 0, st>>>(n_amb, int(T), aoff);
    check_launch("k_scan_counts");
    k_request_fill<<<int(T), 128, 0, st>>>(amb, n_amb, aoff, tau, inv, int(T), int(C), int(kk), int(E), int(M_loc),
                                          row_base, f_owner, f_row, f_key, f_back);
    check_launch("k_request_fill");
}

void shard_requests_sort(cudaStream_t st, int64_t T, int64_t C, int64_t M_loc, int P, int64_t n, int32_t* ws,
                         int32_t* row, int32_t* key, int32_t* back, int32_t* counts) {
    if (n <= 0) return;
    const int64_t cap = T * C;
    int32_t* aoff = ws;
    int32_t* f_owner = aoff + (T + 1);
    int32_t* f_row = f_owner + cap;
    int32_t* f_key = f_row + cap;
    int32_t* f_back = f_key + cap;
    int32_t* pos = f_back + cap;
    k_stable_bucket<<<1, kPlanThreads, 0, st>>>(f_owner, int(n), 1, P, pos, counts);
    check_launch("k_stable_bucket");
    k_request_sort<<<grid_of(n), 256, 0, st>>>(pos, aoff + T, f_row, f_key, f_back, row, key, back);
    check_launch("k_request_sort");
}

void shard_scatter_f64(cudaStream_t st, const double* x, const int32_t* back, int64_t n, double* dst) {
    if (n <= 0) return;
    k_scatter_f64<<<grid_of(n), 256, 0, st>>>(x, back, int(n), dst);
    check_launch("k_scatter_f64");
}

size_t shard_requests_ws_ints(int64_t T, int64_t C) { return size_t(T + 1 + 5 * T * C); }

}  // namespace meft_dev
