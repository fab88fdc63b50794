// Key-Experts selection with reference-exact indices (experts.cpp:47-117, adapter.cpp:42-84).
//
// Scores are fp64 dot products accumulated strictly left to right, one chain per (token, row), exactly
// the reference's dot() (kernels.hpp:37-41). With bf16 inputs every product a_k*b_k is exact in fp64,
// so fma(a,b,acc) == fl(acc + fl(a*b)) and the fast DFMA path is bit-identical to the reference; with
// fp64 inputs the kernel uses __dmul_rn/__dadd_rn (no contraction). Rankings use the reference's total
// order (score desc via operator>/!=, so -0.0 == +0.0; then lower index), and every list is emitted
// ascending, so selected experts, per-token neurons and the union match the CPU reference bit for bit.
//
// Pipeline:
//   router scores [T x N]  -> warp top-kk per token (tau, ascending) -> bucket (token,slot) by expert
//   -> grouped key scoring [T x kk*E] (each expert's key rows are read once per 64-token tile)
//   -> CTA bitonic top-K per token over (score, global index) -> per-token list + union bitmap
//   -> ordered compaction of the bitmap into the ascending union S.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "select.h"

namespace meft_dev {
namespace {

constexpr int ST = 64;   // score tile: entries
constexpr int SC = 64;   // score tile: key rows
constexpr int SK = 16;   // k chunk
constexpr int STHREADS = 256;

__device__ __forceinline__ double ld_in(const double* p, int64_t i) { return p[i]; }
__device__ __forceinline__ double ld_in(const uint16_t* p, int64_t i) { return double(bf16_bits_to_f32(p[i])); }

template <bool EXACT_PRODUCTS>
__device__ __forceinline__ double mac(double acc, double a, double b) {
    if (EXACT_PRODUCTS) return fma(a, b, acc);  // a*b exact => identical to the unfused form
    return __dadd_rn(acc, __dmul_rn(a, b));
}

// The reference's comparator (experts.cpp:36-41): a precedes b.
__device__ __forceinline__ bool beats(double sa, int ia, double sb, int ib) {
    if (sa != sb) return sa > sb;
    return ia < ib;
}

// Grouped score tile. Group g = blockIdx.z-resolved: W rows [g*ncols, (g+1)*ncols), entry list
// entries[off[g] .. off[g+1]) (entry e -> token e / ent_div, output row e). entries == nullptr means
// one group of `n_entries` identity entries.
template <typename In, bool EXACT>
__global__ void __launch_bounds__(STHREADS)
    k_score(const In* __restrict__ h, int d, const In* __restrict__ w, int ncols, const int32_t* __restrict__ entries,
            const int32_t* __restrict__ off, const int32_t* __restrict__ tile_off, int n_groups, int n_entries,
            int ent_div, double* __restrict__ out) {
    __shared__ double sh[SK][ST + 1];
    __shared__ double sw[SK][SC + 1];
    __shared__ int s_tok[ST];
    __shared__ int s_row[ST];

    int g = 0, tile_in_group = blockIdx.x, ebeg = 0, ecount = n_entries;
    if (entries) {
        // locate the group owning this tile (tile_off is the exclusive scan of per-group tile counts)
        int lo = 0, hi = n_groups;  // find last g with tile_off[g] <= blockIdx.x
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (tile_off[mid] <= (int)blockIdx.x) lo = mid; else hi = mid;
        }
        g = lo;
        if ((int)blockIdx.x >= tile_off[n_groups]) return;
        tile_in_group = blockIdx.x - tile_off[g];
        ebeg = off[g];
        ecount = off[g + 1] - off[g];
    }
    const int e0 = tile_in_group * ST;
    if (e0 >= ecount) return;
    const int c0 = blockIdx.y * SC;
    if (c0 >= ncols) return;
    const int tid = threadIdx.x;
    if (tid < ST) {
        const int e = e0 + tid;
        if (e < ecount) {
            const int ent = entries ? entries[ebeg + e] : e;
            s_row[tid] = ent;
            s_tok[tid] = ent / ent_div;
        } else {
            s_row[tid] = -1;
            s_tok[tid] = 0;
        }
    }
    __syncthreads();

    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4 x 4 outputs each
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    const int64_t wrow0 = int64_t(g) * ncols + c0;
    for (int k0 = 0; k0 < d; k0 += SK) {
        const int kn = min(SK, d - k0);
        for (int i = tid; i < ST * SK; i += STHREADS) {
            const int r = i / SK, kk = i % SK;
            sh[kk][r] = (kk < kn) ? ld_in(h, int64_t(s_tok[r]) * d + k0 + kk) : 0.0;
        }
        for (int i = tid; i < SC * SK; i += STHREADS) {
            const int c = i / SK, kk = i % SK;
            sw[kk][c] = (kk < kn && c0 + c < ncols) ? ld_in(w, (wrow0 + c) * d + k0 + kk) : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kn; ++kk) {  // strictly ascending k
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sh[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sw[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = mac<EXACT>(acc[i][j], a[i], b[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
        const int row = s_row[r];
        if (row < 0) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + tx * 4 + j;
            if (c < ncols) out[int64_t(row) * ncols + c] = acc[i][j];
        }
    }
}

// Warp per token: top-kk experts of the router scores (experts.cpp:30-45), written ascending.
__global__ void k_topk_experts(const double* __restrict__ scores, int T, int N, int kk, int32_t* __restrict__ tau,
                               int32_t* __restrict__ counts) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= T) return;
    const double* s = scores + int64_t(warp) * N;
    int32_t* out = tau + int64_t(warp) * kk;
    double ps = 0.0;
    int pi = -1;  // previous pick; -1 = none yet
    for (int r = 0; r < kk; ++r) {
        double bs = -DBL_MAX;
        int bi = -1;
        for (int i = lane; i < N; i += 32) {
            const double v = s[i];
            if (pi >= 0 && !beats(ps, pi, v, i)) continue;  // already taken (ranked at or above prev)
            if (bi < 0 || beats(v, i, bs, bi)) {
                bs = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, bs, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || beats(os, oi, bs, bi))) {
                bs = os;
                bi = oi;
            }
        }
        ps = bs;
        pi = bi;
        if (lane == 0) out[r] = bi;
    }
    __syncwarp();
    if (lane == 0) {
        for (int a = 1; a < kk; ++a) {  // insertion sort ascending (kk is small)
            const int v = out[a];
            int b = a - 1;
            while (b >= 0 && out[b] > v) {
                out[b + 1] = out[b];
                --b;
            }
            out[b + 1] = v;
        }
        if (counts)
            for (int a = 0; a < kk; ++a) atomicAdd(&counts[out[a]], 1);
    }
}

// Single CTA: off = exclusive scan(counts), tile_off = exclusive scan(ceil(counts/ST)), cursor = 0.
__global__ void k_bucket_scan(const int32_t* __restrict__ counts, int N, int32_t* __restrict__ off,
                              int32_t* __restrict__ tile_off, int32_t* __restrict__ cursor, int tile) {
    __shared__ int s_run, s_trun;
    if (threadIdx.x == 0) {
        s_run = 0;
        s_trun = 0;
    }
    __syncthreads();
    for (int base = 0; base < N; base += blockDim.x) {
        const int i = base + threadIdx.x;
        const int c = i < N ? counts[i] : 0;
        const int tcount = (c + tile - 1) / tile;
        // block-wide inclusive scan via warp scans
        int v = c, tv = tcount;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, v, o);
            const int tx = __shfl_up_sync(0xffffffffu, tv, o);
            if (lane >= o) {
                v += x;
                tv += tx;
            }
        }
        __shared__ int ws[32], wts[32];
        if (lane == 31) {
            ws[wid] = v;
            wts[wid] = tv;
        }
        __syncthreads();
        if (wid == 0) {
            const int nw = blockDim.x >> 5;
            int a = lane < nw ? ws[lane] : 0, b = lane < nw ? wts[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, a, o);
                const int y = __shfl_up_sync(0xffffffffu, b, o);
                if (lane >= o) {
                    a += x;
                    b += y;
                }
            }
            ws[lane] = a;
            wts[lane] = b;
        }
        __syncthreads();
        const int wpre = wid > 0 ? ws[wid - 1] : 0, wtpre = wid > 0 ? wts[wid - 1] : 0;
        if (i < N) {
            off[i] = s_run + wpre + v - c;
            tile_off[i] = s_trun + wtpre + tv - tcount;
            cursor[i] = 0;
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) {
            s_run += wpre + v;
            s_trun += wtpre + tv;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        off[N] = s_run;
        tile_off[N] = s_trun;
    }
}

__global__ void k_bucket_fill(const int32_t* __restrict__ tau, int T, int kk, const int32_t* __restrict__ off,
                              int32_t* __restrict__ cursor, int32_t* __restrict__ entries) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= T * kk) return;
    const int e = tau[i];
    const int pos = atomicAdd(&cursor[e], 1);
    entries[off[e] + pos] = i;  // i = t*kk + slot
}

// CTA per token: bitonic sort of the C candidates by the reference order, keep `take`, emit ascending.
__global__ void k_topk_neurons(const double* __restrict__ cand, const int32_t* __restrict__ tau, int kk, int E,
                               int C, int P2, int take, int TP2, int32_t* __restrict__ per_token,
                               uint8_t* __restrict__ flags) {
    extern __shared__ uint8_t sm[];
    double* ks = reinterpret_cast<double*>(sm);
    int* is = reinterpret_cast<int*>(ks + P2);
    const int t = blockIdx.x;
    const double* c = cand + int64_t(t) * C;
    for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        if (i < C) {
            const int slot = i / E, j = i - slot * E;
            ks[i] = c[i];
            is[i] = (tau ? tau[int64_t(t) * kk + slot] : 0) * E + j;
        } else {
            ks[i] = -DBL_MAX;
            is[i] = INT32_MAX;
        }
    }
    __syncthreads();
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const double a = ks[i], b = ks[p];
                    const int ia = is[i], ib = is[p];
                    const bool first = (i & k) == 0;  // this half in "precedes" order
                    bool sw;
                    if (ia == INT32_MAX || ib == INT32_MAX)
                        sw = first ? (ia == INT32_MAX && ib != INT32_MAX) : (ib == INT32_MAX && ia != INT32_MAX);
                    else
                        sw = first ? beats(b, ib, a, ia) : beats(a, ia, b, ib);
                    if (sw) {
                        ks[i] = b;
                        ks[p] = a;
                        is[i] = ib;
                        is[p] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    // the first `take` entries are the selection; sort their indices ascending (reuse ks storage as ints)
    int* sel = reinterpret_cast<int*>(ks);
    for (int i = threadIdx.x; i < TP2; i += blockDim.x) sel[i] = (i < take) ? is[i] : INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= TP2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < TP2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const int a = sel[i], b = sel[p];
                    const bool up = (i & k) == 0;
                    if (up ? (a > b) : (a < b)) {
                        sel[i] = b;
                        sel[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < take; i += blockDim.x) {
        const int v = sel[i];
        per_token[int64_t(t) * take + i] = v;
        flags[v] = 1;
    }
}

// Ordered compaction of the union bitmap (experts.cpp:109-115): pass 1 counts per 1024-block.
__global__ void k_flag_count(const uint8_t* __restrict__ flags, int M, int32_t* __restrict__ bcount) {
    const int i = blockIdx.x * 1024 + threadIdx.x;
    const int f = (i < M) ? (flags[i] != 0) : 0;
    const int c = __syncthreads_count(f);
    if (threadIdx.x == 0) bcount[blockIdx.x] = c;
}

__global__ void k_scan_blocks(int32_t* __restrict__ bcount, int nb, int32_t* __restrict__ total) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int run = 0;
        for (int b = 0; b < nb; ++b) {
            const int c = bcount[b];
            bcount[b] = run;
            run += c;
        }
        *total = run;
    }
}

__global__ void k_flag_write(const uint8_t* __restrict__ flags, int M, const int32_t* __restrict__ boff,
                             int32_t* __restrict__ out) {
    __shared__ int wsum[32];
    const int i = blockIdx.x * 1024 + threadIdx.x;
    const int f = (i < M) ? (flags[i] != 0) : 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
        int v = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += x;
        }
        wsum[lane] = v - wsum[lane];  // exclusive
    }
    __syncthreads();
    if (f) out[boff[blockIdx.x] + wsum[wid] + __popc(bal & ((1u << lane) - 1u))] = i;
}

int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

template <typename In, bool EXACT>
void launch_score(cudaStream_t st, const void* h, int d, const void* w, int ncols, const int32_t* entries,
                  const int32_t* off, const int32_t* tile_off, int n_groups, int grid_x, int n_entries, int ent_div,
                  double* out) {
    dim3 grid(grid_x, (ncols + SC - 1) / SC, 1);
    k_score<In, EXACT><<<grid, STHREADS, 0, st>>>(static_cast<const In*>(h), d, static_cast<const In*>(w), ncols,
                                                  entries, off, tile_off, n_groups, n_entries, ent_div, out);
    check_launch("k_score");
}

void score_dispatch(cudaStream_t st, int dtype, const void* h, int d, const void* w, int ncols,
                    const int32_t* entries, const int32_t* off, const int32_t* tile_off, int n_groups, int grid_x,
                    int n_entries, int ent_div, double* out) {
    if (dtype == 2)
        launch_score<uint16_t, true>(st, h, d, w, ncols, entries, off, tile_off, n_groups, grid_x, n_entries, ent_div,
                                     out);
    else
        launch_score<double, false>(st, h, d, w, ncols, entries, off, tile_off, n_groups, grid_x, n_entries, ent_div,
                                    out);
}

}  // namespace

#include "select_tc.cuh"

void score_rows(cudaStream_t st, int dtype, const void* h, int64_t T, int64_t d, const void* w, int64_t rows,
                double* scores) {
    if (T <= 0 || rows <= 0) return;
    score_dispatch(st, dtype, h, int(d), w, int(rows), nullptr, nullptr, nullptr, 1, int((T + ST - 1) / ST), int(T),
                   1, scores);
}

namespace {
size_t exact_workspace_bytes(int64_t T, int64_t M, int64_t N, int64_t kk_eff) {
    const int64_t E = M / N;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
    add(T * N * 8);             // router scores
    add(T * kk_eff * 4);        // tau (internal copy)
    add(T * kk_eff * E * 8);    // candidate scores
    add(T * kk_eff * 4);        // entries
    add((N + 1) * 4 * 4);       // counts, off, tile_off, cursor
    add(M);                     // union flags
    add(((M + 1023) / 1024 + 1) * 4);  // block offsets
    return b;
}

// K-chunks of the candidate-scoring GEMM: 512-wide chunks tighten the certified bound ~d/512-fold, which cuts the
// exact fp64 re-scoring proportionally (profiles/: 27 -> ~4 ambiguous candidates per token at d = 4096).
int cert_ksplit(int64_t d) {
    static const int forced = [] {  // MEFT_CERT_KSPLIT: developer override for tuning sweeps
        const char* v = std::getenv("MEFT_CERT_KSPLIT");
        return v ? std::max(1, std::min(16, std::atoi(v))) : 0;
    }();
    if (forced) return int(std::min<int64_t>(forced, std::max<int64_t>(1, d / 64)));
    return int(std::max<int64_t>(1, std::min<int64_t>(4, d / 1024)));  // 1024-wide chunks: measured best
}

// K-chunking of the candidate-scoring GEMM and the certified bound that goes with it, shared by the fused
// selection (partials summed inside the classifier) and the sharded protocol (partials summed by the owner):
// both compare float(fp64 sum of the chunk partials) against the same bound.
struct CertSplit {
    int ks;       // chunks actually launched (no empty ones)
    int64_t kbs;  // k-blocks per chunk
    double cb;    // bound coefficient for float(sum of partials)
};
CertSplit cert_split(int64_t d, bool allow) {
    const int req = allow ? cert_ksplit(d) : 1;
    const int64_t nkb = (d + 63) / 64, kbs = (nkb + req - 1) / req;
    const int ks = int((nkb + kbs - 1) / kbs);
    const double cb = ks > 1 ? cert_bound_coeff_split(int(d), int(kbs * 64), ks) : cert_bound_coeff(int(d));
    return CertSplit{ks, kbs, cb};
}

// float(fp64 sum of the ks partial products) of every element
__global__ void k_sum_partials(const float* __restrict__ part, int ks, int64_t n, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < ks; ++p) s += double(part[p * n + i]);
        out[i] = float(s);
    }
}

// Approximate router scores P [T x ldp] = float(fp64 sum of the K-chunk partials of H W_g^T): the split launches
// 4x the tiles of an N = 256 router GEMM (which alone fills under half the SMs) and the certified router bound
// shrinks like the candidate scores'. Returns the bound coefficient for P. `part` holds ks * T * ldp floats.
double router_scores(cudaStream_t st, const uint16_t* h, const uint16_t* wg, int64_t T, int64_t N, int64_t d,
                     int64_t ldp, float* P, float* part) {
    const CertSplit cs = cert_split(d, true);
    GemmEpilogue e;
    e.kind = EPI_STORE_F32;
    e.ldc = ldp;
    if (cs.ks > 1) {
        e.c = part;
        e.ksplit = cs.ks;
        e.split_stride = T * ldp;
    } else {
        e.c = P;
    }
    gemm_bf16(st, T, N, d, GemmOperand{h, d, false}, GemmOperand{wg, d, false}, e);
    if (cs.ks > 1) {
        k_sum_partials<<<int(std::min<int64_t>((T * ldp + 255) / 256, num_sms() * 8)), 256, 0, st>>>(part, cs.ks, T * ldp,
                                                                                                     P);
        check_launch("k_sum_partials");
    }
    return cs.cb;
}

size_t cert_workspace_bytes(int64_t T, int64_t d, int64_t M, int64_t N, int64_t kk_eff) {
    const int64_t E = M / N;
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
    add(T * round_up(N, 4) * 4);  // approximate router scores (fp32)
    add(T * round_up(N, 4) * 4 * cert_split(d, true).ks);  // their K-chunk partials
    add((T + N + M) * 4);         // row norms of h, w_g, keys
    add((T + N + M) * 4);         // their minimum LSB exponents
    add(T * kk_eff * 4);          // tau
    add(T * kk_eff * 4);          // entries
    add((N + 1) * 4 * 4);         // counts, off, tile_off, cursor
    add(T * kk_eff * d * 2);      // token rows bucketed by expert (bf16)
    add(T * kk_eff * E * 4 * cert_ksplit(d));  // approximate candidate scores (fp32 partials per K-chunk)
    add(M);                       // union flags
    add(((M + 1023) / 1024 + 1) * 4);
    const int64_t C = kk_eff * E, take_max = C;
    add(T * take_max * 4 + T * 4);  // certain members + counts
    add(T * C * 4 + T * 4);         // ambiguous candidates + counts
    add(T * C * 8);                 // their exact scores
    add(2 * T * C * 4);             // (token, position) pairs grouped by expert
    add((N + 1) * 4 * 4);           // per-expert ambiguous counts, offsets, tiles, cursor
    return b;
}

bool certified_ok(int dtype, int64_t d, int64_t M, int64_t N, int64_t kk_eff) {
    const int64_t E = M / N;
    return dtype == 2 && d % 8 == 0 && d <= 32768 && E % 4 == 0 && kk_eff * E <= CERT_MAX_C && N <= 2048 &&
           kk_eff <= 64;
}

void ke_select_exact(cudaStream_t st, int dtype, const void* h, const void* w_g, const void* keys, int64_t T,
                     int64_t d, int64_t M, int64_t N, int64_t kk_eff, int64_t take, void* ws, size_t ws_bytes,
                     int32_t* per_token, int32_t* tau_out, int32_t* union_idx, int32_t* union_size);
}  // namespace

size_t select_workspace_bytes(int64_t T, int64_t d, int64_t M, int64_t N, int64_t kk_eff) {
    return std::max(exact_workspace_bytes(T, M, N, kk_eff), cert_workspace_bytes(T, d, M, N, kk_eff));
}

// Certified tensor-core selection (select_tc.cuh): bit-exact with the reference, no fp64 GEMM.
static void ke_select_certified(cudaStream_t st, const void* h_, const void* w_g_, const void* keys_, int64_t T,
                                int64_t d, int64_t M, int64_t N, int64_t kk_eff, int64_t take, void* ws,
                                int32_t* per_token, int32_t* tau_out, int32_t* union_idx, int32_t* union_size,
                                int32_t* stats,
                                const float* key_norms, const int32_t* key_lsb) {
    const uint16_t* h = static_cast<const uint16_t*>(h_);
    const uint16_t* wg = static_cast<const uint16_t*>(w_g_);
    const uint16_t* keys = static_cast<const uint16_t*>(keys_);
    const int64_t E = M / N, C = kk_eff * E, ldp = round_up(N, 4);
    uint8_t* p = static_cast<uint8_t*>(ws);
    auto take_buf = [&](size_t x) {
        void* r = p;
        p += (x + 255) & ~size_t(255);
        return r;
    };
    float* P = static_cast<float*>(take_buf(T * ldp * 4));
    float* Ppart = static_cast<float*>(take_buf(T * ldp * 4 * cert_split(d, true).ks));
    float* hn = static_cast<float*>(take_buf((T + N + M) * 4));
    float* gn = hn + T;
    float* kn = gn + N;
    int32_t* hl = static_cast<int32_t*>(take_buf((T + N + M) * 4));  // per-row minimum LSB exponents
    int32_t* gl = hl + T;
    int32_t* kl = gl + N;
    int32_t* tau = static_cast<int32_t*>(take_buf(T * kk_eff * 4));
    int32_t* entries = static_cast<int32_t*>(take_buf(T * kk_eff * 4));
    int32_t* counts = static_cast<int32_t*>(take_buf((N + 1) * 4 * 4));
    int32_t* off = counts + (N + 1);
    int32_t* tile_off = off + (N + 1);
    int32_t* cursor = tile_off + (N + 1);
    uint16_t* hs = static_cast<uint16_t*>(take_buf(T * kk_eff * d * 2));
    const int ksplit = N == 1 ? 1 : cert_ksplit(d);
    float* cand = static_cast<float*>(take_buf(T * C * 4 * ksplit));
    uint8_t* flags = static_cast<uint8_t*>(take_buf(M));
    int32_t* boff = static_cast<int32_t*>(take_buf(((M + 1023) / 1024 + 1) * 4));
    const double cb = cert_bound_coeff(int(d));

    MEFT_CUDA_CHECK(cudaMemsetAsync(flags, 0, M, st));
    if (stats) MEFT_CUDA_CHECK(cudaMemsetAsync(stats, 0, 2 * sizeof(int32_t), st));
    k_row_norms<<<int((T * 32 + 255) / 256), 256, 0, st>>>(h, T, int(d), hn, hl);
    check_launch("k_row_norms");
    if (key_norms && key_lsb) {  // the store's cached key statistics (kept current by the fused Adam)
        kn = const_cast<float*>(key_norms);
        kl = const_cast<int32_t*>(key_lsb);
    } else {
        k_row_norms<<<int((M * 32 + 255) / 256), 256, 0, st>>>(keys, M, int(d), kn, kl);
        check_launch("k_row_norms");
    }
    if (N == 1) {
        // flat top-K (adapter.cpp:42-84): one candidate block of all M keys per token
        MEFT_CUDA_CHECK(cudaMemsetAsync(tau, 0, T * 4, st));
        GemmEpilogue e;
        e.kind = EPI_STORE_F32;
        e.c = cand;
        e.ldc = M;
        gemm_bf16(st, T, M, d, GemmOperand{h, d, false}, GemmOperand{keys, d, false}, e);
    } else {
        k_row_norms<<<int((N * 32 + 255) / 256), 256, 0, st>>>(wg, N, int(d), gn, gl);
        check_launch("k_row_norms");
        const double cbr = router_scores(st, h, wg, T, N, d, ldp, P, Ppart);  // approximate, on the tensor cores
        MEFT_CUDA_CHECK(cudaMemsetAsync(counts, 0, N * 4, st));
        const int wpb = 4;
        const size_t rsm = size_t(wpb) * (kk_eff + 2 * N) * 4 + size_t(wpb) * N * 8;
        static std::atomic<unsigned long long> rattr{0};
        set_max_smem_once(rattr, reinterpret_cast<const void*>(k_router_certified), 200 * 1024);
        k_router_certified<<<int((T + wpb - 1) / wpb), wpb * 32, rsm, st>>>(P, int(ldp), hn, gn, hl, gl, cbr, h, wg,
                                                                          int(d),
                                                                          int(T), int(N), int(kk_eff), tau, counts,
                                                                          stats);
        check_launch("k_router_certified");
        k_bucket_scan<<<1, 1024, 0, st>>>(counts, int(N), off, tile_off, cursor, 128);
        check_launch("k_bucket_scan");
        k_bucket_fill<<<int((T * kk_eff + 255) / 256), 256, 0, st>>>(tau, int(T), int(kk_eff), off, cursor, entries);
        check_launch("k_bucket_fill");
        const int rows = int(T * kk_eff);
        k_gather_tokens<<<std::max(1, std::min(rows / 8 + 1, num_sms() * 16)), 256, 0, st>>>(h, int(d), entries, rows,
                                                                                              int(kk_eff), hs);
        check_launch("k_gather_tokens");
        GemmEpilogue eg;  // grouped by expert: cand[entry][j] = h_token . key_{g*E + j}
        eg.kind = EPI_ROWS_STORE_F32;
        eg.c = cand;
        eg.ldc = E;
        eg.row_idx = entries;
        eg.ksplit = ksplit;
        eg.split_stride = T * C;
        gemm_bf16_grouped(st, int(N), E, d, GemmOperand{hs, d, false}, rows, GemmOperand{keys, d, false}, M, off,
                          tile_off, eg);
    }
    // certified top-K: classify -> exact re-scoring grouped by expert -> finalize
    int32_t* sure = static_cast<int32_t*>(take_buf(T * C * 4 + T * 4));
    int32_t* n_sure = sure + T * C;
    int32_t* amb = static_cast<int32_t*>(take_buf(T * C * 4 + T * 4));
    int32_t* n_amb = amb + T * C;
    double* xs = static_cast<double*>(take_buf(T * C * 8));
    int32_t* pair_t = static_cast<int32_t*>(take_buf(2 * T * C * 4));
    int32_t* pair_a = pair_t + T * C;
    int32_t* acount = static_cast<int32_t*>(take_buf((N + 1) * 4 * 4));
    int32_t* aoff = acount + (N + 1);
    int32_t* atile = aoff + (N + 1);
    int32_t* acur = atile + (N + 1);
    const int P2 = next_pow2(int(C)), TP2 = next_pow2(int(take));
    const size_t csm = size_t(C) * 9 + 16;  // classify: u32 keys + f32 scores + u8 membership
    if (csm > 200 * 1024) throw MeftError(2, "ke_select: candidate set too large for the certified path");
    // the split GEMM really used kb_split*64-wide chunks (no empty splits): the same arithmetic as base_args
    const CertSplit cs = cert_split(d, ksplit > 1);
    const int ks_eff = cs.ks;
    const double cbk = cs.cb;
    static std::atomic<unsigned long long> cattr{0};
    set_max_smem_once(cattr, reinterpret_cast<const void*>(k_topk_classify), 200 * 1024);
    MEFT_CUDA_CHECK(cudaMemsetAsync(acount, 0, N * 4, st));
    k_topk_classify<<<int(T), 256, csm, st>>>(cand, tau, int(kk_eff), int(E), int(C), P2, int(take), hn, kn, cbk,
                                              sure, n_sure, amb, n_amb, acount, ks_eff, (long long)(T * C));
    check_launch("k_topk_classify");
    k_bucket_scan<<<1, 1024, 0, st>>>(acount, int(N), aoff, atile, acur, 1);
    check_launch("k_bucket_scan");
    k_amb_fill<<<int(T), 128, 0, st>>>(amb, n_amb, int(C), int(E), aoff, acur, pair_t, pair_a);
    check_launch("k_amb_fill");
    static const int rescore_grid = resident_grid(k_rescore_pairs, 256);
    k_rescore_pairs<<<rescore_grid, 256, 0, st>>>(pair_t, pair_a, aoff + N, amb, int(C), h, keys, int(d), hn, kn, hl,
                                                    kl, xs, stats);
    check_launch("k_rescore_pairs");
    k_topk_finalize<<<int(T), 128, size_t(TP2) * 4, st>>>(sure, n_sure, amb, n_amb, xs, int(C), int(take), TP2,
                                                           per_token, flags);
    check_launch("k_topk_finalize");
    if (tau_out) MEFT_CUDA_CHECK(cudaMemcpyAsync(tau_out, tau, T * kk_eff * 4, cudaMemcpyDeviceToDevice, st));
    compact_flags(st, flags, M, union_idx, union_size, boff);
}

void ke_select_device(cudaStream_t st, int dtype, const void* h, const void* w_g, const void* keys, int64_t T,
                      int64_t d, int64_t M, int64_t N, int64_t kk_eff, int64_t take, void* ws, size_t ws_bytes,
                      int32_t* per_token, int32_t* tau_out, int32_t* union_idx, int32_t* union_size,
                      int32_t* stats, bool allow_certified,
                      const float* key_norms, const int32_t* key_lsb) {
    if (ws_bytes < select_workspace_bytes(T, d, M, N, kk_eff)) throw MeftError(6, "ke_select: workspace too small");
    if (allow_certified && certified_ok(dtype, d, M, N, kk_eff)) {
        ke_select_certified(st, h, w_g, keys, T, d, M, N, kk_eff, take, ws, per_token, tau_out, union_idx, union_size,
                            stats, key_norms, key_lsb);
        return;
    }
    if (stats) MEFT_CUDA_CHECK(cudaMemsetAsync(stats, 0, 2 * sizeof(int32_t), st));
    ke_select_exact(st, dtype, h, w_g, keys, T, d, M, N, kk_eff, take, ws, ws_bytes, per_token, tau_out, union_idx,
                    union_size);
}

namespace {
void ke_select_exact(cudaStream_t st, int dtype, const void* h, const void* w_g, const void* keys, int64_t T,
                     int64_t d, int64_t M, int64_t N, int64_t kk_eff, int64_t take, void* ws, size_t ws_bytes,
                     int32_t* per_token, int32_t* tau_out, int32_t* union_idx, int32_t* union_size) {
    (void)ws_bytes;
    const int64_t E = M / N;
    const int64_t C = kk_eff * E;
    uint8_t* p = static_cast<uint8_t*>(ws);
    auto take_buf = [&](size_t x) {
        void* r = p;
        p += (x + 255) & ~size_t(255);
        return r;
    };
    double* rscores = static_cast<double*>(take_buf(T * N * 8));
    int32_t* tau = static_cast<int32_t*>(take_buf(T * kk_eff * 4));
    double* cand = static_cast<double*>(take_buf(T * C * 8));
    int32_t* entries = static_cast<int32_t*>(take_buf(T * kk_eff * 4));
    int32_t* counts = static_cast<int32_t*>(take_buf((N + 1) * 4 * 4));
    int32_t* off = counts + (N + 1);
    int32_t* tile_off = off + (N + 1);
    int32_t* cursor = tile_off + (N + 1);
    uint8_t* flags = static_cast<uint8_t*>(take_buf(M));
    int32_t* boff = static_cast<int32_t*>(take_buf(((M + 1023) / 1024 + 1) * 4));

    const int P2 = next_pow2(int(C));
    const int TP2 = next_pow2(int(take));
    const size_t topk_smem = size_t(P2) * 12;
    if (topk_smem > 200 * 1024) throw MeftError(2, "ke_select: kk*E candidates per token exceed 16384 (unsupported)");

    MEFT_CUDA_CHECK(cudaMemsetAsync(flags, 0, M, st));
    if (N == 1) {
        // single expert: every token sees all M keys (topk_select / ke_select with N=1)
        MEFT_CUDA_CHECK(cudaMemsetAsync(tau, 0, T * 4, st));
        score_rows(st, dtype, h, T, d, keys, M, cand);
    } else {
        score_rows(st, dtype, h, T, d, w_g, N, rscores);
        MEFT_CUDA_CHECK(cudaMemsetAsync(counts, 0, N * 4, st));
        k_topk_experts<<<int((T * 32 + 255) / 256), 256, 0, st>>>(rscores, int(T), int(N), int(kk_eff), tau, counts);
        check_launch("k_topk_experts");
        k_bucket_scan<<<1, 1024, 0, st>>>(counts, int(N), off, tile_off, cursor, ST);
        check_launch("k_bucket_scan");
        k_bucket_fill<<<int((T * kk_eff + 255) / 256), 256, 0, st>>>(tau, int(T), int(kk_eff), off, cursor, entries);
        check_launch("k_bucket_fill");
        const int grid_x = int((T * kk_eff + ST - 1) / ST + N);  // >= total tiles over all groups
        score_dispatch(st, dtype, h, int(d), keys, int(E), entries, off, tile_off, int(N), grid_x, int(T * kk_eff),
                       int(kk_eff), cand);
    }
    static std::atomic<unsigned long long> attr{0};
    set_max_smem_once(attr, reinterpret_cast<const void*>(k_topk_neurons), 200 * 1024);
    k_topk_neurons<<<int(T), 512, topk_smem, st>>>(cand, tau, int(kk_eff), int(E), int(C), P2, int(take), TP2,
                                                   per_token, flags);
    check_launch("k_topk_neurons");
    if (tau_out) MEFT_CUDA_CHECK(cudaMemcpyAsync(tau_out, tau, T * kk_eff * 4, cudaMemcpyDeviceToDevice, st));
    const int nb = int((M + 1023) / 1024);
    k_flag_count<<<nb, 1024, 0, st>>>(flags, int(M), boff);
    k_scan_blocks<<<1, 32, 0, st>>>(boff, nb, union_size);
    k_flag_write<<<nb, 1024, 0, st>>>(flags, int(M), boff, union_idx);
    check_launch("k_flag_write");
}
}  // namespace

void route_topk_device(cudaStream_t st, const double* scores, int64_t T, int64_t N, int64_t kk, int32_t* tau) {
    k_topk_experts<<<int((T * 32 + 255) / 256), 256, 0, st>>>(scores, int(T), int(N), int(kk), tau, nullptr);
    check_launch("k_topk_experts");
}

}  // namespace meft_dev

namespace meft_dev {
// Ascending list of the set entries of flags[M] (used for the staged set of sparse_adam_update).
void compact_flags(cudaStream_t st, const uint8_t* flags, int64_t M, int32_t* out_idx, int32_t* count_dev,
                   int32_t* block_ws) {
    const int nb = int((M + 1023) / 1024);
    k_flag_count<<<nb, 1024, 0, st>>>(flags, int(M), block_ws);
    check_launch("k_flag_count");
    k_scan_blocks<<<1, 32, 0, st>>>(block_ws, nb, count_dev);
    check_launch("k_scan_blocks");
    k_flag_write<<<nb, 1024, 0, st>>>(flags, int(M), block_ws, out_idx);
    check_launch("k_flag_write");
}
}  // namespace meft_dev

// ------------------------------------------------------------------ sharded-selection building blocks
namespace meft_dev {
namespace {
__global__ void k_count_experts(const int32_t* __restrict__ expert, int R, int32_t* __restrict__ counts) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) atomicAdd(&counts[expert[r]], 1);
}

__global__ void k_exact_pairs(const uint16_t* __restrict__ rows, const float* __restrict__ rn,
                              const int32_t* __restrict__ rl, const uint16_t* __restrict__ keys,
                              const float* __restrict__ kn, const int32_t* __restrict__ kl,
                              const int32_t* __restrict__ pair_row, const int32_t* __restrict__ pair_key, int Q, int d,
                              double* __restrict__ out, int* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < Q; p += (gridDim.x * blockDim.x) >> 5) {
        const int r = pair_row[p], k = pair_key[p];
        const double v = exact_dot_rows(rows + int64_t(r) * d, keys + int64_t(k) * d, d, lane, rl[r], kl[k], rn[r],
                                        kn[k], stats ? stats + 1 : nullptr);
        if (lane == 0) out[p] = v;
    }
}
}  // namespace

void row_stats(cudaStream_t st, const uint16_t* x, int64_t rows, int64_t d, float* norms, int32_t* minlsb) {
    if (rows <= 0) return;
    k_row_norms<<<int((rows * 32 + 255) / 256), 256, 0, st>>>(x, rows, int(d), norms, minlsb);
    check_launch("k_row_norms");
}

size_t route_workspace_bytes(int64_t T, int64_t d, int64_t N) {
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
    add(T * round_up(N, 4) * 4);
    add(T * round_up(N, 4) * 4 * cert_split(d, true).ks);
    add((T + N) * 4);
    add((T + N) * 4);
    add((N + 1) * 4);
    return b;
}

void route_certified(cudaStream_t st, const uint16_t* h, const uint16_t* w_g, int64_t T, int64_t d, int64_t N,
                     int64_t kk_eff, void* ws, int32_t* tau, int32_t* stats) {
    if (T <= 0) return;
    const int64_t ldp = round_up(N, 4);
    uint8_t* p = static_cast<uint8_t*>(ws);
    auto take_buf = [&](size_t x) {
        void* r = p;
        p += (x + 255) & ~size_t(255);
        return r;
    };
    float* P = static_cast<float*>(take_buf(T * ldp * 4));
    float* Ppart = static_cast<float*>(take_buf(T * ldp * 4 * cert_split(d, true).ks));
    float* hn = static_cast<float*>(take_buf((T + N) * 4));
    float* gn = hn + T;
    int32_t* hl = static_cast<int32_t*>(take_buf((T + N) * 4));
    int32_t* gl = hl + T;
    int32_t* counts = static_cast<int32_t*>(take_buf((N + 1) * 4));
    row_stats(st, h, T, d, hn, hl);
    row_stats(st, w_g, N, d, gn, gl);
    const double cbr = router_scores(st, h, w_g, T, N, d, ldp, P, Ppart);
    MEFT_CUDA_CHECK(cudaMemsetAsync(counts, 0, N * 4, st));
    const int wpb = 4;
    const size_t rsm = size_t(wpb) * (kk_eff + 2 * N) * 4 + size_t(wpb) * N * 8;
    static std::atomic<unsigned long long> rattr{0};
    set_max_smem_once(rattr, reinterpret_cast<const void*>(k_router_certified), 200 * 1024);
    k_router_certified<<<int((T + wpb - 1) / wpb), wpb * 32, rsm, st>>>(P, int(ldp), hn, gn, hl, gl,
                                                                      cbr, h, w_g, int(d), int(T),
                                                                      int(N), int(kk_eff), tau, counts, stats);
    check_launch("k_router_certified");
}

size_t score_workspace_bytes(int64_t R, int64_t d, int64_t n_experts, int64_t E) {
    size_t b = 0;
    auto add = [&](size_t x) { b += (x + 255) & ~size_t(255); };
    add((n_experts + 1) * 4 * 4);
    add(R * 4);
    add(R * d * 2);
    add(R * E * 4 * cert_split(d, true).ks);  // K-split partial scores
    return b;
}


void score_candidates(cudaStream_t st, const uint16_t* rows, const int32_t* expert, int64_t R, int64_t d,
                      const uint16_t* keys, int64_t n_experts, int64_t E, void* ws, float* cand) {
    if (R <= 0) return;
    uint8_t* p = static_cast<uint8_t*>(ws);
    auto take_buf = [&](size_t x) {
        void* r = p;
        p += (x + 255) & ~size_t(255);
        return r;
    };
    int32_t* counts = static_cast<int32_t*>(take_buf((n_experts + 1) * 4 * 4));
    int32_t* off = counts + (n_experts + 1);
    int32_t* tile_off = off + (n_experts + 1);
    int32_t* cursor = tile_off + (n_experts + 1);
    int32_t* entries = static_cast<int32_t*>(take_buf(R * 4));
    uint16_t* hs = static_cast<uint16_t*>(take_buf(R * d * 2));
    MEFT_CUDA_CHECK(cudaMemsetAsync(counts, 0, n_experts * 4, st));
    k_count_experts<<<int((R + 255) / 256), 256, 0, st>>>(expert, int(R), counts);
    check_launch("k_count_experts");
    k_bucket_scan<<<1, 1024, 0, st>>>(counts, int(n_experts), off, tile_off, cursor, 128);
    check_launch("k_bucket_scan");
    k_bucket_fill<<<int((R + 255) / 256), 256, 0, st>>>(expert, int(R), 1, off, cursor, entries);
    check_launch("k_bucket_fill");
    k_gather_tokens<<<std::max(1, std::min(int(R / 8 + 1), num_sms() * 16)), 256, 0, st>>>(rows, int(d), entries,
                                                                                           int(R), 1, hs);
    check_launch("k_gather_tokens");
    // K-split exactly like the fused selection; the owner returns float(fp64 sum of the partials), which the home
    // classifies against cert_split(d).cb (topk_classify)
    const CertSplit cs = cert_split(d, true);
    float* part = cs.ks > 1 ? static_cast<float*>(take_buf(R * E * 4 * cs.ks)) : cand;
    GemmEpilogue eg;
    eg.kind = EPI_ROWS_STORE_F32;
    eg.c = part;
    eg.ldc = E;
    eg.row_idx = entries;
    eg.ksplit = cs.ks;
    eg.split_stride = R * E;
    gemm_bf16_grouped(st, int(n_experts), E, d, GemmOperand{hs, d, false}, R, GemmOperand{keys, d, false},
                      n_experts * E, off, tile_off, eg);
    if (cs.ks > 1) {
        k_sum_partials<<<int(std::min<int64_t>((R * E + 255) / 256, num_sms() * 8)), 256, 0, st>>>(part, cs.ks, R * E,
                                                                                                  cand);
        check_launch("k_sum_partials");
    }
}

void exact_pair_scores(cudaStream_t st, const uint16_t* rows, const float* rn, const int32_t* rl,
                       const uint16_t* keys, const float* kn, const int32_t* kl, const int32_t* pair_row,
                       const int32_t* pair_key, int64_t Q, int64_t d, double* out, int32_t* stats) {
    if (Q <= 0) return;
    static const int resident = resident_grid(k_exact_pairs, 256);
    const int grid = std::max(1, std::min<int>(int((Q * 32 + 255) / 256), resident));
    k_exact_pairs<<<grid, 256, 0, st>>>(rows, rn, rl, keys, kn, kl, pair_row, pair_key, int(Q), int(d), out, stats);
    check_launch("k_exact_pairs");
}

void topk_classify(cudaStream_t st, const float* cand, const int32_t* tau, int64_t T, int64_t kk, int64_t E,
                   int64_t take, int64_t d, const float* hn, const float* kn, int32_t* sure, int32_t* n_sure,
                   int32_t* amb, int32_t* n_amb, int32_t* amb_count_per_expert) {
    if (T <= 0) return;
    const int64_t C = kk * E;
    const size_t csm = size_t(C) * 9 + 16;
    static std::atomic<unsigned long long> cattr{0};
    set_max_smem_once(cattr, reinterpret_cast<const void*>(k_topk_classify), 200 * 1024);
    k_topk_classify<<<int(T), 256, csm, st>>>(cand, tau, int(kk), int(E), int(C), next_pow2(int(C)), int(take), hn, kn,
                                              cert_split(d, true).cb, sure, n_sure, amb, n_amb, amb_count_per_expert,
                                              1, 0);
    check_launch("k_topk_classify");
}

void topk_finalize(cudaStream_t st, const int32_t* sure, const int32_t* n_sure, const int32_t* amb,
                   const int32_t* n_amb, const double* x, int64_t T, int64_t C, int64_t take, int32_t* per_token,
                   uint8_t* flags) {
    if (T <= 0) return;
    const int TP2 = next_pow2(int(take));
    k_topk_finalize<<<int(T), 128, size_t(TP2) * 4, st>>>(sure, n_sure, amb, n_amb, x, int(C), int(take), TP2,
                                                           per_token, flags);
    check_launch("k_topk_finalize");
}
}  // namespace meft_dev
