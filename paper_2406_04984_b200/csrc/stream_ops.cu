// HBM-streaming kernels of the MEFT layer: row gather of the selected key/value rows
// (adapter.cpp:86-110 / memtier.cpp:117-126), staging of weight gradients (memtier.cpp:128-155),
// the lazy per-pair sparse Adam (memtier.cpp:176-228) and layout/precision conversions used at the
// upload/download boundary. All tables are neuron-major ([pairs x d] rows), so every kernel streams
// whole contiguous rows with 16-byte vector accesses.
#include "common.cuh"
#include "stream_ops.h"

namespace meft_dev {
namespace {

// ---------------------------------------------------------------- gather

// One warp per selected row; both tables in one pass. W is the copy word (uint4 when rows are 16-byte
// multiples, else uint2 / uint16_t).
template <typename W>
__global__ void k_gather2(const W* __restrict__ a, const W* __restrict__ b, int64_t row_words,
                          const int32_t* __restrict__ idx, const int32_t* __restrict__ count_dev, int count,
                          W* __restrict__ oa, W* __restrict__ ob, int pad64) {
    const int n = count_dev ? min(*count_dev, count > 0 ? count : INT32_MAX) : count;
    const int lane = threadIdx.x & 31;
    // pad64: rows [n, next multiple of 64) (capped at count) are written as zeros -- the padding a device-sized
    // GEMM reads past the union (gemm_sm100.cu apply_extent)
    const int n_pad = pad64 ? min((n + 63) & ~63, count) : n;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n_pad; r += (gridDim.x * blockDim.x) >> 5) {
        if (r >= n) {
            W* da = oa + int64_t(r) * row_words;
            W* db = ob + int64_t(r) * row_words;
            for (int64_t v = lane; v < row_words; v += 32) {
                da[v] = W{};
                db[v] = W{};
            }
            continue;
        }
        const W* sa = a + int64_t(idx[r]) * row_words;
        const W* sb = b + int64_t(idx[r]) * row_words;
        W* da = oa + int64_t(r) * row_words;
        W* db = ob + int64_t(r) * row_words;
        for (int64_t v = lane; v < row_words; v += 64) {
            const W x0 = __ldg(sa + v);
            const W y0 = __ldg(sb + v);
            const bool two = v + 32 < row_words;
            W x1 = x0, y1 = y0;
            if (two) {
                x1 = __ldg(sa + v + 32);
                y1 = __ldg(sb + v + 32);
            }
            da[v] = x0;
            db[v] = y0;
            if (two) {
                da[v + 32] = x1;
                db[v + 32] = y1;
            }
        }
    }
}

__global__ void k_check_sorted(const int32_t* __restrict__ idx, int n, int64_t limit, int32_t* __restrict__ err) {
    // err[0]: 0 ok, 3 out of range (err[1] = first bad index), 2 not strictly ascending
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int v = idx[i];
    if (v < 0 || v >= limit) {
        atomicCAS(&err[0], 0, 3);
        atomicMin(&err[1], i);
    } else if (i > 0 && v <= idx[i - 1]) {
        atomicCAS(&err[0], 0, 2);
    }
}

// ---------------------------------------------------------------- staging (scatter_grads)

template <typename G, typename S>
__global__ void k_stage_add(S* __restrict__ stage, int64_t d, const int32_t* __restrict__ idx, int n,
                            const G* __restrict__ g, uint8_t* __restrict__ staged) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const int64_t row = idx[r];
    S* s = stage + row * d;
    const G* gr = g + int64_t(r) * d;
    for (int64_t i = threadIdx.x; i < d; i += blockDim.x) s[i] += S(gr[i]);
    if (staged && threadIdx.x == 0) staged[row] = 1;
}

// fp32 staging, fp32 gradients (the mixed store's scatter_grads): 16-byte vectors, 4 in flight per thread.
__global__ void __launch_bounds__(256) k_stage_add_f32x4(float* __restrict__ stage, int64_t d,
                                                         const int32_t* __restrict__ idx, int n,
                                                         const float* __restrict__ g, uint8_t* __restrict__ staged) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const int64_t row = idx[r];
    float4* s = reinterpret_cast<float4*>(stage + row * d);
    const float4* gr = reinterpret_cast<const float4*>(g + int64_t(r) * d);
    const int d4 = int(d / 4);
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < d4; i0 += blockDim.x * U) {
        float4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < d4) {
                a[u] = s[i];
                b[u] = __ldcs(gr + i);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < d4) s[i] = make_float4(a[u].x + b[u].x, a[u].y + b[u].y, a[u].z + b[u].z, a[u].w + b[u].w);
        }
    }
    if (staged && threadIdx.x == 0) staged[row] = 1;
}

__global__ void k_mark(uint8_t* __restrict__ staged, const int32_t* __restrict__ idx, const int32_t* count_dev,
                       int count) {
    const int n = count_dev ? *count_dev : count;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) staged[idx[i]] = 1;
}

// ---------------------------------------------------------------- sparse Adam (memtier.cpp:187-228)

// Mixed-precision store: fp32 master/m/v/stage, bf16 compute copy. One CTA per staged pair updates the key
// row and/or the value row (`tables`: bit 0 keys, bit 1 values) with the pair's shared step counter
// (memtier.hpp:87-89), zeroes their staging; with `bump` it also advances the counter and clears the flag
// (the layer step updates the value rows first without bump, the key rows afterwards with it).
// With `gpos` the gradients are not staging rows but a dense [count x d] block in `rows` order (the fused layer
// step's weight-grad GEMM output): read once, never zeroed -- 30 B per entry instead of 34.
// Four Adam moments of a row at vector index i: fp32 (float4) or, for COMPACT stores, bf16 (uint2), as floats.
template <bool MOM16>
__device__ __forceinline__ float4 load_mom4(const void* base, int64_t i) {
    if (MOM16) {
        const uint2 u = reinterpret_cast<const uint2*>(base)[i];
        return make_float4(bf16_bits_to_f32(uint16_t(u.x)), bf16_bits_to_f32(uint16_t(u.x >> 16)),
                           bf16_bits_to_f32(uint16_t(u.y)), bf16_bits_to_f32(uint16_t(u.y >> 16)));
    }
    return reinterpret_cast<const float4*>(base)[i];
}
template <bool MOM16>
__device__ __forceinline__ void store_mom4(void* base, int64_t i, float4 v) {
    if (MOM16) {
        reinterpret_cast<uint2*>(base)[i] = make_uint2(pack_bf16x2(f32_to_bf16_bits(v.x), f32_to_bf16_bits(v.y)),
                                                       pack_bf16x2(f32_to_bf16_bits(v.z), f32_to_bf16_bits(v.w)));
    } else {
        reinterpret_cast<float4*>(base)[i] = v;
    }
}

template <bool MOM16>
__global__ void __launch_bounds__(256) k_adam_mixed(const int32_t* __restrict__ rows, const int32_t* count_dev,
                                                    int count, int64_t d, float* __restrict__ wa, void* __restrict__ ma,
                                                    void* __restrict__ va, float* __restrict__ sa,
                                                    uint16_t* __restrict__ ca, float* __restrict__ wb,
                                                    void* __restrict__ mb, void* __restrict__ vb,
                                                    float* __restrict__ sb, uint16_t* __restrict__ cb,
                                                    int32_t* __restrict__ step, uint8_t* __restrict__ staged, float b1,
                                                    float b2, float eps, float lr, int tables, int bump, int gpos,
                                                    float* __restrict__ kn, int32_t* __restrict__ kl) {
    const int n = count_dev ? *count_dev : count;
    __shared__ AdamCoef s_k;
    __shared__ double s_red[8];
    __shared__ int s_lsb[8];
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t j = rows[r];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int t = step[j] + 1;
            if (bump) {
                step[j] = t;
                if (staged) staged[j] = 0;
            }
            s_k = adam_coef(b1, b2, lr, t);
        }
        __syncthreads();
        const AdamCoef k = s_k;
#pragma unroll
        for (int tab = 0; tab < 2; ++tab) {
            if (!(tables & (1 << tab))) continue;
            float4* w4 = reinterpret_cast<float4*>((tab ? wb : wa) + j * d);
            const int64_t esz = MOM16 ? 2 : 4;
            void* m4 = static_cast<uint8_t*>(tab ? mb : ma) + j * d * esz;
            void* v4 = static_cast<uint8_t*>(tab ? vb : va) + j * d * esz;
            float4* g4 = reinterpret_cast<float4*>((tab ? sb : sa) + (gpos ? int64_t(r) : j) * d);
            uint2* c4 = reinterpret_cast<uint2*>((tab ? cb : ca) + j * d);
            const bool stats = tab == 0 && kn != nullptr;  // refresh the key row's selection statistics
            double ss = 0.0;
            int lsb = INT32_MAX;
            for (int64_t i = threadIdx.x; i < d / 4; i += blockDim.x) {
                const float4 g = g4[i];
                float4 m = load_mom4<MOM16>(m4, i), v = load_mom4<MOM16>(v4, i), w = w4[i];
                float* mp = &m.x;
                float* vp = &v.x;
                float* wp = &w.x;
                const float* gp = &g.x;
#pragma unroll
                for (int q = 0; q < 4; ++q) adam_update(wp[q], mp[q], vp[q], gp[q], b1, b2, eps, k);
                store_mom4<MOM16>(m4, i, m);
                store_mom4<MOM16>(v4, i, v);
                w4[i] = w;
                if (!gpos) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                const uint16_t cb4[4] = {f32_to_bf16_bits(w.x), f32_to_bf16_bits(w.y), f32_to_bf16_bits(w.z),
                                         f32_to_bf16_bits(w.w)};
                c4[i] = make_uint2(pack_bf16x2(cb4[0], cb4[1]), pack_bf16x2(cb4[2], cb4[3]));
                if (stats) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double v = double(bf16_bits_to_f32(cb4[q]));
                        ss = fma(v, v, ss);
                        if (cb4[q] & 0x7FFF) lsb = min(lsb, bf16_lsb_exp(cb4[q]));
                    }
                }
            }
            if (stats) {  // same bound as k_row_norms: sqrt of the fp64 sum of squares, rounded up (x(1+2^-20))
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    ss += __shfl_xor_sync(0xffffffffu, ss, o);
                    lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
                }
                if ((threadIdx.x & 31) == 0) {
                    s_red[threadIdx.x >> 5] = ss;
                    s_lsb[threadIdx.x >> 5] = lsb;
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    double t = 0.0;
                    int l = INT32_MAX;
                    for (int w_ = 0; w_ < int(blockDim.x >> 5); ++w_) {
                        t += s_red[w_];
                        l = min(l, s_lsb[w_]);
                    }
                    kn[j] = __double2float_ru(sqrt(t) * (1.0 + 0x1p-20));
                    kl[j] = l;
                }
            }
        }
    }
}

// Adam fused into the weight-gradient GEMM epilogues (EPI_ADAM_F32): the per-pair step of every pair of S advances
// once (memtier.cpp:192-195, the key column and value row share it) and its bias-correction coefficients are
// tabulated by position, before either GEMM runs. Same coefficients as k_adam_mixed (adam_coef).
__global__ void k_adam_coef_bump(const int32_t* __restrict__ rows, int n, int32_t* __restrict__ step,
                                 float2* __restrict__ coef, float b1, float b2, float lr,
                                 const int32_t* __restrict__ n_dev) {
    if (n_dev) n = min(n, max(0, *n_dev));
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const int32_t j = rows[r];
        const int t = step[j] + 1;
        step[j] = t;
        const AdamCoef k = adam_coef(b1, b2, lr, t);
        coef[r] = make_float2(k.scale, k.inv_c2);
    }
}

// Key-row selection statistics from the epilogue's per-256-column partials (fp32 upper bounds of the partial sums
// of squares), summed in column order; same bound form as k_row_norms: sqrt of the sum, rounded up with a 2^-20
// margin (which also covers the fp64 rounding of this 16-term sum).
__global__ void k_adam_stats_finalize(const int32_t* __restrict__ rows, int n, const double* __restrict__ ss,
                                      const int32_t* __restrict__ lsb, int parts, float* __restrict__ kn,
                                      int32_t* __restrict__ kl, const int32_t* __restrict__ n_dev) {
    if (n_dev) n = min(n, max(0, *n_dev));
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double t = 0.0;
        int l = INT32_MAX;
        for (int p = 0; p < parts; ++p) {
            t += ss[int64_t(r) * parts + p];
            l = min(l, lsb[int64_t(r) * parts + p]);
        }
        const int32_t j = rows[r];
        kn[j] = __double2float_ru(sqrt(t) * (1.0 + 0x1p-20));
        kl[j] = l;
    }
}

// fp64 store (API-fidelity mode): the reference's adam_entry in double (memtier.cpp:176-185).
__global__ void __launch_bounds__(256) k_adam_f64(const int32_t* __restrict__ rows, const int32_t* count_dev, int count,
                                                  int64_t d, double* __restrict__ wa, double* __restrict__ ma,
                                                  double* __restrict__ va, double* __restrict__ sa,
                                                  double* __restrict__ wb, double* __restrict__ mb,
                                                  double* __restrict__ vb, double* __restrict__ sb,
                                                  int32_t* __restrict__ step, uint8_t* __restrict__ staged, double b1,
                                                  double b2, double eps, double lr) {
    const int n = count_dev ? *count_dev : count;
    __shared__ double s_c1, s_c2;
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t j = rows[r];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int t = step[j] + 1;
            step[j] = t;
            staged[j] = 0;
            s_c1 = 1.0 - pow(b1, double(t));
            s_c2 = 1.0 - pow(b2, double(t));
        }
        __syncthreads();
        const double c1 = s_c1, c2 = s_c2;
        for (int tab = 0; tab < 2; ++tab) {
            double* w = (tab ? wb : wa) + j * d;
            double* m = (tab ? mb : ma) + j * d;
            double* v = (tab ? vb : va) + j * d;
            double* g = (tab ? sb : sa) + j * d;
            for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
                const double gi = g[i];
                const double mi = b1 * m[i] + (1.0 - b1) * gi;
                const double vi = b2 * v[i] + (1.0 - b2) * gi * gi;
                m[i] = mi;
                v[i] = vi;
                w[i] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
                g[i] = 0.0;
            }
        }
    }
}

// Lazy Adam over one fp64 row table with int64 per-row steps (router rows, memtier.cpp:211-227).
__global__ void __launch_bounds__(256) k_adam_rows_f64(double* __restrict__ w, double* __restrict__ m,
                                                       double* __restrict__ v, double* __restrict__ stage,
                                                       int64_t* __restrict__ step, uint8_t* __restrict__ staged,
                                                       const int32_t* __restrict__ rows, int n, int64_t d, double b1,
                                                       double b2, double eps, double lr) {
    __shared__ double s_c1, s_c2;
    for (int r = blockIdx.x; r < n; r += gridDim.x) {
        const int64_t j = rows[r];
        __syncthreads();
        if (threadIdx.x == 0) {
            const int64_t t = ++step[j];
            staged[j] = 0;
            s_c1 = 1.0 - pow(b1, double(t));
            s_c2 = 1.0 - pow(b2, double(t));
        }
        __syncthreads();
        const double c1 = s_c1, c2 = s_c2;
        for (int64_t i = threadIdx.x; i < d; i += blockDim.x) {
            const int64_t q = j * d + i;
            const double gi = stage[q];
            const double mi = b1 * m[q] + (1.0 - b1) * gi;
            const double vi = b2 * v[q] + (1.0 - b2) * gi * gi;
            m[q] = mi;
            v[q] = vi;
            w[q] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
            stage[q] = 0.0;
        }
    }
}

// ---------------------------------------------------------------- conversions

__global__ void k_f64_to_bf16(const double* __restrict__ s, uint16_t* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = f32_to_bf16_bits(float(s[i]));  // double->float->bf16: exact for bf16-representable inputs
}
__global__ void k_f64_to_f32(const double* __restrict__ s, float* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = float(s[i]);
}
__global__ void k_f32_to_f64(const float* __restrict__ s, double* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = double(s[i]);
}
__global__ void k_f32_to_bf16(const float* __restrict__ s, uint16_t* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = f32_to_bf16_bits(s[i]);
}
__global__ void k_bf16_to_f64(const uint16_t* __restrict__ s, double* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = double(bf16_bits_to_f32(s[i]));
}
__global__ void k_i32_to_i64(const int32_t* __restrict__ s, int64_t* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = s[i];
}
__global__ void k_i64_to_i32(const int64_t* __restrict__ s, int32_t* __restrict__ d, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        d[i] = int32_t(s[i]);
}

// 32x32 tiled transpose of a rows x cols matrix of 8-byte elements.
__global__ void k_transpose8(const uint64_t* __restrict__ s, uint64_t* __restrict__ d, int64_t rows, int64_t cols) {
    __shared__ uint64_t tile[32][33];
    const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = s[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) d[c * rows + r] = tile[threadIdx.x][i];
    }
}

// 32x32 tiled transpose of a rows x cols matrix of 2-byte (bf16) elements.
__global__ void k_transpose2(const uint16_t* __restrict__ s, uint16_t* __restrict__ d, int64_t rows, int64_t cols) {
    __shared__ uint16_t tile[32][34];
    const int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = s[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) d[c * rows + r] = tile[threadIdx.x][i];
    }
}

int grid_for(int64_t n, int per = 256) {
    int64_t g = (n + per - 1) / per;
    const int64_t cap = int64_t(num_sms()) * 16;
    return int(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

// dst[r] = src[idx[r]] for rows of row_bytes (a multiple of 16, 16-byte aligned): warp per row
__global__ void k_gather1(const uint4* __restrict__ src, int64_t row_words, const int32_t* __restrict__ idx, int n,
                          uint4* __restrict__ dst) {
    const int lane = threadIdx.x & 31;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        const uint4* s = src + int64_t(idx[r]) * row_words;
        uint4* d = dst + int64_t(r) * row_words;
        for (int64_t v = lane; v < row_words; v += 32) d[v] = __ldg(s + v);
    }
}

void gather_rows1(cudaStream_t st, const void* src, int64_t row_bytes, const int32_t* idx, int64_t n, void* dst) {
    if (n <= 0) return;
    if (row_bytes % 16 || (reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) % 16)
        throw MeftError(2, "gather_rows: rows must be 16-byte multiples, 16-byte aligned");
    const int grid = std::max(1, std::min<int>(int((n * 32 + 255) / 256), num_sms() * 16));
    k_gather1<<<grid, 256, 0, st>>>(static_cast<const uint4*>(src), row_bytes / 16, idx, int(n),
                                    static_cast<uint4*>(dst));
    check_launch("k_gather1");
}

void gather_rows2(cudaStream_t st, const void* a, const void* b, int64_t row_bytes, const int32_t* idx,
                  const int32_t* count_dev, int64_t count, void* oa, void* ob, bool pad64) {
    if (count <= 0 && !count_dev) return;
    const int64_t warps = count > 0 ? count : int64_t(num_sms()) * 64;
    const int grid = std::max(1, std::min<int>(int((warps * 32 + 255) / 256), num_sms() * 8));
    auto al = [](const void* p, int n) { return (reinterpret_cast<uintptr_t>(p) % n) == 0; };
    if (row_bytes % 16 == 0 && al(a, 16) && al(b, 16) && al(oa, 16) && al(ob, 16))
        k_gather2<uint4><<<grid, 256, 0, st>>>(static_cast<const uint4*>(a), static_cast<const uint4*>(b),
                                               row_bytes / 16, idx, count_dev, int(count), static_cast<uint4*>(oa),
                                               static_cast<uint4*>(ob), pad64 ? 1 : 0);
    else if (row_bytes % 8 == 0)
        k_gather2<uint2><<<grid, 256, 0, st>>>(static_cast<const uint2*>(a), static_cast<const uint2*>(b),
                                               row_bytes / 8, idx, count_dev, int(count), static_cast<uint2*>(oa),
                                               static_cast<uint2*>(ob), pad64 ? 1 : 0);
    else
        k_gather2<uint16_t><<<grid, 256, 0, st>>>(static_cast<const uint16_t*>(a), static_cast<const uint16_t*>(b),
                                                  row_bytes / 2, idx, count_dev, int(count),
                                                  static_cast<uint16_t*>(oa), static_cast<uint16_t*>(ob), pad64 ? 1 : 0);
    check_launch("k_gather2");
}

void check_sorted_unique(cudaStream_t st, const int32_t* idx, int64_t n, int64_t limit, int32_t* err_dev) {
    if (n <= 0) return;
    k_check_sorted<<<int((n + 255) / 256), 256, 0, st>>>(idx, int(n), limit, err_dev);
    check_launch("k_check_sorted");
}

void stage_add(cudaStream_t st, int stage_dtype, void* stage, int64_t d, const int32_t* idx, int64_t n, int g_dtype,
               const void* g, uint8_t* staged) {
    if (n <= 0) return;
    if (stage_dtype == 0 && g_dtype == 0)
        k_stage_add<double, double><<<int(n), 256, 0, st>>>(static_cast<double*>(stage), d, idx, int(n),
                                                            static_cast<const double*>(g), staged);
    else if (stage_dtype == 1 && g_dtype == 1 && d % 4 == 0 && (reinterpret_cast<uintptr_t>(stage) | reinterpret_cast<uintptr_t>(g)) % 16 == 0)
        k_stage_add_f32x4<<<int(n), 256, 0, st>>>(static_cast<float*>(stage), d, idx, int(n),
                                                  static_cast<const float*>(g), staged);
    else if (stage_dtype == 1 && g_dtype == 1)
        k_stage_add<float, float><<<int(n), 256, 0, st>>>(static_cast<float*>(stage), d, idx, int(n),
                                                          static_cast<const float*>(g), staged);
    else if (stage_dtype == 1 && g_dtype == 0)
        k_stage_add<double, float><<<int(n), 256, 0, st>>>(static_cast<float*>(stage), d, idx, int(n),
                                                           static_cast<const double*>(g), staged);
    else
        k_stage_add<float, double><<<int(n), 256, 0, st>>>(static_cast<double*>(stage), d, idx, int(n),
                                                           static_cast<const float*>(g), staged);
    check_launch("k_stage_add");
}

// holes of an ascending index list: (last - first + 1) - n, i.e. how far it is from one contiguous run
__global__ void k_union_holes(const int32_t* __restrict__ idx, const int32_t* __restrict__ n_dev,
                              int32_t* __restrict__ out) {
    const int n = *n_dev;
    *out = n > 0 ? idx[n - 1] - idx[0] + 1 - n : 0;
}

__global__ void k_union_holes_n(const int32_t* __restrict__ idx, int n, int32_t* __restrict__ out) {
    *out = n > 0 ? idx[n - 1] - idx[0] + 1 - n : 0;
}

__global__ void k_hist_add(const int32_t* __restrict__ idx, int n, unsigned long long* __restrict__ hist) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(hist + idx[i], 1ull);
}

void histogram_add(cudaStream_t st, const int32_t* idx, int64_t n, int64_t* hist) {
    if (n <= 0) return;
    k_hist_add<<<int(std::min<int64_t>((n + 255) / 256, 1184)), 256, 0, st>>>(
        idx, int(n), reinterpret_cast<unsigned long long*>(hist));
    check_launch("k_hist_add");
}

// out[i] = recv[0][i] + recv[1][i] + ... in slot order (the home's side of the peer-memory reduce-scatter).
__global__ void k_slot_sum(const float4* __restrict__ recv, int world, int64_t n4, float4* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
        float4 a = recv[i];
        for (int s = 1; s < world; ++s) {
            const float4 b = recv[s * n4 + i];
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        out[i] = a;
    }
}

void slot_sum(cudaStream_t st, const float* recv, int world, int64_t n, float* out) {
    if (n <= 0) return;
    if (n % 4 || (reinterpret_cast<uintptr_t>(recv) | reinterpret_cast<uintptr_t>(out)) % 16)
        throw MeftError(2, "peer_reduce: rows * d must be a multiple of 4 and buffers 16-byte aligned");
    const int64_t n4 = n / 4;
    k_slot_sum<<<int(std::min<int64_t>((n4 + 255) / 256, num_sms() * 8)), 256, 0, st>>>(
        reinterpret_cast<const float4*>(recv), world, n4, reinterpret_cast<float4*>(out));
    check_launch("k_slot_sum");
}

void union_holes(cudaStream_t st, const int32_t* idx, const int32_t* n_dev, int32_t* out) {
    k_union_holes<<<1, 1, 0, st>>>(idx, n_dev, out);
    check_launch("k_union_holes");
}

void union_holes_n(cudaStream_t st, const int32_t* idx, int64_t n, int32_t* out) {
    k_union_holes_n<<<1, 1, 0, st>>>(idx, int(n), out);
    check_launch("k_union_holes");
}

void mark_rows(cudaStream_t st, uint8_t* staged, const int32_t* idx, const int32_t* count_dev, int64_t count) {
    const int grid = grid_for(count > 0 ? count : 1);
    k_mark<<<grid, 256, 0, st>>>(staged, idx, count_dev, int(count));
    check_launch("k_mark");
}

void adam_mixed(cudaStream_t st, const int32_t* rows, const int32_t* count_dev, int64_t count, int64_t d, float* wa,
                void* ma, void* va, float* sa, uint16_t* ca, float* wb, void* mb, void* vb, float* sb,
                uint16_t* cb, int32_t* step, uint8_t* staged, double b1, double b2, double eps, double lr, int tables,
                bool bump, bool grads_by_position, float* key_norms, int32_t* key_lsb, bool moments_bf16) {
    if (d % 4) throw MeftError(2, "adam: d must be a multiple of 4 in mixed precision");
    const int grid = std::max(1, std::min<int>(int(count > 0 ? count : num_sms() * 8), num_sms() * 8));
    auto kern = moments_bf16 ? k_adam_mixed<true> : k_adam_mixed<false>;
    kern<<<grid, 256, 0, st>>>(rows, count_dev, int(count), d, wa, ma, va, sa, ca, wb, mb, vb, sb, cb, step, staged,
                               float(b1), float(b2), float(eps), float(lr), tables, bump ? 1 : 0,
                               grads_by_position ? 1 : 0, key_norms, key_lsb);
    check_launch("k_adam_mixed");
}

void adam_coef_bump(cudaStream_t st, const int32_t* rows, int64_t n, int32_t* step, float2* coef, double b1,
                    double b2, double lr, const int32_t* n_dev) {
    if (n <= 0) return;
    k_adam_coef_bump<<<grid_for(n), 256, 0, st>>>(rows, int(n), step, coef, float(b1), float(b2), float(lr), n_dev);
    check_launch("k_adam_coef_bump");
}

void adam_stats_finalize(cudaStream_t st, const int32_t* rows, int64_t n, const double* ss, const int32_t* lsb,
                         int64_t parts, float* kn, int32_t* kl, const int32_t* n_dev) {
    if (n <= 0) return;
    k_adam_stats_finalize<<<grid_for(n), 256, 0, st>>>(rows, int(n), ss, lsb, int(parts), kn, kl, n_dev);
    check_launch("k_adam_stats_finalize");
}

void adam_f64(cudaStream_t st, const int32_t* rows, const int32_t* count_dev, int64_t count, int64_t d, double* wa,
              double* ma, double* va, double* sa, double* wb, double* mb, double* vb, double* sb, int32_t* step,
              uint8_t* staged, double b1, double b2, double eps, double lr) {
    const int grid = std::max(1, std::min<int>(int(count > 0 ? count : num_sms() * 8), num_sms() * 8));
    k_adam_f64<<<grid, 256, 0, st>>>(rows, count_dev, int(count), d, wa, ma, va, sa, wb, mb, vb, sb, step, staged, b1,
                                     b2, eps, lr);
    check_launch("k_adam_f64");
}

void adam_rows_f64(cudaStream_t st, double* w, double* m, double* v, double* stage, int64_t* step, uint8_t* staged,
                   const int32_t* rows, int64_t n, int64_t d, double b1, double b2, double eps, double lr) {
    if (n <= 0) return;
    const int grid = std::max(1, std::min<int>(int(n), num_sms() * 8));
    k_adam_rows_f64<<<grid, 256, 0, st>>>(w, m, v, stage, step, staged, rows, int(n), d, b1, b2, eps, lr);
    check_launch("k_adam_rows_f64");
}

void convert(cudaStream_t st, int ddt, void* dst, int sdt, const void* src, int64_t n) {
    if (n <= 0) return;
    const int g = grid_for(n);
    if (sdt == 0 && ddt == 2)
        k_f64_to_bf16<<<g, 256, 0, st>>>(static_cast<const double*>(src), static_cast<uint16_t*>(dst), n);
    else if (sdt == 0 && ddt == 1)
        k_f64_to_f32<<<g, 256, 0, st>>>(static_cast<const double*>(src), static_cast<float*>(dst), n);
    else if (sdt == 1 && ddt == 0)
        k_f32_to_f64<<<g, 256, 0, st>>>(static_cast<const float*>(src), static_cast<double*>(dst), n);
    else if (sdt == 1 && ddt == 2)
        k_f32_to_bf16<<<g, 256, 0, st>>>(static_cast<const float*>(src), static_cast<uint16_t*>(dst), n);
    else if (sdt == 2 && ddt == 0)
        k_bf16_to_f64<<<g, 256, 0, st>>>(static_cast<const uint16_t*>(src), static_cast<double*>(dst), n);
    else if (sdt == ddt)
        MEFT_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * (sdt == 0 ? 8 : sdt == 1 ? 4 : 2), cudaMemcpyDeviceToDevice, st));
    else
        throw MeftError(2, "convert: unsupported dtype pair");
    check_launch("convert");
}

void convert_index(cudaStream_t st, bool to64, void* dst, const void* src, int64_t n) {
    if (n <= 0) return;
    const int g = grid_for(n);
    if (to64)
        k_i32_to_i64<<<g, 256, 0, st>>>(static_cast<const int32_t*>(src), static_cast<int64_t*>(dst), n);
    else
        k_i64_to_i32<<<g, 256, 0, st>>>(static_cast<const int64_t*>(src), static_cast<int32_t*>(dst), n);
    check_launch("convert_index");
}

void transpose2(cudaStream_t st, const void* src, void* dst, int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32));
    k_transpose2<<<grid, dim3(32, 8), 0, st>>>(static_cast<const uint16_t*>(src), static_cast<uint16_t*>(dst), rows,
                                                cols);
    check_launch("k_transpose2");
}

void transpose8(cudaStream_t st, const void* src, void* dst, int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0) return;
    dim3 grid(unsigned((cols + 31) / 32), unsigned((rows + 31) / 32));
    k_transpose8<<<grid, dim3(32, 8), 0, st>>>(static_cast<const uint64_t*>(src), static_cast<uint64_t*>(dst), rows,
                                                cols);
    check_launch("k_transpose8");
}

namespace {
// kernels.cpp:15-22: sigmoid(x) = 1/(1+exp(-x)); silu = x*sigmoid(x); silu'(x) = s*(1 + x*(1-s)).
__global__ void k_act_fwd(const double* __restrict__ x, double* __restrict__ y, int64_t n, int act) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double v = x[i];
        y[i] = act == 1 ? (v > 0.0 ? v : 0.0) : v * (1.0 / (1.0 + exp(-v)));
    }
}
__global__ void k_act_bwd(double* __restrict__ g, const double* __restrict__ pre, int64_t n, int act) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double x = pre[i];
        if (act == 1) {
            g[i] = x > 0.0 ? g[i] : 0.0;
        } else {
            const double s = 1.0 / (1.0 + exp(-x));
            g[i] = g[i] * (s * (1.0 + x * (1.0 - s)));
        }
    }
}
__global__ void k_nonfinite(const double* __restrict__ x, int64_t n, int32_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        if (!isfinite(x[i])) *flag = 1;
}
__global__ void k_nonfinite_f32(const float4* __restrict__ x, int64_t n4, int32_t* __restrict__ flag) {
    bool bad = false;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = x[i];
        bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}
__global__ void k_add_f64(double* __restrict__ a, const double* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        a[i] = a[i] + b[i];
}
}  // namespace

void act_forward(cudaStream_t st, const double* x, double* y, int64_t n, int act) {
    if (n <= 0) return;
    k_act_fwd<<<grid_for(n), 256, 0, st>>>(x, y, n, act);
    check_launch("k_act_fwd");
}
void act_backward(cudaStream_t st, double* g, const double* pre, int64_t n, int act) {
    if (n <= 0) return;
    k_act_bwd<<<grid_for(n), 256, 0, st>>>(g, pre, n, act);
    check_launch("k_act_bwd");
}
void flag_nonfinite(cudaStream_t st, const double* x, int64_t n, int32_t* flag_dev) {
    if (n <= 0) return;
    k_nonfinite<<<grid_for(n), 256, 0, st>>>(x, n, flag_dev);
    check_launch("k_nonfinite");
}
void flag_nonfinite_f32(cudaStream_t st, const float* x, int64_t n, int32_t* flag_dev) {
    if (n <= 0) return;
    if (n % 4 || reinterpret_cast<uintptr_t>(x) % 16) throw MeftError(2, "check_finite: f32 rows must be float4 aligned");
    k_nonfinite_f32<<<int(std::min<int64_t>((n / 4 + 255) / 256, num_sms() * 8)), 256, 0, st>>>(
        reinterpret_cast<const float4*>(x), n / 4, flag_dev);
    check_launch("k_nonfinite");
}
void add_f64(cudaStream_t st, double* a, const double* b, int64_t n) {
    if (n <= 0) return;
    k_add_f64<<<grid_for(n), 256, 0, st>>>(a, b, n);
    check_launch("k_add_f64");
}

}  // namespace meft_dev
