// Certified tensor-core Key-Experts selection (bf16 inputs), included by select.cu.
//
// Scores are first computed approximately on the tcgen05 tensor cores (fp32 TMEM accumulation):
// the router as one GEMM, the within-expert key scores as a grouped GEMM over tokens bucketed by expert.
// Every approximate score s carries a rigorous bound |s - x| <= e, where x is the reference's fp64
// left-to-right score (kernels.hpp:37-41):
//     e = CB(d) * ||h_t||_2 * ||w_j||_2,   CB(d) = 32 * 2^-24 * (ceil(d/16) + 1) + d * 2^-52
// (model: each K=16 tcgen05 step adds 16 exact bf16 products to the fp32 accumulator with error at most
// 32 units of 2^-24 * (|acc| + sum|p|), i.e. 16x the worst case of an align-truncate-round adder; the fp64
// reference adds at most d*2^-53*sum|p|; sum|p| <= ||h||*||w|| by Cauchy-Schwarz). With the approximate
// top-K set Top, L_in = min_{Top}(s - e) and U_out = max_{not Top}(s + e):
//   members of Top with s - e > U_out are certainly selected, non-members with s + e < L_in certainly not,
// and the remaining ambiguous candidates A are re-scored EXACTLY. The exact score uses a warp-parallel fp64
// sum that is provably identical to the reference's sequential chain when every partial sum is representable
// (all products are multiples of 2^lsb and sum|p| < 2^(lsb+53)); otherwise it falls back to the sequential
// chain itself. The final choice among A uses the reference's total order, so indices are bit-exact.

namespace {

constexpr int CERT_MAX_C = 8192;  // candidates per token handled by the certified top-K kernel

__host__ __device__ inline double cert_bound_coeff(int d) {
    return 32.0 * 0x1p-24 * double((d + 15) / 16 + 1) + double(d) * 0x1p-52;
}

// Same bound when the tensor-core score is the fp64 sum of `ksplit` partial products over K-chunks of at most
// `chunk` elements, rounded to fp32: per-chunk accumulation error sum_c CB(chunk)*|h_c||k_c| <= CB(chunk)*|h||k|
// (Cauchy-Schwarz), plus the reference's own fp64 rounding over all d terms, the fp64 sum of the partials and
// the final fp32 rounding.
__host__ __device__ inline double cert_bound_coeff_split(int d, int chunk, int ksplit) {
    return 32.0 * 0x1p-24 * double((chunk + 15) / 16 + 1) + double(d) * 0x1p-52 + double(ksplit) * 0x1p-52 +
           0x1p-23;
}


__device__ __forceinline__ double bfd(uint16_t b) { return double(bf16_bits_to_f32(b)); }

// Per-product exactness certificate, fp32 flavour: every bf16 x bf16 product is formed exactly in fp32 (the caller
// guarantees no underflow below 2^-149 and no overflow), its LSB is bounded below by (fp32 exponent field) - 142
// (an exact product has <= 16 significant bits; subnormals: 2^-149), sum|p| is accumulated in fp32 and inflated by
// 2^-10 (its rounding error over <= 2^16 terms per lane and the warp sum is far smaller); the value in fp64.
// ~6 instructions per product and loads 4 deep (the generic path below is ~15 and latency-bound).
// Exponent of the lowest set bit of a finite nonzero double: x is a multiple of 2^lowbit_exp(x).
__device__ __forceinline__ int lowbit_exp(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x)) & 0x7FFFFFFFFFFFFFFFull;
    const int e = int(b >> 52);
    unsigned long long m = b & 0xFFFFFFFFFFFFFull;
    if (e == 0) return -1074 + __ffsll(static_cast<long long>(m)) - 1;  // subnormal: m * 2^-1074
    m |= 1ull << 52;
    return e - 1075 + __ffsll(static_cast<long long>(m)) - 1;
}

__device__ __forceinline__ bool exact_dot_warp_f32(const uint4* __restrict__ a4, const uint4* __restrict__ b4, int d8,
                                                   int lane, double& value) {
    constexpr int U = 4;
    double s = 0.0;
    float sa = 0.0f;
    uint32_t emin = 0x7F800000u;  // min fp32 exponent field (in place) over nonzero products
    for (int v0 = lane; v0 < d8; v0 += 32 * U) {
        uint4 x[U], y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int v = v0 + 32 * u;
            if (v < d8) {
                x[u] = a4[v];
                y[u] = __ldg(b4 + v);
            } else {
                x[u] = make_uint4(0, 0, 0, 0);
                y[u] = x[u];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, ys[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t xw = xs[q >> 1], yw = ys[q >> 1];
                const float xf = __uint_as_float((q & 1) ? (xw & 0xFFFF0000u) : (xw << 16));
                const float yf = __uint_as_float((q & 1) ? (yw & 0xFFFF0000u) : (yw << 16));
                const float p = __fmul_rn(xf, yf);  // exact
                const uint32_t pb = __float_as_uint(p) & 0x7FFFFFFFu;
                emin = min(emin, pb == 0 ? 0x7F800000u : (pb & 0x7F800000u));
                sa += fabsf(p);
                s += double(p);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        emin = min(emin, __shfl_xor_sync(0xffffffffu, emin, o));
    }
    value = s;
    if (emin == 0x7F800000u) return true;  // every product is +-0
    const int e = int(emin >> 23);
    const int lsb = e == 0 ? -149 : e - 142;
    return double(sa) * (1.0 + 0x1p-10) < ldexp(1.0, lsb + 53);
}

// The reference's fp64 score dot(a, b) for bf16 rows, computed by a whole warp; all lanes return it.
__device__ double exact_dot_warp(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b, int d, int lane,
                                 int* fallbacks, bool f32_products = false) {
    double s = 0.0, sa = 0.0;
    int lsb = INT32_MAX;
    const bool vec = (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % 16 == 0);
    if (vec && f32_products) {
        double v;
        if (exact_dot_warp_f32(reinterpret_cast<const uint4*>(a), reinterpret_cast<const uint4*>(b), d / 8, lane, v))
            return v;
        lsb = 0;  // certificate failed: go straight to the sequential chain below
        sa = INFINITY;
    } else if (vec) {
        const uint4* a4 = reinterpret_cast<const uint4*>(a);
        const uint4* b4 = reinterpret_cast<const uint4*>(b);
        for (int v = lane; v < d / 8; v += 32) {
            const uint4 x = a4[v], y = __ldg(b4 + v);
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint16_t xa = uint16_t(xs[q >> 1] >> (16 * (q & 1))), yb = uint16_t(ys[q >> 1] >> (16 * (q & 1)));
                const double p = bfd(xa) * bfd(yb);  // exact: <= 16 significant bits
                if (p != 0.0) {
                    s += p;
                    sa += fabs(p);
                    lsb = min(lsb, bf16_lsb_exp(xa) + bf16_lsb_exp(yb));
                }
            }
        }
    } else {
        for (int k = lane; k < d; k += 32) {
            const double p = bfd(a[k]) * bfd(b[k]);
            if (p != 0.0) {
                s += p;
                sa += fabs(p);
                lsb = min(lsb, bf16_lsb_exp(a[k]) + bf16_lsb_exp(b[k]));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
    }
    // every partial sum (in ANY order) is a multiple of 2^lsb bounded by sum|p|: representable iff < 2^(lsb+53)
    if (lsb == INT32_MAX || sa * (1.0 + 0x1p-30) < ldexp(1.0, lsb + 53)) return s;
    // Certificate failed: the reference's sequential chain acc = fl(acc + a_k b_k), k ascending (products exact, so
    // this equals its fma chain), evaluated 128 terms at a time (lane l holds k = base + 4l .. 4l+3). A chunk whose
    // every prefix sum acc + p_1 + ... + p_i is provably representable -- all are multiples of 2^L, L = the lowest
    // set bit over acc and the chunk's products, and |acc| + sum|p| < 2^(L+53) -- adds no rounding, so the chain
    // through it equals acc + (warp sum of the chunk), which is itself exact (every subset sum obeys the same
    // bound). Only chunks that fail this local test run the dependent add chain over the broadcast products.
    double acc = 0.0;
    for (int base = 0; base < d; base += 128) {
        double p[4];
        double ls = 0.0, la = 0.0;
        int lo = INT32_MAX;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = base + 4 * lane + q;
            p[q] = k < d ? bfd(a[k]) * bfd(b[k]) : 0.0;
            if (p[q] != 0.0) lo = min(lo, lowbit_exp(p[q]));
            ls += p[q];
            la += fabs(p[q]);
        }
        double cs = ls, ca = la;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cs += __shfl_xor_sync(0xffffffffu, cs, o);
            ca += __shfl_xor_sync(0xffffffffu, ca, o);
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        }
        if (lo == INT32_MAX) continue;  // all 128 products are +-0: acc + (+-0) leaves acc unchanged
        const int L = acc != 0.0 ? min(lo, lowbit_exp(acc)) : lo;
        if ((fabs(acc) + ca) * (1.0 + 0x1p-40) < ldexp(1.0, L + 53)) {
            acc += cs;
            continue;
        }
        const int n = min(128, d - base);
        for (int j = 0; j < n; ++j) {
            const double pj = __shfl_sync(0xffffffffu, (j & 3) == 0 ? p[0] : (j & 3) == 1 ? p[1] : (j & 3) == 2 ? p[2] : p[3],
                                          j >> 2);
            acc += pj;
        }
    }
    if (lane == 0 && fallbacks) atomicAdd(fallbacks, 1);
    return acc;
}

// ||row||_2 of bf16 rows (fp64 sum of squares, rounded up), one warp per row.
// Also the row's minimum LSB exponent over its nonzero entries (INT32_MAX for an all-zero row): with
// lsb(h_t) + lsb(w_j) and ||h_t|| ||w_j|| the exactness certificate of a dot can be decided per row pair.
__global__ void k_row_norms(const uint16_t* __restrict__ x, int64_t rows, int d, float* __restrict__ out,
                            int32_t* __restrict__ minlsb) {
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const uint16_t* p = x + r * d;
    double s = 0.0;
    int lsb = INT32_MAX;
    for (int k = lane; k < d; k += 32) {
        const uint16_t b = p[k];
        const double v = bfd(b);
        s = fma(v, v, s);
        if (b & 0x7FFF) lsb = min(lsb, bf16_lsb_exp(b));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        lsb = min(lsb, __shfl_xor_sync(0xffffffffu, lsb, o));
    }
    if (lane == 0) {
        out[r] = __double2float_ru(sqrt(s) * (1.0 + 0x1p-20));
        if (minlsb) minlsb[r] = lsb;
    }
}

// exact_dot_warp with a row-level certificate: when every product is a multiple of 2^(lsb_a + lsb_b) and
// ||a|| ||b|| (>= sum|p|) < 2^(lsb_a + lsb_b + 53), all partial sums in any order are exact, so a plain warp
// fma reduction equals the reference's sequential chain. Otherwise the per-product path decides.
__device__ __forceinline__ double exact_dot_rows(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b, int d,
                                                 int lane, int lsb_a, int lsb_b, float na, float nb, int* fallbacks) {
    if (lsb_a == INT32_MAX || lsb_b == INT32_MAX) return 0.0;  // an all-zero row: every product is +-0
    const int lsb = lsb_a + lsb_b;
    if (lsb + 53 < 1000 && double(na) * double(nb) * (1.0 + 0x1p-30) < ldexp(1.0, lsb + 53) &&
        (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % 16 == 0)) {
        const uint4* a4 = reinterpret_cast<const uint4*>(a);
        const uint4* b4 = reinterpret_cast<const uint4*>(b);
        // Every partial sum is exact, so any order and several accumulators give the reference's value. Loads are
        // issued 4 deep (latency-bound otherwise, ncu). With -149 <= lsb <= 74 each bf16 x bf16 product is exact
        // in fp32 too (a multiple of 2^-149 below 2^127 with <= 16 significant bits): one fp32 multiply and one
        // widening per product instead of two widenings and a DFMA.
        const bool f32_products = lsb >= -149 && lsb <= 74;
        constexpr int U = 4;  // 8 and 16 measured equal (the kernel's tail is the uncertifiable dots, not load depth)
        double s0 = 0.0, s1 = 0.0;
        for (int v0 = lane; v0 < d / 8; v0 += 32 * U) {
            uint4 x[U], y[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int v = v0 + 32 * u;
                if (v < d / 8) {
                    x[u] = a4[v];
                    y[u] = __ldg(b4 + v);
                } else {
                    x[u] = make_uint4(0, 0, 0, 0);
                    y[u] = x[u];
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w}, ys[4] = {y[u].x, y[u].y, y[u].z, y[u].w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float xl = __uint_as_float(xs[q] << 16), yl = __uint_as_float(ys[q] << 16);
                    const float xh = __uint_as_float(xs[q] & 0xFFFF0000u), yh = __uint_as_float(ys[q] & 0xFFFF0000u);
                    if (f32_products) {
                        s0 += double(__fmul_rn(xl, yl));
                        s1 += double(__fmul_rn(xh, yh));
                    } else {
                        s0 = fma(double(xl), double(yl), s0);
                        s1 = fma(double(xh), double(yh), s1);
                    }
                }
            }
        }
        double s = s0 + s1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        return s;
    }
    // fp32-exact products need every product inside fp32's range: all LSBs >= 2^-149 and |p| <= ||a|| ||b|| < 2^127
    const bool f32ok = lsb >= -149 && double(na) * double(nb) < 0x1p126;
    return exact_dot_warp(a, b, d, lane, fallbacks, f32ok);
}

// Warp per token: certified top-kk experts of the approximate router scores P [T x ldp].
__global__ void k_router_certified(const float* __restrict__ P, int ldp, const float* __restrict__ hn,
                                   const float* __restrict__ gn, const int32_t* __restrict__ hl,
                                   const int32_t* __restrict__ gl, double cb, const uint16_t* __restrict__ h,
                                   const uint16_t* __restrict__ wg, int d, int T, int N, int kk,
                                   int32_t* __restrict__ tau, int32_t* __restrict__ counts, int* __restrict__ stats) {
    extern __shared__ uint8_t sm_raw[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = blockIdx.x * (blockDim.x >> 5) + wib;
    if (t >= T) return;
    // per-warp scratch: kk top indices, then up to N ambiguous (idx, exact score)
    int* top = reinterpret_cast<int*>(sm_raw) + wib * (kk + 2 * N);
    int* aidx = top + kk;
    double* ax = reinterpret_cast<double*>(sm_raw + (blockDim.x >> 5) * (kk + 2 * N) * 4) + wib * N;
    const float* s = P + int64_t(t) * ldp;
    const double he = cb * double(hn[t]);

    // approximate top-kk in the reference order (score desc, index asc)
    float ps = 0.f;
    int pi = -1;
    for (int r = 0; r < kk; ++r) {
        float bs = -FLT_MAX;
        int bi = -1;
        for (int i = lane; i < N; i += 32) {
            const float v = s[i];
            if (pi >= 0 && !(v < ps || (v == ps && i > pi))) continue;
            if (bi < 0 || v > bs || (v == bs && i < bi)) {
                bs = v;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float os = __shfl_xor_sync(0xffffffffu, bs, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi >= 0 && (bi < 0 || os > bs || (os == bs && oi < bi))) {
                bs = os;
                bi = oi;
            }
        }
        ps = bs;
        pi = bi;
        if (lane == 0) top[r] = bi;
    }
    __syncwarp();
    // L_in over Top, U_out over the rest (non-Top = ranked after the last Top element)
    double lin = DBL_MAX, uout = -DBL_MAX;
    for (int i = lane; i < N; i += 32) {
        const float v = s[i];
        const double e = he * double(gn[i]);
        const bool in_top = (v > ps) || (v == ps && i <= pi);
        if (in_top) lin = fmin(lin, double(v) - e);
        else uout = fmax(uout, double(v) + e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lin = fmin(lin, __shfl_xor_sync(0xffffffffu, lin, o));
        uout = fmax(uout, __shfl_xor_sync(0xffffffffu, uout, o));
    }
    // ambiguous set A (ordered by warp ballot so the list is deterministic)
    int na = 0, n_in = 0;
    for (int base = 0; base < N; base += 32) {
        const int i = base + lane;
        bool amb = false, sure = false;
        if (i < N) {
            const float v = s[i];
            const double e = he * double(gn[i]);
            const bool in_top = (v > ps) || (v == ps && i <= pi);
            if (in_top) {
                amb = double(v) - e <= uout;
                sure = !amb;
            } else {
                amb = double(v) + e >= lin;
            }
        }
        const unsigned ba = __ballot_sync(0xffffffffu, amb);
        n_in += __popc(__ballot_sync(0xffffffffu, sure));
        if (amb) aidx[na + __popc(ba & ((1u << lane) - 1u))] = i;
        na += __popc(ba);
    }
    __syncwarp();
    int32_t* out = tau + int64_t(t) * kk;
    if (na == 0) {
        if (lane == 0)
            for (int r = 0; r < kk; ++r) out[r] = top[r];
    } else {
        for (int a = 0; a < na; ++a)
            ax[a] = exact_dot_rows(h + int64_t(t) * d, wg + int64_t(aidx[a]) * d, d, lane, hl[t], gl[aidx[a]], hn[t],
                                   gn[aidx[a]], stats ? stats + 1 : nullptr);
        __syncwarp();
        if (lane == 0) {
            if (stats) atomicAdd(stats, na);
            int w = 0;
            for (int r = 0; r < kk; ++r) {  // certain members
                const int i = top[r];
                bool amb = false;
                for (int a = 0; a < na; ++a) amb |= (aidx[a] == i);
                if (!amb) out[w++] = i;
            }
            const int need = kk - w;  // best `need` of A by the exact reference order
            for (int a = 0; a < na && w < kk; ++a) {
                int rank = 0;
                for (int b = 0; b < na; ++b)
                    if (ax[b] > ax[a] || (ax[b] == ax[a] && aidx[b] < aidx[a])) ++rank;
                if (rank < need) out[w++] = aidx[a];
            }
        }
    }
    __syncwarp();
    if (lane == 0) {
        for (int a = 1; a < kk; ++a) {
            const int v = out[a];
            int b = a - 1;
            while (b >= 0 && out[b] > v) {
                out[b + 1] = out[b];
                --b;
            }
            out[b + 1] = v;
        }
        for (int a = 0; a < kk; ++a) atomicAdd(&counts[out[a]], 1);
    }
    (void)n_in;
}

// H_sorted[pos] = h[entries[pos] / kk] (bf16 rows), one warp per row, 16-byte vectors.
__global__ void k_gather_tokens(const uint16_t* __restrict__ h, int d, const int32_t* __restrict__ entries, int n,
                                int kk, uint16_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int nv = d / 8;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        const uint4* src = reinterpret_cast<const uint4*>(h + int64_t(entries[r] / kk) * d);
        uint4* dst = reinterpret_cast<uint4*>(out + int64_t(r) * d);
        for (int v = lane; v < nv; v += 32) dst[v] = __ldg(src + v);
    }
}

// ---- certified per-token top-K, in three kernels so the exact re-scoring can be grouped by expert (key rows
// stay hot in L2) — and, in the expert-sharded layer, executed on the rank that owns the keys.

// orderable uint32 of a float: larger float <=> larger key
__device__ __forceinline__ uint32_t float_key(float f) {
    const uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// K1, CTA per token: radix-select the approximate top-`take` (order: score desc, then candidate position asc —
// positions ascend with the global index because tau is ascending), derive L_in / U_out, and split the
// candidates into certain members (sure[t][0..n_sure)) and ambiguous ones (amb[t][0..n_amb), global indices).
// amb_count[idx / E] counts ambiguous pairs per expert for the grouping.
// smem: key u32[C] | in_top u8[C]
__global__ void __launch_bounds__(256)
    k_topk_classify(const float* __restrict__ cand, const int32_t* __restrict__ tau, int kk, int E, int C, int P2,
                    int take, const float* __restrict__ hn, const float* __restrict__ kn, double cb,
                    int32_t* __restrict__ sure, int32_t* __restrict__ n_sure, int32_t* __restrict__ amb,
                    int32_t* __restrict__ n_amb, int32_t* __restrict__ amb_count, int ksplit,
                    long long split_stride) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint32_t* key = reinterpret_cast<uint32_t*>(sm);
    float* val = reinterpret_cast<float*>(key + C);  // approximate scores (sum of the K-split partials)
    uint8_t* in_top = reinterpret_cast<uint8_t*>(val + C);
    __shared__ double w_lin[32], w_uout[32];
    __shared__ int hist[256], w_cnt[32];
    __shared__ uint32_t s_prefix;
    __shared__ int s_remaining, s_na, s_ns;
    const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const float* c = cand + int64_t(t) * C;
    for (int i = tid; i < C; i += blockDim.x) {
        float v = c[i];
        if (ksplit > 1) {
            double sum = double(v);
            for (int sp = 1; sp < ksplit; ++sp) sum += double(c[sp * split_stride + i]);
            v = float(sum);
        }
        val[i] = v;
        key[i] = float_key(v);
    }
    if (tid == 0) {
        s_na = 0;
        s_ns = 0;
        s_prefix = 0;
        s_remaining = take;
    }
    __syncthreads();
    // radix select of the take-th largest key, 8 bits at a time from the top
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = tid; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        for (int i = tid; i < C; i += blockDim.x)
            if ((key[i] & mask) == prefix) atomicAdd(&hist[(key[i] >> shift) & 255], 1);
        __syncthreads();
        if (warp == 0) {  // digits descending: lane l owns digits 255-8l .. 248-8l
            int part = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) part += hist[255 - 8 * lane - q];
            int incl = part;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += x;
            }
            const int rem = s_remaining;
            const int excl = incl - part;
            if (excl < rem && rem <= incl) {  // exactly one lane
                int cum = excl;
                for (int q = 0; q < 8; ++q) {
                    const int dgt = 255 - 8 * lane - q;
                    if (cum + hist[dgt] >= rem) {
                        s_prefix = prefix | (uint32_t(dgt) << shift);
                        s_remaining = rem - cum;
                        break;
                    }
                    cum += hist[dgt];
                }
            }
        }
        mask |= 255u << shift;
        __syncthreads();
    }
    const uint32_t kth = s_prefix;
    const int need_eq = s_remaining;  // how many candidates equal to the take-th key belong to Top
    // rank among equals by position: block exclusive scan of the equality flags over contiguous chunks
    const int chunk = (C + blockDim.x - 1) / blockDim.x, c0 = tid * chunk, c1 = min(C, c0 + chunk);
    int eq = 0;
    for (int i = c0; i < c1; ++i) eq += key[i] == kth;
    int incl = eq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    if (lane == 31) w_cnt[warp] = incl;
    __syncthreads();
    int before = incl - eq;
    for (int w = 0; w < warp; ++w) before += w_cnt[w];
    for (int i = c0; i < c1; ++i) {
        const bool e_ = key[i] == kth;
        in_top[i] = key[i] > kth || (e_ && before < need_eq);
        before += e_;
    }
    __syncthreads();
    const double he = cb * double(hn[t]);
    const int32_t* my_tau = tau + int64_t(t) * kk;
    double lin = DBL_MAX, uout = -DBL_MAX;
    for (int i = tid; i < C; i += blockDim.x) {
        const int slot = i / E;
        const int gi = my_tau[slot] * E + (i - slot * E);
        const double e = he * double(kn[gi]);
        if (in_top[i]) lin = fmin(lin, double(val[i]) - e);
        else uout = fmax(uout, double(val[i]) + e);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lin = fmin(lin, __shfl_xor_sync(0xffffffffu, lin, o));
        uout = fmax(uout, __shfl_xor_sync(0xffffffffu, uout, o));
    }
    if (lane == 0) {
        w_lin[warp] = lin;
        w_uout[warp] = uout;
    }
    __syncthreads();
    lin = DBL_MAX;
    uout = -DBL_MAX;
    for (int w = 0; w < nwarps; ++w) {
        lin = fmin(lin, w_lin[w]);
        uout = fmax(uout, w_uout[w]);
    }
    int32_t* my_sure = sure + int64_t(t) * take;
    int32_t* my_amb = amb + int64_t(t) * C;
    for (int i = tid; i < C; i += blockDim.x) {
        const int slot = i / E;
        const int gi = my_tau[slot] * E + (i - slot * E);
        const double e = he * double(kn[gi]);
        const bool top = in_top[i];
        const bool ambiguous = top ? (double(val[i]) - e <= uout) : (double(val[i]) + e >= lin);
        if (ambiguous) {
            my_amb[atomicAdd(&s_na, 1)] = gi;
            if (amb_count) atomicAdd(&amb_count[gi / E], 1);
        } else if (top) {
            my_sure[atomicAdd(&s_ns, 1)] = gi;
        }
    }
    __syncthreads();
    if (tid == 0) {
        n_amb[t] = s_na;
        n_sure[t] = s_ns;
    }
}

// K2a, CTA per token: bucket the token's ambiguous pairs by expert (pair_t / pair_a = token, position in amb[t]).
__global__ void k_amb_fill(const int32_t* __restrict__ amb, const int32_t* __restrict__ n_amb, int C, int E,
                           const int32_t* __restrict__ off, int32_t* __restrict__ cursor, int32_t* __restrict__ pair_t,
                           int32_t* __restrict__ pair_a) {
    const int t = blockIdx.x;
    const int n = n_amb[t];
    for (int a = threadIdx.x; a < n; a += blockDim.x) {
        const int e = amb[int64_t(t) * C + a] / E;
        const int pos = off[e] + atomicAdd(&cursor[e], 1);
        pair_t[pos] = t;
        pair_a[pos] = a;
    }
}

// K2b, warp per ambiguous pair, pairs in expert order: the reference's exact fp64 score.
__global__ void k_rescore_pairs(const int32_t* __restrict__ pair_t, const int32_t* __restrict__ pair_a,
                                const int32_t* __restrict__ total, const int32_t* __restrict__ amb, int C,
                                const uint16_t* __restrict__ h, const uint16_t* __restrict__ keys, int d,
                                const float* __restrict__ hn, const float* __restrict__ kn,
                                const int32_t* __restrict__ hl, const int32_t* __restrict__ kl,
                                double* __restrict__ x, int* __restrict__ stats) {
    const int lane = threadIdx.x & 31;
    const int n = *total;
    for (int p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += (gridDim.x * blockDim.x) >> 5) {
        const int t = pair_t[p], a = pair_a[p];
        const int idx = amb[int64_t(t) * C + a];
        const double v = exact_dot_rows(h + int64_t(t) * d, keys + int64_t(idx) * d, d, lane, hl[t], kl[idx], hn[t],
                                        kn[idx], stats ? stats + 1 : nullptr);
        if (lane == 0) x[int64_t(t) * C + a] = v;
    }
    if (stats && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(stats, n);
}

// K3, CTA per token: sure members + the best (take - n_sure) ambiguous ones by the exact reference order,
// emitted ascending (experts.cpp:94-105) into per_token, and marked in the union bitmap.
__global__ void __launch_bounds__(128)
    k_topk_finalize(const int32_t* __restrict__ sure, const int32_t* __restrict__ n_sure,
                    const int32_t* __restrict__ amb, const int32_t* __restrict__ n_amb, const double* __restrict__ x,
                    int C, int take, int TP2, int32_t* __restrict__ per_token, uint8_t* __restrict__ flags) {
    extern __shared__ __align__(16) uint8_t sm[];
    int* sel = reinterpret_cast<int*>(sm);
    __shared__ int s_n;
    const int t = blockIdx.x, tid = threadIdx.x;
    const int ns = n_sure[t], na = n_amb[t], need = take - ns;
    const int32_t* my_amb = amb + int64_t(t) * C;
    const double* my_x = x + int64_t(t) * C;
    for (int i = tid; i < ns; i += blockDim.x) sel[i] = sure[int64_t(t) * take + i];
    if (tid == 0) s_n = ns;
    __syncthreads();
    for (int a = tid; a < na; a += blockDim.x) {
        const double xa = my_x[a];
        const int ia = my_amb[a];
        int rank = 0;
        for (int b = 0; b < na; ++b) rank += (my_x[b] > xa) || (my_x[b] == xa && my_amb[b] < ia);
        if (rank < need) sel[atomicAdd(&s_n, 1)] = ia;
    }
    __syncthreads();
    for (int i = take + tid; i < TP2; i += blockDim.x) sel[i] = INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= TP2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < TP2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const int a = sel[i], b = sel[p];
                    if (((i & k) == 0) ? (a > b) : (a < b)) {
                        sel[i] = b;
                        sel[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = tid; i < take; i += blockDim.x) {
        const int v = sel[i];
        per_token[int64_t(t) * take + i] = v;
        flags[v] = 1;
    }
}

}  // namespace
