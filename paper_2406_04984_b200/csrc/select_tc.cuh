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

// exponent of the least significant mantissa bit of a bf16 value (subnormals: 2^-133)
__device__ __forceinline__ int bf16_lsb_exp(uint16_t b) {
    const int e = (b >> 7) & 0xFF;
    return e == 0 ? -133 : e - 134;
}

__device__ __forceinline__ double bfd(uint16_t b) { return double(bf16_bits_to_f32(b)); }

// The reference's fp64 score dot(a, b) for bf16 rows, computed by a whole warp; all lanes return it.
__device__ double exact_dot_warp(const uint16_t* __restrict__ a, const uint16_t* __restrict__ b, int d, int lane,
                                 int* fallbacks) {
    double s = 0.0, sa = 0.0;
    int lsb = INT32_MAX;
    const bool vec = (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % 16 == 0);
    if (vec) {
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
    double acc = 0.0;  // certificate failed: run the reference's sequential chain (products exact => fma)
    if (lane == 0) {
        for (int k = 0; k < d; ++k) acc = fma(bfd(a[k]), bfd(b[k]), acc);
        if (fallbacks) atomicAdd(fallbacks, 1);
    }
    return __shfl_sync(0xffffffffu, acc, 0);
}

// ||row||_2 of bf16 rows (fp64 sum of squares, rounded up), one warp per row.
__global__ void k_row_norms(const uint16_t* __restrict__ x, int64_t rows, int d, float* __restrict__ out) {
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const uint16_t* p = x + r * d;
    double s = 0.0;
    for (int k = lane; k < d; k += 32) {
        const double v = bfd(p[k]);
        s = fma(v, v, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[r] = __double2float_ru(sqrt(s) * (1.0 + 0x1p-20));
}

// Warp per token: certified top-kk experts of the approximate router scores P [T x ldp].
__global__ void k_router_certified(const float* __restrict__ P, int ldp, const float* __restrict__ hn,
                                   const float* __restrict__ gn, double cb, const uint16_t* __restrict__ h,
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
        for (int a = 0; a < na; ++a) ax[a] = exact_dot_warp(h + int64_t(t) * d, wg + int64_t(aidx[a]) * d, d, lane,
                                                            stats ? stats + 1 : nullptr);
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

// CTA per token: certified top-`take` of the C = kk*E approximate candidate scores.
// smem: ks f32[P2] | is i32[P2] | alist i32[P2] | ax f64[P2] | sel i32[TP2] | hrow bf16[d]
__global__ void __launch_bounds__(256)
    k_topk_certified(const float* __restrict__ cand, const int32_t* __restrict__ tau, int kk, int E, int C, int P2,
                     int take, int TP2, const float* __restrict__ hn, const float* __restrict__ kn, double cb,
                     const uint16_t* __restrict__ h, const uint16_t* __restrict__ keys, int d,
                     int32_t* __restrict__ per_token, uint8_t* __restrict__ flags, int* __restrict__ stats) {
    extern __shared__ __align__(16) uint8_t sm[];
    double* ax = reinterpret_cast<double*>(sm);
    float* ks = reinterpret_cast<float*>(ax + P2);
    int* is = reinterpret_cast<int*>(ks + P2);
    int* alist = is + P2;
    int* sel = alist + P2;
    uint16_t* hrow = reinterpret_cast<uint16_t*>(sel + TP2);
    __shared__ double w_lin[32], w_uout[32];
    __shared__ int s_na, s_nsel, s_nsure;
    const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const float* c = cand + int64_t(t) * C;
    for (int i = tid; i < P2; i += blockDim.x) {
        if (i < C) {
            const int slot = i / E, j = i - slot * E;
            ks[i] = c[i];
            is[i] = tau[int64_t(t) * kk + slot] * E + j;
        } else {
            ks[i] = -FLT_MAX;
            is[i] = INT32_MAX;
        }
    }
    if (tid == 0) {
        s_na = 0;
        s_nsel = 0;
        s_nsure = 0;
    }
    __syncthreads();
    // bitonic sort into the reference order on the approximate scores (padding sorts last)
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const float a = ks[i], b = ks[p];
                    const int ia = is[i], ib = is[p];
                    const bool b_first = (b > a) || (b == a && ib < ia);
                    if (((i & k) == 0) ? b_first : !b_first) {
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
    // L_in = min over Top (s - e), U_out = max over the rest (s + e)
    const double he = cb * double(hn[t]);
    double lin = DBL_MAX, uout = -DBL_MAX;
    for (int i = tid; i < C; i += blockDim.x) {
        const double e = he * double(kn[is[i]]);
        if (i < take) lin = fmin(lin, double(ks[i]) - e);
        else uout = fmax(uout, double(ks[i]) + e);
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
    // classify: certain members go straight to sel; ambiguous ones to alist
    for (int i = tid; i < C; i += blockDim.x) {
        const double e = he * double(kn[is[i]]);
        if (i < take) {
            if (double(ks[i]) - e <= uout) alist[atomicAdd(&s_na, 1)] = is[i];
            else {
                sel[atomicAdd(&s_nsel, 1)] = is[i];
                atomicAdd(&s_nsure, 1);
            }
        } else if (double(ks[i]) + e >= lin) {
            alist[atomicAdd(&s_na, 1)] = is[i];
        }
    }
    __syncthreads();
    const int na = s_na;
    if (na > 0) {
        for (int k = tid; k < d; k += blockDim.x) hrow[k] = h[int64_t(t) * d + k];
        __syncthreads();
        for (int a = warp; a < na; a += nwarps)
            ax[a] = exact_dot_warp(hrow, keys + int64_t(alist[a]) * d, d, lane, stats ? stats + 1 : nullptr);
        __syncthreads();
        const int need = take - s_nsure;
        for (int a = tid; a < na; a += blockDim.x) {  // rank within A by the exact reference order
            const double xa = ax[a];
            const int ia = alist[a];
            int rank = 0;
            for (int b = 0; b < na; ++b) rank += (ax[b] > xa) || (ax[b] == xa && alist[b] < ia);
            if (rank < need) sel[atomicAdd(&s_nsel, 1)] = ia;
        }
        if (tid == 0 && stats) atomicAdd(stats, na);
    }
    __syncthreads();
    for (int i = take + tid; i < TP2; i += blockDim.x) sel[i] = INT32_MAX;
    __syncthreads();
    for (int k = 2; k <= TP2; k <<= 1) {  // ascending output (experts.cpp:104)
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
