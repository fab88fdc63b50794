// fp64 SIMT GEMM for the API-fidelity (float64 Matrix) path of the drop-in shim.
// Each output is one fma chain over ascending k that skips a(m,k) == 0 — the compiled form of the
// reference's matmul_row (kernels.cpp:34-41, FMA-contracted under -march=native) —
// so results are bitwise identical to the reference matmul. Arbitrary element strides give transposed
// views (transpose(w_b_k), transpose(relu(z)), ...) without materialising them.
#include "common.cuh"
#include "kernels.h"

namespace meft_dev {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256)
    k_dgemm(int64_t M, int64_t N, int64_t K, const double* __restrict__ A, int64_t as0, int64_t as1,
            const double* __restrict__ B, int64_t bs0, int64_t bs1, double* __restrict__ C, int64_t ldc, int epi,
            const double* __restrict__ mk, int64_t ms0, int64_t ms1, int a_relu) {
    __shared__ double sa[TK][TM + 1];
    __shared__ double sb[TK][TN + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t m0 = int64_t(blockIdx.y) * TM, n0 = int64_t(blockIdx.x) * TN;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t k0 = 0; k0 < K; k0 += TK) {
        const int kn = int(K - k0 < TK ? K - k0 : TK);
        for (int i = tid; i < TM * TK; i += 256) {
            const int r = i / TK, kk = i % TK;
            const int64_t m = m0 + r;
            double v = (kk < kn && m < M) ? A[m * as0 + (k0 + kk) * as1] : 0.0;
            if (a_relu) v = v > 0.0 ? v : 0.0;
            sa[kk][r] = v;
        }
        for (int i = tid; i < TN * TK; i += 256) {
            const int c = i % TN, kk = i / TN;
            const int64_t n = n0 + c;
            sb[kk][c] = (kk < kn && n < N) ? B[(k0 + kk) * bs0 + n * bs1] : 0.0;
        }
        __syncthreads();
        for (int kk = 0; kk < kn; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (a[i] == 0.0) continue;  // matmul_row skips zero a-entries
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int64_t m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t n = n0 + tx * 4 + j;
            if (n >= N) continue;
            double v = acc[i][j];
            double* c = C + m * ldc + n;
            switch (epi) {
                case DEPI_ADD: v = *c + v; break;
                case DEPI_RELU_STORE: v = v > 0.0 ? v : 0.0; break;
                case DEPI_MASK_STORE: v = (mk[m * ms0 + n * ms1] > 0.0) ? v : 0.0; break;
                default: break;
            }
            *c = v;
        }
    }
}

}  // namespace

void dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, const DOperand& A, const DOperand& B, double* C,
           int64_t ldc, int epi, const DOperand* mask) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) {
        if (epi != DEPI_ADD) {
            for (int64_t m = 0; m < M; ++m) MEFT_CUDA_CHECK(cudaMemsetAsync(C + m * ldc, 0, N * 8, st));
        }
        return;
    }
    dim3 grid(unsigned(ceil_div(N, TN)), unsigned(ceil_div(M, TM)));
    k_dgemm<<<grid, 256, 0, st>>>(M, N, K, A.ptr, A.s0, A.s1, B.ptr, B.s0, B.s1, C, ldc, epi,
                                  mask ? mask->ptr : nullptr, mask ? mask->s0 : 0, mask ? mask->s1 : 0, A.relu ? 1 : 0);
    check_launch("k_dgemm");
}

}  // namespace meft_dev
