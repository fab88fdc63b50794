// Internal host-side launch API of the sm_100a kernels (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace meft_dev {

// ---------------------------------------------------------------- bf16 tcgen05 GEMM
// C[M x N] (epilogue) of  sum_k A(m,k) * B(n,k)  with bf16 operands and fp32 accumulation in TMEM.
//   K-major operand:  X(i,k) = ptr[i*ld + k]
//   MN-major operand: X(i,k) = ptr[k*ld + i]
struct GemmOperand {
    const void* ptr;
    int64_t ld;     // elements
    bool mn_major;
    // B only: row gather. Row p of the logical B (p < N when K-major, p < K when MN-major) is row rows[p] of the
    // table at ptr ([table_rows x ld]); loaded with TMA tile::gather4 straight into the operand tile.
    const int32_t* rows = nullptr;
    int64_t table_rows = 0;
    int32_t* run_ws = nullptr;  // MN-major gathered B: scratch of ceil(K / 64) ints (per-k-block run table)
    // Panelled A (gemm_bf16 only): the dimension gemm_bf16 chunks (K of a K-major A, M of an MN-major A) is stored
    // as consecutive panels of kGemmPanel columns, panel p at ptr + p * panel_stride, each with leading dimension
    // ld, so every sub-GEMM reads one dense [rows x kGemmPanel] panel. 0 = one plain matrix.
    int64_t panel_stride = 0;
    // L2 eviction priority of this operand's TMA loads: 0 default, 1 evict_first, 2 evict_last (plain boxes only).
    int l2_hint = 0;
};
constexpr int64_t kGemmPanel = 65536;  // = gemm_bf16's chunk width

enum GemmEpi : int {
    EPI_STORE_F32 = 0,     // C f32 [M x ldc] = acc            (or += acc when accumulate)
    EPI_RELU_BF16 = 1,     // C bf16 = relu(acc), positive never rounds to zero; with `bits` also the bitmask acc > 0
    EPI_MASK_BF16 = 2,     // C bf16 = mask(m,n) > 0 ? acc : 0 ; mask bf16 [M x ldm], or the bitmask `bits`
    EPI_ROWS_ADD_F32 = 3,  // C f32: C[row_idx[m]*ldc + n] += acc (row_idx unique -> no atomics)
    EPI_ROWS_STORE_F32 = 4,  // C f32: C[row_idx[m]*ldc + n] = acc
    // Push to peers: global row g = row0 + m belongs to home h = g / peer_rows; the f32 row is stored into that
    // home's receive buffer peer[h] (device pointer, NVLink peer-mapped for h != this rank) at slot peer_slot:
    // peer[h][(peer_slot * peer_rows + g % peer_rows) * ldc + col0 + n]. A reduce-scatter fused into the epilogue.
    EPI_PEER_F32 = 5,
    // Frozen base FFN (adapter.cpp:118-120, 153-164): act = 0 SiLU, 1 ReLU.
    EPI_ACT_BF16 = 6,   // C bf16 = act(acc); aux bf16 [M x ldaux] = acc (the pre-activation, kept for backward)
    EPI_DACT_BF16 = 7,  // C bf16 = acc * act'(aux)   (aux: the stored pre-activation)
    // Lazy sparse Adam fused into a weight-gradient GEMM (memtier.cpp:187-210 on the fused step): acc row m is the
    // gradient of table row j = row_idx[m]; the epilogue applies adam_update to adam_w/m/v[j*ldc + n] with the
    // per-position coefficients adam_coef[m] (scale, inv_c2) and writes the bf16 compute copy adam_c. With stat_ss
    // it also emits the selection statistics of the new bf16 row per 256-column tile nb:
    // stat_ss[m*stat_ld + nb] = an upper bound of the sum of squares (fp32 sums rounded up, stored as double),
    // stat_lsb[...] = minimum LSB exponent of the nonzero entries.
    // No K split (the update needs the finished gradient); N <= 65536.
    EPI_ADAM_F32 = 8,
};
constexpr int kMaxPeers = 8;

struct GemmEpilogue {
    int kind = EPI_STORE_F32;
    void* c = nullptr;
    int64_t ldc = 0;
    const void* mask = nullptr;
    int64_t ldm = 0;
    // EPI_RELU_BF16 (written) / EPI_MASK_BF16 (read instead of `mask`): bit (n % 32) of bits[m * ldbits + n / 32]
    // is acc(m, n) > 0 -- 1/16 of the bytes of the bf16 activation as the backward's mask.
    uint32_t* bits = nullptr;
    int64_t ldbits = 0;
    const int32_t* row_idx = nullptr;
    bool accumulate = false;
    // K split (f32 store epilogues, 1-CTA kernel): split s of `ksplit` multiplies K-chunk s only and writes its
    // partial product to c + s * split_stride (elements); the caller sums the partials.
    int ksplit = 1;
    int64_t split_stride = 0;
    // EPI_ACT_BF16 / EPI_DACT_BF16
    void* aux = nullptr;
    int64_t ldaux = 0;
    int act = 0;
    // EPI_PEER_F32
    float* peer[kMaxPeers] = {};
    int peer_count = 0;
    int peer_slot = 0;
    int64_t peer_rows = 0;
    int64_t row0 = 0, col0 = 0;
    // EPI_ADAM_F32 (ldc = table row pitch in elements)
    float* adam_w = nullptr;
    void* adam_m = nullptr;  // fp32, or bf16 with adam_mom16 (COMPACT store)
    void* adam_v = nullptr;
    bool adam_mom16 = false;
    uint16_t* adam_c = nullptr;
    const float2* adam_coef = nullptr;
    float b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
    double* stat_ss = nullptr;
    int32_t* stat_lsb = nullptr;
    int64_t stat_ld = 0;  // >= ceil(N / 256)
    // Panelled C of the bf16 epilogues (EPI_RELU_BF16 / EPI_MASK_BF16 with bits): N stored as kGemmPanel-wide panels
    // at c + p * panel_stride, leading dimension ldc (see GemmOperand::panel_stride).
    int64_t panel_stride = 0;
    // Launch option, CTA-pair kernel tile order: 0 = the default policy, -1 = sweep N first (the co-running tiles
    // share their A panels; B is re-read every wave), g > 0 = groups of g 256-row M tiles per streamed B panel.
    int raster = 0;
    // Device-sized extent: M / N / K as passed is a capacity; the kernels read the real size of dimension
    // extent_dim (1 = M, 2 = N, 3 = K) from device memory, so the launch needs no host read-back (see apply_extent).
    const int32_t* extent = nullptr;
    int extent_dim = 0;
};
constexpr int kAdamStatTile = 256;  // columns per EPI_ADAM_F32 statistics partial

void gemm_bf16(cudaStream_t st, int64_t M, int64_t N, int64_t K, const GemmOperand& A, const GemmOperand& B,
               const GemmEpilogue& epi);

// Leave n SMs free of persistent GEMM CTAs (for overlapped NCCL kernels); 0 restores the full machine.
void gemm_reserve_sms(int n);

// Grouped variant (K-major operands): group g computes rows [row_off[g], row_off[g+1]) of A against the N rows
// [g*N, (g+1)*N) of B; tile_off = exclusive scan of ceil(rows_g / 128) (device arrays, no host sync). The
// epilogue sees the global A row m (use EPI_ROWS_STORE_F32 with row_idx to place it) and column n < N.
void gemm_bf16_grouped(cudaStream_t st, int G, int64_t N, int64_t K, const GemmOperand& A, int64_t a_rows,
                       const GemmOperand& B, int64_t b_rows, const int32_t* row_off, const int32_t* tile_off,
                       const GemmEpilogue& epi);

// ---------------------------------------------------------------- fp64 SIMT GEMM (API-fidelity path)
// C[M x N] = sum_k A(m,k) * B(k,n) over ascending k (fma chain, reference kernels.cpp:34-41), with
// arbitrary element strides so transposed views need no copies.
struct DOperand {
    const double* ptr;
    int64_t s0, s1;     // element strides for (row, col) of the logical matrix
    bool relu = false;  // load max(x, 0) (A operand only: ReLU(z) without materialising it)
};
enum DEpi : int {
    DEPI_STORE = 0,        // C = acc
    DEPI_ADD = 1,          // C += acc
    DEPI_RELU_STORE = 2,   // C = relu(acc)   (unused by the shim; kept for symmetry)
    DEPI_MASK_STORE = 3,   // C = mask(m,n) > 0 ? acc : 0   (mask f64 with strides)
};
void dgemm(cudaStream_t st, int64_t M, int64_t N, int64_t K, const DOperand& A, const DOperand& B, double* C,
           int64_t ldc, int epi, const DOperand* mask);

// ---------------------------------------------------------------- exact selection (fp64 scores)
// dtype: 0 = f64 inputs (unfused mul/add, reference's compiled dot()), 2 = bf16 inputs (exact products:
// fma == unfused).
void score_rows(cudaStream_t st, int dtype, const void* h, int64_t T, int64_t d, const void* w, int64_t rows,
                double* scores);  // scores[T x rows] = dot(h_t, w_row)
}  // namespace meft_dev
