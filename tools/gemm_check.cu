// Developer harness (not part of the product): numerics + throughput of the tcgen05 GEMM variants
// used by the MEFT FFN, against a naive fp32 SIMT reference. Built by tools/Makefile.
//   ./gemm_check            small shapes, every (A,B) major combination and epilogue
//   ./gemm_check perf       cfg2-shaped GEMMs (T=8192, |S|=65536, d=4096), CUDA-event timed
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2406_04984_b200/csrc/kernels.h"

using namespace meft_dev;

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__global__ void k_fill(uint16_t* p, int64_t n, uint32_t seed, float scale) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    for (; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t x = uint32_t(i) * 2654435761u ^ seed;
        x ^= x >> 15;
        x *= 2246822519u;
        x ^= x >> 13;
        float f = (float(x & 0xFFFFFF) / float(0x1000000) * 2.0f - 1.0f) * scale;
        p[i] = __bfloat16_as_ushort(__float2bfloat16_rn(f));
    }
}

__device__ float ld_bf(const uint16_t* p) { return __uint_as_float(uint32_t(*p) << 16); }

// ref C[m,n] = sum_k A(m,k) B(n,k)
__global__ void k_ref(int M, int N, int K, const uint16_t* A, int64_t lda, int amn, const uint16_t* B, int64_t ldb,
                      int bmn, float* C) {
    int m = blockIdx.y, n = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= M || n >= N) return;
    float acc = 0.f;
    for (int k = 0; k < K; ++k) {
        float a = ld_bf(amn ? A + (int64_t)k * lda + m : A + (int64_t)m * lda + k);
        float b = ld_bf(bmn ? B + (int64_t)k * ldb + n : B + (int64_t)n * ldb + k);
        acc = fmaf(a, b, acc);
    }
    C[(int64_t)m * N + n] = acc;
}

static uint16_t* alloc_fill(int64_t n, uint32_t seed, float scale = 1.0f) {
    uint16_t* p;
    CK(cudaMalloc(&p, n * 2));
    k_fill<<<1024, 256>>>(p, n, seed, scale);
    CK(cudaGetLastError());
    return p;
}

static float bf2f(uint16_t b) {
    uint32_t u = uint32_t(b) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

static int check_case(int M, int N, int K, bool amn, bool bmn, int epi) {
    const int64_t lda = amn ? (M + 7) / 8 * 8 + 8 : (K + 7) / 8 * 8 + 8;
    const int64_t ldb = bmn ? (N + 7) / 8 * 8 + 8 : (K + 7) / 8 * 8 + 8;
    const int64_t arows = amn ? K : M, brows = bmn ? K : N;
    uint16_t* A = alloc_fill(arows * lda, 17 + M, 1.0f);
    uint16_t* B = alloc_fill(brows * ldb, 91 + N, 1.0f);
    float* R;
    CK(cudaMalloc(&R, (int64_t)M * N * 4));
    k_ref<<<dim3((N + 127) / 128, M), 128>>>(M, N, K, A, lda, amn, B, ldb, bmn, R);
    CK(cudaGetLastError());
    const int64_t ldc = (N + 7) / 8 * 8;
    std::vector<float> ref((size_t)M * N);
    CK(cudaMemcpy(ref.data(), R, ref.size() * 4, cudaMemcpyDeviceToHost));

    GemmEpilogue e;
    e.kind = epi;
    e.ldc = ldc;
    void* C = nullptr;
    int32_t* rows = nullptr;
    uint16_t* mask = nullptr;
    const int64_t crow = (epi == EPI_ROWS_ADD_F32) ? 2 * M + 3 : M;
    const int64_t celt = (epi == EPI_STORE_F32 || epi == EPI_ROWS_ADD_F32) ? 4 : 2;
    CK(cudaMalloc(&C, crow * ldc * celt));
    CK(cudaMemset(C, 0, crow * ldc * celt));
    e.c = C;
    std::vector<int32_t> hrows(M);
    if (epi == EPI_ROWS_ADD_F32) {
        for (int i = 0; i < M; ++i) hrows[i] = 2 * i + 1;
        CK(cudaMalloc(&rows, M * 4));
        CK(cudaMemcpy(rows, hrows.data(), M * 4, cudaMemcpyHostToDevice));
        e.row_idx = rows;
    }
    if (epi == EPI_MASK_BF16) {
        mask = alloc_fill((int64_t)M * ldc, 5, 1.0f);  // random signs; we treat bits != 0 as "on"
        // zero out negatives so mask = relu-like
        std::vector<uint16_t> hm((size_t)M * ldc);
        CK(cudaMemcpy(hm.data(), mask, hm.size() * 2, cudaMemcpyDeviceToHost));
        for (auto& v : hm)
            if (v & 0x8000) v = 0;
        CK(cudaMemcpy(mask, hm.data(), hm.size() * 2, cudaMemcpyHostToDevice));
        e.mask = mask;
        e.ldm = ldc;
    }
    gemm_bf16(0, M, N, K, GemmOperand{A, lda, amn}, GemmOperand{B, ldb, bmn}, e);
    CK(cudaDeviceSynchronize());

    double max_err = 0, max_ref = 0;
    std::vector<uint8_t> hc(crow * ldc * celt);
    CK(cudaMemcpy(hc.data(), C, hc.size(), cudaMemcpyDeviceToHost));
    std::vector<uint16_t> hm;
    if (mask) {
        hm.resize((size_t)M * ldc);
        CK(cudaMemcpy(hm.data(), mask, hm.size() * 2, cudaMemcpyDeviceToHost));
    }
    int bad_relu = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double want = ref[(size_t)m * N + n], got = 0;
            if (epi == EPI_STORE_F32)
                got = reinterpret_cast<float*>(hc.data())[(size_t)m * ldc + n];
            else if (epi == EPI_ROWS_ADD_F32)
                got = reinterpret_cast<float*>(hc.data())[(size_t)hrows[m] * ldc + n];
            else if (epi == EPI_RELU_BF16) {
                got = bf2f(reinterpret_cast<uint16_t*>(hc.data())[(size_t)m * ldc + n]);
                if ((want > 0) != (got > 0) && std::fabs(want) > 1e-3) bad_relu++;
                want = want > 0 ? want : 0;
            } else {
                got = bf2f(reinterpret_cast<uint16_t*>(hc.data())[(size_t)m * ldc + n]);
                if (!hm[(size_t)m * ldc + n]) want = 0;
            }
            max_err = std::fmax(max_err, std::fabs(got - want));
            max_ref = std::fmax(max_ref, std::fabs(want));
        }
    const double rel = max_err / (max_ref > 0 ? max_ref : 1);
    const double tol = (epi == EPI_STORE_F32 || epi == EPI_ROWS_ADD_F32) ? 1e-4 : 1e-2;
    const bool ok = rel < tol && bad_relu == 0;
    std::printf("check M=%5d N=%5d K=%5d amn=%d bmn=%d epi=%d  max_rel_err=%.3e  %s\n", M, N, K, amn, bmn, epi, rel,
                ok ? "OK" : "FAIL");
    cudaFree(A);
    cudaFree(B);
    cudaFree(R);
    cudaFree(C);
    if (rows) cudaFree(rows);
    if (mask) cudaFree(mask);
    return ok ? 0 : 1;
}

static void perf_case(const char* name, int M, int N, int K, bool amn, bool bmn, int epi) {
    const int64_t lda = amn ? M : K, ldb = bmn ? N : K;
    uint16_t* A = alloc_fill((amn ? (int64_t)K : M) * lda, 3);
    uint16_t* B = alloc_fill((bmn ? (int64_t)K : N) * ldb, 4);
    void* C;
    const int64_t celt = (epi == EPI_STORE_F32) ? 4 : 2;
    CK(cudaMalloc(&C, (int64_t)M * N * celt));
    uint16_t* mask = nullptr;
    GemmEpilogue e;
    e.kind = epi;
    e.c = C;
    e.ldc = N;
    if (epi == EPI_MASK_BF16) {
        mask = alloc_fill((int64_t)M * N, 9);
        e.mask = mask;
        e.ldm = N;
    }
    for (int i = 0; i < 2; ++i) gemm_bf16(0, M, N, K, GemmOperand{A, lda, amn}, GemmOperand{B, ldb, bmn}, e);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 5;
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) gemm_bf16(0, M, N, K, GemmOperand{A, lda, amn}, GemmOperand{B, ldb, bmn}, e);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    const double tf = 2.0 * M * N * (double)K / (ms * 1e-3) / 1e12;
    std::printf("perf %-28s M=%5d N=%6d K=%5d  %8.3f ms  %7.1f TFLOP/s\n", name, M, N, K, ms, tf);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    if (mask) cudaFree(mask);
}

// K split: partials of `ks` K-chunks written to C + s*stride, summed here and compared with the reference.
static int check_split(int M, int N, int K, int ks) {
    const int64_t lda = (K + 7) / 8 * 8 + 8, ldb = lda;
    uint16_t* A = alloc_fill(M * lda, 7 + M, 1.0f);
    uint16_t* B = alloc_fill(N * ldb, 3 + N, 1.0f);
    float* R;
    CK(cudaMalloc(&R, (int64_t)M * N * 4));
    k_ref<<<dim3((N + 127) / 128, M), 128>>>(M, N, K, A, lda, false, B, ldb, false, R);
    CK(cudaGetLastError());
    std::vector<float> ref((size_t)M * N);
    CK(cudaMemcpy(ref.data(), R, ref.size() * 4, cudaMemcpyDeviceToHost));
    const int64_t ldc = (N + 7) / 8 * 8, stride = (int64_t)M * ldc;
    float* C;
    CK(cudaMalloc(&C, ks * stride * 4));
    CK(cudaMemset(C, 0, ks * stride * 4));
    GemmEpilogue e;
    e.kind = EPI_STORE_F32;
    e.c = C;
    e.ldc = ldc;
    e.ksplit = ks;
    e.split_stride = stride;
    gemm_bf16(0, M, N, K, GemmOperand{A, lda, false}, GemmOperand{B, ldb, false}, e);
    CK(cudaDeviceSynchronize());
    std::vector<float> hc(ks * stride);
    CK(cudaMemcpy(hc.data(), C, hc.size() * 4, cudaMemcpyDeviceToHost));
    double max_err = 0, max_ref = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double got = 0;
            for (int s = 0; s < ks; ++s) got += hc[s * stride + (size_t)m * ldc + n];
            max_err = std::fmax(max_err, std::fabs(got - ref[(size_t)m * N + n]));
            max_ref = std::fmax(max_ref, std::fabs(ref[(size_t)m * N + n]));
        }
    const double rel = max_err / (max_ref > 0 ? max_ref : 1);
    const bool ok = rel < 1e-4;
    std::printf("split M=%5d N=%5d K=%5d ks=%d  max_rel_err=%.3e  %s\n", M, N, K, ks, rel, ok ? "OK" : "FAIL");
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    cudaFree(R);
    return ok ? 0 : 1;
}

// Gathered B (TMA tile::gather4): logical row p of B = table row idx[p]; compared with a materialised gather.
static int check_gather(int M, int N, int K, bool bmn, int table_rows) {
    const int64_t lda = (K + 7) / 8 * 8 + 8;
    const int cols = bmn ? N : K, nidx = bmn ? K : N;
    const int64_t ldt = (cols + 7) / 8 * 8 + 8;
    uint16_t* A = alloc_fill((int64_t)M * lda, 11 + M, 1.0f);
    uint16_t* tab = alloc_fill((int64_t)table_rows * ldt, 29 + N, 1.0f);
    std::vector<int32_t> idx(nidx);
    uint32_t x = 12345;
    for (int p = 0; p < nidx; ++p) {  // ascending with random gaps, like a union
        x = x * 1664525u + 1013904223u;
        idx[p] = (p == 0 ? 0 : idx[p - 1] + 1) + int((x >> 24) % 3);
    }
    if (idx[nidx - 1] >= table_rows) { std::printf("gather: table too small\n"); return 1; }
    int32_t* didx;
    CK(cudaMalloc(&didx, nidx * 4));
    CK(cudaMemcpy(didx, idx.data(), nidx * 4, cudaMemcpyHostToDevice));
    // materialise logical B
    std::vector<uint16_t> ht((size_t)table_rows * ldt), hb((size_t)nidx * ldt);
    CK(cudaMemcpy(ht.data(), tab, ht.size() * 2, cudaMemcpyDeviceToHost));
    for (int p = 0; p < nidx; ++p) std::memcpy(&hb[(size_t)p * ldt], &ht[(size_t)idx[p] * ldt], ldt * 2);
    uint16_t* Bm;
    CK(cudaMalloc(&Bm, hb.size() * 2));
    CK(cudaMemcpy(Bm, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
    float* R;
    CK(cudaMalloc(&R, (int64_t)M * N * 4));
    k_ref<<<dim3((N + 127) / 128, M), 128>>>(M, N, K, A, lda, false, Bm, ldt, bmn, R);
    CK(cudaGetLastError());
    std::vector<float> ref((size_t)M * N), got((size_t)M * N);
    CK(cudaMemcpy(ref.data(), R, ref.size() * 4, cudaMemcpyDeviceToHost));
    float* C;
    CK(cudaMalloc(&C, (int64_t)M * N * 4));
    GemmEpilogue e;
    e.kind = EPI_STORE_F32;
    e.c = C;
    e.ldc = N;
    GemmOperand b{tab, ldt, bmn};
    b.rows = didx;
    b.table_rows = table_rows;
    CK(cudaMalloc(&b.run_ws, (K / 64 + 2) * 4));
    gemm_bf16(0, M, N, K, GemmOperand{A, lda, false}, b, e);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(got.data(), C, got.size() * 4, cudaMemcpyDeviceToHost));
    double max_err = 0, max_ref = 0;
    for (size_t i = 0; i < got.size(); ++i) {
        max_err = std::fmax(max_err, std::fabs(double(got[i]) - ref[i]));
        max_ref = std::fmax(max_ref, std::fabs(double(ref[i])));
    }
    const double rel = max_err / (max_ref > 0 ? max_ref : 1);
    const bool ok = rel < 1e-4;
    std::printf("gather M=%5d N=%5d K=%5d bmn=%d table=%d  max_rel_err=%.3e  %s\n", M, N, K, bmn, table_rows, rel,
                ok ? "OK" : "FAIL");
    cudaFree(A);
    cudaFree(tab);
    cudaFree(didx);
    cudaFree(Bm);
    cudaFree(R);
    cudaFree(C);
    return ok ? 0 : 1;
}

static void perf_gather(const char* name, int M, int N, int K, bool bmn, int epi, bool hole = true) {
    const int cols = bmn ? N : K, nidx = bmn ? K : N, table = nidx + 1;
    uint16_t* A = alloc_fill((int64_t)M * K, 3);
    uint16_t* tab = alloc_fill((int64_t)table * cols, 4);
    std::vector<int32_t> idx(nidx);
    for (int p = 0; p < nidx; ++p) idx[p] = p + (hole && p >= nidx / 2);  // the union minus one row
    int32_t* didx;
    CK(cudaMalloc(&didx, nidx * 4));
    CK(cudaMemcpy(didx, idx.data(), nidx * 4, cudaMemcpyHostToDevice));
    void* C;
    CK(cudaMalloc(&C, (int64_t)M * N * 4));
    GemmEpilogue e;
    e.kind = epi;
    e.c = C;
    e.ldc = N;
    GemmOperand b{tab, cols, bmn};
    b.rows = didx;
    b.table_rows = table;
    CK(cudaMalloc(&b.run_ws, (K / 64 + 2) * 4));
    for (int i = 0; i < 2; ++i) gemm_bf16(0, M, N, K, GemmOperand{A, K, false}, b, e);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    const int reps = 5;
    cudaEventRecord(t0);
    for (int i = 0; i < reps; ++i) gemm_bf16(0, M, N, K, GemmOperand{A, K, false}, b, e);
    cudaEventRecord(t1);
    CK(cudaEventSynchronize(t1));
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    ms /= reps;
    std::printf("perf %-28s M=%5d N=%6d K=%5d  %8.3f ms  %7.1f TFLOP/s\n", name, M, N, K, ms,
                2.0 * M * N * K / (ms * 1e-3) / 1e12);
    cudaFree(A);
    cudaFree(tab);
    cudaFree(didx);
    cudaFree(C);
}

int main(int argc, char** argv) {
    const bool perf = argc > 1 && std::strcmp(argv[1], "perf") == 0;
    if (argc > 1 && std::strcmp(argv[1], "perf4") == 0) {  // cfg4-like: |S| = 640k of M = 1M neurons
        const int T = 8192, S = 655360, D = 4096;
        perf_case("z=h.keys^T relu (K,K)", T, S, D, false, false, EPI_RELU_BF16);
        perf_case("out=act.values (K,MN)", T, D, S, false, true, EPI_STORE_F32);
        perf_case("gW=act^T.g (MN,MN)", S, D, T, true, true, EPI_STORE_F32);
        return 0;
    }
    if (argc > 1 && std::strcmp(argv[1], "perfmaj") == 0) {  // the out / grad_h shape with every operand major
        const int T = 8192, S = 65536, D = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            perf_case("out-shape (K,K)", T, D, S, false, false, EPI_STORE_F32);
            perf_case("out-shape (K,MN)", T, D, S, false, true, EPI_STORE_F32);
            perf_case("out-shape (MN,K)", T, D, S, true, false, EPI_STORE_F32);
            perf_case("out-shape (MN,MN)", T, D, S, true, true, EPI_STORE_F32);
            perf_case("z-shape (K,K)", T, S, D, false, false, EPI_STORE_F32);
            perf_case("gW-shape (MN,MN)", S, D, T, true, true, EPI_STORE_F32);
            perf_case("gW-shape (K,K)", S, D, T, false, false, EPI_STORE_F32);
        }
        return 0;
    }
    if (argc > 1 && std::strcmp(argv[1], "perfg") == 0) {
        const int T = 8192, S = 65536, D = 4096;
        perf_case("z dense", T, S, D, false, false, EPI_RELU_BF16);
        perf_gather("z gathered, no hole", T, S, D, false, EPI_RELU_BF16, false);
        perf_gather("z gathered, one hole", T, S, D, false, EPI_RELU_BF16, true);
        perf_case("z dense", T, S, D, false, false, EPI_RELU_BF16);
        perf_case("out dense", T, D, S, false, true, EPI_STORE_F32);
        perf_gather("out gathered, no hole", T, D, S, true, EPI_STORE_F32, false);
        perf_gather("out gathered, one hole", T, D, S, true, EPI_STORE_F32, true);
        perf_case("out dense", T, D, S, false, true, EPI_STORE_F32);
        return 0;
    }
    int fails = 0;
    if (!perf) {
        const int shapes[][3] = {{128, 256, 64}, {256, 512, 256}, {200, 300, 130}, {1000, 700, 520}, {64, 48, 40}};
        const bool majors[][2] = {{false, false}, {false, true}, {true, true}, {true, false}};
        for (auto& s : shapes)
            for (auto& mj : majors) fails += check_case(s[0], s[1], s[2], mj[0], mj[1], EPI_STORE_F32);
        for (int epi : {EPI_RELU_BF16, EPI_MASK_BF16, EPI_ROWS_ADD_F32}) {
            fails += check_case(384, 512, 256, false, false, epi);
            fails += check_case(300, 260, 200, true, true, epi);
        }
        // shapes large enough for the CTA-pair (256x256) kernel, incl. ragged M/N/K edges
        const int pshapes[][3] = {{2304, 2304, 320}, {2200, 2500, 200}, {4096, 2048, 1024}};
        for (auto& s : pshapes)
            for (auto& mj : majors) fails += check_case(s[0], s[1], s[2], mj[0], mj[1], EPI_STORE_F32);
        for (int epi : {EPI_RELU_BF16, EPI_MASK_BF16, EPI_ROWS_ADD_F32}) {
            fails += check_case(2304, 2304, 256, false, false, epi);
            fails += check_case(2200, 2500, 130, true, true, epi);
        }
        for (bool bmn : {false, true}) {
            fails += check_gather(300, 260, 200, bmn, 1200);    // 1-CTA, ragged
            fails += check_gather(2304, 2304, 320, bmn, 9000);  // CTA pair
            fails += check_gather(2200, 2500, 136, bmn, 9000);  // CTA pair, ragged
        }
        fails += check_split(300, 260, 1024, 8);
        fails += check_split(512, 256, 4096, 8);
        fails += check_split(200, 300, 650, 3);
        std::printf("gemm_check: %d failures\n", fails);
        return fails ? 1 : 0;
    }
    const int T = 8192, S = 65536, D = 4096;
    perf_case("z=h.keys^T relu (K,K)", T, S, D, false, false, EPI_RELU_BF16);
    perf_case("out=act.values (K,MN)", T, D, S, false, true, EPI_STORE_F32);
    perf_case("dA=g.values^T mask (K,K)", T, S, D, false, false, EPI_MASK_BF16);
    perf_case("gW=act^T.g (MN,MN)", S, D, T, true, true, EPI_STORE_F32);
    perf_gather("z gathered keys (K,K)", T, S, D, false, EPI_RELU_BF16);
    perf_gather("out gathered values (K,MN)", T, D, S, true, EPI_STORE_F32);
    return 0;
}
