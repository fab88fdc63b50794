// Developer probe (not part of the product): semantics of TMA tile::gather4 on sm_100a -- which tensor-map box
// it needs, how the 4 gathered rows land in shared memory under 128B swizzle, and what an out-of-range row
// index yields. Built by tools/Makefile; prints one line per experiment.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

__global__ void k_probe(const __grid_constant__ CUtensorMap m, int r0, int r1, int r2, int r3, int col, int bytes,
                        uint16_t* out) {
    __shared__ __align__(1024) uint16_t buf[2048];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(buf), b = (uint32_t)__cvta_generic_to_shared(&bar);
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = 0xDEAD;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d),
            "l"(&m), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
        uint32_t done = 0;
        for (int it = 0; it < 1000000 && !done; ++it)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(b)
                : "memory");
        out[2048] = done;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int R = 64, C = 128;
    std::vector<uint16_t> h(R * C);
    for (int r = 0; r < R; ++r)
        for (int c = 0; c < C; ++c) h[r * C + c] = uint16_t(r * 256 + c);  // row in the high byte, column low
    uint16_t *dt, *dout;
    CK(cudaMalloc(&dt, h.size() * 2));
    CK(cudaMalloc(&dout, 2049 * 2));
    CK(cudaMemcpy(dt, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
    for (int boxh : {1, 4}) {
        for (int sw : {0, 1}) {
            CUtensorMap m;
            const cuuint64_t dims[2] = {cuuint64_t(C), cuuint64_t(R)}, strides[1] = {cuuint64_t(C * 2)};
            const cuuint32_t box[2] = {64, cuuint32_t(boxh)}, es[2] = {1, 1};
            CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, dt, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE,
                             sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                std::printf("boxh=%d sw128=%d: encode failed (%d)\n", boxh, sw, int(r));
                continue;
            }
            for (int oob : {0, 1}) {
                const int rows[4] = {5, 17, oob ? 70 : 2, 40};
                k_probe<<<1, 128>>>(m, rows[0], rows[1], rows[2], rows[3], 64, 512, dout);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    std::printf("boxh=%d sw128=%d oob=%d: launch error %s\n", boxh, sw, oob, cudaGetErrorString(e));
                    return 1;
                }
                std::vector<uint16_t> o(2049);
                CK(cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost));
                std::printf("boxh=%d sw128=%d oob=%d done=%d  first elem of each 16B chunk (row:col) for 4 smem rows:\n",
                            boxh, sw, oob, int(o[2048]));
                for (int sr = 0; sr < 5; ++sr) {
                    std::printf("   smem row %d:", sr);
                    for (int ch = 0; ch < 8; ++ch) {
                        const uint16_t v = o[sr * 64 + ch * 8];
                        if (v == 0xDEAD) std::printf("  ----");
                        else std::printf("  %2d:%-3d", v >> 8, v & 255);
                    }
                    std::printf("\n");
                }
            }
        }
    }
    return 0;
}
