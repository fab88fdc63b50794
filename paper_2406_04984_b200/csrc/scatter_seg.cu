// scatter_grads with repeated neuron ids (memtier.cpp:128-155): an atomic-free segmented scatter-add. The entry
// positions are sorted by neuron id (stable radix sort, so equal ids keep their position order); each run of equal
// ids is one segment, and one CTA per segment adds its gradient rows into the staging row in position order:
// stage = fl(...fl(fl(stage + g_j1) + g_j2)...), exactly the reference's sequential loop, with no atomics and every
// segment in parallel. (Strictly ascending index lists -- every call the trainer makes -- take the one-CTA-per-row
// kernel in stream_ops.cu directly.)
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include "common.cuh"
#include "stream_ops.h"

namespace meft_dev {
namespace {

template <typename G, typename S>
__global__ void __launch_bounds__(256) k_stage_segments(S* __restrict__ stage, int64_t d,
                                                        const int32_t* __restrict__ ids,   // sorted ids
                                                        const int32_t* __restrict__ pos,   // their positions
                                                        const int32_t* __restrict__ seg_off,  // exclusive offsets
                                                        const int32_t* __restrict__ n_seg, const G* __restrict__ g,
                                                        uint8_t* __restrict__ staged) {
    const int ns = *n_seg;
    for (int sgi = blockIdx.x; sgi < ns; sgi += gridDim.x) {
        const int b = seg_off[sgi], e = seg_off[sgi + 1];
        const int64_t row = ids[b];
        S* srow = stage + row * d;
        for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
            S acc = srow[c];
            for (int k = b; k < e; ++k) acc += S(g[int64_t(pos[k]) * d + c]);
            srow[c] = acc;
        }
        if (staged && threadIdx.x == 0) staged[row] = 1;
    }
}

__global__ void k_iota(int32_t* __restrict__ p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// seg_off[i] = exclusive scan of the run lengths (n_seg runs), seg_off[n_seg] = n
__global__ void __launch_bounds__(1024) k_run_offsets(const int32_t* __restrict__ len, const int32_t* __restrict__ n_seg,
                                                      int32_t* __restrict__ off) {
    __shared__ int s_base;
    const int ns = *n_seg;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (int c0 = 0; c0 < ns; c0 += blockDim.x) {  // chunked block scan, chunks in order
        const int i = c0 + threadIdx.x;
        int v = i < ns ? len[i] : 0;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        __shared__ int ws[32];
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) ws[w] = x;
        __syncthreads();
        if (w == 0) {
            int t = ws[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        const int excl = x - v + (w > 0 ? ws[w - 1] : 0) + s_base;
        if (i < ns) off[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_base = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) off[ns] = s_base;
}

template <typename G, typename S>
void run_segments(cudaStream_t st, S* stage, int64_t d, const int32_t* ids, const int32_t* pos, const int32_t* off,
                  const int32_t* n_seg, int64_t n, const void* g, uint8_t* staged) {
    const int grid = int(std::max<int64_t>(1, std::min<int64_t>(n, int64_t(num_sms()) * 8)));
    k_stage_segments<G, S><<<grid, 256, 0, st>>>(stage, d, ids, pos, off, n_seg, static_cast<const G*>(g), staged);
    check_launch("k_stage_segments");
}

}  // namespace

size_t stage_add_segmented_ws(int64_t n) {
    size_t sort_b = 0, rle_b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_b, static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr), static_cast<int32_t*>(nullptr), int(n));
    cub::DeviceRunLengthEncode::Encode(nullptr, rle_b, static_cast<const int32_t*>(nullptr),
                                       static_cast<int32_t*>(nullptr), static_cast<int32_t*>(nullptr),
                                       static_cast<int32_t*>(nullptr), int(n));
    const size_t slot = ((size_t(n + 1) * 4) + 255) & ~size_t(255);  // every carved buffer is 256-byte aligned
    return std::max(sort_b, rle_b) + 6 * slot + 256 + 256;
}

void stage_add_segmented(cudaStream_t st, int stage_dtype, void* stage, int64_t d, const int32_t* idx, int64_t n,
                         int g_dtype, const void* g, uint8_t* staged, void* ws, size_t ws_bytes) {
    if (n <= 0) return;
    if (ws_bytes < stage_add_segmented_ws(n)) throw MeftError(6, "stage_add_segmented: workspace too small");
    auto align = [](size_t b) { return (b + 255) & ~size_t(255); };
    uint8_t* p = static_cast<uint8_t*>(ws);
    int32_t* iota = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n) * 4);
    int32_t* ids = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n) * 4);
    int32_t* pos = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n) * 4);
    int32_t* uniq = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n) * 4);
    int32_t* len = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n) * 4);
    int32_t* off = reinterpret_cast<int32_t*>(p);
    p += align(size_t(n + 1) * 4);
    int32_t* n_seg = reinterpret_cast<int32_t*>(p);
    p += 256;
    void* tmp = p;
    size_t tmp_b = ws_bytes - size_t(p - static_cast<uint8_t*>(ws));
    k_iota<<<int((n + 255) / 256), 256, 0, st>>>(iota, int(n));
    check_launch("k_iota");
    // stable LSD radix sort of (id, position): equal ids keep ascending positions
    MEFT_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp, tmp_b, idx, ids, iota, pos, int(n), 0, 32, st));
    tmp_b = ws_bytes - size_t(p - static_cast<uint8_t*>(ws));
    MEFT_CUDA_CHECK(cub::DeviceRunLengthEncode::Encode(tmp, tmp_b, ids, uniq, len, n_seg, int(n), st));
    k_run_offsets<<<1, 1024, 0, st>>>(len, n_seg, off);
    check_launch("k_run_offsets");
    if (stage_dtype == 0 && g_dtype == 0)
        run_segments<double, double>(st, static_cast<double*>(stage), d, ids, pos, off, n_seg, n, g, staged);
    else if (stage_dtype == 1 && g_dtype == 1)
        run_segments<float, float>(st, static_cast<float*>(stage), d, ids, pos, off, n_seg, n, g, staged);
    else if (stage_dtype == 1 && g_dtype == 0)
        run_segments<double, float>(st, static_cast<float*>(stage), d, ids, pos, off, n_seg, n, g, staged);
    else
        run_segments<float, double>(st, static_cast<double*>(stage), d, ids, pos, off, n_seg, n, g, staged);
}

}  // namespace meft_dev
