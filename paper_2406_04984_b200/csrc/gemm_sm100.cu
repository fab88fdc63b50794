// bf16 x bf16 -> fp32 GEMM on the 5th-generation tensor cores (sm_100a).
//
// Persistent, warp-specialised kernel, one CTA per SM:
//   warp 0   : TMA producer (cp.async.bulk.tensor, 128B swizzle) into a STAGES-deep smem ring
//   warp 1   : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=256, K=16 per instruction)
//   warps 2-5: epilogue — tcgen05.ld from a double-buffered TMEM accumulator, fused elementwise op,
//              vectorised stores. Double buffering lets tile i's epilogue overlap tile i+1's MMAs.
// Both operands may be K-major or MN-major (UMMA descriptor major bits), so the six FFN GEMMs of the
// MEFT layer read their operands in place with no transposes.
#include <cudaTypedefs.h>

#include <atomic>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace meft_dev {
namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
#ifndef MEFT_STAGES  // 1-CTA kernel ring depth (A/B knob)
#define MEFT_STAGES 4
#endif
constexpr int STAGES = MEFT_STAGES;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int TMEM_COLS = 512;  // 2 accumulators x 256 fp32 columns
constexpr int GROUP_M = 16;     // raster: 16 M-tiles share each resident B panel in L2
// grouped mode: the group offset tables (tile and row offsets, G + 1 each) are staged in shared memory
constexpr int MAX_SMEM_GROUPS = 2048;
constexpr int GROUP_TABLE_BYTES = 2 * (MAX_SMEM_GROUPS + 1) * 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256 + GROUP_TABLE_BYTES;

struct KArgs {
    int M, N, K;
    int tiles_m, tiles_n, num_kb;
    int epi;
    int accumulate;
    void* c;
    long long ldc;
    const uint16_t* mask;
    long long ldm;
    uint32_t* bits;
    long long ldbits;
    const int32_t* row_idx;
    // grouped mode: G groups; group g owns A rows [g_row_off[g], g_row_off[g+1]) and B rows
    // [g*g_brows, (g+1)*g_brows); g_tile_off = exclusive scan of its BM-tiles (device arrays).
    int grouped;
    int G, g_ntiles, g_brows;
    const int32_t* g_row_off;
    const int32_t* g_tile_off;
    // pair-kernel raster: m-tiles per group (tiles_m = sweep all of M first); n_fast = sweep N first
    int raster_group, raster_n_fast;
    // K split: tile index = split * base_tiles + base tile; split s runs k-blocks [s*kb_split, (s+1)*kb_split)
    int ksplit, kb_split;
    long long split_stride;
    // gathered B: logical B row p < b_idx_n is table row b_idx[p]; rows past it read as zeros (OOB index)
    const int32_t* b_idx;
    int b_idx_n, b_oob_row;
    const int32_t* kb_run;  // MN-major gathered B: per k-block first table row of a contiguous run, or -1
    // EPI_ACT_BF16 / EPI_DACT_BF16
    uint16_t* aux;
    long long ldaux;
    int act;
    // EPI_PEER_F32 (see kernels.h)
    float* peer[kMaxPeers];
    long long peer_rows, row0, col0;
    int peer_slot;
    // EPI_ADAM_F32 (see kernels.h)
    float* adam_w;
    void* adam_m;  // fp32, or bf16 when mom16
    void* adam_v;
    int mom16;
    uint16_t* adam_c;
    const float2* adam_coef;
    float b1, b2, eps;
    double* stat_ss;
    int32_t* stat_lsb;
    long long stat_ld;
    // L2 eviction priority of the A / B TMA loads (GemmOperand::l2_hint)
    int hint_a, hint_b;
    // device-sized extent (GemmEpilogue::extent): the launch is sized for the static M / N / K (a capacity); the
    // kernel reads the real size of dimension extent_dim (1 = M, 2 = N, 3 = K) from *extent before its first tile
    const int32_t* extent;
    int extent_dim, extent_tile_m;
    int b_gather_k;  // gathered B rows index K (MN-major B) rather than N
};

// Shrink the capacity-sized problem to the device-resident extent (every thread, before any tile is resolved).
// N: tiles past the extent do not run, and the output columns up to the next multiple of 64 are stored -- exact
// zeros, because B's rows there read as zeros (a gathered B: out-of-bounds rows; a materialised B: the caller pads
// it, gather_rows2 pad64), so a K-extent consumer of this output reads zeros there just as TMA's out-of-bounds
// fill gives a host-sized launch. K: k-blocks past the extent are not issued. M: tiles past it do not run.
__device__ __forceinline__ void apply_extent(KArgs& a) {
    if (a.extent_dim == 0) return;
    const int v = max(0, __ldg(a.extent));
    if (a.extent_dim == 1) {
        a.M = min(v, a.M);
        a.tiles_m = (a.M + a.extent_tile_m - 1) / a.extent_tile_m;
    } else if (a.extent_dim == 2) {
        const int n = min(v, a.N);
        a.tiles_n = (n + BN - 1) / BN;
        if (a.b_idx && !a.b_gather_k) a.b_idx_n = n;
        a.N = min((n + 63) & ~63, a.N);
    } else {
        a.K = min(v, a.K);
        a.num_kb = (a.K + BK - 1) / BK;
        a.kb_split = a.num_kb;
        if (a.b_idx && a.b_gather_k) a.b_idx_n = a.K;
    }
}

__device__ __forceinline__ int gather_row(const KArgs& a, int p) {
    return p < a.b_idx_n ? __ldg(a.b_idx + p) : a.b_oob_row;
}

// Gathered-B indices in the producer warp. A piece of B rows whose table rows form one contiguous run (the
// common case for a dense union) is loaded as ONE plain 2-D box at the run's first table row; only broken
// pieces fall back to tile::gather4 (~4x more TMA issue per stage). Indices are fetched with one coalesced warp
// load per piece, one piece ahead, so the producer never waits on them.
// MN-major B (gathered along K): the 64 k-rows of a k-block, lane l holds rows 2l and 2l+1.
struct KRows {
    int v0, v1;
};
__device__ __forceinline__ KRows load_krows(const KArgs& a, int k0, int lane) {
    return KRows{gather_row(a, k0 + 2 * lane), gather_row(a, k0 + 2 * lane + 1)};
}
__device__ __forceinline__ void krows_four(const KRows& x, int r, int& i0, int& i1, int& i2, int& i3) {
    const int l = r >> 1;  // rows r..r+3 (r % 4 == 0) live in lanes r/2 and r/2 + 1
    i0 = __shfl_sync(0xffffffffu, x.v0, l);
    i1 = __shfl_sync(0xffffffffu, x.v1, l);
    i2 = __shfl_sync(0xffffffffu, x.v0, l + 1);
    i3 = __shfl_sync(0xffffffffu, x.v1, l + 1);
}
// Per-k-block run table (identical for every tile): k_kb_runs builds it before the GEMM; the producer reads it
// 32 k-blocks per warp load, one aligned batch ahead, so the latency of the read never reaches the TMA issue.
struct RunBatch {
    int cur = 0, cur_base = -1 << 30, nxt = 0, nxt_base = -1 << 30;
    __device__ __forceinline__ int fetch(const KArgs& a, int base, int lane) const {
        const int kb = base + lane;
        return (kb >= 0 && kb < a.num_kb) ? __ldg(a.kb_run + kb) : -1;
    }
    // run of k-block kb (warp-uniform); next_start = first k-block of the following tile (prefetch target)
    __device__ __forceinline__ int get(const KArgs& a, int kb, int kb_end, int next_start, int lane) {
        if (kb < cur_base || kb >= cur_base + 32) {
            const int base = kb & ~31;
            if (base == nxt_base) {
                cur = nxt;
            } else {
                cur = fetch(a, base, lane);
            }
            cur_base = base;
            const int nb = (base + 32 < kb_end) ? base + 32 : (next_start & ~31);
            nxt = fetch(a, nb, lane);
            nxt_base = nb;
        }
        return __shfl_sync(0xffffffffu, cur, kb - cur_base);
    }
};

__global__ void k_kb_runs(const int32_t* __restrict__ idx, int n, int num_kb, int32_t* __restrict__ out,
                          const int32_t* __restrict__ n_dev) {
    const int kb = blockIdx.x * blockDim.x + threadIdx.x;
    if (kb >= num_kb) return;
    if (n_dev) n = min(n, max(0, *n_dev));
    const int p = kb * BK;
    out[kb] = (p + BK <= n && idx[p + BK - 1] - idx[p] == BK - 1) ? idx[p] : -1;
}

// K-major B (gathered along N): the tile's R = 32 * 4 * H rows, lane l holds rows h*128 + 4l + j.
template <int H>
__device__ __forceinline__ void load_nrows(const KArgs& a, int n0, int lane, int (&g)[4 * H]) {
#pragma unroll
    for (int j = 0; j < 4 * H; ++j) g[j] = gather_row(a, n0 + (j >> 2) * 128 + 4 * lane + (j & 3));
}
template <int H>
__device__ __forceinline__ int nrows_run(const KArgs& a, const int (&g)[4 * H], int n0) {  // warp-uniform
    const int first = __shfl_sync(0xffffffffu, g[0], 0), last = __shfl_sync(0xffffffffu, g[4 * H - 1], 31);
    return (n0 + 128 * H <= a.b_idx_n && last - first == 128 * H - 1) ? first : -1;
}

__device__ __forceinline__ int base_tile_count(const KArgs& a) {
    return a.grouped ? a.g_tile_off[a.G] * a.g_ntiles : a.tiles_m * a.tiles_n;
}

struct TileInfo {
    int a_row0;  // first A row (global)
    int b_row0;  // first B row (global)
    int m_lim;   // A rows >= m_lim are not part of this tile's problem
    int n_col0;  // output column of the tile's first B row
};

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& m_blk, int& n_blk);

// s_toff / s_roff: the group tables in shared memory (grouped mode; nullptr = read them from global memory).
__device__ __forceinline__ TileInfo resolve_tile(const KArgs& a, int tile, const int* s_toff = nullptr,
                                                 const int* s_roff = nullptr) {
    TileInfo t;
    if (!a.grouped) {
        int mb, nb;
        tile_coords(tile, a.tiles_m, a.tiles_n, mb, nb);
        t.a_row0 = mb * BM;
        t.b_row0 = nb * BN;
        t.m_lim = a.M;
        t.n_col0 = t.b_row0;
    } else {
        const int mt_global = tile / a.g_ntiles, nt = tile - mt_global * a.g_ntiles;
        const int* toff = s_toff ? s_toff : a.g_tile_off;
        const int* roff = s_roff ? s_roff : a.g_row_off;
        int lo = 0, hi = a.G;  // last g with g_tile_off[g] <= mt_global (a dependent chain: keep it on-chip)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (toff[mid] <= mt_global) lo = mid; else hi = mid;
        }
        t.a_row0 = roff[lo] + (mt_global - toff[lo]) * BM;
        t.m_lim = roff[lo + 1];
        t.n_col0 = nt * BN;
        t.b_row0 = lo * a.g_brows + t.n_col0;
    }
    return t;
}

__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int& m_blk, int& n_blk) {
    const int group_size = GROUP_M * tiles_n;
    const int g = tile / group_size;
    const int first_m = g * GROUP_M;
    const int gm = min(GROUP_M, tiles_m - first_m);
    const int local = tile - g * group_size;
    m_blk = first_m + local % gm;
    n_blk = local / gm;
}

__device__ __forceinline__ void epilogue_chunk(const KArgs& a, int m, int n, const uint32_t (&r)[32],
                                               long long c_off = 0) {
    const int cnt = min(32, a.N - n);
    switch (a.epi) {
        case EPI_STORE_F32:
        case EPI_ROWS_ADD_F32:
        case EPI_ROWS_STORE_F32:
        case EPI_PEER_F32: {
            const bool acc = a.accumulate || a.epi == EPI_ROWS_ADD_F32;
            float* c;
            if (a.epi == EPI_PEER_F32) {  // this row's home rank and the slot reserved for us in its buffer
                const long long g = a.row0 + m;
                const long long home = g / a.peer_rows;
                c = a.peer[home] + (a.peer_slot * a.peer_rows + (g - home * a.peer_rows)) * a.ldc + a.col0 + n;
            } else {
                const long long row = (a.epi != EPI_STORE_F32) ? (long long)a.row_idx[m] : (long long)m;
                c = reinterpret_cast<float*>(a.c) + c_off + row * a.ldc + n;
            }
            if (cnt == 32) {
                float4* c4 = reinterpret_cast<float4*>(c);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float4 v = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                           __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
                    if (acc) {
                        const float4 o = c4[j];
                        v.x += o.x;
                        v.y += o.y;
                        v.z += o.z;
                        v.w += o.w;
                    }
                    c4[j] = v;
                }
            } else {
                for (int j = 0; j < cnt; ++j) c[j] = (acc ? c[j] : 0.0f) + __uint_as_float(r[j]);
            }
            break;
        }
        case EPI_RELU_BF16: {
            uint16_t* c = reinterpret_cast<uint16_t*>(a.c) + (long long)m * a.ldc + n;
            if (a.bits) {
                uint32_t w = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) w |= (j < cnt && __uint_as_float(r[j]) > 0.0f) ? (1u << j) : 0u;
                a.bits[(long long)m * a.ldbits + (n >> 5)] = w;
            }
            if (cnt == 32) {
                uint4* c4 = reinterpret_cast<uint4*>(c);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    uint4 v;
                    v.x = pack_bf16x2(relu_bf16_bits(__uint_as_float(r[8 * j + 0])),
                                      relu_bf16_bits(__uint_as_float(r[8 * j + 1])));
                    v.y = pack_bf16x2(relu_bf16_bits(__uint_as_float(r[8 * j + 2])),
                                      relu_bf16_bits(__uint_as_float(r[8 * j + 3])));
                    v.z = pack_bf16x2(relu_bf16_bits(__uint_as_float(r[8 * j + 4])),
                                      relu_bf16_bits(__uint_as_float(r[8 * j + 5])));
                    v.w = pack_bf16x2(relu_bf16_bits(__uint_as_float(r[8 * j + 6])),
                                      relu_bf16_bits(__uint_as_float(r[8 * j + 7])));
                    c4[j] = v;
                }
            } else {
                for (int j = 0; j < cnt; ++j) c[j] = relu_bf16_bits(__uint_as_float(r[j]));
            }
            break;
        }
        case EPI_MASK_BF16: {
            uint16_t* c = reinterpret_cast<uint16_t*>(a.c) + (long long)m * a.ldc + n;
            if (a.bits) {  // bitmask of act > 0 (written by the z GEMM's EPI_RELU_BF16)
                const uint32_t w = a.bits[(long long)m * a.ldbits + (n >> 5)];
                if (cnt == 32) {
                    uint4* c4 = reinterpret_cast<uint4*>(c);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t o[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const int e = 8 * j + 2 * q;
                            const uint16_t lo = (w >> e) & 1u ? f32_to_bf16_bits(__uint_as_float(r[e])) : 0;
                            const uint16_t hi = (w >> (e + 1)) & 1u ? f32_to_bf16_bits(__uint_as_float(r[e + 1])) : 0;
                            o[q] = pack_bf16x2(lo, hi);
                        }
                        c4[j] = make_uint4(o[0], o[1], o[2], o[3]);
                    }
                } else {
                    for (int j = 0; j < cnt; ++j) c[j] = (w >> j) & 1u ? f32_to_bf16_bits(__uint_as_float(r[j])) : 0;
                }
                break;
            }
            const uint16_t* mk = a.mask + (long long)m * a.ldm + n;
            if (cnt == 32) {
                uint4* c4 = reinterpret_cast<uint4*>(c);
                const uint4* m4 = reinterpret_cast<const uint4*>(mk);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 mm = m4[j];
                    const uint32_t mw[4] = {mm.x, mm.y, mm.z, mm.w};
                    uint32_t o[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint16_t lo = (mw[q] & 0xFFFFu) ? f32_to_bf16_bits(__uint_as_float(r[8 * j + 2 * q])) : 0;
                        const uint16_t hi = (mw[q] >> 16) ? f32_to_bf16_bits(__uint_as_float(r[8 * j + 2 * q + 1])) : 0;
                        o[q] = pack_bf16x2(lo, hi);
                    }
                    c4[j] = make_uint4(o[0], o[1], o[2], o[3]);
                }
            } else {
                for (int j = 0; j < cnt; ++j) c[j] = mk[j] ? f32_to_bf16_bits(__uint_as_float(r[j])) : 0;
            }
            break;
        }
        case EPI_ACT_BF16:
        case EPI_DACT_BF16: {  // frozen base FFN: activation forward / its derivative times the incoming gradient
            uint16_t* c = reinterpret_cast<uint16_t*>(a.c) + (long long)m * a.ldc + n;
            uint16_t* x = a.aux + (long long)m * a.ldaux + n;
            auto act_f = [&](float p) { return a.act == 1 ? (p > 0.f ? p : 0.f) : p / (1.f + __expf(-p)); };
            auto dact_f = [&](float v, float p) {
                if (a.act == 1) return p > 0.f ? v : 0.f;
                const float sg = 1.f / (1.f + __expf(-p));
                return v * (sg * (1.f + p * (1.f - sg)));
            };
            const bool vec = cnt == 32 && ((reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(x)) % 16 == 0);
            if (vec) {  // 4 x 16-byte accesses of 8 bf16 per row chunk
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t cw[4], xw[4];
                    if (a.epi == EPI_DACT_BF16) {
                        const uint4 xv = reinterpret_cast<const uint4*>(x)[q];
                        xw[0] = xv.x, xw[1] = xv.y, xw[2] = xv.z, xw[3] = xv.w;
                    }
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const float v0 = __uint_as_float(r[8 * q + 2 * w]), v1 = __uint_as_float(r[8 * q + 2 * w + 1]);
                        if (a.epi == EPI_ACT_BF16) {
                            xw[w] = pack_bf16x2(f32_to_bf16_bits(v0), f32_to_bf16_bits(v1));
                            cw[w] = pack_bf16x2(f32_to_bf16_bits(act_f(v0)), f32_to_bf16_bits(act_f(v1)));
                        } else {
                            const float p0 = bf16_bits_to_f32(uint16_t(xw[w])), p1 = bf16_bits_to_f32(uint16_t(xw[w] >> 16));
                            cw[w] = pack_bf16x2(f32_to_bf16_bits(dact_f(v0, p0)), f32_to_bf16_bits(dact_f(v1, p1)));
                        }
                    }
                    reinterpret_cast<uint4*>(c)[q] = make_uint4(cw[0], cw[1], cw[2], cw[3]);
                    if (a.epi == EPI_ACT_BF16) reinterpret_cast<uint4*>(x)[q] = make_uint4(xw[0], xw[1], xw[2], xw[3]);
                }
            } else {
                for (int j = 0; j < cnt; ++j) {
                    const float v = __uint_as_float(r[j]);
                    if (a.epi == EPI_ACT_BF16) {
                        x[j] = f32_to_bf16_bits(v);
                        c[j] = f32_to_bf16_bits(act_f(v));
                    } else {
                        c[j] = f32_to_bf16_bits(dact_f(v, bf16_bits_to_f32(x[j])));
                    }
                }
            }
            break;
        }
        default:
            break;
    }
}

// ---------------------------------------------------------------- EPI_ADAM_F32: sparse Adam in the epilogue
// Four entries of one table row: the shared adam_update (bit-identical to k_adam_mixed), bf16 copy, statistics.
// Key statistics (sum of squares of the new bf16 row) as an fp32 UPPER bound: every bf16 square is exact in fp32
// and every addition rounds toward +inf, so the bound holds with no fp64 work in the epilogue (measured: the fp64
// form made the key-table GEMM 0.5 ms slower and doubled its operand re-reads).
using stat_t = float;
__device__ __forceinline__ float stat_sq_add(float x, float s) { return __fmaf_ru(x, x, s); }
__device__ __forceinline__ float stat_add(float a, float b) { return __fadd_ru(a, b); }

template <bool STATS>
__device__ __forceinline__ uint2 adam4(float4& w, float4& m, float4& v, const float4& g, const KArgs& a, AdamCoef k,
                                       stat_t& ss, int& lsb) {
    adam_update(w.x, m.x, v.x, g.x, a.b1, a.b2, a.eps, k);
    adam_update(w.y, m.y, v.y, g.y, a.b1, a.b2, a.eps, k);
    adam_update(w.z, m.z, v.z, g.z, a.b1, a.b2, a.eps, k);
    adam_update(w.w, m.w, v.w, g.w, a.b1, a.b2, a.eps, k);
    const uint16_t c[4] = {f32_to_bf16_bits(w.x), f32_to_bf16_bits(w.y), f32_to_bf16_bits(w.z), f32_to_bf16_bits(w.w)};
    if (STATS) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            ss = stat_sq_add(bf16_bits_to_f32(c[q]), ss);
            if (c[q] & 0x7FFF) lsb = min(lsb, bf16_lsb_exp(c[q]));
        }
    }
    return make_uint2(pack_bf16x2(c[0], c[1]), pack_bf16x2(c[2], c[3]));
}

// Pair kernel: the warp's 32 accumulator rows (one per lane, 32 columns per tcgen05.ld) are transposed through a
// 32 x 36 fp32 shared scratch so that 8 lanes cover one table row's 128 contiguous bytes: every w/m/v load and
// store is a full 128-byte segment. All 8 rows' loads of a chunk are issued before any update (24 x 16 B in flight
// per lane) to cover DRAM latency behind the mainloop of the next tile (an L2 prefetch one chunk ahead measured
// neutral).
__device__ __forceinline__ void st_shared_f4(uint32_t addr, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
#ifndef MEFT_ADAM_STREAMING
#define MEFT_ADAM_STREAMING 1
#endif
#if MEFT_ADAM_STREAMING  // the tables are touched once per step: evict-first loads and stores
#define ADAM_LD(p) __ldcs(p)
#define ADAM_ST(p, v) __stcs(p, v)
#else
#define ADAM_LD(p) (*(p))
#define ADAM_ST(p, v) (*(p) = (v))
#endif
// Adam moments of 4 consecutive entries at element offset `off`: fp32 tables, or bf16 ones (COMPACT stores; rounded
// to nearest even on store).
template <bool MOM16>
__device__ __forceinline__ float4 adam_ld_mom(const void* base, long long off) {
    if (MOM16) {
        const uint2 u = ADAM_LD(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(base) + off));
        return make_float4(bf16_bits_to_f32(uint16_t(u.x)), bf16_bits_to_f32(uint16_t(u.x >> 16)),
                           bf16_bits_to_f32(uint16_t(u.y)), bf16_bits_to_f32(uint16_t(u.y >> 16)));
    }
    return ADAM_LD(reinterpret_cast<const float4*>(static_cast<const float*>(base) + off));
}
template <bool MOM16>
__device__ __forceinline__ void adam_st_mom(void* base, long long off, float4 v) {
    if (MOM16) {
        ADAM_ST(reinterpret_cast<uint2*>(static_cast<uint16_t*>(base) + off),
                make_uint2(pack_bf16x2(f32_to_bf16_bits(v.x), f32_to_bf16_bits(v.y)),
                           pack_bf16x2(f32_to_bf16_bits(v.z), f32_to_bf16_bits(v.w))));
    } else {
        ADAM_ST(reinterpret_cast<float4*>(static_cast<float*>(base) + off), v);
    }
}
constexpr int ADAM_SCRATCH_LD = 36;  // floats per scratch row (16-byte aligned, conflict-free quarter-warp phases)
constexpr int ADAM_SCRATCH_BYTES = 4 * 32 * ADAM_SCRATCH_LD * 4;

// MEFT_ADAM_EXP_* (developer A/B builds only, tools/ab_variants.sh; results are NOT an Adam update):
//   NOTRAFFIC: no w/m/v loads or stores (constants in their place); NOMATH: no Adam arithmetic (the gradient passed
//   through); NOTRANSPOSE: no shared-memory transpose (the accumulator registers used in place); NOSTORE: nothing
//   written at all (the stores sit behind a condition that is never true at run time, so the tables -- and hence the
//   next step's union -- stay as they are while the code stays in the kernel).
#ifndef MEFT_ADAM_EXP_NOTRAFFIC
#define MEFT_ADAM_EXP_NOTRAFFIC 0
#endif
#ifndef MEFT_ADAM_EXP_NOMATH
#define MEFT_ADAM_EXP_NOMATH 0
#endif
#ifndef MEFT_ADAM_EXP_NOTRANSPOSE
#define MEFT_ADAM_EXP_NOTRANSPOSE 0
#endif
#ifndef MEFT_ADAM_EXP_NOSTORE
#define MEFT_ADAM_EXP_NOSTORE 0
#endif
template <bool STATS, bool MOM16>
__device__ __forceinline__ void adam_tile_transposed(const KArgs& a, uint32_t taddr, int m0, int n_col0, float* sw,
                                                     int lane) {
    const int mrow = m0 + lane;
    const int jl = mrow < a.M ? __ldg(a.row_idx + mrow) : -1;
    const float2 kl = mrow < a.M ? __ldg(a.adam_coef + mrow) : make_float2(0.f, 0.f);
    const int sub = lane >> 3, c4 = (lane & 7) * 4;
    int j[8];
    AdamCoef k[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const int row = it * 4 + sub;
        j[it] = __shfl_sync(0xffffffffu, jl, row);
        k[it] = AdamCoef{__shfl_sync(0xffffffffu, kl.x, row), __shfl_sync(0xffffffffu, kl.y, row)};
    }
    stat_t ss[8];
    int lsb[8];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        ss[it] = 0;
        lsb[it] = INT32_MAX;
    }
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
        const int n = n_col0 + c * 32;
        if (n >= a.N) break;  // warp-uniform (N % 32 == 0)
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        float4 w[8], m[8], v[8];
#pragma unroll
        for (int it = 0; it < 8; ++it) {  // invalid rows (past M: j < 0) read row 0 and never store
            const long long off = (long long)max(j[it], 0) * a.ldc + n + c4;
#if MEFT_ADAM_EXP_NOTRAFFIC
            w[it] = m[it] = v[it] = make_float4(1e-3f, 0.f, 0.f, 0.f);
            (void)off;
#else
            w[it] = ADAM_LD(reinterpret_cast<const float4*>(a.adam_w + off));
            m[it] = adam_ld_mom<MOM16>(a.adam_m, off);
            v[it] = adam_ld_mom<MOM16>(a.adam_v, off);
#endif
        }
        tmem_ld_wait();
        const uint32_t sbase = smem_u32(sw);
#if !MEFT_ADAM_EXP_NOTRANSPOSE
#pragma unroll
        for (int q = 0; q < 8; ++q)
            st_shared_f4(sbase + (lane * ADAM_SCRATCH_LD + 4 * q) * 4,
                         make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                     __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
        __syncwarp();
#endif
#pragma unroll
        for (int it = 0; it < 8; ++it) {
#if MEFT_ADAM_EXP_NOTRANSPOSE
            const float4 g = make_float4(__uint_as_float(r[4 * it]), __uint_as_float(r[4 * it + 1]),
                                         __uint_as_float(r[4 * it + 2]), __uint_as_float(r[4 * it + 3]));
#else
            const float4 g = ld_shared_f4(sbase + ((it * 4 + sub) * ADAM_SCRATCH_LD + c4) * 4);
#endif
#if MEFT_ADAM_EXP_NOMATH  // no Adam arithmetic: the gradient passed through
            w[it] = m[it] = v[it] = g;
            const uint2 cb = make_uint2(__float_as_uint(g.x), __float_as_uint(g.y));
#else
            const uint2 cb = adam4<STATS>(w[it], m[it], v[it], g, a, k[it], ss[it], lsb[it]);
#endif
            if (MEFT_ADAM_EXP_NOSTORE ? j[it] < -1 : j[it] >= 0) {
                const long long off = (long long)max(j[it], 0) * a.ldc + n + c4;
#if !MEFT_ADAM_EXP_NOTRAFFIC
                ADAM_ST(reinterpret_cast<float4*>(a.adam_w + off), w[it]);
                adam_st_mom<MOM16>(a.adam_m, off, m[it]);
                adam_st_mom<MOM16>(a.adam_v, off, v[it]);
#endif
                *reinterpret_cast<uint2*>(a.adam_c + off) = cb;
            }
        }
        __syncwarp();  // the scratch is rewritten by the next chunk
    }
    if (STATS) {  // the 8 lanes of each row reduce in a fixed butterfly; lane 8*sub writes the row's partial
        const int nb = n_col0 / kAdamStatTile;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
            stat_t t = ss[it];
            int l = lsb[it];
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                t = stat_add(t, __shfl_xor_sync(0xffffffffu, t, o));
                l = min(l, __shfl_xor_sync(0xffffffffu, l, o));
            }
            const int mr = m0 + it * 4 + sub;
            if ((lane & 7) == 0 && mr < a.M && (!MEFT_ADAM_EXP_NOSTORE || j[it] < -1)) {
                a.stat_ss[mr * a.stat_ld + nb] = t;
                a.stat_lsb[mr * a.stat_ld + nb] = l;
            }
        }
    }
}

// 1-CTA kernel (MEFT_GEMM_PAIR=0 only; the Adam GEMMs otherwise always run on CTA pairs): thread = accumulator row,
// same arithmetic without the transpose.
template <bool MOM16>
__device__ __forceinline__ void adam_tile_rows(const KArgs& a, uint32_t taddr, int m, int n_col0) {
    const bool ok = m < a.M;
    const int j = ok ? __ldg(a.row_idx + m) : 0;
    const float2 kl = ok ? __ldg(a.adam_coef + m) : make_float2(0.f, 0.f);
    const AdamCoef k{kl.x, kl.y};
    stat_t ss = 0;
    int lsb = INT32_MAX;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
        const int n = n_col0 + c * 32;
        if (n >= a.N) break;
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        if (!ok) continue;
        const long long off = (long long)j * a.ldc + n;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float4 w = reinterpret_cast<const float4*>(a.adam_w + off)[q];
            float4 mm = adam_ld_mom<MOM16>(a.adam_m, off + 4 * q);
            float4 v = adam_ld_mom<MOM16>(a.adam_v, off + 4 * q);
            const float4 g = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                         __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
            const uint2 cb = adam4<true>(w, mm, v, g, a, k, ss, lsb);
            reinterpret_cast<float4*>(a.adam_w + off)[q] = w;
            adam_st_mom<MOM16>(a.adam_m, off + 4 * q, mm);
            adam_st_mom<MOM16>(a.adam_v, off + 4 * q, v);
            reinterpret_cast<uint2*>(a.adam_c + off)[q] = cb;
        }
    }
    if (a.stat_ss && ok) {
        const int nb = n_col0 / kAdamStatTile;
        a.stat_ss[m * a.stat_ld + nb] = ss;
        a.stat_lsb[m * a.stat_ld + nb] = lsb;
    }
}

template <bool A_MN, bool B_MN>
__device__ __forceinline__ void gemm_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmG,
                                          const KArgs& args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* s_toff = reinterpret_cast<int*>(smem + STAGES * STAGE_BYTES + 256);
    int* s_roff = s_toff + (MAX_SMEM_GROUPS + 1);
    const bool tables = args.grouped && args.G <= MAX_SMEM_GROUPS;
    if (tables) {
        for (int i = threadIdx.x; i <= args.G; i += blockDim.x) {
            s_toff[i] = args.g_tile_off[i];
            s_roff[i] = args.g_row_off[i];
        }
    } else {
        s_toff = s_roff = nullptr;
    }

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + b, 1);
            mbar_init(tempty + b, 4);  // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmG);
    }
    if (warp == 1) tmem_alloc(tmem_slot, TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int base_tiles = base_tile_count(args);
    const int num_tiles = base_tiles * args.ksplit;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (lane 0; all lanes for gathered B rows)
        const bool gather = args.b_idx != nullptr;
        const uint64_t pol_a = l2_policy(args.hint_a), pol_b = l2_policy(args.hint_b);
        int stage = 0;
        uint32_t phase = 0;
        int gn[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // K-major gathered B: the NEXT tile's rows (prefetched)
        RunBatch rb;                            // MN-major gathered B: k-block run table reader
        auto tile_n0 = [&](int t) {
            const int sp_ = t / base_tiles;
            return resolve_tile(args, t - sp_ * base_tiles, s_toff, s_roff).b_row0;
        };
        if (gather && !B_MN && blockIdx.x < num_tiles) load_nrows<2>(args, tile_n0(blockIdx.x), lane, gn);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int sp = tile / base_tiles;
            const TileInfo ti = resolve_tile(args, tile - sp * base_tiles, s_toff, s_roff);
            const int m0 = ti.a_row0, n0 = ti.b_row0;
            const int kb0 = sp * args.kb_split, kb1 = min(args.num_kb, kb0 + args.kb_split);
            const int next = tile + int(gridDim.x);
            int gi[8];
            int run = -1;
            if (gather && !B_MN) {
#pragma unroll
                for (int j = 0; j < 8; ++j) gi[j] = gn[j];
                run = nrows_run<2>(args, gi, n0);
                if (next < num_tiles) load_nrows<2>(args, tile_n0(next), lane, gn);
            }
            for (int kb = kb0; kb < kb1; ++kb) {
                uint8_t* sa = smem + stage * STAGE_BYTES;
                uint8_t* sb = sa + A_BYTES;
                const int k0 = kb * BK;
                if (gather && B_MN)
                    run = rb.get(args, kb, kb1, next < num_tiles ? (next / base_tiles) * args.kb_split : 0, lane);
                if (lane == 0) {
                    mbar_wait(empty + stage, phase ^ 1);
                    mbar_arrive_expect_tx(full + stage, STAGE_BYTES);
                    auto ld_a = [&](void* dst, int c0, int c1) {
                        if (args.hint_a) tma_load_2d_hint(dst, &tmA, full + stage, c0, c1, pol_a);
                        else tma_load_2d(dst, &tmA, full + stage, c0, c1);
                    };
                    auto ld_b = [&](void* dst, int c0, int c1) {
                        if (args.hint_b) tma_load_2d_hint(dst, &tmB, full + stage, c0, c1, pol_b);
                        else tma_load_2d(dst, &tmB, full + stage, c0, c1);
                    };
                    if (!A_MN) {
                        ld_a(sa, k0, m0);
                    } else {
#pragma unroll
                        for (int j = 0; j < BM / 64; ++j) ld_a(sa + j * 8192, m0 + 64 * j, k0);
                    }
                    if (!gather || run >= 0) {  // plain box (gathered B: at the run's table row)
                        const int brow = gather ? run : (B_MN ? k0 : n0);
                        if (!B_MN) {
                            ld_b(sb, k0, brow);
                        } else {
#pragma unroll
                            for (int j = 0; j < BN / 64; ++j) ld_b(sb + j * 8192, n0 + 64 * j, brow);
                        }
                    }
                }
                if (gather && run < 0) {
                    __syncwarp();  // the stage is free (lane 0 waited on it)
                    if (!B_MN) {   // 256 B rows x 64 k: lane owns rows 4l..4l+3 and 128+4l..
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            tma_gather4(sb + (h * 128 + 4 * lane) * 128, &tmG, full + stage, k0, gi[4 * h],
                                        gi[4 * h + 1], gi[4 * h + 2], gi[4 * h + 3]);
                    } else {  // 4 chunks of 64 n x 64 k-rows: lane owns k-rows 4(l%16).. of chunks l/16, l/16+2
                        const int r = (lane & 15) * 4;
                        int i0, i1, i2, i3;
                        krows_four(load_krows(args, k0, lane), r, i0, i1, i2, i3);  // broken k-block: rare
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int ch = (lane >> 4) + 2 * h;
                            tma_gather4(sb + ch * 8192 + r * 128, &tmG, full + stage, n0 + 64 * ch, i0, i1, i2, i3);
                        }
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(BM, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait(tempty + acc, aphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                const int kb0 = (tile / base_tiles) * args.kb_split, kb1 = min(args.num_kb, kb0 + args.kb_split);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
                    const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        // K-major SW128: a 16-element K step is +32 B inside the swizzle atom, SBO = 8 rows * 128 B.
                        // MN-major SW128: a 16-row K step is +2048 B; LBO = 8 KB between 64-wide MN chunks.
                        const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                                 : umma_desc_sw128(a_addr + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                                 : umma_desc_sw128(b_addr + k * 32, 16, 1024);
                        umma_bf16(d_tmem, ad, bd, idesc, (kb != kb0 || k != 0));
                    }
                    umma_commit(empty + stage);  // frees this smem stage once the MMAs above retire
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(tfull + acc);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5)
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const int sp = tile / base_tiles;
            const TileInfo ti = resolve_tile(args, tile - sp * base_tiles, s_toff, s_roff);
            const long long c_off = sp * args.split_stride;
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            mbar_wait(tfull + acc, aphase);
            tc_fence_after();
            const int m = ti.a_row0 + q * 32 + lane;
            if (args.epi == EPI_ADAM_F32) {
                const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
                if (args.mom16)
                    adam_tile_rows<true>(args, ta, m, ti.n_col0);
                else
                    adam_tile_rows<false>(args, ta, m, ti.n_col0);
            } else {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * BN + c * 32, r);
                    tmem_ld_wait();
                    if (args.num_kb == 0)  // empty K (a zero extent): nothing was accumulated
                        for (int j = 0; j < 32; ++j) r[j] = 0u;
                    const int n = ti.n_col0 + c * 32;
                    if (m < ti.m_lim && n < args.N) epilogue_chunk(args, m, n, r, c_off);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
        }
    }

    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ==================================================================================================== CTA pair
// 2-CTA variant (cta_group::2, cluster of 2 on one TPC): the pair computes a 256 x 256 tile with one
// tcgen05.mma M=256 per K=16 step, issued by the leader CTA. Each CTA stages its own 128 A rows and its own
// 128 B rows (half of the tile's N), so per-SM shared-memory operand traffic drops by a third versus the 1-CTA
// 128x256 tile, and each CTA's TMEM accumulates its 128 rows x all 256 columns.
//   warp 0 (both CTAs): TMA into the local ring, completion counted on the leader's full barrier
//   warp 1 (leader)   : MMA issue; commits multicast to both CTAs' empty / tmem-full barriers
//   warps 2-5 (both)  : epilogue of the local 128 rows; release the accumulator on the leader's tmem-empty
// 4 x 32 KB stages. Measured against 6 (round 2, tools/r2_call45.sh / r2_call46.sh, alternating on one box): the
// step 23.83-23.91 -> 23.47-23.48 ms, the co-running tiles' operand streams stay closer together (ncu: z / dA DRAM
// 2.8-3.5 -> 1.6 GB, grad-W 14.1-14.5 -> 8.3-8.4 GB per launch) and the power-capped clock rises (1.28 -> 1.41 GHz
// on the grad-W GEMMs); 3 stages starve the MMA (24.79 ms), 5 sit between.
#ifndef MEFT_P_STAGES
#define MEFT_P_STAGES 4
#endif
constexpr int P_STAGES = MEFT_P_STAGES;
constexpr int P_A_BYTES = 128 * BK * 2;
constexpr int P_B_BYTES = 128 * BK * 2;
constexpr int P_STAGE_BYTES = P_A_BYTES + P_B_BYTES;
constexpr int P_SMEM_BYTES = P_STAGES * P_STAGE_BYTES + 1024 + 256;
constexpr int P_TILE_M = 256;

__device__ __forceinline__ void tile_coords_pair(int tile, const KArgs& args, int& m_blk, int& n_blk) {
    const int tiles_m = args.tiles_m, tiles_n = args.tiles_n;
    if (args.raster_n_fast) {  // B resident in L2, A streamed once
        m_blk = tile / tiles_n;
        n_blk = tile % tiles_n;
        return;
    }
    const int group = args.raster_group;  // pair-tiles of M that share each B panel while resident
    const int group_size = group * tiles_n;
    const int g = tile / group_size;
    const int first_m = g * group;
    const int gm = min(group, tiles_m - first_m);
    const int local = tile - g * group_size;
    m_blk = first_m + local % gm;
    n_blk = local / gm;
}

template <bool A_MN, bool B_MN>
__device__ __forceinline__ void pair_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmG,
                                          const KArgs& args) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_STAGES * P_STAGE_BYTES);
    uint64_t* empty = full + P_STAGES;
    uint64_t* tfull = empty + P_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < P_STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull + b, 1);
            mbar_init(tempty + b, 8);  // 4 epilogue warps in each of the two CTAs
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmG);
    }
    if (warp == 1) tmem_alloc_pair(tmem_slot, TMEM_COLS);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int num_tiles = args.tiles_m * args.tiles_n;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs; all lanes for gathered B rows)
        const bool gather = args.b_idx != nullptr;
        const uint64_t pol_a = l2_policy(args.hint_a), pol_b = l2_policy(args.hint_b);
        int stage = 0;
        uint32_t phase = 0;
        int gn[4] = {0, 0, 0, 0};  // K-major gathered B: the NEXT tile's rows of this CTA's half (prefetched)
        RunBatch rb;               // MN-major gathered B: k-block run table reader
        auto tile_n0 = [&](int t) {
            int mb_, nb_;
            tile_coords_pair(t, args, mb_, nb_);
            return nb_ * BN + int(rank) * 128;
        };
        if (gather && !B_MN && pair < num_tiles) load_nrows<1>(args, tile_n0(pair), lane, gn);
        for (int tile = pair; tile < num_tiles; tile += npairs) {
            int mb, nb;
            tile_coords_pair(tile, args, mb, nb);
            const int m0 = mb * P_TILE_M + int(rank) * 128;  // this CTA's A rows
            const int n0 = nb * BN + int(rank) * 128;        // this CTA's half of the B rows
            const int next = tile + npairs;
            int gi[4];
            int run = -1;
            if (gather && !B_MN) {
#pragma unroll
                for (int j = 0; j < 4; ++j) gi[j] = gn[j];
                run = nrows_run<1>(args, gi, n0);
                if (next < num_tiles) load_nrows<1>(args, tile_n0(next), lane, gn);
            }
            for (int kb = 0; kb < args.num_kb; ++kb) {
                uint8_t* sa = smem + stage * P_STAGE_BYTES;
                uint8_t* sb = sa + P_A_BYTES;
                const int k0 = kb * BK;
                if (gather && B_MN) run = rb.get(args, kb, args.num_kb, 0, lane);
                if (lane == 0) {
                    mbar_wait(empty + stage, phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(full + stage, 2 * P_STAGE_BYTES);
                    auto ld_a = [&](void* dst, int c0, int c1) {
                        if (args.hint_a) tma_load_2d_pair_hint(dst, &tmA, full + stage, c0, c1, pol_a);
                        else tma_load_2d_pair(dst, &tmA, full + stage, c0, c1);
                    };
                    auto ld_b = [&](void* dst, int c0, int c1) {
                        if (args.hint_b) tma_load_2d_pair_hint(dst, &tmB, full + stage, c0, c1, pol_b);
                        else tma_load_2d_pair(dst, &tmB, full + stage, c0, c1);
                    };
                    if (!A_MN) {
                        ld_a(sa, k0, m0);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j) ld_a(sa + j * 8192, m0 + 64 * j, k0);
                    }
                    if (!gather || run >= 0) {  // plain box (gathered B: at the run's table row)
                        const int brow = gather ? run : (B_MN ? k0 : n0);
                        if (!B_MN) {
                            ld_b(sb, k0, brow);
                        } else {
#pragma unroll
                            for (int j = 0; j < 2; ++j) ld_b(sb + j * 8192, n0 + 64 * j, brow);
                        }
                    }
                }
                if (gather && run < 0) {
                    __syncwarp();  // the stage is free (lane 0 waited on it)
                    if (!B_MN) {   // 128 B rows x 64 k: lane owns rows 4l..4l+3
                        tma_gather4_pair(sb + 4 * lane * 128, &tmG, full + stage, k0, gi[0], gi[1], gi[2], gi[3]);
                    } else {  // 2 chunks of 64 n x 64 k-rows: lane owns k-rows 4(l%16).. of chunk l/16
                        const int r = (lane & 15) * 4, ch = lane >> 4;
                        int i0, i1, i2, i3;
                        krows_four(load_krows(args, k0, lane), r, i0, i1, i2, i3);  // broken k-block: rare
                        tma_gather4_pair(sb + ch * 8192 + r * 128, &tmG, full + stage, n0 + 64 * ch, i0, i1, i2, i3);
                    }
                }
                if (++stage == P_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA)
        if (leader && lane == 0) {
            constexpr uint32_t idesc = umma_idesc_bf16(P_TILE_M, BN, A_MN, B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
                const int acc = it & 1;
                const uint32_t aphase = (it >> 1) & 1;
                mbar_wait_cluster(tempty + acc, aphase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * BN;
                for (int kb = 0; kb < args.num_kb; ++kb) {
                    mbar_wait(full + stage, phase);
                    tc_fence_after();
                    const uint32_t a_addr = smem_u32(smem + stage * P_STAGE_BYTES);
                    const uint32_t b_addr = a_addr + P_A_BYTES;
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = A_MN ? umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                                 : umma_desc_sw128(a_addr + k * 32, 16, 1024);
                        const uint64_t bd = B_MN ? umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                                 : umma_desc_sw128(b_addr + k * 32, 16, 1024);
                        umma_bf16_pair(d_tmem, ad, bd, idesc, (kb | k) != 0);
                    }
                    umma_commit_pair(empty + stage);  // frees this stage in both CTAs
                    if (++stage == P_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_pair(tfull + acc);  // both CTAs' accumulators ready
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5, both CTAs)
        const int q = warp & 3;
        int it = 0;
        for (int tile = pair; tile < num_tiles; tile += npairs, ++it) {
            int mb, nb;
            tile_coords_pair(tile, args, mb, nb);
            const int acc = it & 1;
            const uint32_t aphase = (it >> 1) & 1;
            mbar_wait(tfull + acc, aphase);
            tc_fence_after();
            const int m = mb * P_TILE_M + int(rank) * 128 + q * 32 + lane;
            if (args.epi == EPI_ADAM_F32) {
                float* sw = reinterpret_cast<float*>(smem + P_STAGES * P_STAGE_BYTES + 256) + q * 32 * ADAM_SCRATCH_LD;
                const uint32_t ta = tmem_base + (uint32_t(q * 32) << 16) + acc * BN;
                if (args.mom16) {
                    if (args.stat_ss)
                        adam_tile_transposed<true, true>(args, ta, m - lane, nb * BN, sw, lane);
                    else
                        adam_tile_transposed<false, true>(args, ta, m - lane, nb * BN, sw, lane);
                } else {
                    if (args.stat_ss)
                        adam_tile_transposed<true, false>(args, ta, m - lane, nb * BN, sw, lane);
                    else
                        adam_tile_transposed<false, false>(args, ta, m - lane, nb * BN, sw, lane);
                }
            } else {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem_base + (uint32_t(q * 32) << 16) + acc * BN + c * 32, r);
                    tmem_ld_wait();
                    if (args.num_kb == 0)  // empty K (a zero extent): nothing was accumulated
                        for (int j = 0; j < 32; ++j) r[j] = 0u;
                    const int n = nb * BN + c * 32;
                    if (m < args.M && n < args.N) epilogue_chunk(args, m, n, r);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty + acc, 0);
        }
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair(tmem_base, TMEM_COLS);
    }
}

// The kernels. The *_ext variants first shrink a capacity-sized launch to its device-resident extent
// (apply_extent; a private copy of the arguments); the plain ones read the arguments straight from parameter space.
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmG, const KArgs args) {
    gemm_body<A_MN, B_MN>(tmA, tmB, tmG, args);
}
template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    k_gemm_bf16_ext(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmG, const KArgs args_in) {
    KArgs args = args_in;
    apply_extent(args);
    gemm_body<A_MN, B_MN>(tmA, tmB, tmG, args);
}
template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_gemm_bf16_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmG, const KArgs args) {
    pair_body<A_MN, B_MN>(tmA, tmB, tmG, args);
}
template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    k_gemm_bf16_pair_ext(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const __grid_constant__ CUtensorMap tmG, const KArgs args_in) {
    KArgs args = args_in;
    apply_extent(args);
    pair_body<A_MN, B_MN>(tmA, tmB, tmG, args);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw MeftError(6, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows of pitch ld elements.
#ifndef MEFT_L2_PROMOTION  // A/B knob (tools/ab_variants.sh)
#define MEFT_L2_PROMOTION CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
CUtensorMap make_map(const void* base, int64_t inner, int64_t outer, int64_t ld, uint32_t box_inner,
                     uint32_t box_outer) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, MEFT_L2_PROMOTION,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw MeftError(6, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// SMs the persistent GEMMs may occupy. A communication-overlapped caller reserves a few for concurrently running
// NCCL kernels, which otherwise only get an SM once a whole chain of persistent GEMMs has drained.
std::atomic<int> g_reserved_sms{0};
int gemm_sms() {
    static const int env_reserve = [] {  // MEFT_GEMM_SM_RESERVE: A/B knob (SMs left idle by every persistent GEMM)
        const char* v = std::getenv("MEFT_GEMM_SM_RESERVE");
        return v ? std::max(0, std::atoi(v)) : 0;
    }();
    return std::max(2, num_sms() - std::max(env_reserve, g_reserved_sms.load(std::memory_order_relaxed)));
}

template <bool A_MN, bool B_MN>
void launch(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tg, const KArgs& args,
            int tiles_bound) {
    static std::atomic<unsigned long long> attr_done{0}, attr_done_ext{0};
    const int grid = std::max(1, std::min(tiles_bound, gemm_sms()));
    if (args.extent_dim) {
        set_max_smem_once(attr_done_ext, reinterpret_cast<const void*>(k_gemm_bf16_ext<A_MN, B_MN>), SMEM_BYTES);
        k_gemm_bf16_ext<A_MN, B_MN><<<grid, NUM_THREADS, SMEM_BYTES, st>>>(ta, tb, tg, args);
    } else {
        set_max_smem_once(attr_done, reinterpret_cast<const void*>(k_gemm_bf16<A_MN, B_MN>), SMEM_BYTES);
        k_gemm_bf16<A_MN, B_MN><<<grid, NUM_THREADS, SMEM_BYTES, st>>>(ta, tb, tg, args);
    }
    check_launch("k_gemm_bf16");
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

void check_epilogue(const GemmEpilogue& epi) {
    if (epi.kind == EPI_PEER_F32) {
        if (epi.peer_count < 1 || epi.peer_count > kMaxPeers || epi.peer_rows < 1 || epi.ldc % 4 || epi.col0 % 4 ||
            epi.peer_slot < 0 || epi.peer_slot >= epi.peer_count)
            throw MeftError(2, "gemm_bf16: peer epilogue arguments");
        for (int i = 0; i < epi.peer_count; ++i)
            if (!aligned16(epi.peer[i])) throw MeftError(2, "gemm_bf16: peer buffers must be 16-byte aligned");
        return;
    }
    if (epi.kind == EPI_ADAM_F32) {
        if (!epi.row_idx || !epi.adam_coef || !aligned16(epi.adam_w) || !aligned16(epi.adam_m) ||
            !aligned16(epi.adam_v) || !aligned16(epi.adam_c) || epi.ldc % 32 || epi.ksplit > 1 || epi.accumulate ||
            (epi.stat_ss && (!epi.stat_lsb || epi.stat_ld < 1)))
            throw MeftError(2, "gemm_bf16: Adam epilogue arguments (row_idx, coef, 16-byte aligned tables, ldc % 32)");
        return;
    }
    if (epi.kind == EPI_STORE_F32 || epi.kind == EPI_ROWS_ADD_F32 || epi.kind == EPI_ROWS_STORE_F32) {
        if (!aligned16(epi.c) || (epi.ldc % 4)) throw MeftError(2, "gemm_bf16: f32 output alignment");
    } else {
        if (!aligned16(epi.c) || (epi.ldc % 8)) throw MeftError(2, "gemm_bf16: bf16 output alignment");
    }
    if (epi.kind == EPI_MASK_BF16 && !epi.bits && (!aligned16(epi.mask) || (epi.ldm % 8)))
        throw MeftError(2, "gemm_bf16: mask alignment");
    if ((epi.kind == EPI_ACT_BF16 || epi.kind == EPI_DACT_BF16) && (!epi.aux || epi.ldaux < 1 || epi.act < 0 ||
                                                                   epi.act > 1))
        throw MeftError(2, "gemm_bf16: activation epilogue needs aux [M x ldaux] and act in {0: SiLU, 1: ReLU}");
}

KArgs base_args(int64_t M, int64_t N, int64_t K, const GemmEpilogue& epi) {
    KArgs args{};
    args.M = int(M);
    args.N = int(N);
    args.K = int(K);
    args.tiles_m = int(ceil_div(M, BM));
    args.tiles_n = int(ceil_div(N, BN));
    args.num_kb = int(ceil_div(K, BK));
    args.epi = epi.kind;
    args.accumulate = epi.accumulate ? 1 : 0;
    args.c = epi.c;
    args.ldc = epi.ldc;
    args.mask = static_cast<const uint16_t*>(epi.mask);
    args.ldm = epi.ldm;
    args.bits = epi.bits;
    args.ldbits = epi.ldbits;
    args.row_idx = epi.row_idx;
    args.grouped = 0;
    args.b_idx = nullptr;
    args.kb_run = nullptr;
    for (int i = 0; i < kMaxPeers; ++i) args.peer[i] = i < epi.peer_count ? epi.peer[i] : nullptr;
    args.aux = static_cast<uint16_t*>(epi.aux);
    args.ldaux = epi.ldaux;
    args.act = epi.act;
    args.peer_rows = epi.peer_rows;
    args.row0 = epi.row0;
    args.col0 = epi.col0;
    args.peer_slot = epi.peer_slot;
    args.adam_w = epi.adam_w;
    args.adam_m = epi.adam_m;
    args.adam_v = epi.adam_v;
    args.mom16 = epi.adam_mom16 ? 1 : 0;
    args.adam_c = epi.adam_c;
    args.adam_coef = epi.adam_coef;
    args.b1 = epi.b1;
    args.b2 = epi.b2;
    args.eps = epi.eps;
    args.stat_ss = epi.stat_ss;
    args.stat_lsb = epi.stat_lsb;
    args.stat_ld = epi.stat_ld;
    args.b_idx_n = 0;
    args.b_oob_row = 0;
    args.extent = epi.extent;
    args.extent_dim = epi.extent ? epi.extent_dim : 0;
    args.extent_tile_m = BM;
    if (args.extent_dim && (args.extent_dim < 1 || args.extent_dim > 3 || epi.ksplit > 1))
        throw MeftError(2, "gemm_bf16: extent_dim must be 1 (M), 2 (N) or 3 (K), without a K split");
    args.ksplit = 1;
    args.kb_split = args.num_kb;
    args.split_stride = 0;
    if (epi.ksplit > 1) {
        if (!(epi.kind == EPI_STORE_F32 || epi.kind == EPI_ROWS_STORE_F32) || epi.accumulate)
            throw MeftError(2, "gemm_bf16: K split needs a plain f32 store epilogue");
        args.kb_split = int(ceil_div(args.num_kb, epi.ksplit));
        args.ksplit = int(ceil_div(args.num_kb, args.kb_split));  // no empty splits
        args.split_stride = epi.split_stride;
    }
    return args;
}

void dispatch(cudaStream_t st, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tg,
              const KArgs& args,
              int tiles_bound) {
    if (!a_mn && !b_mn)
        launch<false, false>(st, ta, tb, tg, args, tiles_bound);
    else if (!a_mn && b_mn)
        launch<false, true>(st, ta, tb, tg, args, tiles_bound);
    else if (a_mn && b_mn)
        launch<true, true>(st, ta, tb, tg, args, tiles_bound);
    else
        launch<true, false>(st, ta, tb, tg, args, tiles_bound);
}

template <bool A_MN, bool B_MN>
void launch_pair(cudaStream_t st, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tg, const KArgs& args,
                 int pair_tiles) {
    static std::atomic<unsigned long long> attr_done{0}, attr_done_ext{0};
    const int pairs = std::max(1, std::min(pair_tiles, gemm_sms() / 2));
    const int smem = P_SMEM_BYTES + (args.epi == EPI_ADAM_F32 ? ADAM_SCRATCH_BYTES : 0);
    if (args.extent_dim) {
        set_max_smem_once(attr_done_ext, reinterpret_cast<const void*>(k_gemm_bf16_pair_ext<A_MN, B_MN>),
                          P_SMEM_BYTES + ADAM_SCRATCH_BYTES);
        k_gemm_bf16_pair_ext<A_MN, B_MN><<<2 * pairs, NUM_THREADS, smem, st>>>(ta, tb, tg, args);
    } else {
        set_max_smem_once(attr_done, reinterpret_cast<const void*>(k_gemm_bf16_pair<A_MN, B_MN>),
                          P_SMEM_BYTES + ADAM_SCRATCH_BYTES);
        k_gemm_bf16_pair<A_MN, B_MN><<<2 * pairs, NUM_THREADS, smem, st>>>(ta, tb, tg, args);
    }
    check_launch("k_gemm_bf16_pair");
}

void launch_pair_dispatch(cudaStream_t st, bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb,
                          const CUtensorMap& tg,
                          const KArgs& args, int pair_tiles) {
    if (!a_mn && !b_mn)
        launch_pair<false, false>(st, ta, tb, tg, args, pair_tiles);
    else if (!a_mn && b_mn)
        launch_pair<false, true>(st, ta, tb, tg, args, pair_tiles);
    else if (a_mn && b_mn)
        launch_pair<true, true>(st, ta, tb, tg, args, pair_tiles);
    else
        launch_pair<true, false>(st, ta, tb, tg, args, pair_tiles);
}

// MEFT_GEMM_PAIR=0 forces the 1-CTA kernel (A/B comparisons in tools/gemm_check).
bool pair_mode_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("MEFT_GEMM_PAIR");
        return !(v && v[0] == '0');
    }();
    return on;
}

}  // namespace

namespace {

void gemm_bf16_one(cudaStream_t st, int64_t M, int64_t N, int64_t K, const GemmOperand& A, const GemmOperand& B,
                   const GemmEpilogue& epi) {
    if (M <= 0 || N <= 0) return;
    if (K <= 0) throw MeftError(2, "gemm_bf16: K must be positive");
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) throw MeftError(1, "gemm_bf16: dimension too large");
    if (!aligned16(A.ptr) || !aligned16(B.ptr) || (A.ld % 8) || (B.ld % 8))
        throw MeftError(2, "gemm_bf16: operands need 16-byte aligned base and leading dimension % 8 == 0");
    check_epilogue(epi);
    KArgs args = base_args(M, N, K, epi);
    args.hint_a = A.l2_hint;
    args.hint_b = B.l2_hint;
    const CUtensorMap ta = A.mn_major ? make_map(A.ptr, M, K, A.ld, 64, 64) : make_map(A.ptr, K, M, A.ld, 64, BM);
    CUtensorMap tg;
    if (B.rows) {  // gathered B rows: a {64 x 1} box over the whole table, rows fetched by tile::gather4
        if (B.table_rows <= 0 || B.table_rows >= INT32_MAX) throw MeftError(2, "gemm_bf16: gather table rows");
        tg = make_map(B.ptr, B.mn_major ? N : K, B.table_rows, B.ld, 64, 1);
        args.b_idx = B.rows;
        args.b_gather_k = B.mn_major ? 1 : 0;
        args.b_idx_n = int(B.mn_major ? K : N);
        args.b_oob_row = int(B.table_rows);
        if (B.mn_major) {
            if (!B.run_ws) throw MeftError(2, "gemm_bf16: MN-major gathered B needs run_ws");
            k_kb_runs<<<int((args.num_kb + 255) / 256), 256, 0, st>>>(B.rows, args.b_idx_n, args.num_kb, B.run_ws,
                                                                     args.extent_dim == 3 ? args.extent : nullptr);
            check_launch("k_kb_runs");
            args.kb_run = B.run_ws;
        }
    }
    // large problems: 256x256 tiles on CTA pairs (enough pair-tiles to fill the machine at least once); the Adam
    // epilogue always (its transposed, coalesced table stream lives in the pair kernel: at cfg1 the two grad-W
    // GEMMs took 85 us each with the 1-CTA kernel's row-per-thread epilogue)
    const int64_t pair_tiles = ceil_div(M, P_TILE_M) * ceil_div(N, BN);
    if ((pair_tiles >= num_sms() / 2 || epi.kind == EPI_ADAM_F32) && pair_mode_enabled() && args.ksplit == 1) {
        const CUtensorMap tb = B.mn_major ? make_map(B.ptr, N, B.rows ? B.table_rows : K, B.ld, 64, 64)
                                          : make_map(B.ptr, K, B.rows ? B.table_rows : N, B.ld, 64, 128);
        args.tiles_m = int(ceil_div(M, P_TILE_M));
        args.extent_tile_m = P_TILE_M;
        // G pair-tiles of M share each streamed B panel.  Measured (ncu dram bytes + time, tools/gemm_check):
        // K-major x K-major (z, dA: K = d) likes 16 (dA 3.31 -> 3.08 ms); the long-K / MN-major GEMMs 8.
        // Sweeping all of M first doubles DRAM reads: a 64 MB 'resident' operand does not survive per-die L2.
        static const int forced = [] {
            const char* v = std::getenv("MEFT_PAIR_GROUP");  // A/B experiments
            return v ? std::max(1, std::atoi(v)) : 0;
        }();
        static const int forced_amn = [] {
            const char* v = std::getenv("MEFT_PAIR_GROUP_AMN");  // A/B experiments (grad-W GEMMs)
            return v ? std::max(1, std::atoi(v)) : 0;
        }();
        static const int forced_bmn = [] {
            const char* v = std::getenv("MEFT_PAIR_GROUP_BMN");  // A/B experiments (out / grad_h GEMMs)
            return v ? std::max(1, std::atoi(v)) : 0;
        }();
        args.raster_group = forced ? forced : (!A.mn_major && !B.mn_major ? 16 : 8);
        if (A.mn_major && forced_amn) args.raster_group = forced_amn;
        if (!A.mn_major && B.mn_major && forced_bmn) args.raster_group = forced_bmn;
        if (epi.raster > 0) args.raster_group = epi.raster;
        args.raster_n_fast = epi.raster < 0 ? 1 : 0;
        launch_pair_dispatch(st, A.mn_major, B.mn_major, ta, tb, B.rows ? tg : tb, args, int(pair_tiles));
        return;
    }
    const CUtensorMap tb = B.mn_major ? make_map(B.ptr, N, B.rows ? B.table_rows : K, B.ld, 64, 64)
                                      : make_map(B.ptr, K, B.rows ? B.table_rows : N, B.ld, 64, BN);
    dispatch(st, A.mn_major, B.mn_major, ta, tb, B.rows ? tg : tb, args, args.tiles_m * args.tiles_n * args.ksplit);
}

int64_t env_elems(const char* name) {
    const char* v = std::getenv(name);
    return v ? std::max<int64_t>(0, std::atoll(v)) : 0;
}

const void* advance(const void* p, int64_t elems, int64_t esize) {
    return static_cast<const uint8_t*>(p) + elems * esize;
}

}  // namespace

// Large problems run as a grid of sub-GEMMs (chunks of M / N / K, each a persistent launch): co-running CTA
// pairs then stay within an L2-sized window of shared operand panels. M/N chunks are bitwise neutral (every
// output tile is computed exactly as before); K chunks (f32 store epilogues only) add the chunk partials in the
// epilogue. Chunk sizes: MEFT_GEMM_{M,N,K}CHUNK (elements), else the policy below. K chunks change the fp32
// summation order of long-K products (within the bf16 tolerance) and are applied identically on every path.
void gemm_bf16(cudaStream_t st, int64_t M, int64_t N, int64_t K, const GemmOperand& A, const GemmOperand& B,
               const GemmEpilogue& epi) {
    static const int64_t mc_env = env_elems("MEFT_GEMM_MCHUNK"), nc_env = env_elems("MEFT_GEMM_NCHUNK"),
                         kc_env = env_elems("MEFT_GEMM_KCHUNK");
    const bool f32_out = epi.kind == EPI_STORE_F32 || epi.kind == EPI_ROWS_ADD_F32 || epi.kind == EPI_PEER_F32;
    // policy: 65536 per dimension (measured on |S| = 640k GEMMs: z 37.5 -> 33.8 ms, out 46.7 -> 38.5,
    // gW 45.2 -> 39.2; 32768 is equivalent, cfg2's |S| = 65536 stays one launch)
    constexpr int64_t kChunk = 65536;
    // panelled operands fix the chunk width to the panel width
    const bool panels = A.panel_stride || epi.panel_stride;
    if (panels && (epi.mask && !epi.bits)) throw MeftError(2, "gemm_bf16: a panelled C needs the bitmask, not a mask");
    const int64_t mc = panels ? kGemmPanel : round_up(mc_env ? mc_env : kChunk, P_TILE_M);
    const int64_t nc = panels ? kGemmPanel : round_up(nc_env ? nc_env : kChunk, BN);
    const int64_t kc = f32_out ? (panels ? kGemmPanel : round_up(kc_env ? kc_env : kChunk, BK)) : K;
    static_assert(kChunk == kGemmPanel, "panel width = chunk width");
    if (epi.kind == EPI_ADAM_F32 && (N > nc || N != epi.ldc))
        throw MeftError(2, "gemm_bf16: the Adam epilogue covers whole table rows of at most 65536 columns");
    if (epi.extent && ((epi.extent_dim == 1 && M > mc) || (epi.extent_dim == 2 && N > nc) ||
                       (epi.extent_dim == 3 && K > kc)))
        throw MeftError(2, "gemm_bf16: a device-sized dimension must fit one launch (at most 65536)");
    if ((mc >= M && nc >= N && kc >= K) || epi.ksplit > 1) return gemm_bf16_one(st, M, N, K, A, B, epi);
    const int64_t ce = (epi.kind == EPI_STORE_F32 || epi.kind == EPI_ROWS_ADD_F32 || epi.kind == EPI_ROWS_STORE_F32)
                           ? 4 : 2;
    const bool rows_epi = epi.kind == EPI_ROWS_ADD_F32 || epi.kind == EPI_ROWS_STORE_F32;
    for (int64_t m0 = 0; m0 < M; m0 += mc) {
        for (int64_t n0 = 0; n0 < N; n0 += nc) {
            for (int64_t k0 = 0; k0 < K; k0 += kc) {
                const int64_t ml = std::min(mc, M - m0), nl = std::min(nc, N - n0), kl = std::min(kc, K - k0);
                GemmOperand a = A;
                if (A.panel_stride) {  // the chunked dimension steps through whole panels
                    a.ptr = advance(A.ptr, A.mn_major ? (m0 / kGemmPanel) * A.panel_stride + k0 * A.ld
                                                      : (k0 / kGemmPanel) * A.panel_stride + m0 * A.ld, 2);
                    a.panel_stride = 0;
                } else {
                    a.ptr = advance(A.ptr, A.mn_major ? k0 * A.ld + m0 : m0 * A.ld + k0, 2);
                }
                GemmOperand b = B;
                if (!B.rows) {
                    b.ptr = advance(B.ptr, B.mn_major ? k0 * B.ld + n0 : n0 * B.ld + k0, 2);
                } else if (B.mn_major) {  // logical rows = K positions; table columns = N
                    b.rows = B.rows + k0;
                    b.ptr = advance(B.ptr, n0, 2);
                } else {  // logical rows = N positions; table columns = K
                    b.rows = B.rows + n0;
                    b.ptr = advance(B.ptr, k0, 2);
                }
                GemmEpilogue e = epi;
                if (k0 > 0) e.accumulate = true;
                if (epi.kind == EPI_PEER_F32) {  // logical offsets: the addresses are resolved per row
                    e.row0 = epi.row0 + m0;
                    e.col0 = epi.col0 + n0;
                } else if (epi.kind == EPI_ADAM_F32) {
                    e.row_idx = epi.row_idx + m0;
                    e.adam_coef = epi.adam_coef + m0;
                    if (epi.stat_ss) {
                        e.stat_ss = epi.stat_ss + m0 * epi.stat_ld;
                        e.stat_lsb = epi.stat_lsb + m0 * epi.stat_ld;
                    }
                } else if (rows_epi) {
                    e.row_idx = epi.row_idx + m0;
                    e.c = const_cast<void*>(advance(epi.c, n0, ce));
                } else if (epi.panel_stride) {
                    e.c = const_cast<void*>(advance(epi.c, (n0 / kGemmPanel) * epi.panel_stride + m0 * epi.ldc, ce));
                    e.panel_stride = 0;
                } else {
                    e.c = const_cast<void*>(advance(epi.c, m0 * epi.ldc + n0, ce));
                }
                if (epi.mask) e.mask = advance(epi.mask, m0 * epi.ldm + n0, 2);
                if (epi.bits) e.bits = epi.bits + m0 * epi.ldbits + n0 / 32;
                if (epi.aux) e.aux = const_cast<void*>(advance(epi.aux, m0 * epi.ldaux + n0, 2));
                gemm_bf16_one(st, ml, nl, kl, a, b, e);
            }
        }
    }
}

void gemm_bf16_grouped(cudaStream_t st, int G, int64_t N, int64_t K, const GemmOperand& A, int64_t a_rows,
                       const GemmOperand& B, int64_t b_rows, const int32_t* row_off, const int32_t* tile_off,
                       const GemmEpilogue& epi) {
    if (G <= 0 || N <= 0 || a_rows <= 0) return;
    if (A.mn_major || B.mn_major) throw MeftError(2, "gemm_bf16_grouped: K-major operands only");
    if (B.rows) throw MeftError(2, "gemm_bf16_grouped: gathered B is not supported");
    if (epi.extent) throw MeftError(2, "gemm_bf16_grouped: no device-sized extent");
    if (!aligned16(A.ptr) || !aligned16(B.ptr) || (A.ld % 8) || (B.ld % 8))
        throw MeftError(2, "gemm_bf16_grouped: operand alignment");
    check_epilogue(epi);
    const CUtensorMap ta = make_map(A.ptr, K, a_rows, A.ld, 64, BM);
    const CUtensorMap tb = make_map(B.ptr, K, b_rows, B.ld, 64, BN);
    KArgs args = base_args(a_rows, N, K, epi);
    args.grouped = 1;
    args.G = G;
    args.g_ntiles = int(ceil_div(N, BN));
    args.g_brows = int(N);
    args.g_row_off = row_off;
    args.g_tile_off = tile_off;
    const int64_t bound = (ceil_div(a_rows, BM) + G) * args.g_ntiles * args.ksplit;  // >= device tile count
    dispatch(st, false, false, ta, tb, tb, args, int(std::min<int64_t>(bound, INT32_MAX)));
}

void gemm_reserve_sms(int n) { g_reserved_sms.store(std::max(0, n), std::memory_order_relaxed); }

}  // namespace meft_dev
