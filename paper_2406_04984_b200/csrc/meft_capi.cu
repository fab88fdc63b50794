// libmeft_cuda.so — C ABI of the B200 MEFT layer (declarations and reference citations: include/meft_cuda.h).
// Host orchestration only: every numeric step is a kernel in gemm_sm100.cu / select.cu / stream_ops.cu /
// dgemm.cu. There is no CPU compute path.
#include <algorithm>
#include <array>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <functional>
#include <optional>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/meft_cuda.h"
#include "common.cuh"
#include "kernels.h"
#include "select.h"
#include "stream_ops.h"
#include "shard_plan.h"
#include "trunk.h"

using namespace meft_dev;

namespace {
thread_local std::string t_err;
thread_local int64_t t_err_index = -1;
}  // namespace

// ---- guard zones (MEFT_GUARD_ZONES=1): the out-of-bounds-write check that stands in for compute-sanitizer, which
// this pool does not allow. Every context scratch buffer is followed by a 4 KB guard region and every store table by
// a 4 KB gap, all filled with 0xA5; after each C-ABI call the regions are verified on the device and a damaged one
// fails the call (MEFT_E_CUDA, naming the buffer) -- so a test suite run with the variable set proves no kernel wrote
// past a buffer it was given.
namespace {
constexpr size_t kGuard = 4096;
constexpr int kGuardByte = 0xA5;
bool guard_mode() {
    static const bool on = [] {
        const char* v = std::getenv("MEFT_GUARD_ZONES");
        return v && v[0] == '1';
    }();
    return on;
}
struct GuardRegion {
    const void* p;
    size_t n;
    std::string label;
};
std::mutex g_guard_mu;
std::vector<GuardRegion>& guard_regions() {  // store tables' guard gaps (global: stores outlive contexts)
    static std::vector<GuardRegion>* v = new std::vector<GuardRegion>();
    return *v;
}
void forget_guards(const void* store) {  // drop a store's table guards (caller holds g_guard_mu)
    const std::string prefix = "store " + std::to_string(reinterpret_cast<uintptr_t>(store)) + " ";
    auto& v = guard_regions();
    v.erase(std::remove_if(v.begin(), v.end(),
                           [&](const GuardRegion& g) { return g.label.compare(0, prefix.size(), prefix) == 0; }),
            v.end());
}
__global__ void k_guard_check(const uint8_t* __restrict__ p, size_t n, int* __restrict__ bad) {
    int c = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        c += p[i] != kGuardByte;
    if (c) atomicAdd(bad, c);
}
}  // namespace

struct meft_graph {
    cudaGraphExec_t exec = nullptr;
};

struct meft_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;  // overlaps host transfers with compute in the _host step
    // small FFNs: out and grad_h run on a side stream beside dA / the grad-W GEMMs (SmallFfnStreams)
    cudaStream_t side_stream = nullptr;
    cudaEvent_t ev_z = nullptr, ev_side_out = nullptr, ev_da = nullptr, ev_side_gh = nullptr;
    bool own_stream = false;
    cudaEvent_t ev_in = nullptr, ev_fwd = nullptr, ev_out = nullptr, ev_h_in = nullptr;
    std::string err;
    int64_t err_index = -1;
    int32_t* dev_small = nullptr;   // 128 device ints (validation flags, counts; [32, 96): sharded plan counts)
    int32_t* host_small = nullptr;  // 64 pinned ints
    struct Buf {
        void* p = nullptr;
        size_t n = 0;
        size_t req = 0;  // bytes last requested (guard mode: [req, n + kGuard) is the guard region)
    };
    int* guard_bad = nullptr;  // guard mode: per-region damage counts
    std::unordered_map<std::string, Buf> scratch;

    int selection_mode = MEFT_SELECT_AUTO;
    int adam_mode = -1;  // MEFT_ADAM_*; -1 = not set (environment MEFT_ADAM_EPILOGUE, else EPILOGUE)
    int gather_mode = -1;  // MEFT_GATHER_*; -1 = not set (environment MEFT_GATHER, else AUTO)
    bool check_finite = false;  // fused step: raise MEFT_E_NONFINITE like check_finite (kernels.cpp:7-13)
    // meft_ctx_set_host_sync: 1 = read |S| back mid-step, 0 = device-sized FFN GEMMs (no read-back), -1 = AUTO (the
    // default; environment MEFT_HOST_SYNC=0|1|auto for new contexts): device-sized when the union is expected dense
    int host_sync = MEFT_HOST_SYNC_AUTO;

    bool capturing() const {  // the context stream is being captured into a CUDA graph
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        MEFT_CUDA_CHECK(cudaStreamIsCapturing(stream, &cs));
        return cs != cudaStreamCaptureStatusNone;
    }

    // phase timing (meft_ctx_set_timing)
    bool timing = false;
    struct PhaseRec {
        int phase;
        cudaEvent_t a, b;
        long long launches;
    };
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<PhaseRec> recs;

    cudaEvent_t next_event() {
        if (ev_used == ev_pool.size()) {
            cudaEvent_t e;
            MEFT_CUDA_CHECK(cudaEventCreate(&e));
            ev_pool.push_back(e);
        }
        return ev_pool[ev_used++];
    }

    void* get(const std::string& name, size_t bytes) {
        Buf& b = scratch[name];
        const size_t extra = guard_mode() ? kGuard : 0;
        if (b.n < bytes) {
            if (capturing())
                throw MeftError(MEFT_E_INVALID, "scratch '" + name + "' would grow while capturing a graph: run the "
                                                "same calls once eagerly before meft_graph_begin");
            if (b.p) MEFT_CUDA_CHECK(cudaFree(b.p));
            b.p = nullptr;
            b.n = 0;
            const size_t want = std::max<size_t>(bytes, 256);
            cudaError_t e = cudaMalloc(&b.p, want + extra);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw MeftError(MEFT_E_OOM, "device allocation of " + std::to_string(want) + " bytes for '" + name +
                                                "' failed: " + cudaGetErrorString(e));
            }
            b.n = want;
        }
        if (extra) {  // everything past the requested bytes is guard
            b.req = bytes;
            MEFT_CUDA_CHECK(cudaMemsetAsync(static_cast<uint8_t*>(b.p) + bytes, kGuardByte, b.n + extra - bytes, stream));
        }
        return b.p;
    }

    // guard mode: verify every scratch guard region and the stores' table gaps; throws naming the damaged buffer
    void check_guards() {
        if (!guard_mode() || capturing()) return;
        if (!guard_bad) MEFT_CUDA_CHECK(cudaMalloc(&guard_bad, 64 * sizeof(int)));
        int* bad = guard_bad;
        std::vector<std::string> labels;
        std::vector<std::pair<const void*, size_t>> regions;
        for (auto& kv : scratch)
            if (kv.second.p) {
                labels.push_back("scratch '" + kv.first + "'");
                regions.push_back({static_cast<uint8_t*>(kv.second.p) + kv.second.req, kv.second.n + kGuard - kv.second.req});
            }
        // held until the check has run: another thread's meft_store_destroy frees its tables under the same lock, so
        // no store guard region is read after its memory is gone
        std::lock_guard<std::mutex> lk(g_guard_mu);
        for (auto& g : guard_regions()) {
            labels.push_back(g.label);
            regions.push_back({g.p, g.n});
        }
        MEFT_CUDA_CHECK(cudaMemsetAsync(bad, 0, std::min<size_t>(regions.size(), 64) * 4, stream));
        for (size_t i = 0; i < regions.size(); ++i) {
            k_guard_check<<<8, 256, 0, stream>>>(static_cast<const uint8_t*>(regions[i].first), regions[i].second,
                                                  bad + std::min<size_t>(i, 63));
        }
        std::vector<int> h(std::min<size_t>(regions.size(), 64));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(h.data(), bad, h.size() * 4, cudaMemcpyDeviceToHost, stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(stream));
        for (size_t i = 0; i < h.size(); ++i)
            if (h[i]) {
                const std::string who = i < 63 ? labels[i] : std::string("one of the later regions");
                throw MeftError(MEFT_E_CUDA, "guard zone after " + who + " overwritten (" + std::to_string(h[i]) +
                                                 " bytes): an out-of-bounds write");
            }
    }
};

namespace {

struct LayerBufs {
    void* w_a = nullptr;  // [r x d] master (f64 or f32)
    void* w_b = nullptr;
    void* w_g = nullptr;  // [N x d]
    void* m_a = nullptr;
    void* v_a = nullptr;
    void* m_b = nullptr;
    void* v_b = nullptr;
    void* st_a = nullptr;
    void* st_b = nullptr;
    void* c_a = nullptr;  // compute copies (bf16 in MIXED; alias of the masters in F64)
    void* c_b = nullptr;
    void* c_g = nullptr;
    int32_t* step = nullptr;  // [r]
    uint8_t* staged = nullptr;
    float* kn = nullptr;      // MIXED: cached norms of the bf16 compute keys
    int32_t* kl = nullptr;    // MIXED: cached minimum LSB exponents of the bf16 compute keys
    void* base = nullptr;
    void* stage_base = nullptr;  // staging tables, allocated on first use (scatter_grads / staging access)
    // router training state (memtier.cpp:86-91), allocated by meft_store_enable_router
    void* m_g = nullptr;
    void* v_g = nullptr;
    int32_t* rstep = nullptr;
    void* router_base = nullptr;
    int64_t* ehist = nullptr;  // [N] routed-token counts per expert (trainer.cpp:240), accumulated by the step
};

}  // namespace

struct meft_store {
    int64_t layers = 0, d = 0, pairs = 0, experts = 0;
    meft_precision prec = MEFT_STORE_MIXED;  // F64 or MIXED (COMPACT stores are MIXED with bf16 moments)
    bool mom16 = false;                      // COMPACT: Adam moments m_a, v_a, m_b, v_b in bf16
    int device = 0;
    std::vector<LayerBufs> L;
    std::vector<char> key_stats_valid;  // per layer: kn/kl match the current compute keys
    // per layer: staging may hold gradients (scatter_grads / caller access) that the next Adam must consume.
    // While clear, staging is all zero and the fused layer step bypasses it entirely.
    std::vector<char> pending;
    // host-sync AUTO: per layer, whether the last read-back union was dense (1) or not (0), -1 before the first;
    // and the steps since (AUTO re-reads |S| every kUnionRecheck steps, so a drifting union is noticed)
    std::vector<signed char> union_dense;
    std::vector<int> since_check;
    bool train_router = false;
};

namespace {

// One phase of the layer step: an NVTX range (host-side enqueue; nsys / ncu --nvtx show it, a no-op without a
// tool attached) and, when timing is enabled, CUDA events on the context stream around its kernels.
const char* const kPhaseNames[] = {"meft/select (ke_select)", "meft/gather (fetch)", "meft/ffn_forward (sparse_ffn_pa)",
                                   "meft/ffn_backward (sparse_backward + fused Adam)", "meft/adam (sparse_adam_update)"};
struct PhaseScope {
    meft_ctx* c;
    int phase;
    cudaEvent_t a = nullptr;
    long long l0 = 0;
    PhaseScope(meft_ctx* ctx, int p) : c(ctx), phase(p) {
        nvtxRangePushA(kPhaseNames[p]);
        if (!c->timing) return;
        a = c->next_event();
        MEFT_CUDA_CHECK(cudaEventRecord(a, c->stream));
        l0 = launch_counter();
    }
    ~PhaseScope() {
        nvtxRangePop();
        if (!c->timing) return;
        cudaEvent_t b = c->next_event();
        cudaEventRecord(b, c->stream);
        c->recs.push_back({phase, a, b, launch_counter() - l0});
    }
};

meft_status fail(meft_ctx* ctx, int code, const std::string& msg, int64_t index = -1) {
    t_err = msg;
    t_err_index = index;
    if (ctx) {
        ctx->err = msg;
        ctx->err_index = index;
    }
    return static_cast<meft_status>(code);
}

}  // namespace

// For the other C-ABI translation units (checkpoint.cu): record an error the way guarded() does.
meft_status meft_internal_fail(meft_ctx* ctx, int code, const char* msg) { return fail(ctx, code, msg); }

namespace {

template <class F>
meft_status guarded(meft_ctx* ctx, F&& f) {
    try {
        if (ctx) MEFT_CUDA_CHECK(cudaSetDevice(ctx->device));
        f();
        if (ctx && guard_mode()) ctx->check_guards();
        return MEFT_OK;
    } catch (const MeftError& e) {
        return fail(ctx, e.code, e.what(), e.index);
    } catch (const std::bad_alloc&) {
        return fail(ctx, MEFT_E_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(ctx, MEFT_E_CUDA, e.what());
    }
}

int esize(meft_dtype dt) { return dt == MEFT_F64 ? 8 : dt == MEFT_F32 ? 4 : 2; }
int dcode(meft_dtype dt) { return int(dt); }

void require(bool ok, int code, const std::string& msg) {
    if (!ok) throw MeftError(code, msg);
}

void require_ctx(meft_ctx* ctx) { require(ctx != nullptr, MEFT_E_INVALID, "null context"); }

const LayerBufs& layer_of(const meft_store* s, int64_t layer) {
    require(s != nullptr, MEFT_E_INVALID, "null store");
    if (layer < 0 || layer >= s->layers)
        throw MeftError(MEFT_E_RANGE, "layer " + std::to_string(layer) + " out of range", layer);
    return s->L[size_t(layer)];
}

// Reads the device validation flags written by check_sorted_unique (err[0] code, err[1] first bad position).
void raise_index_error(meft_ctx* ctx, const int32_t* S, const char* who, bool order_matters) {
    MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small, ctx->dev_small, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost,
                                    ctx->stream));
    MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    const int code = ctx->host_small[0];
    if (code == 3) {
        int32_t bad = 0;
        MEFT_CUDA_CHECK(cudaMemcpy(&bad, S + ctx->host_small[1], sizeof(int32_t), cudaMemcpyDeviceToHost));
        throw MeftError(MEFT_E_RANGE, std::string(who) + ": index " + std::to_string(bad) + " out of range", bad);
    }
    if (code == 2 && order_matters)
        throw MeftError(MEFT_E_INVALID, std::string(who) + ": indices not sorted ascending");
}

int validate_indices(meft_ctx* ctx, const int32_t* S, int64_t s, int64_t limit, const char* who,
                     bool order_matters) {
    if (s <= 0) return 0;
    const int32_t init[2] = {0, INT32_MAX};
    MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->dev_small, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    check_sorted_unique(ctx->stream, S, s, limit, ctx->dev_small);
    raise_index_error(ctx, S, who, order_matters);
    return ctx->host_small[0];
}

int64_t selection_take(int64_t M, int64_t N, int64_t kk, int64_t k, int64_t* kk_eff, int* warned) {
    if (k < 1) throw MeftError(MEFT_E_INVALID, "ke_select: K must be >= 1");
    if (N < 1 || M < 1) throw MeftError(MEFT_E_INVALID, "ExpertPartition: N and r must be >= 1");
    if (M % N) throw MeftError(MEFT_E_INVALID, "ExpertPartition: N=" + std::to_string(N) + " does not divide r=" +
                                                   std::to_string(M));
    if (kk < 1) throw MeftError(MEFT_E_INVALID, "select_experts: budget must be >= 1");
    const int64_t ke = std::min(kk, N);
    const int64_t visible = ke * (M / N);
    if (kk_eff) *kk_eff = ke;
    if (warned) *warned = k > visible ? 1 : 0;
    return std::min(k, visible);
}

// Per-GEMM launch knobs of the six FFN GEMMs: CTA-pair tile order (GemmEpilogue::raster) and the L2 eviction
// priority of each operand's TMA stream (GemmOperand::l2_hint). The defaults are the measured choices (DESIGN.md
// §4); MEFT_GEMM_<Z|OUT|DA|GH|GWB|GWA>="raster,hint_a,hint_b" overrides one GEMM for A/B experiments.
struct GemmKnob {
    int raster = 0, hint_a = 0, hint_b = 0;
};
enum FfnGemm { G_Z = 0, G_OUT, G_DA, G_GH, G_GWB, G_GWA, G_COUNT };
GemmKnob gemm_knob(int which) {
    static const std::array<GemmKnob, G_COUNT> knobs = [] {
        static const char* names[G_COUNT] = {"MEFT_GEMM_Z", "MEFT_GEMM_OUT", "MEFT_GEMM_DA",
                                             "MEFT_GEMM_GH", "MEFT_GEMM_GWB", "MEFT_GEMM_GWA"};
        std::array<GemmKnob, G_COUNT> k{};
        for (int i = 0; i < G_COUNT; ++i) {
            const char* v = std::getenv(names[i]);
            if (v) std::sscanf(v, "%d,%d,%d", &k[i].raster, &k[i].hint_a, &k[i].hint_b);
        }
        return k;
    }();
    return knobs[which];
}
GemmOperand knob_a(GemmOperand op, int which) {
    op.l2_hint = gemm_knob(which).hint_a;
    return op;
}
GemmOperand knob_b(GemmOperand op, int which) {
    op.l2_hint = gemm_knob(which).hint_b;
    return op;
}
GemmEpilogue knob_e(GemmEpilogue e, int which) {
    e.raster = gemm_knob(which).raster;
    return e;
}

// ---- FFN building blocks (adapter.cpp:122-126, 166-175)

// Selected key/value rows either materialised ([s x d], rows == nullptr) or gathered by the GEMMs themselves:
// keys_s/values_s are then the whole [table_rows x d] compute tables and rows[0..s) the selected row ids
// (TMA tile::gather4 / contiguous-run boxes into the operand tiles; the fetch kernel disappears).
struct RowGather {
    const int32_t* rows = nullptr;
    int64_t table_rows = 0;
};

GemmOperand kv_operand(meft_ctx* ctx, const void* p, int64_t d, bool mn_major, const RowGather& rg, int64_t s) {
    GemmOperand op{p, d, mn_major};
    if (rg.rows) {
        op.rows = rg.rows;
        op.table_rows = rg.table_rows;
        if (mn_major) op.run_ws = static_cast<int32_t*>(ctx->get("kb_run", size_t(s / 64 + 2) * 4));
    }
    return op;
}

// A rank whose part of the union is empty still owes every token home its slot of the fused reduce-scatter: the
// homes fold all `world` slots of their receive buffers, which are never cleared between steps, so the slot is
// written as zeros (the GEMM epilogue's row layout: home h, slot = this rank, rows [0, rows) x d).
void zero_peer_slots(cudaStream_t st, const meft_peer_out& po, bool grad_h, int64_t d) {
    for (int h = 0; h < po.world; ++h) {
        float* base = grad_h ? po.grad_h_recv[h] : po.out_recv[h];
        require(base != nullptr, MEFT_E_INVALID, "peer_out: null receive buffer");
        MEFT_CUDA_CHECK(cudaMemsetAsync(base + size_t(po.rank) * size_t(po.rows) * size_t(d), 0,
                                        size_t(po.rows) * size_t(d) * 4, st));
    }
}

// The out / grad_h GEMMs' epilogue when their rows are pushed to the token homes (meft_peer_out).
GemmEpilogue peer_epilogue(const meft_peer_out& po, bool grad_h, int64_t d) {
    require(po.world >= 1 && po.world <= kMaxPeers && po.rank >= 0 && po.rank < po.world && po.rows >= 1,
            MEFT_E_INVALID, "peer_out: world in [1, 8], rank < world, rows >= 1");
    GemmEpilogue e;
    e.kind = EPI_PEER_F32;
    e.ldc = d;
    e.peer_count = po.world;
    e.peer_slot = po.rank;
    e.peer_rows = po.rows;
    for (int i = 0; i < po.world; ++i) e.peer[i] = grad_h ? po.grad_h_recv[i] : po.out_recv[i];
    return e;
}

// Small FFNs (the GEMMs cannot fill the machine, e.g. BASELINE config 1): the out GEMM runs on the context's side
// stream beside dA, and grad_h beside the value-table grad-W GEMM. Dependencies: out and dA need z; grad_h needs
// dA; the value grad-W GEMM's Adam epilogue rewrites the bf16 values out and dA read, so it waits for out; the
// key grad-W GEMM rewrites the keys grad_h reads, so it waits for grad_h (the main stream then also covers all
// side work). Same kernels on the same inputs: bit-identical to the serial order.
struct SmallFfnStreams {
    cudaStream_t side = nullptr;
    cudaEvent_t ev_z = nullptr, ev_out = nullptr, ev_da = nullptr, ev_gh = nullptr;
};

void ffn_forward_impl(meft_ctx* ctx, meft_dtype dt, const void* h, const void* keys_s, const void* values_s,
                      int64_t T, int64_t d, int64_t s, int64_t ld_z, void* z, void* out, bool accumulate,
                      const RowGather& rg = RowGather(), const meft_peer_out* peer = nullptr,
                      uint32_t* act_bits = nullptr, int64_t panel = 0, const int32_t* s_dev = nullptr,
                      const SmallFfnStreams* cc = nullptr) {
    cudaStream_t st = ctx->stream;
    if (dt == MEFT_F64) {
        double* outd = static_cast<double*>(out);
        if (!accumulate) MEFT_CUDA_CHECK(cudaMemsetAsync(outd, 0, size_t(T * d) * 8, st));
        if (s == 0) return;
        // z = h * w_a_k   (w_a_k(k=c, n=j) = keys_s[j*d + c])
        dgemm(st, T, s, d, DOperand{static_cast<const double*>(h), d, 1}, DOperand{static_cast<const double*>(keys_s), 1, d},
              static_cast<double*>(z), ld_z, DEPI_STORE, nullptr);
        // out += ReLU(z) * w_b_k   (a separate chain added afterwards, like add_inplace)
        double* tmp = static_cast<double*>(ctx->get("ffn_tmp", size_t(T * d) * 8));
        DOperand A{static_cast<const double*>(z), ld_z, 1};
        A.relu = true;
        dgemm(st, T, d, s, A, DOperand{static_cast<const double*>(values_s), d, 1}, tmp, d, DEPI_STORE, nullptr);
        add_f64(st, outd, tmp, T * d);
        return;
    }
    require(dt == MEFT_BF16, MEFT_E_INVALID, "ffn_forward: dtype must be F64 or BF16");
    require(d % 8 == 0 && ld_z % 8 == 0 && (panel ? ld_z == kGemmPanel : ld_z >= s), MEFT_E_INVALID,
            "ffn_forward(bf16): d and ld_z must be multiples of 8");
    if (s == 0) {
        if (peer) {
            zero_peer_slots(st, *peer, false, d);
        } else if (!accumulate) {
            MEFT_CUDA_CHECK(cudaMemsetAsync(out, 0, size_t(T * d) * 4, st));
        }
        return;
    }
    GemmEpilogue e1;
    e1.kind = EPI_RELU_BF16;
    e1.c = z;
    e1.ldc = ld_z;
    e1.bits = act_bits;  // [T x ceil(s / 32)] bitmask of z > 0 for the backward's mask
    e1.ldbits = (s + 31) / 32;
    e1.panel_stride = panel;  // act in kGemmPanel-wide panels (|S| > 65536)
    // s_dev: s is a capacity, the union size is read on the device (z: N, out: K)
    e1.extent = s_dev;
    e1.extent_dim = 2;
    gemm_bf16(st, T, s, d, knob_a(GemmOperand{h, d, false}, G_Z), knob_b(kv_operand(ctx, keys_s, d, false, rg, s), G_Z),
              knob_e(e1, G_Z));
    GemmEpilogue e2;
    if (peer) {
        e2 = peer_epilogue(*peer, false, d);
    } else {
        e2.kind = EPI_STORE_F32;
        e2.c = out;
        e2.ldc = d;
        e2.accumulate = accumulate;
    }
    e2.extent = s_dev;
    e2.extent_dim = 3;
    GemmOperand za{z, ld_z, false};
    za.panel_stride = panel;
    cudaStream_t so = st;
    if (cc) {  // out beside dA (SmallFfnStreams)
        MEFT_CUDA_CHECK(cudaEventRecord(cc->ev_z, st));
        MEFT_CUDA_CHECK(cudaStreamWaitEvent(cc->side, cc->ev_z, 0));
        so = cc->side;
    }
    gemm_bf16(so, T, d, s, knob_a(za, G_OUT), knob_b(kv_operand(ctx, values_s, d, true, rg, s), G_OUT),
              knob_e(e2, G_OUT));
    if (cc) MEFT_CUDA_CHECK(cudaEventRecord(cc->ev_out, so));
}

// stage_keys/stage_values non-null => weight grads are row-added into the store staging at S (fused scatter).
void ffn_backward_impl(meft_ctx* ctx, meft_dtype dt, const void* g, const void* h, const void* z, const void* keys_s,
                       const void* values_s, int64_t T, int64_t d, int64_t s, int64_t ld_z, void* masked,
                       void* grad_keys_s, void* grad_values_s, void* grad_h, bool acc_h, const int32_t* S_rows,
                       void* stage_keys, void* stage_values, const RowGather& rg = RowGather(),
                       cudaEvent_t grad_h_done = nullptr, const std::function<void()>* between = nullptr,
                       const meft_peer_out* peer = nullptr, const GemmEpilogue* epi_values = nullptr,
                       const GemmEpilogue* epi_keys = nullptr, const uint32_t* act_bits = nullptr,
                       int64_t panel = 0, const void* gT = nullptr, const void* hT = nullptr,
                       const int32_t* s_dev = nullptr, const SmallFfnStreams* cc = nullptr) {
    cudaStream_t st = ctx->stream;
    if (dt == MEFT_F64) {
        const double* gd = static_cast<const double*>(g);
        const double* hd = static_cast<const double*>(h);
        const double* zd = static_cast<const double*>(z);
        double* md = static_cast<double*>(masked);
        double* ghd = static_cast<double*>(grad_h);
        if (!acc_h && ghd) MEFT_CUDA_CHECK(cudaMemsetAsync(ghd, 0, size_t(T * d) * 8, st));
        if (s == 0) return;
        // masked = (G * w_b_k^T) .* 1[z>0]
        DOperand mk{zd, ld_z, 1};
        dgemm(st, T, s, d, DOperand{gd, d, 1}, DOperand{static_cast<const double*>(values_s), 1, d}, md, ld_z,
              DEPI_MASK_STORE, &mk);
        // grad_values = ReLU(z)^T G
        DOperand rz{zd, 1, ld_z};
        rz.relu = true;
        dgemm(st, s, d, T, rz, DOperand{gd, d, 1}, static_cast<double*>(grad_values_s), d, DEPI_STORE, nullptr);
        // grad_keys (neuron-major) = masked^T h
        dgemm(st, s, d, T, DOperand{md, 1, ld_z}, DOperand{hd, d, 1}, static_cast<double*>(grad_keys_s), d,
              DEPI_STORE, nullptr);
        // grad_h += masked * w_a_k^T, as a separate chain (add_inplace, adapter.cpp:174)
        if (ghd) {
            double* tmp = static_cast<double*>(ctx->get("ffn_tmp", size_t(T * d) * 8));
            dgemm(st, T, d, s, DOperand{md, ld_z, 1}, DOperand{static_cast<const double*>(keys_s), d, 1}, tmp, d,
                  DEPI_STORE, nullptr);
            add_f64(st, ghd, tmp, T * d);
        }
        return;
    }
    require(dt == MEFT_BF16, MEFT_E_INVALID, "ffn_backward: dtype must be F64 or BF16");
    require(d % 8 == 0 && ld_z % 8 == 0 && (panel ? ld_z == kGemmPanel && act_bits : ld_z >= s), MEFT_E_INVALID,
            "ffn_backward(bf16): alignment");
    auto op = [panel](const void* p, int64_t ld, bool mn) {  // act / masked operands, panelled when |S| > 65536
        GemmOperand o{p, ld, mn};
        o.panel_stride = panel;
        return o;
    };
    if (s == 0) {  // nothing selected here: grad_h is zero (or this rank's peer slots are), and final now
        if (peer) {
            zero_peer_slots(st, *peer, true, d);
        } else if (!acc_h && grad_h) {
            MEFT_CUDA_CHECK(cudaMemsetAsync(grad_h, 0, size_t(T * d) * 4, st));
        }
        if (grad_h_done) MEFT_CUDA_CHECK(cudaEventRecord(grad_h_done, st));
        return;
    }
    GemmEpilogue e3;  // masked = mask(act) .* (G * values_s^T)
    e3.kind = EPI_MASK_BF16;
    e3.c = masked;
    e3.ldc = ld_z;
    e3.mask = z;
    e3.ldm = ld_z;
    e3.bits = const_cast<uint32_t*>(act_bits);  // the forward's bitmask instead of re-reading act (1/16 the bytes)
    e3.ldbits = (s + 31) / 32;
    e3.panel_stride = panel;
    e3.extent = s_dev;  // s_dev: s is a capacity (dA: N, grad_h: K, grad-W: M)
    e3.extent_dim = 2;
    gemm_bf16(st, T, s, d, knob_a(GemmOperand{g, d, false}, G_DA),
              knob_b(kv_operand(ctx, values_s, d, false, rg, s), G_DA), knob_e(e3, G_DA));
    if (grad_h || peer) {  // first after masked, so grad_h can stream back while the weight-gradient GEMMs run
        GemmEpilogue e6;  // grad_h (+)= masked * keys_s
        if (peer) {
            e6 = peer_epilogue(*peer, true, d);
        } else {
            e6.kind = EPI_STORE_F32;
            e6.c = grad_h;
            e6.ldc = d;
            e6.accumulate = acc_h;
        }
        e6.extent = s_dev;
        e6.extent_dim = 3;
        cudaStream_t sg = st;
        if (cc) {  // grad_h beside the value grad-W GEMM (SmallFfnStreams)
            MEFT_CUDA_CHECK(cudaEventRecord(cc->ev_da, st));
            MEFT_CUDA_CHECK(cudaStreamWaitEvent(cc->side, cc->ev_da, 0));
            sg = cc->side;
        }
        gemm_bf16(sg, T, d, s, knob_a(op(masked, ld_z, false), G_GH),
                  knob_b(kv_operand(ctx, keys_s, d, true, rg, s), G_GH), knob_e(e6, G_GH));
        if (cc) MEFT_CUDA_CHECK(cudaEventRecord(cc->ev_gh, sg));
    }
    if (grad_h_done) MEFT_CUDA_CHECK(cudaEventRecord(grad_h_done, cc ? cc->side : st));
    GemmEpilogue e4;  // grad_values = act^T G   (M = s, N = d, K = T)
    if (S_rows) {
        e4.kind = EPI_ROWS_ADD_F32;
        e4.c = stage_values;
        e4.row_idx = S_rows;
    } else {
        e4.kind = EPI_STORE_F32;
        e4.c = grad_values_s;
    }
    e4.ldc = d;
    // grad-W B operands: g / h as stored ([T x d], MN-major) or their [d x T] transposes (K-major) when given
    const GemmOperand gB = gT ? GemmOperand{gT, T, false} : GemmOperand{g, d, true};
    const GemmOperand hB = hT ? GemmOperand{hT, T, false} : GemmOperand{h, d, true};
    auto rows_extent = [s_dev](GemmEpilogue e) {
        e.extent = s_dev;
        e.extent_dim = 1;
        return e;
    };
    if (cc) MEFT_CUDA_CHECK(cudaStreamWaitEvent(st, cc->ev_out, 0));  // out has read the values this rewrites
    gemm_bf16(st, s, d, T, knob_a(op(z, ld_z, true), G_GWB), knob_b(gB, G_GWB),
              knob_e(rows_extent(epi_values ? *epi_values : e4), G_GWB));
    if (between) (*between)();  // e.g. consume grad_values before grad_keys reuses its buffer
    GemmEpilogue e5 = e4;  // grad_keys = masked^T h
    e5.c = S_rows ? stage_keys : grad_keys_s;
    if (cc) MEFT_CUDA_CHECK(cudaStreamWaitEvent(st, cc->ev_gh, 0));  // grad_h has read the keys this rewrites
    gemm_bf16(st, s, d, T, knob_a(op(masked, ld_z, true), G_GWA), knob_b(hB, G_GWA),
              knob_e(rows_extent(epi_keys ? *epi_keys : e5), G_GWA));
}

// ---- store helpers

bool is_a_family(meft_tensor t) {
    return t == MEFT_T_W_A || t == MEFT_T_M_A || t == MEFT_T_V_A || t == MEFT_T_STAGE_A || t == MEFT_T_W_A_COMPUTE;
}

void* tensor_ptr(const meft_store* s, const LayerBufs& L, meft_tensor t, meft_dtype* dt, int64_t* rows,
                 int64_t* cols) {
    const meft_dtype master = s->prec == MEFT_STORE_F64 ? MEFT_F64 : MEFT_F32;
    const meft_dtype comp = s->prec == MEFT_STORE_F64 ? MEFT_F64 : MEFT_BF16;
    *rows = s->pairs;
    *cols = s->d;
    switch (t) {
        case MEFT_T_W_A: *dt = master; return L.w_a;
        case MEFT_T_W_B: *dt = master; return L.w_b;
        case MEFT_T_W_G: *dt = master; *rows = s->experts; return L.w_g;
        case MEFT_T_M_A: *dt = s->mom16 ? MEFT_BF16 : master; return L.m_a;
        case MEFT_T_V_A: *dt = s->mom16 ? MEFT_BF16 : master; return L.v_a;
        case MEFT_T_M_B: *dt = s->mom16 ? MEFT_BF16 : master; return L.m_b;
        case MEFT_T_V_B: *dt = s->mom16 ? MEFT_BF16 : master; return L.v_b;
        case MEFT_T_STAGE_A: *dt = master; return L.st_a;
        case MEFT_T_STAGE_B: *dt = master; return L.st_b;
        case MEFT_T_W_A_COMPUTE: *dt = comp; return L.c_a;
        case MEFT_T_W_B_COMPUTE: *dt = comp; return L.c_b;
        case MEFT_T_W_G_COMPUTE: *dt = comp; *rows = s->experts; return L.c_g;
        case MEFT_T_PAIR_STEP: *dt = MEFT_F32; *cols = 1; return L.step;  // int32 storage
        case MEFT_T_STAGED: *dt = MEFT_BF16; *cols = 1; return L.staged;  // uint8 storage
        case MEFT_T_M_G:
        case MEFT_T_V_G:
        case MEFT_T_ROUTER_STEP:
            if (!s->train_router) throw MeftError(MEFT_E_LOGIC, "router state: the router is frozen");
            *rows = s->experts;
            if (t == MEFT_T_ROUTER_STEP) {
                *dt = MEFT_F32;  // int32 storage
                *cols = 1;
                return L.rstep;
            }
            *dt = master;
            return t == MEFT_T_M_G ? L.m_g : L.v_g;
        default: throw MeftError(MEFT_E_INVALID, "unknown store tensor");
    }
}

// Uploads a float64 host matrix in the reference layout into the device tensor (converting layout/precision),
// refreshing the bf16 compute copy when a MIXED master weight changes.
// Host <-> store transfers in reference layouts, converted on the device through two fixed 64 MB fp64 scratch
// buffers (chunks of whole columns of a d x r table, or of whole rows), so an M = 1M table (34 GB in fp64) never
// needs a table-sized staging copy in HBM.
constexpr int64_t kXferElems = int64_t(8) << 20;

void* elem_offset(void* base, meft_dtype dt, int64_t elems) {
    return static_cast<uint8_t*>(base) + elems * esize(dt);
}

void upload_f64(meft_ctx* ctx, meft_store* s, const LayerBufs& L, meft_tensor t, const double* host) {
    cudaStream_t st = ctx->stream;
    meft_dtype dt;
    int64_t rows, cols;
    void* dst = tensor_ptr(s, L, t, &dt, &rows, &cols);
    void* comp = nullptr;  // the bf16 compute copy that follows the master (mixed stores)
    if (s->prec == MEFT_STORE_MIXED)
        comp = t == MEFT_T_W_A ? L.c_a : t == MEFT_T_W_B ? L.c_b : t == MEFT_T_W_G ? L.c_g : nullptr;
    double* tmp = static_cast<double*>(ctx->get("xfer_a", size_t(kXferElems) * 8));
    if (is_a_family(t)) {  // host d x r -> device r x d, a block of whole columns at a time
        double* tr = static_cast<double*>(ctx->get("xfer_b", size_t(kXferElems) * 8));
        const int64_t d = s->d, r = s->pairs, cw = std::max<int64_t>(1, kXferElems / d);
        for (int64_t c0 = 0; c0 < r; c0 += cw) {
            const int64_t w = std::min(cw, r - c0);
            MEFT_CUDA_CHECK(cudaMemcpy2DAsync(tmp, size_t(w) * 8, host + c0, size_t(r) * 8, size_t(w) * 8, size_t(d),
                                              cudaMemcpyHostToDevice, st));
            transpose8(st, tmp, tr, d, w);  // d x w -> w x d
            convert(st, dcode(dt), elem_offset(dst, dt, c0 * d), 0, tr, w * d);
            if (comp) convert(st, 2, elem_offset(comp, MEFT_BF16, c0 * d), 0, tr, w * d);
            MEFT_CUDA_CHECK(cudaStreamSynchronize(st));  // the scratch is reused by the next block
        }
    } else {
        const int64_t rc = std::max<int64_t>(1, kXferElems / std::max<int64_t>(cols, 1));
        for (int64_t r0 = 0; r0 < rows; r0 += rc) {
            const int64_t nr = std::min(rc, rows - r0), n = nr * cols;
            MEFT_CUDA_CHECK(cudaMemcpyAsync(tmp, host + r0 * cols, size_t(n) * 8, cudaMemcpyHostToDevice, st));
            convert(st, dcode(dt), elem_offset(dst, dt, r0 * cols), 0, tmp, n);
            if (comp) convert(st, 2, elem_offset(comp, MEFT_BF16, r0 * cols), 0, tmp, n);
            MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    }
    if (t == MEFT_T_W_A) {
        for (size_t l = 0; l < s->L.size(); ++l)
            if (&s->L[l] == &L) s->key_stats_valid[l] = 0;
    }
}

void download_f64(meft_ctx* ctx, meft_store* s, const LayerBufs& L, meft_tensor t, double* host) {
    cudaStream_t st = ctx->stream;
    meft_dtype dt;
    int64_t rows, cols;
    const void* srcp = tensor_ptr(s, L, t, &dt, &rows, &cols);
    double* tmp = static_cast<double*>(ctx->get("xfer_a", size_t(kXferElems) * 8));
    if (is_a_family(t)) {  // device r x d -> host d x r, a block of whole columns at a time
        double* tr = static_cast<double*>(ctx->get("xfer_b", size_t(kXferElems) * 8));
        const int64_t d = s->d, r = s->pairs, cw = std::max<int64_t>(1, kXferElems / d);
        for (int64_t c0 = 0; c0 < r; c0 += cw) {
            const int64_t w = std::min(cw, r - c0);
            convert(st, 0, tmp, dcode(dt), elem_offset(const_cast<void*>(srcp), dt, c0 * d), w * d);
            transpose8(st, tmp, tr, w, d);  // w x d -> d x w
            MEFT_CUDA_CHECK(cudaMemcpy2DAsync(host + c0, size_t(r) * 8, tr, size_t(w) * 8, size_t(w) * 8, size_t(d),
                                              cudaMemcpyDeviceToHost, st));
            MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    } else {
        const int64_t rc = std::max<int64_t>(1, kXferElems / std::max<int64_t>(cols, 1));
        for (int64_t r0 = 0; r0 < rows; r0 += rc) {
            const int64_t nr = std::min(rc, rows - r0), n = nr * cols;
            convert(st, 0, tmp, dcode(dt), elem_offset(const_cast<void*>(srcp), dt, r0 * cols), n);
            MEFT_CUDA_CHECK(cudaMemcpyAsync(host + r0 * cols, tmp, size_t(n) * 8, cudaMemcpyDeviceToHost, st));
            MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    }
}

// HostStore::init streams (memtier.cpp:67-77) with the reference RNG (rng.hpp:13-36, 62-66).
uint64_t mix_seed(uint64_t seed, uint64_t stream) {
    uint64_t x = seed ^ (0x9E3779B97F4A7C15ull * (stream + 1));
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

void uniform_fill(uint64_t seed, double lo, double hi, double* out, int64_t n) {
    std::mt19937_64 gen(seed);
    for (int64_t i = 0; i < n; ++i) {
        const double u = double(gen() >> 11) * 0x1.0p-53;
        out[i] = std::fma(hi - lo, u, lo);  // the compiled reference contracts lo + (hi-lo)*u
    }
}

// Staging tables (the reference's stage_a/stage_b, memtier.hpp:110-113) are allocated zeroed on first use: the
// fused layer step never needs them, which keeps 2 x pairs x d fp32 per layer out of HBM.
void ensure_staging(meft_store* s, int64_t layer) {
    LayerBufs& L = s->L[size_t(layer)];
    if (L.stage_base) return;
    const size_t mb = s->prec == MEFT_STORE_F64 ? 8 : 4;
    const size_t one = (size_t(s->pairs) * size_t(s->d) * mb + 255) & ~size_t(255);
    int prev = 0;
    MEFT_CUDA_CHECK(cudaGetDevice(&prev));
    MEFT_CUDA_CHECK(cudaSetDevice(s->device));
    cudaError_t e = cudaMalloc(&L.stage_base, 2 * one);
    if (e != cudaSuccess) {
        cudaGetLastError();
        L.stage_base = nullptr;
        cudaSetDevice(prev);
        throw MeftError(MEFT_E_OOM, "staging: cannot allocate " + std::to_string(2 * one) + " bytes for layer " +
                                        std::to_string(layer));
    }
    MEFT_CUDA_CHECK(cudaMemset(L.stage_base, 0, 2 * one));
    L.st_a = L.stage_base;
    L.st_b = static_cast<uint8_t*>(L.stage_base) + one;
    MEFT_CUDA_CHECK(cudaSetDevice(prev));
}

bool is_staging(meft_tensor t) { return t == MEFT_T_STAGE_A || t == MEFT_T_STAGE_B || t == MEFT_T_STAGED; }

// ---- sparse Adam over the staged set (memtier.cpp:187-210)

void adam_impl(meft_ctx* ctx, meft_store* s, int64_t layer, double b1, double b2, double eps, double lr) {
    const LayerBufs& L = s->L[size_t(layer)];
    s->pending[size_t(layer)] = 0;
    if (!L.stage_base) return;  // staging never touched: nothing is staged (flags are only set with it)
    cudaStream_t st = ctx->stream;
    int32_t* rows = static_cast<int32_t*>(ctx->get("adam_rows", size_t(s->pairs) * 4));
    int32_t* bws = static_cast<int32_t*>(ctx->get("adam_bws", size_t((s->pairs + 1023) / 1024 + 1) * 4));
    int32_t* cnt = ctx->dev_small + 8;
    compact_flags(st, L.staged, s->pairs, rows, cnt, bws);
    if (s->prec == MEFT_STORE_MIXED)
        adam_mixed(st, rows, cnt, 0, s->d, static_cast<float*>(L.w_a), L.m_a, L.v_a, static_cast<float*>(L.st_a),
                   static_cast<uint16_t*>(L.c_a), static_cast<float*>(L.w_b), L.m_b, L.v_b,
                   static_cast<float*>(L.st_b), static_cast<uint16_t*>(L.c_b), L.step, L.staged, b1, b2, eps, lr, 3,
                   true, false, nullptr, nullptr, s->mom16);
    else
        adam_f64(st, rows, cnt, 0, s->d, static_cast<double*>(L.w_a), static_cast<double*>(L.m_a),
                 static_cast<double*>(L.v_a), static_cast<double*>(L.st_a), static_cast<double*>(L.w_b),
                 static_cast<double*>(L.m_b), static_cast<double*>(L.v_b), static_cast<double*>(L.st_b), L.step,
                 L.staged, b1, b2, eps, lr);
}

}  // namespace

// =========================================================================================== C ABI

extern "C" {

const char* meft_version(void) { return "meft-b200 0.1 (sm_100a)"; }

meft_status meft_ctx_create(int device, void* stream, meft_ctx** out) {
    if (!out) return fail(nullptr, MEFT_E_INVALID, "null output pointer");
    std::unique_ptr<meft_ctx> c(new meft_ctx());
    c->device = device;
    meft_status st = guarded(c.get(), [&] {
        // NULL is the legacy default stream (what torch reports for its default stream), so work stays
        // ordered with the caller's framework; pass MEFT_OWN_STREAM to get a private non-blocking stream.
        if (stream == MEFT_OWN_STREAM) {
            MEFT_CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        } else {
            c->stream = static_cast<cudaStream_t>(stream);
        }
        MEFT_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        MEFT_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
        MEFT_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_fwd, cudaEventDisableTiming));
        MEFT_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
        MEFT_CUDA_CHECK(cudaEventCreateWithFlags(&c->ev_h_in, cudaEventDisableTiming));
        MEFT_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&c->ev_z, &c->ev_side_out, &c->ev_da, &c->ev_side_gh})
            MEFT_CUDA_CHECK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        MEFT_CUDA_CHECK(cudaMalloc(&c->dev_small, 128 * sizeof(int32_t)));
        MEFT_CUDA_CHECK(cudaMallocHost(&c->host_small, 64 * sizeof(int32_t)));
        if (const char* v = std::getenv("MEFT_HOST_SYNC"))  // the default of new contexts
            c->host_sync = v[0] == '0' ? 0 : v[0] == '1' ? 1 : MEFT_HOST_SYNC_AUTO;
    });
    if (st != MEFT_OK) return st;
    *out = c.release();
    return MEFT_OK;
}

void meft_ctx_destroy(meft_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->scratch)
        if (kv.second.p) cudaFree(kv.second.p);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->dev_small) cudaFree(ctx->dev_small);
    if (ctx->guard_bad) cudaFree(ctx->guard_bad);
    if (ctx->host_small) cudaFreeHost(ctx->host_small);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->ev_fwd) cudaEventDestroy(ctx->ev_fwd);
    if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
    if (ctx->ev_h_in) cudaEventDestroy(ctx->ev_h_in);
    for (cudaEvent_t e : {ctx->ev_z, ctx->ev_side_out, ctx->ev_da, ctx->ev_side_gh})
        if (e) cudaEventDestroy(e);
    if (ctx->side_stream) {
        cudaStreamSynchronize(ctx->side_stream);
        cudaStreamDestroy(ctx->side_stream);
    }
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

void* meft_ctx_stream(meft_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }
const char* meft_last_error(const meft_ctx* ctx) { return ctx ? ctx->err.c_str() : t_err.c_str(); }
int64_t meft_last_error_index(const meft_ctx* ctx) { return ctx ? ctx->err_index : t_err_index; }

meft_status meft_synchronize(meft_ctx* ctx) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

int64_t meft_kernel_launches(void) { return launch_counter(); }

meft_status meft_ctx_set_timing(meft_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        ctx->timing = enable != 0;
    });
}

meft_status meft_ctx_set_selection(meft_ctx* ctx, int mode) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(mode == MEFT_SELECT_AUTO || mode == MEFT_SELECT_EXACT, MEFT_E_INVALID, "unknown selection mode");
        ctx->selection_mode = mode;
    });
}

meft_status meft_ctx_set_check_finite(meft_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        ctx->check_finite = enable != 0;
    });
}

meft_status meft_ctx_set_host_sync(meft_ctx* ctx, int enable) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(enable == 0 || enable == 1 || enable == MEFT_HOST_SYNC_AUTO, MEFT_E_INVALID,
                "set_host_sync: 0, 1 or MEFT_HOST_SYNC_AUTO");
        ctx->host_sync = enable;
    });
}

meft_status meft_graph_begin(meft_ctx* ctx) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(!ctx->capturing(), MEFT_E_INVALID, "graph_begin: the context stream is already being captured");
        require(!ctx->timing, MEFT_E_INVALID, "graph_begin: phase timing (meft_ctx_set_timing) cannot be captured");
        // thread-local: an unsafe call (allocation, synchronisation) from this thread fails the capture loudly
        MEFT_CUDA_CHECK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    });
}

meft_status meft_graph_end(meft_ctx* ctx, meft_graph** graph) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(graph != nullptr, MEFT_E_INVALID, "graph_end: null output");
        *graph = nullptr;
        cudaGraph_t g = nullptr;
        const cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
        if (e != cudaSuccess || !g) {
            cudaGetLastError();
            if (g) cudaGraphDestroy(g);
            throw MeftError(MEFT_E_CUDA, std::string("graph_end: the capture failed (") + cudaGetErrorString(e) +
                                             "): a call synchronised or allocated while capturing");
        }
        cudaGraphExec_t x = nullptr;
        const cudaError_t ei = cudaGraphInstantiate(&x, g, 0);
        cudaGraphDestroy(g);
        if (ei != cudaSuccess) throw MeftError(MEFT_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
        *graph = new meft_graph{x};
    });
}

meft_status meft_graph_launch(meft_ctx* ctx, meft_graph* graph) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(graph != nullptr && graph->exec != nullptr, MEFT_E_INVALID, "graph_launch: null graph");
        MEFT_CUDA_CHECK(cudaGraphLaunch(graph->exec, ctx->stream));
    });
}

void meft_graph_destroy(meft_graph* graph) {
    if (!graph) return;
    if (graph->exec) cudaGraphExecDestroy(graph->exec);
    delete graph;
}

meft_status meft_set_gemm_sm_reserve(int sms) {
    return guarded(nullptr, [&] {
        require(sms >= 0 && sms <= 64, MEFT_E_INVALID, "gemm SM reserve must be in [0, 64]");
        gemm_reserve_sms(sms);
    });
}

meft_status meft_ctx_set_gather(meft_ctx* ctx, int mode) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(mode == MEFT_GATHER_AUTO || mode == MEFT_GATHER_KERNEL || mode == MEFT_GATHER_TMA, MEFT_E_INVALID,
                "unknown gather mode");
        ctx->gather_mode = mode;
    });
}

meft_status meft_ctx_set_adam(meft_ctx* ctx, int mode) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(mode == MEFT_ADAM_EPILOGUE || mode == MEFT_ADAM_PASS, MEFT_E_INVALID, "unknown Adam mode");
        ctx->adam_mode = mode;
    });
}

meft_status meft_ctx_read_timing(meft_ctx* ctx, double* ms5, int64_t* launches5) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        double ms[5] = {0, 0, 0, 0, 0};
        int64_t ln[5] = {0, 0, 0, 0, 0};
        for (const auto& r : ctx->recs) {
            float e = 0.f;
            MEFT_CUDA_CHECK(cudaEventElapsedTime(&e, r.a, r.b));
            if (r.phase >= 0 && r.phase < 5) {
                ms[r.phase] += e;
                ln[r.phase] += r.launches;
            }
        }
        ctx->recs.clear();
        ctx->ev_used = 0;
        for (int i = 0; i < 5; ++i) {
            if (ms5) ms5[i] = ms[i];
            if (launches5) launches5[i] = ln[i];
        }
    });
}

meft_status meft_device_alloc(meft_ctx* ctx, size_t bytes, void** out) {
    return guarded(ctx, [&] {
        cudaError_t e = cudaMalloc(out, std::max<size_t>(bytes, 1));
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw MeftError(MEFT_E_OOM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
    });
}
meft_status meft_device_free(meft_ctx* ctx, void* ptr) {
    return guarded(ctx, [&] { MEFT_CUDA_CHECK(cudaFree(ptr)); });
}
meft_status meft_host_alloc(meft_ctx* ctx, size_t bytes, void** out) {
    return guarded(ctx, [&] { MEFT_CUDA_CHECK(cudaMallocHost(out, std::max<size_t>(bytes, 1))); });
}
meft_status meft_host_free(meft_ctx* ctx, void* ptr) {
    return guarded(ctx, [&] { MEFT_CUDA_CHECK(cudaFreeHost(ptr)); });
}
meft_status meft_copy_to_device(meft_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        if (bytes) MEFT_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    });
}
meft_status meft_copy_to_host(meft_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        if (bytes) MEFT_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}
meft_status meft_memset(meft_ctx* ctx, void* dst, int value, size_t bytes) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        if (bytes) MEFT_CUDA_CHECK(cudaMemsetAsync(dst, value, bytes, ctx->stream));
    });
}
meft_status meft_convert(meft_ctx* ctx, void* dst, meft_dtype dst_dt, const void* src, meft_dtype src_dt, int64_t n) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        convert(ctx->stream, dcode(dst_dt), dst, dcode(src_dt), src, n);
    });
}

// ------------------------------------------------------------------ selection

meft_status meft_selection_shape(int64_t M, int64_t N, int64_t kk, int64_t k, int64_t* take, int64_t* kk_eff,
                                 int* warn) {
    return guarded(nullptr, [&] {
        const int64_t t = selection_take(M, N, kk, k, kk_eff, warn);
        if (take) *take = t;
    });
}

meft_status meft_route_scores(meft_ctx* ctx, meft_dtype dt, const void* h, const void* w_g, int64_t T, int64_t d,
                              int64_t N, double* scores) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(dt == MEFT_F64 || dt == MEFT_BF16, MEFT_E_INVALID, "route_scores: dtype must be F64 or BF16");
        require(T >= 0 && d >= 0 && N >= 0, MEFT_E_SHAPE, "route_scores: negative dimension");
        score_rows(ctx->stream, dcode(dt), h, T, d, w_g, N, scores);
    });
}

meft_status meft_select_experts(meft_ctx* ctx, const double* scores, int64_t T, int64_t N, int64_t kk, int32_t* tau) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        if (kk < 1) throw MeftError(MEFT_E_INVALID, "select_experts: budget must be >= 1");
        if (T > 0 && N > 0) route_topk_device(ctx->stream, scores, T, N, std::min(kk, N), tau);
    });
}

meft_status meft_ke_select(meft_ctx* ctx, meft_dtype dt, const void* h, const void* w_g, const void* keys, int64_t T,
                           int64_t d, int64_t M, int64_t N, int64_t kk, int64_t k, int32_t* per_token, int32_t* tau,
                           int32_t* union_idx, int32_t* union_size_dev) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(dt == MEFT_F64 || dt == MEFT_BF16, MEFT_E_INVALID, "ke_select: dtype must be F64 or BF16");
        int64_t kk_eff = 0;
        const int64_t take = selection_take(M, N, kk, k, &kk_eff, nullptr);
        if (T == 0) {
            MEFT_CUDA_CHECK(cudaMemsetAsync(union_size_dev, 0, 4, ctx->stream));
            return;
        }
        const size_t wsb = select_workspace_bytes(T, d, M, N, kk_eff);
        void* ws = ctx->get("select_ws", wsb);
        ke_select_device(ctx->stream, dcode(dt), h, w_g, keys, T, d, M, N, kk_eff, take, ws, wsb, per_token, tau,
                         union_idx, union_size_dev, nullptr, ctx->selection_mode == MEFT_SELECT_AUTO);
    });
}

meft_status meft_topk_select(meft_ctx* ctx, meft_dtype dt, const void* h, const void* keys, int64_t T, int64_t d,
                             int64_t M, int64_t k, int32_t* per_token, int32_t* union_idx, int32_t* union_size_dev) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(dt == MEFT_F64 || dt == MEFT_BF16, MEFT_E_INVALID, "topk_select: dtype must be F64 or BF16");
        if (k < 1) throw MeftError(MEFT_E_INVALID, "topk_select: K must be >= 1");
        require(M >= 1, MEFT_E_SHAPE, "topk_select: no keys");
        const int64_t take = std::min(k, M);
        if (T == 0) {
            MEFT_CUDA_CHECK(cudaMemsetAsync(union_size_dev, 0, 4, ctx->stream));
            return;
        }
        const size_t wsb = select_workspace_bytes(T, d, M, 1, 1);
        void* ws = ctx->get("select_ws", wsb);
        ke_select_device(ctx->stream, dcode(dt), h, nullptr, keys, T, d, M, 1, 1, take, ws, wsb, per_token, nullptr,
                         union_idx, union_size_dev, nullptr, ctx->selection_mode == MEFT_SELECT_AUTO);
    });
}

// ------------------------------------------------------------------ gather

meft_status meft_gather_adapter(meft_ctx* ctx, meft_dtype dt, const void* keys, const void* values, int64_t M,
                                int64_t d, const int32_t* S, int64_t s, void* keys_s, void* values_s) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        validate_indices(ctx, S, s, M, "gather_adapter", true);
        if (s > 0 && d > 0) gather_rows2(ctx->stream, keys, values, d * esize(dt), S, nullptr, s, keys_s, values_s);
    });
}

// ------------------------------------------------------------------ FFN

meft_status meft_ffn_forward(meft_ctx* ctx, meft_dtype dt, const void* h, const void* keys_s, const void* values_s,
                             int64_t T, int64_t d, int64_t s, int64_t ld_z, void* z, void* out, int accumulate) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(T >= 0 && d >= 0 && s >= 0 && ld_z >= s, MEFT_E_SHAPE, "ffn_forward: bad shape");
        ffn_forward_impl(ctx, dt, h, keys_s, values_s, T, d, s, ld_z, z, out, accumulate != 0);
    });
}

meft_status meft_ffn_backward(meft_ctx* ctx, meft_dtype dt, const void* grad_out, const void* h, const void* z,
                              const void* keys_s, const void* values_s, int64_t T, int64_t d, int64_t s,
                              int64_t ld_z, void* masked_ws, void* grad_keys_s, void* grad_values_s, void* grad_h,
                              int accumulate_grad_h) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(T >= 0 && d >= 0 && s >= 0 && ld_z >= s, MEFT_E_SHAPE, "ffn_backward: bad shape");
        ffn_backward_impl(ctx, dt, grad_out, h, z, keys_s, values_s, T, d, s, ld_z, masked_ws, grad_keys_s,
                          grad_values_s, grad_h, accumulate_grad_h != 0, nullptr, nullptr, nullptr);
    });
}

meft_status meft_base_ffn_forward(meft_ctx* ctx, const double* h, const double* w_in, const double* w_out, int64_t T,
                                  int64_t d, int64_t n, int act, double* base_pre, double* out) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        cudaStream_t st = ctx->stream;
        dgemm(st, T, n, d, DOperand{h, d, 1}, DOperand{w_in, n, 1}, base_pre, n, DEPI_STORE, nullptr);
        double* a = static_cast<double*>(ctx->get("base_act", size_t(std::max<int64_t>(T * n, 1)) * 8));
        act_forward(st, base_pre, a, T * n, act);
        dgemm(st, T, d, n, DOperand{a, n, 1}, DOperand{w_out, d, 1}, out, d, DEPI_STORE, nullptr);
    });
}

meft_status meft_base_ffn_backward(meft_ctx* ctx, const double* grad_out, const double* base_pre, const double* w_in,
                                   const double* w_out, int64_t T, int64_t d, int64_t n, int act, double* grad_h) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        cudaStream_t st = ctx->stream;
        double* da = static_cast<double*>(ctx->get("base_act", size_t(std::max<int64_t>(T * n, 1)) * 8));
        // d_act = G * w_out^T ; d_pre = d_act .* f'(base_pre) ; grad_h = d_pre * w_in^T
        dgemm(st, T, n, d, DOperand{grad_out, d, 1}, DOperand{w_out, 1, d}, da, n, DEPI_STORE, nullptr);
        act_backward(st, da, base_pre, T * n, act);
        dgemm(st, T, d, n, DOperand{da, n, 1}, DOperand{w_in, 1, n}, grad_h, d, DEPI_STORE, nullptr);
    });
}

// ------------------------------------------------------------------ sharded-selection bookkeeping

static void copy_counts(meft_ctx* ctx, const int32_t* dev, int world, int64_t* host) {
    std::vector<int32_t> tmp(static_cast<size_t>(world));
    MEFT_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), dev, size_t(world) * 4, cudaMemcpyDeviceToHost, ctx->stream));
    MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < world; ++r) host[r] = tmp[size_t(r)];
}

meft_status meft_shard_dispatch(meft_ctx* ctx, const int32_t* tau, int64_t T, int64_t kk, int64_t n_loc, int world,
                                const uint16_t* h, int64_t d, uint16_t* send_rows, int32_t* send_exp, int32_t* order,
                                int32_t* inv, int64_t* counts) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(world >= 1 && world <= 64 && n_loc >= 1 && kk >= 1 && T >= 0 && d % 8 == 0 && counts, MEFT_E_INVALID,
                "shard_dispatch: 1 <= world <= 64, n_loc >= 1, d % 8 == 0");
        int32_t* pos = static_cast<int32_t*>(ctx->get("shard_pos", size_t(std::max<int64_t>(T * kk, 1)) * 4));
        int32_t* cnt = ctx->dev_small + 32;
        MEFT_CUDA_CHECK(cudaMemsetAsync(cnt, 0, size_t(world) * 4, ctx->stream));
        shard_dispatch(ctx->stream, tau, T, kk, n_loc, world, h, d, pos, send_rows, send_exp, order, inv, cnt);
        copy_counts(ctx, cnt, world, counts);
    });
}

meft_status meft_shard_unpermute_rows(meft_ctx* ctx, const float* src, const int32_t* order, int64_t n, int64_t cols,
                                      float* dst) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        shard_unpermute_rows(ctx->stream, src, order, n, cols, dst);
    });
}

meft_status meft_shard_requests(meft_ctx* ctx, const int32_t* amb, const int32_t* n_amb, const int32_t* tau,
                                const int32_t* inv, int64_t T, int64_t C, int64_t kk, int64_t E, int64_t M_loc,
                                int world, const int64_t* row_base, int32_t* row, int32_t* key, int32_t* back,
                                int64_t* counts, int64_t* total) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(world >= 1 && world <= 64 && E >= 1 && M_loc >= 1 && counts && total && row_base, MEFT_E_INVALID,
                "shard_requests: arguments");
        cudaStream_t st = ctx->stream;
        int32_t* ws = static_cast<int32_t*>(ctx->get("shard_req", shard_requests_ws_ints(T, C) * 4 + 256));
        int32_t* rb = ctx->dev_small + 32;
        std::vector<int32_t> base(static_cast<size_t>(world));
        for (int r = 0; r < world; ++r) base[size_t(r)] = int32_t(row_base[r]);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(rb, base.data(), size_t(world) * 4, cudaMemcpyHostToDevice, st));
        shard_requests_fill(st, amb, n_amb, tau, inv, T, C, kk, E, M_loc, rb, ws);
        int32_t n = 0;
        MEFT_CUDA_CHECK(cudaMemcpyAsync(&n, ws + T, 4, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        *total = n;
        int32_t* cnt = ctx->dev_small + 32;
        MEFT_CUDA_CHECK(cudaMemsetAsync(cnt, 0, size_t(world) * 4, st));
        shard_requests_sort(st, T, C, M_loc, world, n, ws, row, key, back, cnt);
        copy_counts(ctx, cnt, world, counts);
    });
}

meft_status meft_gather_rows(meft_ctx* ctx, const void* src, int64_t row_bytes, const int32_t* idx, int64_t n,
                             void* dst) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(n >= 0 && row_bytes >= 0, MEFT_E_INVALID, "gather_rows: n, row_bytes >= 0");
        gather_rows1(ctx->stream, src, row_bytes, idx, n, dst);
    });
}

meft_status meft_shard_scatter_f64(meft_ctx* ctx, const double* x, const int32_t* back, int64_t n, double* dst) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        shard_scatter_f64(ctx->stream, x, back, n, dst);
    });
}

// ------------------------------------------------------------------ toy trunk (model.cpp:50-218), fp64

meft_status meft_embed_f64(meft_ctx* ctx, const double* emb, int64_t vocab, const double* pos, int64_t max_seq,
                           int64_t d, const int32_t* tokens, int64_t batch, int64_t seq, double* h) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(vocab >= 1 && d >= 1 && batch >= 0 && seq >= 0, MEFT_E_INVALID, "embed: dimensions");
        if (seq > max_seq) throw MeftError(MEFT_E_RANGE, "embed: sequence longer than max_seq");
        embed_f64(ctx->stream, emb, pos, tokens, batch * seq, seq, d, h);
    });
}

meft_status meft_attention_forward_f64(meft_ctx* ctx, const double* h, const double* wq, const double* wk,
                                       const double* wv, const double* wo, const int32_t* segments, int64_t batch,
                                       int64_t seq, int64_t d, double* out, double* q, double* k, double* v,
                                       double* probs) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(batch >= 0 && seq >= 1 && d >= 1, MEFT_E_INVALID, "attention_forward: dimensions");
        const int64_t T = batch * seq;
        double* c = static_cast<double*>(ctx->get("trunk_ctx", size_t(std::max<int64_t>(T * d, 1)) * 8));
        attention_forward_f64(ctx->stream, h, wq, wk, wv, wo, segments, T, seq, d, q, k, v, probs, c, out);
    });
}

meft_status meft_attention_backward_f64(meft_ctx* ctx, const double* wq, const double* wk, const double* wv,
                                        const double* wo, const int32_t* segments, int64_t batch, int64_t seq,
                                        int64_t d, const double* q, const double* k, const double* v,
                                        const double* probs, const double* dh_out, double* dh) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(batch >= 0 && seq >= 1 && d >= 1, MEFT_E_INVALID, "attention_backward: dimensions");
        const int64_t T = batch * seq, n = std::max<int64_t>(T * d, 1);
        double* w = static_cast<double*>(ctx->get("trunk_bwd", size_t(4 * n + std::max<int64_t>(T * seq, 1)) * 8));
        attention_backward_f64(ctx->stream, wq, wk, wv, wo, segments, T, seq, d, q, k, v, probs, dh_out, w,
                               w + 4 * n, w + n, w + 2 * n, w + 3 * n, dh);
    });
}

meft_status meft_lm_loss_f64(meft_ctx* ctx, const double* emb, int64_t vocab, int64_t d, const double* h, int64_t T,
                             const int32_t* targets, const uint8_t* loss_mask, double loss_scale, double* loss_sum,
                             double* dh) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(vocab >= 1 && d >= 1 && T >= 0 && loss_sum, MEFT_E_INVALID, "lm_loss: dimensions / loss_sum");
        cudaStream_t st = ctx->stream;
        *loss_sum = 0.0;
        if (T == 0) return;
        double* logits = static_cast<double*>(ctx->get("trunk_logits", size_t(2 * T * vocab + T) * 8));
        double* dlogits = logits + T * vocab;
        double* term = dlogits + T * vocab;
        // logits = h emb^T ; rows ; dh = dlogits emb
        dgemm(st, T, vocab, d, DOperand{h, d, 1}, DOperand{emb, 1, d}, logits, vocab, DEPI_STORE, nullptr);
        lm_loss_rows_f64(st, logits, T, vocab, targets, loss_mask, loss_scale, dlogits, term);
        dgemm(st, T, d, vocab, DOperand{dlogits, vocab, 1}, DOperand{emb, d, 1}, dh, d, DEPI_STORE, nullptr);
        std::vector<double> terms(static_cast<size_t>(T));
        std::vector<uint8_t> mask(static_cast<size_t>(T));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(terms.data(), term, size_t(T) * 8, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(mask.data(), loss_mask, size_t(T), cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        double loss = 0.0;  // model.cpp:193, contracted: loss = fma(log_denom - logit[target], scale, loss)
        for (int64_t t = 0; t < T; ++t)
            if (mask[size_t(t)]) loss = std::fma(terms[size_t(t)], loss_scale, loss);
        *loss_sum = loss;
    });
}

meft_status meft_argmax_logits_f64(meft_ctx* ctx, const double* emb, int64_t vocab, int64_t d, const double* h_row,
                                   int64_t* token) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(vocab >= 1 && d >= 1 && token, MEFT_E_INVALID, "argmax_logits: dimensions / token");
        int64_t* dev = reinterpret_cast<int64_t*>(ctx->dev_small + 24);
        argmax_logits_f64(ctx->stream, emb, vocab, d, h_row, dev);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(token, dev, 8, cudaMemcpyDeviceToHost, ctx->stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

meft_status meft_matmul_f64(meft_ctx* ctx, const double* A, const double* B, int64_t m, int64_t k, int64_t n,
                            double* C) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        cudaStream_t st = ctx->stream;
        dgemm(st, m, n, k, DOperand{A, k, 1}, DOperand{B, n, 1}, C, n, DEPI_STORE, nullptr);
        MEFT_CUDA_CHECK(cudaMemsetAsync(ctx->dev_small + 16, 0, 4, st));
        flag_nonfinite(st, C, m * n, ctx->dev_small + 16);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small + 16, ctx->dev_small + 16, 4, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        if (ctx->host_small[16]) throw MeftError(MEFT_E_NONFINITE, "matmul: non-finite entry");
    });
}

meft_status meft_transpose_f64(meft_ctx* ctx, const double* src, double* dst, int64_t rows, int64_t cols) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        transpose8(ctx->stream, src, dst, rows, cols);
    });
}

meft_status meft_activation_f64(meft_ctx* ctx, int act, const double* x, double* y, int64_t n) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(act == 0 || act == 1, MEFT_E_INVALID, "activation: 0 SiLU or 1 ReLU");
        act_forward(ctx->stream, x, y, n, act);
    });
}

meft_status meft_rows_add(meft_ctx* ctx, meft_dtype dt, void* table, int64_t d, const int32_t* idx, int64_t n,
                          const void* rows, uint8_t* flags) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(dt == MEFT_F64 || dt == MEFT_F32, MEFT_E_INVALID, "rows_add: dtype must be F64 or F32");
        require(d >= 1 && n >= 0 && (n == 0 || (table && idx && rows)), MEFT_E_INVALID, "rows_add: arguments");
        if (n == 0) return;
        // strictly ascending indices: one CTA per row; otherwise the segmented (sorted, run-length) add
        const int32_t init[2] = {0, INT32_MAX};
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->dev_small, init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
        check_sorted_unique(ctx->stream, idx, n, INT32_MAX, ctx->dev_small);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small, ctx->dev_small, 4, cudaMemcpyDeviceToHost, ctx->stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (ctx->host_small[0] == 0) {
            stage_add(ctx->stream, dcode(dt), table, d, idx, n, dcode(dt), rows, flags);
        } else {
            const size_t wb = stage_add_segmented_ws(n);
            stage_add_segmented(ctx->stream, dcode(dt), table, d, idx, n, dcode(dt), rows, flags,
                                ctx->get("scatter_seg", wb), wb);
        }
    });
}

meft_status meft_adam_rows_f64(meft_ctx* ctx, double* w, double* m, double* v, double* stage, int64_t* step,
                               uint8_t* staged, const int32_t* rows, int64_t n, int64_t d, double beta1, double beta2,
                               double eps, double lr) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        adam_rows_f64(ctx->stream, w, m, v, stage, step, staged, rows, n, d, beta1, beta2, eps, lr);
    });
}

// ------------------------------------------------------------------ store

meft_status meft_store_create(meft_ctx* ctx, int64_t layers, int64_t d, int64_t pairs, int64_t experts,
                              meft_precision precision, meft_store** out) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(out != nullptr, MEFT_E_INVALID, "null output pointer");
        require(layers >= 1 && d >= 1 && pairs >= 1 && experts >= 1, MEFT_E_SHAPE, "store_create: non-positive shape");
        require(precision == MEFT_STORE_F64 || precision == MEFT_STORE_MIXED || precision == MEFT_STORE_COMPACT,
                MEFT_E_INVALID, "store_create: unknown precision");
        std::unique_ptr<meft_store> s(new meft_store());
        s->layers = layers;
        s->d = d;
        s->pairs = pairs;
        s->experts = experts;
        s->mom16 = precision == MEFT_STORE_COMPACT;
        s->prec = s->mom16 ? MEFT_STORE_MIXED : precision;
        precision = s->prec;
        s->device = ctx->device;
        const int mb = precision == MEFT_STORE_F64 ? 8 : 4;
        const int momb = s->mom16 ? 2 : mb;  // Adam moment element size
        const size_t pd = size_t(pairs) * size_t(d), nd = size_t(experts) * size_t(d);
        auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t gap = guard_mode() ? kGuard : 0;  // guard mode: a 4 KB guard after every table
        std::vector<GuardRegion> new_guards;
        size_t bytes = 2 * al(pd * mb) + 4 * al(pd * momb) + al(nd * mb) + al(size_t(pairs) * 4) + al(size_t(pairs));
        if (precision == MEFT_STORE_MIXED) bytes += 2 * al(pd * 2) + al(nd * 2) + 2 * al(size_t(pairs) * 4);
        bytes += al(size_t(experts) * 8);
        bytes += 16 * gap;
        for (int64_t l = 0; l < layers; ++l) {
            LayerBufs L;
            cudaError_t e = cudaMalloc(&L.base, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                for (auto& p : s->L) cudaFree(p.base);
                throw MeftError(MEFT_E_OOM, "store_create: cannot allocate " + std::to_string(bytes) +
                                                " bytes for layer " + std::to_string(l));
            }
            MEFT_CUDA_CHECK(cudaMemsetAsync(L.base, 0, bytes, ctx->stream));
            uint8_t* p = static_cast<uint8_t*>(L.base);
            int table = 0;
            auto take = [&](size_t n) {
                void* r = p;
                p += al(n);
                if (gap) {  // the guard after this table (registered once the fill has run, below)
                    MEFT_CUDA_CHECK(cudaMemsetAsync(p, kGuardByte, gap, ctx->stream));
                    new_guards.push_back({p, gap, "store " + std::to_string(reinterpret_cast<uintptr_t>(s.get())) +
                                                      " layer " + std::to_string(l) + " table " + std::to_string(table)});
                    p += gap;
                }
                ++table;
                return r;
            };
            L.w_a = take(pd * mb);
            L.w_b = take(pd * mb);
            L.m_a = take(pd * momb);
            L.v_a = take(pd * momb);
            L.m_b = take(pd * momb);
            L.v_b = take(pd * momb);
            L.w_g = take(nd * mb);
            L.step = static_cast<int32_t*>(take(size_t(pairs) * 4));
            L.staged = static_cast<uint8_t*>(take(size_t(pairs)));
            L.ehist = static_cast<int64_t*>(take(size_t(experts) * 8));
            if (precision == MEFT_STORE_MIXED) {
                L.c_a = take(pd * 2);
                L.c_b = take(pd * 2);
                L.c_g = take(nd * 2);
                L.kn = static_cast<float*>(take(size_t(pairs) * 4));
                L.kl = static_cast<int32_t*>(take(size_t(pairs) * 4));
            } else {
                L.c_a = L.w_a;
                L.c_b = L.w_b;
                L.c_g = L.w_g;
            }
            s->L.push_back(L);
            s->key_stats_valid.push_back(0);
            s->pending.push_back(0);
            s->union_dense.push_back(-1);
            s->since_check.push_back(0);
        }
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (!new_guards.empty()) {  // the gaps are filled now: other threads' checks may read them
            std::lock_guard<std::mutex> lk(g_guard_mu);
            for (auto& g : new_guards) guard_regions().push_back(g);
        }
        *out = s.release();
    });
}

void meft_store_destroy(meft_store* store) {
    if (!store) return;
    std::unique_lock<std::mutex> lk(g_guard_mu, std::defer_lock);
    if (guard_mode()) {  // no guard check may be reading this store's gaps while they are freed
        lk.lock();
        forget_guards(store);
    }
    cudaSetDevice(store->device);
    for (auto& L : store->L) {
        cudaFree(L.base);
        if (L.stage_base) cudaFree(L.stage_base);
        if (L.router_base) cudaFree(L.router_base);
    }
    delete store;
}

meft_status meft_store_enable_router(meft_ctx* ctx, meft_store* s) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(s != nullptr, MEFT_E_INVALID, "null store");
        if (s->train_router) return;
        const size_t mb = s->prec == MEFT_STORE_F64 ? 8 : 4;
        const size_t nd = (size_t(s->experts) * size_t(s->d) * mb + 255) & ~size_t(255);
        const size_t bytes = 2 * nd + size_t(s->experts) * 4;
        for (auto& L : s->L) {
            cudaError_t e = cudaMalloc(&L.router_base, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                L.router_base = nullptr;
                throw MeftError(MEFT_E_OOM, "enable_router: cannot allocate router state");
            }
            MEFT_CUDA_CHECK(cudaMemsetAsync(L.router_base, 0, bytes, ctx->stream));
            L.m_g = L.router_base;
            L.v_g = static_cast<uint8_t*>(L.router_base) + nd;
            L.rstep = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(L.router_base) + 2 * nd);
        }
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        s->train_router = true;
    });
}

meft_status meft_store_expert_histogram(meft_ctx* ctx, meft_store* s, int64_t layer, int64_t* host_out, int reset) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        if (host_out)
            MEFT_CUDA_CHECK(cudaMemcpyAsync(host_out, L.ehist, size_t(s->experts) * 8, cudaMemcpyDeviceToHost,
                                            ctx->stream));
        if (reset) MEFT_CUDA_CHECK(cudaMemsetAsync(L.ehist, 0, size_t(s->experts) * 8, ctx->stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    });
}

meft_status meft_store_train_router(const meft_store* s, int* on) {
    return guarded(nullptr, [&] {
        require(s != nullptr && on != nullptr, MEFT_E_INVALID, "null store / output");
        *on = s->train_router ? 1 : 0;
    });
}

meft_status meft_store_info(const meft_store* s, int64_t* layers, int64_t* d, int64_t* pairs, int64_t* experts,
                            meft_precision* precision) {
    return guarded(nullptr, [&] {
        require(s != nullptr, MEFT_E_INVALID, "null store");
        if (layers) *layers = s->layers;
        if (d) *d = s->d;
        if (pairs) *pairs = s->pairs;
        if (experts) *experts = s->experts;
        if (precision) *precision = s->mom16 ? MEFT_STORE_COMPACT : s->prec;
    });
}

meft_status meft_store_init_reference(meft_ctx* ctx, meft_store* s, uint64_t seed) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(s != nullptr, MEFT_E_INVALID, "null store");
        const double bound = 1.0 / std::sqrt(double(s->d));
        std::vector<double> buf(size_t(s->d * std::max(s->pairs, s->experts)));
        for (int64_t l = 0; l < s->layers; ++l) {
            const LayerBufs& L = s->L[size_t(l)];
            uniform_fill(mix_seed(seed, 0x5000 + 2 * uint64_t(l)), -bound, bound, buf.data(), s->d * s->pairs);
            upload_f64(ctx, s, L, MEFT_T_W_A, buf.data());
            uniform_fill(mix_seed(seed, 0x5001 + 2 * uint64_t(l)), -bound, bound, buf.data(), s->experts * s->d);
            upload_f64(ctx, s, L, MEFT_T_W_G, buf.data());
        }
    });
}

meft_status meft_reference_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, int round_bf16,
                                   double* host_out) {
    return guarded(nullptr, [&] {
        require(n >= 0 && (n == 0 || host_out != nullptr), MEFT_E_INVALID, "reference_uniform: n >= 0, output");
        uniform_fill(mix_seed(seed, stream), lo, hi, host_out, n);
        if (round_bf16) {
            for (int64_t i = 0; i < n; ++i) {  // RNE to bf16 (finite inputs): add half an ulp plus the tie bit
                const float f = float(host_out[i]);  // the doubles here are far from any float rounding tie
                uint32_t u;
                std::memcpy(&u, &f, 4);
                u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u;
                float r;
                std::memcpy(&r, &u, 4);
                host_out[i] = double(r);
            }
        }
    });
}

meft_status meft_store_upload_host(meft_ctx* ctx, meft_store* s, int64_t layer, meft_tensor t, const void* host,
                                   int64_t rows, int64_t cols) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        if (is_staging(t)) {
            ensure_staging(s, layer);
            s->pending[size_t(layer)] = 1;
        }
        if (t == MEFT_T_PAIR_STEP || t == MEFT_T_STAGED || t == MEFT_T_ROUTER_STEP) {
            const int64_t n = t == MEFT_T_ROUTER_STEP ? s->experts : s->pairs;
            require(rows * cols == n, MEFT_E_SHAPE, "store_upload: counter length");
            if (t != MEFT_T_STAGED) {
                meft_dtype dt_;
                int64_t r_, c_;
                int32_t* dst = static_cast<int32_t*>(tensor_ptr(s, L, t, &dt_, &r_, &c_));
                int64_t* tmp = static_cast<int64_t*>(ctx->get("upload_a", size_t(n) * 8));
                MEFT_CUDA_CHECK(cudaMemcpyAsync(tmp, host, size_t(n) * 8, cudaMemcpyHostToDevice, ctx->stream));
                convert_index(ctx->stream, false, dst, tmp, n);
            } else {
                MEFT_CUDA_CHECK(cudaMemcpyAsync(L.staged, host, size_t(s->pairs), cudaMemcpyHostToDevice, ctx->stream));
            }
            MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            return;
        }
        require(t != MEFT_T_W_A_COMPUTE && t != MEFT_T_W_B_COMPUTE && t != MEFT_T_W_G_COMPUTE, MEFT_E_INVALID,
                "store_upload: compute copies are derived from the masters");
        meft_dtype dt;
        int64_t dr, dc;
        tensor_ptr(s, L, t, &dt, &dr, &dc);
        const int64_t er = is_a_family(t) ? s->d : dr, ec = is_a_family(t) ? s->pairs : dc;
        if (rows != er || cols != ec)
            throw MeftError(MEFT_E_SHAPE, "store_upload: expected " + std::to_string(er) + "x" + std::to_string(ec));
        upload_f64(ctx, s, L, t, static_cast<const double*>(host));
    });
}

meft_status meft_store_download_host(meft_ctx* ctx, meft_store* s, int64_t layer, meft_tensor t, void* host,
                                     int64_t rows, int64_t cols) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        if (is_staging(t)) ensure_staging(s, layer);
        if (t == MEFT_T_PAIR_STEP || t == MEFT_T_STAGED || t == MEFT_T_ROUTER_STEP) {
            const int64_t n = t == MEFT_T_ROUTER_STEP ? s->experts : s->pairs;
            require(rows * cols == n, MEFT_E_SHAPE, "store_download: counter length");
            if (t != MEFT_T_STAGED) {
                meft_dtype dt_;
                int64_t r_, c_;
                int32_t* src = static_cast<int32_t*>(tensor_ptr(s, L, t, &dt_, &r_, &c_));
                int64_t* tmp = static_cast<int64_t*>(ctx->get("upload_a", size_t(n) * 8));
                convert_index(ctx->stream, true, tmp, src, n);
                MEFT_CUDA_CHECK(cudaMemcpyAsync(host, tmp, size_t(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
            } else {
                MEFT_CUDA_CHECK(cudaMemcpyAsync(host, L.staged, size_t(s->pairs), cudaMemcpyDeviceToHost, ctx->stream));
            }
            MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
            return;
        }
        meft_dtype dt;
        int64_t dr, dc;
        tensor_ptr(s, L, t, &dt, &dr, &dc);
        const int64_t er = is_a_family(t) ? s->d : dr, ec = is_a_family(t) ? s->pairs : dc;
        if (rows != er || cols != ec)
            throw MeftError(MEFT_E_SHAPE, "store_download: expected " + std::to_string(er) + "x" + std::to_string(ec));
        download_f64(ctx, s, L, t, static_cast<double*>(host));
    });
}

meft_status meft_store_tensor(meft_store* s, int64_t layer, meft_tensor t, void** dev, meft_dtype* dt, int64_t* rows,
                              int64_t* cols) {
    return guarded(nullptr, [&] {
        const LayerBufs& L = layer_of(s, layer);
        if (is_staging(t)) {  // the caller may write through the view: the next Adam must consume staging
            ensure_staging(s, layer);
            s->pending[size_t(layer)] = 1;
        }
        meft_dtype d0;
        int64_t r0, c0;
        void* p = tensor_ptr(s, L, t, &d0, &r0, &c0);
        if (dev) *dev = p;
        if (dt) *dt = d0;
        if (rows) *rows = r0;
        if (cols) *cols = c0;
    });
}

meft_status meft_fetch(meft_ctx* ctx, meft_store* s, int64_t layer, const int32_t* S, int64_t n, void* keys_s,
                       void* values_s) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        validate_indices(ctx, S, n, s->pairs, "gather_adapter", true);
        const int es = s->prec == MEFT_STORE_F64 ? 8 : 2;
        if (n > 0) gather_rows2(ctx->stream, L.c_a, L.c_b, s->d * es, S, nullptr, n, keys_s, values_s);
    });
}

meft_status meft_scatter_grads(meft_ctx* ctx, meft_store* s, int64_t layer, const int32_t* S, int64_t n,
                               const void* gk, const void* gv, meft_dtype gdt) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        require(gdt == MEFT_F64 || gdt == MEFT_F32, MEFT_E_INVALID, "scatter_grads: gradient dtype must be F64/F32");
        if (n <= 0) return;
        const int code = validate_indices(ctx, S, n, s->pairs, "scatter_grads", false);
        ensure_staging(s, layer);
        s->pending[size_t(layer)] = 1;
        const int sdt = s->prec == MEFT_STORE_F64 ? 0 : 1;
        if (code == 0) {  // strictly ascending => unique rows => one CTA per row, no atomics
            stage_add(ctx->stream, sdt, L.st_a, s->d, S, n, dcode(gdt), gk, L.staged);
            stage_add(ctx->stream, sdt, L.st_b, s->d, S, n, dcode(gdt), gv, nullptr);
        } else {  // repeated indices (memtier.cpp:139-149 sums them in entry order): segmented by neuron id
            const size_t wb = stage_add_segmented_ws(n);
            void* ws = ctx->get("scatter_seg", wb);
            stage_add_segmented(ctx->stream, sdt, L.st_a, s->d, S, n, dcode(gdt), gk, L.staged, ws, wb);
            stage_add_segmented(ctx->stream, sdt, L.st_b, s->d, S, n, dcode(gdt), gv, nullptr, ws, wb);
        }
    });
}

meft_status meft_sparse_adam_update(meft_ctx* ctx, meft_store* s, int64_t layer, double beta1, double beta2,
                                    double eps, double lr) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        layer_of(s, layer);
        adam_impl(ctx, s, layer, beta1, beta2, eps, lr);
        s->key_stats_valid[size_t(layer)] = 0;
    });
}

// ------------------------------------------------------------------ fused layer step

static void ffn_update_impl(meft_ctx* ctx, meft_store* s, int64_t layer, const void* h, const void* g, int64_t T,
                            const int32_t* uni, int64_t su, int64_t holes, double b1, double b2, double eps,
                            double lr, float* out, float* grad_h, cudaEvent_t g_ready, cudaEvent_t fwd_done,
                            cudaEvent_t gh_done = nullptr, const int32_t* tau = nullptr, int64_t kk_eff = 0,
                            const meft_peer_out* peer = nullptr, const meft_base_ffn* base = nullptr,
                            const int32_t* su_dev = nullptr);

static void ensure_key_stats(meft_ctx* ctx, meft_store* s, int64_t layer);
static bool adam_epilogue_enabled(const meft_ctx* ctx);
static void finish_info(meft_ctx* ctx, const meft_store* s, int64_t T, int64_t k, meft_step_info* info);

static void layer_step_impl(meft_ctx* ctx, meft_store* s, int64_t layer, const void* h, const void* g, int64_t T,
                            int64_t kk, int64_t k, double b1, double b2, double eps, double lr, float* out,
                            float* grad_h, int32_t* per_token_user, int32_t* union_user, meft_step_info* info,
                            cudaEvent_t g_ready, cudaEvent_t fwd_done, cudaEvent_t gh_done = nullptr,
                            const meft_base_ffn* base = nullptr, bool defer_info = false) {
    // defer_info (enqueue-only step): the caller synchronises the stream later and then calls finish_info
    const long long launches0 = launch_counter();
    const LayerBufs& L = layer_of(s, layer);
    require(s->prec == MEFT_STORE_MIXED, MEFT_E_INVALID, "layer_step: requires a MIXED precision store");
    const int64_t d = s->d, M = s->pairs, N = s->experts;
    require(d % 8 == 0, MEFT_E_INVALID, "layer_step: d must be a multiple of 8");
    int64_t kk_eff = 0;
    int warned = 0;
    const int64_t take = selection_take(M, N, kk, k, &kk_eff, &warned);
    cudaStream_t st = ctx->stream;

    int32_t* per_token = per_token_user ? per_token_user
                                        : static_cast<int32_t*>(ctx->get("per_token", size_t(T * take) * 4));
    int32_t* uni = union_user ? union_user : static_cast<int32_t*>(ctx->get("union", size_t(M) * 4));
    int32_t* usize = ctx->dev_small + 4;
    // the routed experts: expert histogram, and the router's straight-through gradient when it trains
    int32_t* tau = static_cast<int32_t*>(ctx->get("tau_step", size_t(T * kk_eff) * 4));
    const size_t wsb = select_workspace_bytes(T, d, M, N, kk_eff);
    void* ws = ctx->get("select_ws", wsb);

    // meft_ffn: ke_select (experts.cpp:47-117)
    {
        PhaseScope ps(ctx, 0);
        ensure_key_stats(ctx, s, layer);  // cached across steps: the fused Adam refreshes the rows it updates
        ke_select_device(st, 2, h, L.c_g, L.c_a, T, d, M, N, kk_eff, take, ws, wsb, per_token, tau, uni, usize,
                         ctx->dev_small + 5, ctx->selection_mode == MEFT_SELECT_AUTO, L.kn, L.kl);
    }
    histogram_add(st, tau, T * kk_eff, L.ehist);
    // Enqueue-only step (host sync off): the FFN GEMMs are launched for the capacity M and read |S| from usize on
    // the device, so nothing here waits for the selection; otherwise |S| (and the union's hole count, which picks
    // the gather) is read back once and the GEMMs are sized exactly. Bit-identical either way.
    // AUTO host sync takes the device-sized step for a layer whose last read-back union was dense (one TMA run up to
    // a hole per 12,800 rows and at least 3/4 of M, so the capacity launch is ~|S|: cfg2, cfg3), re-reading |S| every
    // kUnionRecheck steps; any other union keeps the read-back (cfg1: capacity-sized launches and the padded gather
    // cost ~10% there). A forced device-sized step (host sync 0) with no dense read-back yet picks its gather from
    // the hole count of T * take uniform draws over M, M p (1 - p) with p = exp(-T take / M) (TMA from T take / M
    // >= ~9.5).
    constexpr int kUnionRecheck = 64;
    const size_t li = size_t(layer);
    const bool known_dense = s->union_dense[li] == 1;
    const bool recheck = !ctx->capturing() && (s->union_dense[li] < 0 || s->since_check[li] >= kUnionRecheck);
    const double p_miss = std::exp(-double(T) * double(take) / double(M));
    const int64_t holes_est = known_dense ? 0 : int64_t(std::ceil(double(M) * p_miss * (1.0 - p_miss)));
    const bool device_sized = (ctx->host_sync == 0 || (ctx->host_sync == MEFT_HOST_SYNC_AUTO && known_dense &&
                                                       !recheck)) &&
                              !s->pending[li] && !s->train_router && !(base && base->n > 0) && !ctx->check_finite &&
                              adam_epilogue_enabled(ctx) && d % 32 == 0 && M <= kGemmPanel;
    int64_t su = -1;
    if (device_sized && info && !defer_info)
        require(!ctx->capturing(), MEFT_E_INVALID,
                "layer_step: pass a NULL meft_step_info while capturing a graph (it is read back at the step's end)");
    if (device_sized) {
        ++s->since_check[li];
        ffn_update_impl(ctx, s, layer, h, g, T, uni, M, holes_est, b1, b2, eps, lr, out, grad_h, g_ready, fwd_done,
                        gh_done, nullptr, kk_eff, nullptr, nullptr, usize);
        if (info) {  // the step is fully enqueued: read |S| and the selection counters at its end
            MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small + 4, usize, 16, cudaMemcpyDeviceToHost, st));
            if (!defer_info) MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        }
    } else {
        require(!ctx->capturing(), MEFT_E_INVALID,
                "layer_step: this step reads the union size back (host sync on, or a step outside the enqueue-only "
                "conditions of meft_ctx_set_host_sync) and cannot be captured");
        union_holes(st, uni, usize, usize + 3);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small + 4, usize, 16, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        su = ctx->host_small[4];
        const int64_t holes = ctx->host_small[7];
        s->union_dense[li] = (holes >= 0 && holes * 12800 <= su && 4 * su >= 3 * M) ? 1 : 0;
        s->since_check[li] = 0;
        ffn_update_impl(ctx, s, layer, h, g, T, uni, su, ctx->host_small[7], b1, b2, eps, lr, out, grad_h, g_ready,
                        fwd_done, gh_done, s->train_router ? tau : nullptr, kk_eff, nullptr, base);
    }
    if (ctx->check_finite) {  // the reference's check_finite on its matmul outputs (kernels.cpp:7-13)
        int32_t* flag = ctx->dev_small + 20;
        MEFT_CUDA_CHECK(cudaMemsetAsync(flag, 0, 4, st));
        if (out) flag_nonfinite_f32(st, out, T * d, flag);
        if (grad_h) flag_nonfinite_f32(st, grad_h, T * d, flag);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small + 20, flag, 4, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        if (ctx->host_small[20]) throw MeftError(MEFT_E_NONFINITE, "layer_step: non-finite entry in out / grad_h");
    }

    if (info) {
        info->take = take;
        info->kk_eff = kk_eff;
        info->warned = warned;
        info->gpu_launches = int(launch_counter() - launches0);
        info->meter_hidden = T * d;
        info->router_flops = T * N * d;
        info->expert_scoring_flops = T * kk * (M / N) * d;
        if (!(device_sized && defer_info)) finish_info(ctx, s, T, k, info);
    }
    (void)su;
}

// The union-dependent fields of meft_step_info from the read-back |S| and selection counters (host_small[4..6]),
// once the stream has passed the step's read-back copy.
static void finish_info(meft_ctx* ctx, const meft_store* s, int64_t T, int64_t k, meft_step_info* info) {
    const int64_t su = ctx->host_small[4], d = s->d;
    info->union_size = su;
    info->rescored = ctx->host_small[5];
    info->fallbacks = ctx->host_small[6];
    info->meter_h2d = 2 * d * su;
    info->meter_d2h = 2 * d * su;
    info->beta_paper = double(su) / double(k);
    info->dedup_ratio = double(su) / double(T * k);
    info->activated_fraction = double(su) / double(s->pairs);
}

// fetch -> sparse_ffn_pa -> sparse_backward -> scatter_grads -> sparse_adam_update for T tokens against the union S
// (uni: ascending store-local pair ids, su of them), on a MIXED store.
// How the FFN GEMMs get the selected key/value rows (meft_ctx_set_gather; default from MEFT_GATHER=kernel|tma).
// TMA lets the GEMM producers fetch them (contiguous runs as plain boxes, the rest by tile::gather4) -- bitwise
// the same operand tiles as the materialised copy; AUTO picks it when the union is nearly one run (a broken
// 128-row piece costs ~4x its TMA issue), i.e. at most one hole per 12800 selected rows.
// meft_ctx_set_adam; default from MEFT_ADAM_EPILOGUE=0 (separate pass) for A/B comparisons (bitwise identical).
static bool adam_epilogue_enabled(const meft_ctx* ctx) {
    static const bool env_on = [] {
        const char* v = std::getenv("MEFT_ADAM_EPILOGUE");
        return !(v && v[0] == '0');
    }();
    return ctx->adam_mode < 0 ? env_on : ctx->adam_mode == MEFT_ADAM_EPILOGUE;
}

static bool use_tma_gather(const meft_ctx* ctx, int64_t su, int64_t holes) {
    static const int env_mode = [] {
        const char* v = std::getenv("MEFT_GATHER");
        if (!v) return int(MEFT_GATHER_AUTO);
        return std::strcmp(v, "kernel") == 0 ? int(MEFT_GATHER_KERNEL)
                                             : std::strcmp(v, "tma") == 0 ? int(MEFT_GATHER_TMA) : int(MEFT_GATHER_AUTO);
    }();
    const int mode = ctx->gather_mode >= 0 ? ctx->gather_mode : env_mode;
    if (mode == MEFT_GATHER_KERNEL || su <= 0) return false;
    if (mode == MEFT_GATHER_TMA) return true;
    return holes >= 0 && holes * 12800 <= su;
}

// Trainable router (train_router): straight-through gradient (trainer.cpp:140-181, router.cu) staged for the
// touched experts and applied by the router rows' lazy Adam with their own step counters (memtier.cpp:157-172,
// 211-227); the bf16 router copy the next selection reads is refreshed by the same kernel.
static void router_update_impl(meft_ctx* ctx, meft_store* s, int64_t layer, const uint16_t* h, const uint16_t* act,
                               const uint16_t* masked, int64_t ld, const int32_t* uni, int64_t su, const int32_t* tau,
                               int64_t T, int64_t kk, double b1, double b2, double eps, double lr) {
    const LayerBufs& L = layer_of(s, layer);
    cudaStream_t st = ctx->stream;
    const int64_t N = s->experts, d = s->d, E = s->pairs / s->experts;
    if (su <= 0) return;  // no union: every y_e is empty, nothing is touched
    PhaseScope ps(ctx, 4);
    int32_t* lo = static_cast<int32_t*>(ctx->get("rt_lo", size_t(N + 1) * 4));
    float* dldp = static_cast<float*>(ctx->get("rt_dldp", size_t(T * kk) * 4));
    uint8_t* live = static_cast<uint8_t*>(ctx->get("rt_live", size_t(T * kk)));
    float* gg = static_cast<float*>(ctx->get("rt_grad", size_t(N * d) * 4));
    uint8_t* touched = static_cast<uint8_t*>(ctx->get("rt_touched", size_t(N)));
    int32_t* rows = static_cast<int32_t*>(ctx->get("rt_rows", size_t(N) * 4));
    int32_t* bws = static_cast<int32_t*>(ctx->get("rt_bws", size_t((N + 1023) / 1024 + 1) * 4));
    router_ste_grads(st, uni, su, E, N, act, masked, ld, tau, T, kk, h, d, lo, dldp, live, gg, touched);
    compact_flags(st, touched, N, rows, ctx->dev_small + 9, bws);
    adam_mixed(st, rows, ctx->dev_small + 9, 0, d, static_cast<float*>(L.w_g), static_cast<float*>(L.m_g),
               static_cast<float*>(L.v_g), gg, static_cast<uint16_t*>(L.c_g), nullptr, nullptr, nullptr, nullptr,
               nullptr, L.rstep, nullptr, b1, b2, eps, lr, 1, true, false);
}

static void ffn_update_impl(meft_ctx* ctx, meft_store* s, int64_t layer, const void* h, const void* g, int64_t T,
                            const int32_t* uni, int64_t su, int64_t holes, double b1, double b2, double eps,
                            double lr, float* out, float* grad_h, cudaEvent_t g_ready, cudaEvent_t fwd_done,
                            cudaEvent_t gh_done, const int32_t* tau, int64_t kk_eff, const meft_peer_out* peer,
                            const meft_base_ffn* base, const int32_t* su_dev) {
    // su_dev != nullptr: su is the capacity (the store's M) and the union size lives on the device (the
    // enqueue-only step of layer_step_impl): every union-sized launch reads it there
    const LayerBufs& L = layer_of(s, layer);
    const int64_t d = s->d;
    cudaStream_t st = ctx->stream;
    // the z GEMM also writes the bitmask z > 0; the masked GEMM reads it instead of the bf16 act (64 MB instead of
    // 1 GB at cfg2). MEFT_ACT_BITS=0 reads act (A/B; bitwise identical).
    static const bool use_bits = [] {
        const char* v = std::getenv("MEFT_ACT_BITS");
        return !(v && v[0] == '0');
    }();
    // |S| > 65536: act and masked are stored as 65536-column panels ([T x 65536] each), so every chunked sub-GEMM
    // streams one dense panel instead of a strided window of a T x |S| matrix (MEFT_ACT_PANELS=0: one matrix)
    static const bool panels_on = [] {
        const char* v = std::getenv("MEFT_ACT_PANELS");
        return !(v && v[0] == '0');
    }();
    const bool panels = panels_on && use_bits && su > kGemmPanel && !s->train_router && !base;
    const int64_t ld = panels ? kGemmPanel : round_up(std::max<int64_t>(su, 1), 64);
    const int64_t panel = panels ? T * kGemmPanel : 0;
    const int64_t z_elems = panels ? ceil_div(su, kGemmPanel) * panel : T * ld;
    if (holes < 0 && su > 0 && use_tma_gather(ctx, su, 0)) {  // caller does not know: measure (one read-back)
        union_holes_n(st, uni, su, ctx->dev_small + 12);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(ctx->host_small + 12, ctx->dev_small + 12, 4, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        holes = ctx->host_small[12];
    }

    uint16_t* act = static_cast<uint16_t*>(ctx->get("act", size_t(z_elems) * 2));
    uint16_t* masked = static_cast<uint16_t*>(ctx->get("masked", size_t(z_elems) * 2));
    uint32_t* act_bits = use_bits ? static_cast<uint32_t*>(ctx->get(
                                        "act_bits", size_t(std::max<int64_t>(T * ((su + 31) / 32), 1)) * 4))
                                  : nullptr;
    float* outb = out ? out : static_cast<float*>(ctx->get("out", size_t(T * d) * 4));
    float* ghb = grad_h ? grad_h : static_cast<float*>(ctx->get("grad_h", size_t(T * d) * 4));
    // fetch (memtier.cpp:117-126): the selected key/value rows of the bf16 compute tables, either gathered inside
    // the GEMM operand loads (rg) or materialised by the gather kernel
    RowGather rg;
    const void* ks = L.c_a;
    const void* vs = L.c_b;
    if (use_tma_gather(ctx, su, holes)) {  // device-sized: `holes` is layer_step_impl's estimate
        rg.rows = uni;
        rg.table_rows = s->pairs;
    } else {
        uint16_t* ksb = static_cast<uint16_t*>(ctx->get("keys_s", size_t(std::max<int64_t>(su, 1) * d) * 2));
        uint16_t* vsb = static_cast<uint16_t*>(ctx->get("values_s", size_t(std::max<int64_t>(su, 1) * d) * 2));
        if (su > 0) {
            PhaseScope ps(ctx, 1);
            // device-sized: the union's rows plus zero rows up to the next multiple of 64 (apply_extent)
            gather_rows2(st, L.c_a, L.c_b, d * 2, uni, su_dev, su, ksb, vsb, su_dev != nullptr);
        }
        ks = ksb;
        vs = vsb;
    }

    // sparse_ffn_pa: the frozen base FFN first (adapter.cpp:118-120), then the adapter term (122-126) added onto
    // it; every token against the whole union
    if (base && base->n == 0) base = nullptr;
    // small fused-Adam steps: out / grad_h beside dA / the grad-W GEMMs (SmallFfnStreams; MEFT_SMALL_STREAMS=0 off)
    static const bool small_streams_env = [] {
        const char* v = std::getenv("MEFT_SMALL_STREAMS");
        return !(v && v[0] == '0');
    }();
    const bool fused_adam = !s->pending[size_t(layer)] && adam_epilogue_enabled(ctx) && d % 32 == 0 && d <= 65536;
    const bool small = ceil_div(T, int64_t(256)) * ceil_div(std::max<int64_t>(su, 1), int64_t(256)) < num_sms() / 2;
    const SmallFfnStreams ccs{ctx->side_stream, ctx->ev_z, ctx->ev_side_out, ctx->ev_da, ctx->ev_side_gh};
    const SmallFfnStreams* cc =
        small_streams_env && fused_adam && small && !base && !peer && !s->train_router && ctx->side_stream ? &ccs
                                                                                                          : nullptr;
    require(!(base && peer), MEFT_E_INVALID, "layer step: the base FFN runs on the token home, not with peer outputs");
    const int64_t ldn = base ? round_up(base->n, 8) : 0;
    uint16_t* base_pre = base ? static_cast<uint16_t*>(ctx->get("base_pre", size_t(T * ldn) * 2)) : nullptr;
    {
        PhaseScope ps(ctx, 2);
        if (base) {
            require(base->w_in && base->w_out && base->n % 8 == 0 && (base->act == 0 || base->act == 1),
                    MEFT_E_INVALID, "base FFN: w_in / w_out, n % 8 == 0, act 0 (SiLU) or 1 (ReLU)");
            uint16_t* base_act = static_cast<uint16_t*>(ctx->get("base_act", size_t(T * ldn) * 2));
            GemmEpilogue e1;  // pre = h w_in (kept for the backward), act(pre)
            e1.kind = EPI_ACT_BF16;
            e1.c = base_act;
            e1.ldc = ldn;
            e1.aux = base_pre;
            e1.ldaux = ldn;
            e1.act = base->act;
            gemm_bf16(st, T, base->n, d, GemmOperand{h, d, false}, GemmOperand{base->w_in, base->n, true}, e1);
            GemmEpilogue e2;  // out = act(pre) w_out
            e2.kind = EPI_STORE_F32;
            e2.c = outb;
            e2.ldc = d;
            gemm_bf16(st, T, d, base->n, GemmOperand{base_act, ldn, false}, GemmOperand{base->w_out, d, true}, e2);
        }
        ffn_forward_impl(ctx, MEFT_BF16, h, ks, vs, T, d, su, ld, act, outb, base != nullptr, rg, peer, act_bits,
                         panel, su_dev, cc);
    }
    if (fwd_done) MEFT_CUDA_CHECK(cudaEventRecord(fwd_done, cc ? cc->side : st));  // out is done
    if (g_ready) MEFT_CUDA_CHECK(cudaStreamWaitEvent(st, g_ready, 0));

    const bool stats_valid = s->key_stats_valid[size_t(layer)] != 0;
    require(!s->train_router || tau != nullptr, MEFT_E_LOGIC, "router training runs on the single-GPU layer step");
    if (base) {  // frozen-base backward (adapter.cpp:153-164): grad_h = ((G w_out^T) .* act'(pre)) w_in^T, first
        PhaseScope ps(ctx, 3);
        uint16_t* dpre = static_cast<uint16_t*>(ctx->get("base_dpre", size_t(T * ldn) * 2));
        GemmEpilogue e1;
        e1.kind = EPI_DACT_BF16;
        e1.c = dpre;
        e1.ldc = ldn;
        e1.aux = base_pre;
        e1.ldaux = ldn;
        e1.act = base->act;
        gemm_bf16(st, T, base->n, d, GemmOperand{g, d, false}, GemmOperand{base->w_out, d, false}, e1);
        GemmEpilogue e2;
        e2.kind = EPI_STORE_F32;
        e2.c = ghb;
        e2.ldc = d;
        gemm_bf16(st, T, d, base->n, GemmOperand{dpre, ldn, false}, GemmOperand{base->w_in, base->n, false}, e2);
    }
    auto train_router = [&] {  // after the backward: it reads act and masked
        if (s->train_router)
            router_update_impl(ctx, s, layer, static_cast<const uint16_t*>(h), act, masked, ld, uni, su, tau, T,
                               kk_eff, b1, b2, eps, lr);
    };
    require(!su_dev || (!s->pending[size_t(layer)] && !s->train_router && !base && !peer && !panels &&
                        adam_epilogue_enabled(ctx) && d % 32 == 0),
            MEFT_E_LOGIC, "device-sized layer step outside the fused-Adam path");
    if (s->pending[size_t(layer)]) {
        // earlier scatter_grads are pending: sparse_backward + scatter_grads fused, the weight-grad GEMM epilogues
        // add straight into the stage rows at S, then Adam consumes every staged pair (memtier.cpp:187-210)
        ensure_staging(s, layer);
        {
            PhaseScope ps(ctx, 3);
            ffn_backward_impl(ctx, MEFT_BF16, g, h, act, ks, vs, T, d, su, ld, masked, nullptr, nullptr, ghb,
                              base != nullptr, uni, L.st_a, L.st_b, rg, gh_done, nullptr, peer, nullptr, nullptr,
                              act_bits, panel);
        }
        train_router();
        PhaseScope ps(ctx, 4);
        if (su > 0) mark_rows(st, L.staged, uni, nullptr, su);
        adam_impl(ctx, s, layer, b1, b2, eps, lr);
    } else if (adam_epilogue_enabled(ctx) && d % 32 == 0 && d <= 65536) {
        // staging is all zero, so staged == S exactly and each weight-gradient row is final when its GEMM tile
        // drains: the sparse Adam (memtier.cpp:187-210) runs in those GEMMs' epilogues (EPI_ADAM_F32) on the
        // fp32 accumulator, overlapping the HBM-bound update with the tensor-bound mainloop -- no gradient block,
        // no separate pass. Per-pair steps advance once, before either GEMM (the key and value rows share them).
        float2* coef = static_cast<float2*>(ctx->get("adam_coef", size_t(std::max<int64_t>(su, 1)) * 8));
        const int64_t parts = ceil_div(d, int64_t(kAdamStatTile));
        const bool stats = stats_valid && su > 0;
        double* kss = stats ? static_cast<double*>(ctx->get("adam_kss", size_t(su * parts) * 8)) : nullptr;
        int32_t* klsb = stats ? static_cast<int32_t*>(ctx->get("adam_klsb", size_t(su * parts) * 4)) : nullptr;
        if (su > 0) adam_coef_bump(st, uni, su, L.step, coef, b1, b2, lr, su_dev);
        auto adam_epi = [&](bool keys) {
            GemmEpilogue e;
            e.kind = EPI_ADAM_F32;
            e.ldc = d;
            e.row_idx = uni;
            e.adam_w = static_cast<float*>(keys ? L.w_a : L.w_b);
            e.adam_m = keys ? L.m_a : L.m_b;
            e.adam_v = keys ? L.v_a : L.v_b;
            e.adam_mom16 = s->mom16;
            e.adam_c = static_cast<uint16_t*>(keys ? L.c_a : L.c_b);
            e.adam_coef = coef;
            e.b1 = float(b1);
            e.b2 = float(b2);
            e.eps = float(eps);
            if (keys && stats) {
                e.stat_ss = kss;
                e.stat_lsb = klsb;
                e.stat_ld = parts;
            }
            return e;
        };
        const GemmEpilogue ev = adam_epi(false), ek = adam_epi(true);
        {
            PhaseScope ps(ctx, 3);
            // MEFT_GW_KMAJOR=1: the grad-W GEMMs read [d x T] transposes of g and h (K-major B) -- an A/B knob
            static const bool kmajor = [] {
                const char* v = std::getenv("MEFT_GW_KMAJOR");
                return v && v[0] == '1';
            }();
            void* gT = nullptr;
            void* hT = nullptr;
            if (kmajor && su > 0) {
                gT = ctx->get("gT", size_t(T * d) * 2);
                hT = ctx->get("hT", size_t(T * d) * 2);
                transpose2(st, g, gT, T, d);
                transpose2(st, h, hT, T, d);
            }
            ffn_backward_impl(ctx, MEFT_BF16, g, h, act, ks, vs, T, d, su, ld, masked, nullptr, nullptr, ghb,
                              base != nullptr, nullptr, nullptr, nullptr, rg, gh_done, nullptr, peer, &ev, &ek,
                              act_bits, panel, gT, hT, su_dev, cc);
        }
        train_router();
        if (stats) {
            PhaseScope p4(ctx, 4);
            adam_stats_finalize(st, uni, su, kss, klsb, parts, L.kn, L.kl, su_dev);
        }
        return;  // key statistics stay valid (refreshed for exactly the rows that changed)
    } else {
        // staging is all zero, so staged == S exactly: the weight grads go to a dense [|S| x d] step block that
        // Adam reads in place of the staging rows (same values, no staging traffic, nothing to zero). ONE block
        // serves both tables: the value rows are updated right after their gradient GEMM (no counter bump), then
        // the key gradient overwrites the block and the key rows are updated with the shared step counter.
        float* gblk = static_cast<float*>(ctx->get("step_grad", size_t(std::max<int64_t>(su, 1) * d) * 4));
        auto adam_table = [&](int table) {
            PhaseScope p4(ctx, 4);
            const bool keys = table == 1;
            adam_mixed(st, uni, nullptr, su, d, static_cast<float*>(L.w_a), L.m_a, L.v_a, gblk,
                       static_cast<uint16_t*>(L.c_a), static_cast<float*>(L.w_b), L.m_b, L.v_b, gblk,
                       static_cast<uint16_t*>(L.c_b), L.step, nullptr, b1, b2, eps, lr, table, keys, true,
                       keys && stats_valid ? L.kn : nullptr, keys && stats_valid ? L.kl : nullptr, s->mom16);
        };
        std::optional<PhaseScope> p3;
        p3.emplace(ctx, 3);
        const std::function<void()> values_step = [&] {
            p3.reset();
            if (su > 0) adam_table(2);
            p3.emplace(ctx, 3);
        };
        ffn_backward_impl(ctx, MEFT_BF16, g, h, act, ks, vs, T, d, su, ld, masked, gblk, gblk, ghb, base != nullptr,
                          nullptr, nullptr, nullptr, rg, gh_done, &values_step, peer, nullptr, nullptr, act_bits,
                          panel);
        p3.reset();
        train_router();
        if (su > 0) adam_table(1);
        return;  // key statistics stay valid (refreshed for exactly the rows that changed)
    }
    s->key_stats_valid[size_t(layer)] = 0;
}

// Cached norms / minimum LSB exponents of a layer's bf16 compute keys (the certified selection's inputs).
static void ensure_key_stats(meft_ctx* ctx, meft_store* s, int64_t layer) {
    const LayerBufs& L = layer_of(s, layer);
    require(s->prec == MEFT_STORE_MIXED, MEFT_E_INVALID, "key stats: requires a MIXED precision store");
    if (s->key_stats_valid[size_t(layer)]) return;
    row_stats(ctx->stream, static_cast<const uint16_t*>(L.c_a), s->pairs, s->d, L.kn, L.kl);
    s->key_stats_valid[size_t(layer)] = 1;
}

// ------------------------------------------------------------------ expert-sharded layer building blocks

meft_status meft_route_select(meft_ctx* ctx, const uint16_t* h, const uint16_t* w_g, int64_t T, int64_t d, int64_t N,
                              int64_t kk, int32_t* tau) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        if (kk < 1) throw MeftError(MEFT_E_INVALID, "select_experts: budget must be >= 1");
        require(N >= 1 && d % 8 == 0, MEFT_E_INVALID, "route_select: N >= 1 and d % 8 == 0 required");
        void* ws = ctx->get("route_ws", route_workspace_bytes(T, d, N));
        route_certified(ctx->stream, h, w_g, T, d, N, std::min(kk, N), ws, tau, nullptr);
    });
}

meft_status meft_row_stats(meft_ctx* ctx, const uint16_t* rows, int64_t n, int64_t d, float* norms, int32_t* minlsb) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        row_stats(ctx->stream, rows, n, d, norms, minlsb);
    });
}

meft_status meft_store_key_stats(meft_ctx* ctx, meft_store* s, int64_t layer, float* norms, int32_t* minlsb) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        ensure_key_stats(ctx, s, layer);
        if (norms)
            MEFT_CUDA_CHECK(cudaMemcpyAsync(norms, L.kn, size_t(s->pairs) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        if (minlsb)
            MEFT_CUDA_CHECK(cudaMemcpyAsync(minlsb, L.kl, size_t(s->pairs) * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    });
}

meft_status meft_score_candidates(meft_ctx* ctx, meft_store* s, int64_t layer, const uint16_t* rows,
                                  const int32_t* expert_local, int64_t R, float* cand) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        require(s->prec == MEFT_STORE_MIXED && s->d % 8 == 0, MEFT_E_INVALID, "score_candidates: MIXED store, d % 8");
        const int64_t E = s->pairs / s->experts;
        require(E % 4 == 0, MEFT_E_INVALID, "score_candidates: expert size must be a multiple of 4");
        void* ws = ctx->get("score_ws", score_workspace_bytes(R, s->d, s->experts, E));
        score_candidates(ctx->stream, rows, expert_local, R, s->d, static_cast<const uint16_t*>(L.c_a), s->experts, E,
                         ws, cand);
    });
}

meft_status meft_exact_scores(meft_ctx* ctx, meft_store* s, int64_t layer, const uint16_t* rows, int64_t R,
                              const int32_t* pair_row, const int32_t* pair_key, int64_t Q, double* out) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        const LayerBufs& L = layer_of(s, layer);
        ensure_key_stats(ctx, s, layer);
        float* rn = static_cast<float*>(ctx->get("rows_norm", size_t(std::max<int64_t>(R, 1)) * 4));
        int32_t* rl = static_cast<int32_t*>(ctx->get("rows_lsb", size_t(std::max<int64_t>(R, 1)) * 4));
        row_stats(ctx->stream, rows, R, s->d, rn, rl);
        exact_pair_scores(ctx->stream, rows, rn, rl, static_cast<const uint16_t*>(L.c_a), L.kn, L.kl, pair_row,
                          pair_key, Q, s->d, out, nullptr);
    });
}

meft_status meft_topk_classify(meft_ctx* ctx, const float* cand, const int32_t* tau, int64_t T, int64_t kk, int64_t E,
                               int64_t take, int64_t d, const float* hn, const float* kn, int32_t* sure,
                               int32_t* n_sure, int32_t* amb, int32_t* n_amb) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(take >= 1 && take <= kk * E, MEFT_E_INVALID, "topk_classify: 1 <= take <= kk*E");
        topk_classify(ctx->stream, cand, tau, T, kk, E, take, d, hn, kn, sure, n_sure, amb, n_amb, nullptr);
    });
}

meft_status meft_topk_finalize(meft_ctx* ctx, const int32_t* sure, const int32_t* n_sure, const int32_t* amb,
                               const int32_t* n_amb, const double* x, int64_t T, int64_t C, int64_t take,
                               int32_t* per_token, uint8_t* union_flags) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        topk_finalize(ctx->stream, sure, n_sure, amb, n_amb, x, T, C, take, per_token, union_flags);
    });
}

meft_status meft_layer_ffn_local(meft_ctx* ctx, meft_store* s, int64_t layer, const uint16_t* h_all,
                                 const uint16_t* g_all, int64_t T, const int32_t* S_local, int64_t su, double beta1,
                                 double beta2, double eps, double lr, float* out_partial, float* grad_h_partial,
                                 void* g_ready, void* fwd_done, void* grad_h_done, const meft_peer_out* peer) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        layer_of(s, layer);
        require(s->prec == MEFT_STORE_MIXED && s->d % 8 == 0, MEFT_E_INVALID, "layer_ffn_local: MIXED store, d % 8");
        if (peer)
            require(peer->rows * peer->world == T, MEFT_E_SHAPE, "layer_ffn_local: peer rows * world must equal T");
        ffn_update_impl(ctx, s, layer, h_all, g_all, T, S_local, su, -1, beta1, beta2, eps, lr, out_partial,
                        grad_h_partial, static_cast<cudaEvent_t>(g_ready), static_cast<cudaEvent_t>(fwd_done),
                        static_cast<cudaEvent_t>(grad_h_done), nullptr, 0, peer);
    });
}

meft_status meft_peer_reduce(meft_ctx* ctx, const float* recv, int world, int64_t rows, int64_t d, float* out) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(world >= 1 && world <= kMaxPeers && rows >= 0 && d >= 0, MEFT_E_INVALID, "peer_reduce: arguments");
        slot_sum(ctx->stream, recv, world, rows * d, out);
    });
}

meft_status meft_ipc_handle(meft_ctx* ctx, void* dev_ptr, void* handle64) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
        cudaIpcMemHandle_t hnd;
        MEFT_CUDA_CHECK(cudaIpcGetMemHandle(&hnd, dev_ptr));
        std::memcpy(handle64, &hnd, sizeof(hnd));
    });
}

meft_status meft_ipc_open(meft_ctx* ctx, const void* handle64, void** dev_ptr) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        cudaIpcMemHandle_t hnd;
        std::memcpy(&hnd, handle64, sizeof(hnd));
        MEFT_CUDA_CHECK(cudaIpcOpenMemHandle(dev_ptr, hnd, cudaIpcMemLazyEnablePeerAccess));
    });
}

meft_status meft_ipc_close(meft_ctx* ctx, void* dev_ptr) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        MEFT_CUDA_CHECK(cudaIpcCloseMemHandle(dev_ptr));
    });
}

meft_status meft_layer_step(meft_ctx* ctx, meft_store* s, int64_t layer, const void* h, const void* grad_out,
                            int64_t T, int64_t kk, int64_t k, double beta1, double beta2, double eps, double lr,
                            float* out, float* grad_h, int32_t* per_token, int32_t* union_idx, meft_step_info* info) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(T >= 1, MEFT_E_SHAPE, "layer_step: no tokens");
        layer_step_impl(ctx, s, layer, h, grad_out, T, kk, k, beta1, beta2, eps, lr, out, grad_h, per_token, union_idx,
                        info, nullptr, nullptr);
    });
}

meft_status meft_layer_step_base(meft_ctx* ctx, meft_store* s, int64_t layer, const void* h, const void* grad_out,
                                 int64_t T, int64_t kk, int64_t k, double beta1, double beta2, double eps, double lr,
                                 float* out, float* grad_h, int32_t* per_token, int32_t* union_idx,
                                 meft_step_info* info, const meft_base_ffn* base) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(T >= 1, MEFT_E_SHAPE, "layer_step: no tokens");
        layer_step_impl(ctx, s, layer, h, grad_out, T, kk, k, beta1, beta2, eps, lr, out, grad_h, per_token, union_idx,
                        info, nullptr, nullptr, nullptr, base);
    });
}

meft_status meft_layer_step_host(meft_ctx* ctx, meft_store* s, int64_t layer, const uint16_t* h_host,
                                 const uint16_t* g_host, int64_t T, int64_t kk, int64_t k, double beta1, double beta2,
                                 double eps, double lr, float* out_host, float* grad_h_host, meft_step_info* info) {
    return guarded(ctx, [&] {
        require_ctx(ctx);
        require(T >= 1, MEFT_E_SHAPE, "layer_step: no tokens");
        require(s != nullptr, MEFT_E_INVALID, "null store");
        const int64_t d = s->d;
        const size_t in_bytes = size_t(T * d) * 2, out_bytes = size_t(T * d) * 4;
        void* hd = ctx->get("h_in", in_bytes);
        void* gd = ctx->get("g_in", in_bytes);
        float* od = static_cast<float*>(ctx->get("out_dev", out_bytes));
        float* ghd = static_cast<float*>(ctx->get("gh_dev", out_bytes));
        // h on the compute stream; grad_out on the copy stream, overlapping selection + forward. grad_out starts
        // after h has arrived (MEFT_H2D_SERIAL=0: at once), so h -- on the critical path of the selection -- gets
        // the whole host link instead of sharing it with a transfer needed only by the backward.
        static const bool h_first = [] {
            const char* v = std::getenv("MEFT_H2D_SERIAL");
            return !(v && v[0] == '0');
        }();
        MEFT_CUDA_CHECK(cudaMemcpyAsync(hd, h_host, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
        if (h_first) {
            MEFT_CUDA_CHECK(cudaEventRecord(ctx->ev_h_in, ctx->stream));
            MEFT_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_h_in, 0));
        }
        MEFT_CUDA_CHECK(cudaMemcpyAsync(gd, g_host, in_bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
        MEFT_CUDA_CHECK(cudaEventRecord(ctx->ev_in, ctx->copy_stream));
        // The copy stream carries both results back while compute continues: out after the forward, grad_h as soon
        // as its GEMM (scheduled right after `masked`) is done -- overlapping the weight-gradient GEMMs and Adam.
        // The copies are enqueued after the step is (the events are recorded inside it).
        layer_step_impl(ctx, s, layer, hd, gd, T, kk, k, beta1, beta2, eps, lr, od, ghd, nullptr, nullptr, info,
                        ctx->ev_in, ctx->ev_fwd, ctx->ev_out, nullptr, /*defer_info=*/true);
        if (out_host) {
            MEFT_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_fwd, 0));
            MEFT_CUDA_CHECK(cudaMemcpyAsync(out_host, od, out_bytes, cudaMemcpyDeviceToHost, ctx->copy_stream));
        }
        if (grad_h_host) {
            MEFT_CUDA_CHECK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_out, 0));
            MEFT_CUDA_CHECK(cudaMemcpyAsync(grad_h_host, ghd, out_bytes, cudaMemcpyDeviceToHost, ctx->copy_stream));
        }
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->copy_stream));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (info) finish_info(ctx, s, T, k, info);  // idempotent when the step already synchronised
    });
}

}  // extern "C"
