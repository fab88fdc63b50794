// The expert-sharded MEFT layer step behind the C ABI (include/meft_cuda.h meft_layer_step_sharded):
// the protocol of paper_2406_04984_b200/sharded.py composed from the library's own building blocks (certified
// routing, grouped tcgen05 candidate scoring, exact re-scoring, certified classification, the fused FFN + lazy
// Adam of the local union) with the exchanges issued here, over NCCL or host callbacks.
//
// Per step, rank r of P (T tokens each, shard = experts [r*N/P, (r+1)*N/P) and pairs [r*M/P, (r+1)*M/P)):
//   all-gather h, grad_out -> route (exact tau) -> dispatch plan (device) -> counts all-gather -> all-to-all of
//   (token id, owner-local expert) entries -> owners gather the token rows from the all-gathered h and score them ->
//   candidate scores all-to-all back -> key norms all-gather -> certified classification -> exact re-scoring
//   requests all-to-all -> exact scores back -> finalize -> MAX all-reduce of the union bitmap -> FFN + Adam of the
//   local union over all P*T tokens, its out / grad_h GEMMs storing every row straight into the row's home over peer
//   memory (the reduce-scatter fused into the epilogue) -> barrier -> each home folds its slots.
// Every host-visible count is read once per exchange (the all-to-all sizes), exactly where sharded.py reads them.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/meft_cuda.h"
#include "common.cuh"
#include "select.h"

using namespace meft_dev;

meft_status meft_internal_fail(meft_ctx* ctx, int code, const char* msg);  // meft_capi.cu

namespace {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;  // optional (>= 2.18)
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // the copy already mapped into the process (e.g. torch's) first, so both share one NCCL
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.CommSplit = reinterpret_cast<decltype(api.CommSplit)>(sym("ncclCommSplit"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.AllReduce &&
                 api.ReduceScatter && api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    if (!api.ok) throw MeftError(MEFT_E_NCCL, "NCCL unavailable: " + api.why);
    return api;
}

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw MeftError(MEFT_E_NCCL, std::string(what) + ": " + (nccl().GetErrorString(r) ?: "nccl error"));
}

// ---------------------------------------------------------------- communicators
struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    // device buffers, stream-ordered on `st`
    virtual void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
    virtual void all_to_all_v(const void* send, const std::vector<size_t>& send_bytes, void* recv,
                              const std::vector<size_t>& recv_bytes, cudaStream_t st) = 0;
    virtual void all_reduce_max_u8(uint8_t* buf, size_t n, cudaStream_t st) = 0;
    virtual void reduce_scatter_sum_f32(const float* send, float* recv, size_t n_per_rank, cudaStream_t st) = 0;
    // host metadata: every rank's `bytes` in rank order (synchronous)
    virtual void all_gather_host(const void* send, size_t bytes, void* recv, cudaStream_t st) = 0;
    // every rank's work enqueued on `st` before the barrier is complete before any rank's work after it
    virtual void barrier(cudaStream_t st) = 0;
    // the ranks share one process (device pointers are valid across them; no IPC)
    virtual bool same_process() const = 0;
    // All-gather on a second communicator and stream, started once `ready` (recorded on the caller's stream) has
    // fired; returns the event that fires when it is done, or nullptr when this communicator cannot overlap (the
    // caller then all-gathers in stream order).
    virtual cudaEvent_t all_gather_behind(const void*, void*, size_t, cudaEvent_t, cudaStream_t) { return nullptr; }
};

std::vector<size_t> offsets(const std::vector<size_t>& n) {
    std::vector<size_t> o(n.size() + 1, 0);
    for (size_t i = 0; i < n.size(); ++i) o[i + 1] = o[i] + n[i];
    return o;
}

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    bool owned = false;
    void* meta = nullptr;  // device scratch for host metadata all-gathers
    size_t meta_bytes = 0;
    int32_t* word = nullptr;  // the barrier's one-word all-reduce
    // bulk exchanges that overlap the step: a communicator split off `comm` (collective: every rank creates it in its
    // first step) with its own stream, so its kernels never queue behind the selection's collectives
    ncclComm_t bulk = nullptr;
    cudaStream_t bulk_stream = nullptr;
    cudaEvent_t bulk_done = nullptr;
    bool bulk_tried = false;
    ~NcclComm() override {
        if (meta) cudaFree(meta);
        if (word) cudaFree(word);
        if (bulk) nccl().CommDestroy(bulk);
        if (bulk_done) cudaEventDestroy(bulk_done);
        if (bulk_stream) cudaStreamDestroy(bulk_stream);
        if (owned && comm) nccl().CommDestroy(comm);
    }
    cudaEvent_t all_gather_behind(const void* send, void* recv, size_t bytes, cudaEvent_t ready,
                                  cudaStream_t st) override {
        if (!bulk_tried) {  // every rank takes this branch in the same (first) step
            bulk_tried = true;
            int32_t ok = 0;
            if (nccl().CommSplit && nccl().CommSplit(comm, 0, rank, &bulk, nullptr) == ncclSuccess) {
                ok = cudaStreamCreateWithFlags(&bulk_stream, cudaStreamNonBlocking) == cudaSuccess &&
                     cudaEventCreateWithFlags(&bulk_done, cudaEventDisableTiming) == cudaSuccess;
                if (!ok) cudaGetLastError();
            } else {
                bulk = nullptr;
            }
            // all ranks use the split communicator, or none does (a rank without it would never join its collectives)
            std::vector<int32_t> every(static_cast<size_t>(world));
            all_gather_host(&ok, 4, every.data(), st);
            for (int32_t e : every) ok &= e;
            if (!ok && bulk) {
                nccl().CommDestroy(bulk);
                bulk = nullptr;
            }
        }
        if (!bulk) return nullptr;
        MEFT_CUDA_CHECK(cudaStreamWaitEvent(bulk_stream, ready, 0));
        nck(nccl().AllGather(send, recv, bytes, ncclInt8, bulk, bulk_stream), "ncclAllGather (bulk)");
        MEFT_CUDA_CHECK(cudaEventRecord(bulk_done, bulk_stream));
        return bulk_done;
    }
    bool same_process() const override { return false; }
    void barrier(cudaStream_t st) override {
        if (!word) MEFT_CUDA_CHECK(cudaMalloc(&word, 4));
        nck(nccl().AllReduce(word, word, 1, ncclInt32, ncclSum, comm, st), "ncclAllReduce (barrier)");
    }
    void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        nck(nccl().AllGather(send, recv, bytes, ncclInt8, comm, st), "ncclAllGather");
    }
    void all_to_all_v(const void* send, const std::vector<size_t>& sb, void* recv, const std::vector<size_t>& rb,
                      cudaStream_t st) override {
        const auto so = offsets(sb), ro = offsets(rb);
        nck(nccl().GroupStart(), "ncclGroupStart");
        for (int p = 0; p < world; ++p) {
            if (sb[size_t(p)])
                nck(nccl().Send(static_cast<const uint8_t*>(send) + so[size_t(p)], sb[size_t(p)], ncclInt8, p, comm, st),
                    "ncclSend");
            if (rb[size_t(p)])
                nck(nccl().Recv(static_cast<uint8_t*>(recv) + ro[size_t(p)], rb[size_t(p)], ncclInt8, p, comm, st),
                    "ncclRecv");
        }
        nck(nccl().GroupEnd(), "ncclGroupEnd");
    }
    void all_reduce_max_u8(uint8_t* buf, size_t n, cudaStream_t st) override {
        nck(nccl().AllReduce(buf, buf, n, ncclUint8, ncclMax, comm, st), "ncclAllReduce");
    }
    void reduce_scatter_sum_f32(const float* send, float* recv, size_t n, cudaStream_t st) override {
        nck(nccl().ReduceScatter(send, recv, n, ncclFloat32, ncclSum, comm, st), "ncclReduceScatter");
    }
    void all_gather_host(const void* send, size_t bytes, void* recv, cudaStream_t st) override {
        const size_t need = bytes * size_t(world + 1);
        if (meta_bytes < need) {
            if (meta) MEFT_CUDA_CHECK(cudaFree(meta));
            meta = nullptr;
            MEFT_CUDA_CHECK(cudaMalloc(&meta, need));
            meta_bytes = need;
        }
        uint8_t* mine = static_cast<uint8_t*>(meta) + bytes * size_t(world);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(mine, send, bytes, cudaMemcpyHostToDevice, st));
        all_gather(mine, meta, bytes, st);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(recv, meta, bytes * size_t(world), cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
    }
};

struct HostComm final : Comm {
    meft_host_comm cb{};
    void call(int rc, const char* what) {
        if (rc != 0) throw MeftError(MEFT_E_NCCL, std::string("host communicator: ") + what + " failed");
    }
    bool same_process() const override { return true; }
    void barrier(cudaStream_t st) override {
        const uint8_t b = 1;
        std::vector<uint8_t> all(static_cast<size_t>(world));
        all_gather_host(&b, 1, all.data(), st);  // synchronises this rank's stream first
    }
    void all_gather_host(const void* send, size_t bytes, void* recv, cudaStream_t st) override {
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        call(cb.all_gather(cb.user, send, bytes, recv), "all_gather");
    }
    void all_gather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
        std::vector<uint8_t> hs(bytes), hr(bytes * size_t(world));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, bytes, cudaMemcpyDeviceToHost, st));
        all_gather_host(hs.data(), bytes, hr.data(), st);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    void all_to_all_v(const void* send, const std::vector<size_t>& sb, void* recv, const std::vector<size_t>& rb,
                      cudaStream_t st) override {
        const size_t ns = std::accumulate(sb.begin(), sb.end(), size_t(0));
        const size_t nr = std::accumulate(rb.begin(), rb.end(), size_t(0));
        std::vector<uint8_t> hs(std::max<size_t>(ns, 1)), hr(std::max<size_t>(nr, 1));
        if (ns) MEFT_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, ns, cudaMemcpyDeviceToHost, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        call(cb.all_to_all_v(cb.user, hs.data(), sb.data(), hr.data(), rb.data()), "all_to_all_v");
        if (nr) MEFT_CUDA_CHECK(cudaMemcpyAsync(recv, hr.data(), nr, cudaMemcpyHostToDevice, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    void all_reduce_max_u8(uint8_t* buf, size_t n, cudaStream_t st) override {
        std::vector<uint8_t> hs(n), hr(n * size_t(world));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(hs.data(), buf, n, cudaMemcpyDeviceToHost, st));
        all_gather_host(hs.data(), n, hr.data(), st);
        for (int p = 1; p < world; ++p)
            for (size_t i = 0; i < n; ++i) hr[i] = std::max(hr[i], hr[size_t(p) * n + i]);
        MEFT_CUDA_CHECK(cudaMemcpyAsync(buf, hr.data(), n, cudaMemcpyHostToDevice, st));
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
    }
    void reduce_scatter_sum_f32(const float* send, float* recv, size_t n, cudaStream_t st) override {
        // every rank's partial rows of this home (slot order), summed on the device in slot order like the fold of
        // the fused peer path (the exchange itself is the host all-gather)
        std::vector<float> hs(n * size_t(world)), hr(n * size_t(world) * size_t(world));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(hs.data(), send, hs.size() * 4, cudaMemcpyDeviceToHost, st));
        all_gather_host(hs.data(), hs.size() * 4, hr.data(), st);
        std::vector<float> mine(n * size_t(world));  // [slot p][n] = rank p's partial rows of home `rank`
        for (int p = 0; p < world; ++p)
            std::memcpy(mine.data() + size_t(p) * n, hr.data() + (size_t(p) * size_t(world) + size_t(rank)) * n, n * 4);
        float* dev = nullptr;
        MEFT_CUDA_CHECK(cudaMalloc(&dev, mine.size() * 4));
        MEFT_CUDA_CHECK(cudaMemcpyAsync(dev, mine.data(), mine.size() * 4, cudaMemcpyHostToDevice, st));
        slot_sum_launch(dev, n, recv, st);
        MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
        MEFT_CUDA_CHECK(cudaFree(dev));
    }
    void slot_sum_launch(const float* slots, size_t n, float* out, cudaStream_t st);
};

// ---------------------------------------------------------------- per-context state
struct Scratch {
    std::unordered_map<std::string, std::pair<void*, size_t>> bufs;
    ~Scratch() {
        for (auto& kv : bufs) cudaFree(kv.second.first);
    }
    template <class T>
    T* get(const std::string& name, size_t count) {
        auto& b = bufs[name];
        const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
        if (b.second < bytes) {
            if (b.first) MEFT_CUDA_CHECK(cudaFree(b.first));
            b.first = nullptr;
            b.second = 0;
            const cudaError_t e = cudaMalloc(&b.first, bytes);
            if (e != cudaSuccess) {
                cudaGetLastError();
                throw MeftError(MEFT_E_OOM, "sharded step: cannot allocate " + std::to_string(bytes) + " bytes for " +
                                                name);
            }
            b.second = bytes;
        }
        return static_cast<T*>(b.first);
    }
};

// Receive buffers of the reduce-scatter fused into the out / grad_h GEMM epilogues (EPI_PEER_F32, meft_peer_out):
// each home owns [world x rows x d] fp32 for out and for grad_h; every rank maps every home's pair (CUDA IPC across
// processes, plain pointers when the ranks share a process) and its GEMMs store each output row straight into the
// row's home at slot = its rank; the home folds the slots in slot order (meft_peer_reduce) after a barrier.
struct PeerSet {
    int world = 0;
    int64_t rows = 0, d = 0;
    bool ready = false, failed = false;
    void* own[2] = {nullptr, nullptr};
    std::vector<void*> opened;
    meft_peer_out desc{};
    void release() {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        opened.clear();
        for (void*& p : own) {
            if (p) cudaFree(p);
            p = nullptr;
        }
        ready = false;
    }
    ~PeerSet() { release(); }
};

struct ShardCtx {
    std::unique_ptr<Comm> comm;
    Scratch scratch;
    PeerSet peers;
    int last_peer = 0, last_overlap = 0;  // meft_ctx_sharded_paths
    cudaEvent_t in_ready = nullptr;  // the step's inputs are ready (start of the overlapped grad_out all-gather)
    ~ShardCtx() {
        if (in_ready) cudaEventDestroy(in_ready);
    }
};

// Map every home's receive buffers on every rank; all ranks agree (twice: after allocation / export and after
// opening) so that either all use the fused path or all fall back to the reduce-scatter collectives.
bool setup_peers(Comm& cm, PeerSet& ps, int64_t rows, int64_t d, cudaStream_t st, bool wanted) {
    if (ps.world == cm.world && ps.rows == rows && ps.d == d && (ps.ready || ps.failed)) return ps.ready;
    ps.release();
    ps.failed = false;
    ps.world = cm.world;
    ps.rows = rows;
    ps.d = d;
    const size_t bytes = size_t(cm.world) * size_t(rows) * size_t(d) * 4;
    struct Rec {
        int32_t ok, pad;
        uint64_t ptr[2];
        unsigned char handle[2][64];
    };
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
    Rec mine{};
    mine.ok = wanted ? 1 : 0;  // a rank that opts out (MEFT_SHARDED_PEER=0) takes every rank to the fallback
    for (int i = 0; i < 2 && mine.ok; ++i) {
        if (cudaMalloc(&ps.own[i], bytes) != cudaSuccess) {
            cudaGetLastError();
            ps.own[i] = nullptr;
            mine.ok = 0;
            break;
        }
        mine.ptr[i] = reinterpret_cast<uint64_t>(ps.own[i]);
        if (!cm.same_process()) {
            cudaIpcMemHandle_t h;
            if (cudaIpcGetMemHandle(&h, ps.own[i]) != cudaSuccess) {
                cudaGetLastError();
                mine.ok = 0;
            } else {
                std::memcpy(mine.handle[i], &h, 64);
            }
        }
    }
    std::vector<Rec> all(static_cast<size_t>(cm.world));
    cm.all_gather_host(&mine, sizeof(Rec), all.data(), st);
    int32_t mapped = 1;
    for (const Rec& r : all) mapped &= r.ok;
    if (mapped) {
        ps.desc = meft_peer_out{};
        ps.desc.world = cm.world;
        ps.desc.rank = cm.rank;
        ps.desc.rows = rows;
        for (int p = 0; p < cm.world && mapped; ++p) {
            float* base[2];
            for (int i = 0; i < 2; ++i) {
                if (p == cm.rank || cm.same_process()) {
                    base[i] = reinterpret_cast<float*>(all[size_t(p)].ptr[i]);
                    continue;
                }
                cudaIpcMemHandle_t h;
                std::memcpy(&h, all[size_t(p)].handle[i], 64);
                void* q = nullptr;
                if (cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    mapped = 0;
                    break;
                }
                ps.opened.push_back(q);
                base[i] = static_cast<float*>(q);
            }
            if (mapped) {
                ps.desc.out_recv[p] = base[0];
                ps.desc.grad_h_recv[p] = base[1];
            }
        }
    }
    std::vector<int32_t> every(static_cast<size_t>(cm.world));
    cm.all_gather_host(&mapped, 4, every.data(), st);
    for (int32_t m : every) mapped &= m;
    if (!mapped) {
        ps.release();
        ps.failed = true;
        return false;
    }
    ps.ready = true;
    return true;
}

std::mutex g_mu;
std::unordered_map<const meft_ctx*, std::unique_ptr<ShardCtx>> g_shard;

ShardCtx& shard_of(meft_ctx* ctx) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& p = g_shard[ctx];
    if (!p) p.reset(new ShardCtx());
    return *p;
}

// errors are recorded the way every other entry point records them (meft_last_error of the context / thread)
template <class F>
meft_status guard(meft_ctx* ctx, F&& f) {
    try {
        f();
        return MEFT_OK;
    } catch (const MeftError& e) {
        return meft_internal_fail(ctx, e.code, e.what());
    } catch (const std::bad_alloc&) {
        return meft_internal_fail(ctx, MEFT_E_OOM, "host allocation failed");
    } catch (const std::exception& e) {
        return meft_internal_fail(ctx, MEFT_E_CUDA, e.what());
    }
}

void ok(meft_status st, meft_ctx* ctx) {
    if (st != MEFT_OK) throw MeftError(int(st), meft_last_error(ctx));
}

// ---------------------------------------------------------------- small kernels of the protocol
// dispatch entry p: (global token row base + order[p] / kk, owner-local expert)
__global__ void k_dispatch_entries(const int32_t* __restrict__ order, const int32_t* __restrict__ send_exp, int n,
                                   int kk, int base, int2* __restrict__ out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = make_int2(base + order[p] / kk, send_exp[p]);
}

// owner side: rows[i] = h_all[entries[i].x] (bf16, 16-byte vectors, warp per row), experts[i] = entries[i].y
__global__ void k_gather_entries(const uint16_t* __restrict__ h_all, int d, const int2* __restrict__ entries, int n,
                                 uint16_t* __restrict__ rows, int32_t* __restrict__ experts) {
    const int lane = threadIdx.x & 31, nv = d / 8;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
        const int2 e = entries[r];
        const uint4* s = reinterpret_cast<const uint4*>(h_all + int64_t(e.x) * d);
        uint4* o = reinterpret_cast<uint4*>(rows + int64_t(r) * d);
        for (int v = lane; v < nv; v += 32) o[v] = __ldg(s + v);
        if (lane == 0) experts[r] = e.y;
    }
}

__global__ void k_pack_pairs(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int n, int2* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = make_int2(a[i], b[i]);
}

__global__ void k_unpack_pairs(const int2* __restrict__ in, int n, int32_t* __restrict__ a, int32_t* __restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        a[i] = in[i].x;
        b[i] = in[i].y;
    }
}

__global__ void k_count_nonzero(const uint8_t* __restrict__ f, int64_t n, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        c += f[i] != 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_slot_sum(const float* __restrict__ slots, int world, int64_t n, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        float s = slots[i];
        for (int p = 1; p < world; ++p) s += slots[int64_t(p) * n + i];
        out[i] = s;
    }
}

int blocks(int64_t n, int per = 256) { return int(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 65535))); }

void HostComm::slot_sum_launch(const float* slots, size_t n, float* out, cudaStream_t st) {
    k_slot_sum<<<blocks(int64_t(n)), 256, 0, st>>>(slots, world, int64_t(n), out);
    check_launch("k_slot_sum");
}

// ---------------------------------------------------------------- the step
void sharded_step(meft_ctx* ctx, ShardCtx& sc, meft_store* store, int64_t layer, const uint16_t* w_g,
                  const uint16_t* h, const uint16_t* g, int64_t T, int64_t kk, int64_t k, double b1, double b2,
                  double eps, double lr, float* out, float* grad_h, int32_t* per_token_user, meft_step_info* info) {
    Comm& cm = *sc.comm;
    Scratch& S = sc.scratch;
    const int P = cm.world, r = cm.rank;
    int64_t layers = 0, d = 0, M_loc = 0, N_loc = 0;
    meft_precision prec;
    ok(meft_store_info(store, &layers, &d, &M_loc, &N_loc, &prec), ctx);
    if (prec == MEFT_STORE_F64) throw MeftError(MEFT_E_INVALID, "layer_step_sharded: needs a MIXED or COMPACT store");
    if (T < 1) throw MeftError(MEFT_E_SHAPE, "layer_step_sharded: no tokens");
    if (d % 8) throw MeftError(MEFT_E_INVALID, "layer_step_sharded: d must be a multiple of 8");
    if (!h || !g || !w_g || !out || !grad_h) throw MeftError(MEFT_E_INVALID, "layer_step_sharded: null buffer");
    const int64_t N = N_loc * P, M = M_loc * P, E = M / N;
    int64_t take = 0, kk_eff = 0;
    int warned = 0;
    ok(meft_selection_shape(M, N, kk, k, &take, &kk_eff, &warned), ctx);
    const int64_t C = kk_eff * E, n = T * kk_eff, TT = T * P;
    cudaStream_t st = static_cast<cudaStream_t>(meft_ctx_stream(ctx));
    const long long launches0 = meft_kernel_launches();

    {  // every rank must bring the same number of tokens (the homes' row blocks of the P*T-row products)
        std::vector<int64_t> ts(static_cast<size_t>(P));
        cm.all_gather_host(&T, 8, ts.data(), st);
        for (int p = 0; p < P; ++p)
            if (ts[size_t(p)] != T)
                throw MeftError(MEFT_E_SHAPE, "layer_step_sharded: rank " + std::to_string(p) + " brings " +
                                                  std::to_string(ts[size_t(p)]) + " tokens, this rank " +
                                                  std::to_string(T) + " (all ranks need the same T)");
    }
    // all-gather the hidden states and the incoming gradient (rank order: rank p's tokens are rows [p*T, (p+1)*T)).
    // grad_out is needed only by the backward: over NCCL it travels on the bulk communicator behind the selection
    // and the forward, and the FFN waits for it (g_ready) just before its backward GEMMs. Its buffer's previous
    // readers (the last step's backward) precede `in_ready` on this stream.
    uint16_t* h_all = S.get<uint16_t>("h_all", size_t(TT * d));
    uint16_t* g_all = S.get<uint16_t>("g_all", size_t(TT * d));
    if (!sc.in_ready) MEFT_CUDA_CHECK(cudaEventCreateWithFlags(&sc.in_ready, cudaEventDisableTiming));
    MEFT_CUDA_CHECK(cudaEventRecord(sc.in_ready, st));
    cudaEvent_t g_ready = cm.all_gather_behind(g, g_all, size_t(T * d) * 2, sc.in_ready, st);
    cm.all_gather(h, h_all, size_t(T * d) * 2, st);
    if (!g_ready) cm.all_gather(g, g_all, size_t(T * d) * 2, st);
    sc.last_overlap = g_ready ? 1 : 0;

    // 1. route this rank's tokens (certified, exact tau)
    int32_t* tau = S.get<int32_t>("tau", size_t(n));
    ok(meft_route_select(ctx, h, w_g, T, d, N, kk, tau), ctx);
    // 2. dispatch plan; owners receive (token id, owner-local expert) entries and gather the rows themselves
    int32_t* send_exp = S.get<int32_t>("send_exp", size_t(n));
    int32_t* order = S.get<int32_t>("order", size_t(n));
    int32_t* inv = S.get<int32_t>("inv", size_t(n));
    std::vector<int64_t> send_cnt(static_cast<size_t>(P));
    ok(meft_shard_dispatch(ctx, tau, T, kk_eff, N_loc, P, h, d, nullptr, send_exp, order, inv, send_cnt.data()), ctx);
    std::vector<int64_t> cmat(static_cast<size_t>(P) * P);  // cmat[src * P + dst]: entries src dispatches to dst
    cm.all_gather_host(send_cnt.data(), size_t(P) * 8, cmat.data(), st);
    std::vector<int64_t> recv_cnt(static_cast<size_t>(P));
    for (int s = 0; s < P; ++s) recv_cnt[size_t(s)] = cmat[size_t(s) * P + size_t(r)];
    const int64_t R = std::accumulate(recv_cnt.begin(), recv_cnt.end(), int64_t(0));
    int2* entries = S.get<int2>("entries", size_t(n));
    k_dispatch_entries<<<blocks(n), 256, 0, st>>>(order, send_exp, int(n), int(kk_eff), int(r * T), entries);
    check_launch("k_dispatch_entries");
    std::vector<size_t> sb(static_cast<size_t>(P)), rb(static_cast<size_t>(P));
    for (int p = 0; p < P; ++p) {
        sb[size_t(p)] = size_t(send_cnt[size_t(p)]) * 8;
        rb[size_t(p)] = size_t(recv_cnt[size_t(p)]) * 8;
    }
    int2* recv_entries = S.get<int2>("recv_entries", size_t(std::max<int64_t>(R, 1)));
    cm.all_to_all_v(entries, sb, recv_entries, rb, st);
    uint16_t* recv_rows = S.get<uint16_t>("recv_rows", size_t(std::max<int64_t>(R, 1) * d));
    int32_t* recv_exp = S.get<int32_t>("recv_exp", size_t(std::max<int64_t>(R, 1)));
    if (R) {
        k_gather_entries<<<std::max(1, std::min(int(R / 8 + 1), num_sms() * 16)), 256, 0, st>>>(
            h_all, int(d), recv_entries, int(R), recv_rows, recv_exp);
        check_launch("k_gather_entries");
    }
    // 3-4. owners score the received rows against their experts' keys; scores travel back in dispatch order
    float* cand_recv = S.get<float>("cand_recv", size_t(std::max<int64_t>(R, 1) * E));
    if (R) ok(meft_score_candidates(ctx, store, layer, recv_rows, recv_exp, R, cand_recv), ctx);
    for (int p = 0; p < P; ++p) {
        sb[size_t(p)] = size_t(recv_cnt[size_t(p)] * E) * 4;  // answers go back to the sources
        rb[size_t(p)] = size_t(send_cnt[size_t(p)] * E) * 4;
    }
    float* cand_back = S.get<float>("cand_back", size_t(n * E));
    cm.all_to_all_v(cand_recv, sb, cand_back, rb, st);
    float* cand = S.get<float>("cand", size_t(n * E));
    ok(meft_shard_unpermute_rows(ctx, cand_back, order, n, E, cand), ctx);
    float* hn = S.get<float>("hn", size_t(T));
    int32_t* hl = S.get<int32_t>("hl", size_t(T));
    ok(meft_row_stats(ctx, h, T, d, hn, hl), ctx);
    float* kn_loc = S.get<float>("kn_loc", size_t(M_loc));
    float* kn = S.get<float>("kn", size_t(M));
    ok(meft_store_key_stats(ctx, store, layer, kn_loc, nullptr), ctx);
    cm.all_gather(kn_loc, kn, size_t(M_loc) * 4, st);
    // 5. certified classification at the token home
    int32_t* sure = S.get<int32_t>("sure", size_t(T * take));
    int32_t* n_sure = S.get<int32_t>("n_sure", size_t(T));
    int32_t* amb = S.get<int32_t>("amb", size_t(T * C));
    int32_t* n_amb = S.get<int32_t>("n_amb", size_t(T));
    ok(meft_topk_classify(ctx, cand, tau, T, kk_eff, E, take, d, hn, kn, sure, n_sure, amb, n_amb), ctx);
    // 6. exact re-scoring of the ambiguous candidates by their owners: a request names the owner's receive row of the
    // token's dispatched entry (this rank's block starts after the entries of lower source ranks) and the local key
    std::vector<int64_t> send_off(static_cast<size_t>(P), 0), row_base(static_cast<size_t>(P));
    for (int o = 1; o < P; ++o) send_off[size_t(o)] = send_off[size_t(o - 1)] + send_cnt[size_t(o - 1)];
    for (int o = 0; o < P; ++o) {
        int64_t before = 0;
        for (int s = 0; s < r; ++s) before += cmat[size_t(s) * P + size_t(o)];
        row_base[size_t(o)] = before - send_off[size_t(o)];
    }
    int32_t* req_row = S.get<int32_t>("req_row", size_t(T * C));
    int32_t* req_key = S.get<int32_t>("req_key", size_t(T * C));
    int32_t* back = S.get<int32_t>("back", size_t(T * C));
    std::vector<int64_t> rsend(static_cast<size_t>(P));
    int64_t n_req = 0;
    ok(meft_shard_requests(ctx, amb, n_amb, tau, inv, T, C, kk_eff, E, M_loc, P, row_base.data(), req_row, req_key,
                           back, rsend.data(), &n_req),
       ctx);
    std::vector<int64_t> rmat(static_cast<size_t>(P) * P);
    cm.all_gather_host(rsend.data(), size_t(P) * 8, rmat.data(), st);
    std::vector<int64_t> rrecv(static_cast<size_t>(P));
    for (int s = 0; s < P; ++s) rrecv[size_t(s)] = rmat[size_t(s) * P + size_t(r)];
    const int64_t Q = std::accumulate(rrecv.begin(), rrecv.end(), int64_t(0));
    int2* req = S.get<int2>("req", size_t(std::max<int64_t>(n_req, 1)));
    if (n_req) {
        k_pack_pairs<<<blocks(n_req), 256, 0, st>>>(req_row, req_key, int(n_req), req);
        check_launch("k_pack_pairs");
    }
    for (int p = 0; p < P; ++p) {
        sb[size_t(p)] = size_t(rsend[size_t(p)]) * 8;
        rb[size_t(p)] = size_t(rrecv[size_t(p)]) * 8;
    }
    int2* in_req = S.get<int2>("in_req", size_t(std::max<int64_t>(Q, 1)));
    cm.all_to_all_v(req, sb, in_req, rb, st);
    int32_t* in_row = S.get<int32_t>("in_row", size_t(std::max<int64_t>(Q, 1)));
    int32_t* in_key = S.get<int32_t>("in_key", size_t(std::max<int64_t>(Q, 1)));
    double* x_out = S.get<double>("x_out", size_t(std::max<int64_t>(Q, 1)));
    if (Q) {
        k_unpack_pairs<<<blocks(Q), 256, 0, st>>>(in_req, int(Q), in_row, in_key);
        check_launch("k_unpack_pairs");
        ok(meft_exact_scores(ctx, store, layer, recv_rows, R, in_row, in_key, Q, x_out), ctx);
    }
    for (int p = 0; p < P; ++p) {  // exact fp64 scores back to the requesters (same byte counts)
        sb[size_t(p)] = size_t(rrecv[size_t(p)]) * 8;
        rb[size_t(p)] = size_t(rsend[size_t(p)]) * 8;
    }
    double* x_back = S.get<double>("x_back", size_t(std::max<int64_t>(n_req, 1)));
    cm.all_to_all_v(x_out, sb, x_back, rb, st);
    double* xs = S.get<double>("xs", size_t(T * C));
    MEFT_CUDA_CHECK(cudaMemsetAsync(xs, 0, size_t(T * C) * 8, st));
    if (n_req) ok(meft_shard_scatter_f64(ctx, x_back, back, n_req, xs), ctx);
    // 7. final per-token selection (global pair ids) and the global union: MAX all-reduce of the M-byte bitmap
    int32_t* per_token = per_token_user ? per_token_user : S.get<int32_t>("per_token", size_t(T * take));
    uint8_t* flags = S.get<uint8_t>("flags", size_t(M));
    MEFT_CUDA_CHECK(cudaMemsetAsync(flags, 0, size_t(M), st));
    ok(meft_topk_finalize(ctx, sure, n_sure, amb, n_amb, xs, T, C, take, per_token, flags), ctx);
    cm.all_reduce_max_u8(flags, size_t(M), st);
    // this owner's part of the union, as ascending local pair ids
    int32_t* S_loc = S.get<int32_t>("S_loc", size_t(M_loc));
    int32_t* cnt = S.get<int32_t>("cnt", 4);
    int32_t* bws = S.get<int32_t>("bws", size_t(M_loc / 1024 + 2));
    compact_flags(st, flags + size_t(r) * size_t(M_loc), M_loc, S_loc, cnt, bws);
    unsigned long long* ucount = reinterpret_cast<unsigned long long*>(cnt + 2);
    MEFT_CUDA_CHECK(cudaMemsetAsync(ucount, 0, 8, st));
    k_count_nonzero<<<blocks(M, 1024), 256, 0, st>>>(flags, M, ucount);
    check_launch("k_count_nonzero");
    int32_t host_cnt[4] = {0, 0, 0, 0};
    MEFT_CUDA_CHECK(cudaMemcpyAsync(host_cnt, cnt, 16, cudaMemcpyDeviceToHost, st));
    MEFT_CUDA_CHECK(cudaStreamSynchronize(st));
    const int64_t su = host_cnt[0];
    unsigned long long union_size = 0;
    std::memcpy(&union_size, host_cnt + 2, 8);
    // 8-9. FFN over all P*T tokens on the local part of the union (fused scatter + lazy Adam), partial sums home:
    // pushed by the out / grad_h GEMM epilogues straight into the homes' receive buffers over peer memory and
    // folded there in slot order (MEFT_SHARDED_PEER=0, or a rank that cannot map the buffers: reduce-scatters)
    static const bool peer_env = [] {
        const char* v = std::getenv("MEFT_SHARDED_PEER");
        return !(v && v[0] == '0');
    }();
    sc.last_peer = setup_peers(cm, sc.peers, T, d, st, peer_env) ? 1 : 0;
    if (sc.last_peer) {
        ok(meft_layer_ffn_local(ctx, store, layer, h_all, g_all, TT, S_loc, su, b1, b2, eps, lr, nullptr, nullptr,
                                g_ready, nullptr, nullptr, &sc.peers.desc),
           ctx);
        cm.barrier(st);  // every rank's rows are in this home's slots
        ok(meft_peer_reduce(ctx, static_cast<const float*>(sc.peers.own[0]), P, T, d, out), ctx);
        ok(meft_peer_reduce(ctx, static_cast<const float*>(sc.peers.own[1]), P, T, d, grad_h), ctx);
    } else {
        float* out_p = S.get<float>("out_p", size_t(TT * d));
        float* gh_p = S.get<float>("gh_p", size_t(TT * d));
        ok(meft_layer_ffn_local(ctx, store, layer, h_all, g_all, TT, S_loc, su, b1, b2, eps, lr, out_p, gh_p, g_ready,
                                nullptr, nullptr, nullptr),
           ctx);
        cm.reduce_scatter_sum_f32(out_p, out, size_t(T * d), st);
        cm.reduce_scatter_sum_f32(gh_p, grad_h, size_t(T * d), st);
    }
    if (info) {
        std::memset(info, 0, sizeof(*info));
        info->union_size = int64_t(union_size);
        info->take = take;
        info->kk_eff = kk_eff;
        info->warned = warned;
        info->gpu_launches = int(meft_kernel_launches() - launches0);
        info->rescored = int(n_req);
        info->meter_h2d = 2 * d * int64_t(union_size);
        info->meter_d2h = 2 * d * int64_t(union_size);
        info->meter_hidden = TT * d;
        info->beta_paper = double(union_size) / double(k);
        info->dedup_ratio = double(union_size) / double(TT * k);
        info->activated_fraction = double(union_size) / double(M);
        info->router_flops = TT * N * d;
        info->expert_scoring_flops = TT * kk * E * d;
    }
}

}  // namespace

extern "C" {

meft_status meft_nccl_unique_id(void* id128) {
    return guard(nullptr, [&] {
        if (!id128) throw MeftError(MEFT_E_INVALID, "nccl_unique_id: null output");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
    });
}

meft_status meft_ctx_comm_init(meft_ctx* ctx, const void* id128, int rank, int world) {
    return guard(ctx, [&] {
        if (!ctx || !id128 || world < 1 || rank < 0 || rank >= world)
            throw MeftError(MEFT_E_INVALID, "ctx_comm_init: ctx, id, 0 <= rank < world");
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        std::unique_ptr<NcclComm> c(new NcclComm());
        nck(nccl().CommInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
        c->owned = true;
        c->rank = rank;
        c->world = world;
        shard_of(ctx).comm = std::move(c);
    });
}

meft_status meft_ctx_set_comm(meft_ctx* ctx, void* nccl_comm, int rank, int world) {
    return guard(ctx, [&] {
        if (!ctx || !nccl_comm || world < 1 || rank < 0 || rank >= world)
            throw MeftError(MEFT_E_INVALID, "ctx_set_comm: ctx, comm, 0 <= rank < world");
        nccl();  // fail now if NCCL cannot be loaded
        std::unique_ptr<NcclComm> c(new NcclComm());
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        c->rank = rank;
        c->world = world;
        shard_of(ctx).comm = std::move(c);
    });
}

meft_status meft_ctx_set_host_comm(meft_ctx* ctx, const meft_host_comm* cb, int rank, int world) {
    return guard(ctx, [&] {
        if (!ctx || !cb || !cb->all_gather || !cb->all_to_all_v || world < 1 || rank < 0 || rank >= world)
            throw MeftError(MEFT_E_INVALID, "ctx_set_host_comm: ctx, callbacks, 0 <= rank < world");
        std::unique_ptr<HostComm> c(new HostComm());
        c->cb = *cb;
        c->rank = rank;
        c->world = world;
        shard_of(ctx).comm = std::move(c);
    });
}

meft_status meft_ctx_clear_comm(meft_ctx* ctx) {
    return guard(ctx, [&] {
        std::lock_guard<std::mutex> lk(g_mu);
        g_shard.erase(ctx);
    });
}

meft_status meft_layer_step_sharded(meft_ctx* ctx, meft_store* shard, int64_t layer, const uint16_t* w_g,
                                    const uint16_t* h, const uint16_t* grad_out, int64_t T, int64_t kk, int64_t k,
                                    double beta1, double beta2, double eps, double lr, float* out, float* grad_h,
                                    int32_t* per_token, meft_step_info* info) {
    return guard(ctx, [&] {
        if (!ctx || !shard) throw MeftError(MEFT_E_INVALID, "layer_step_sharded: null context or store");
        ShardCtx& sc = shard_of(ctx);
        if (!sc.comm) throw MeftError(MEFT_E_LOGIC, "layer_step_sharded: the context has no communicator");
        sharded_step(ctx, sc, shard, layer, w_g, h, grad_out, T, kk, k, beta1, beta2, eps, lr, out, grad_h, per_token,
                     info);
    });
}

meft_status meft_ctx_sharded_paths(meft_ctx* ctx, int* peer, int* overlap) {
    return guard(ctx, [&] {
        if (!ctx) throw MeftError(MEFT_E_INVALID, "sharded_paths: null context");
        const ShardCtx& sc = shard_of(ctx);
        if (peer) *peer = sc.last_peer;
        if (overlap) *overlap = sc.last_overlap;
    });
}

}  // extern "C"
