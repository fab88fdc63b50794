/* meft_cuda.h — C ABI of libmeft_cuda.so, the B200 (sm_100a) implementation of the MEFT sparse
 * Key-Experts adapter layer (arXiv 2406.04984).
 *
 * This is the thin layer under the drop-in C++ host API (include/meft/<name>.hpp, the same declarations as
 * the reference's proj/include/meft headers). Every entry point names the reference function it replaces
 * (paths relative to /root/reference/proj). Plain pointers and sizes only — no torch or CUDA types.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers unless a function name ends in _host.
 *  - Work is enqueued on the context's stream; only calls that must return a host-visible size
 *    synchronise (documented per function).
 *  - Key tables are NEURON-MAJOR: row j of `keys` [pairs x d] is column j of the reference's w_a (d x r,
 *    adapter.hpp:20-26). Values [pairs x d] are the reference's w_b rows unchanged. The *_host store
 *    transfers convert from/to the reference layouts.
 *  - Indices on device are int32 (pairs < 2^31); the drop-in shim widens to index_t (int64).
 *  - Errors map to the reference's exception taxonomy: MEFT_E_SHAPE -> ShapeError,
 *    MEFT_E_INVALID -> std::invalid_argument, MEFT_E_RANGE -> std::out_of_range (offending index via
 *    meft_last_error_index), MEFT_E_LOGIC -> std::logic_error, MEFT_E_NONFINITE -> runtime_error("...non-finite...").
 *  - One host thread per context at a time.
 */
#ifndef MEFT_CUDA_H
#define MEFT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum meft_status {
    MEFT_OK = 0,
    MEFT_E_SHAPE = 1,
    MEFT_E_INVALID = 2,
    MEFT_E_RANGE = 3,
    MEFT_E_LOGIC = 4,
    MEFT_E_NONFINITE = 5,
    MEFT_E_CUDA = 6,
    MEFT_E_NCCL = 7,
    MEFT_E_OOM = 8,
    /* MEFT1 checkpoints (memtier.hpp:172-183): CheckpointHeaderError, CheckpointShapeError,
     * CheckpointTruncatedError; I/O failures map to std::runtime_error. */
    MEFT_E_CKPT_HEADER = 9,
    MEFT_E_CKPT_SHAPE = 10,
    MEFT_E_CKPT_TRUNCATED = 11,
    MEFT_E_IO = 12
} meft_status;

typedef enum meft_dtype { MEFT_F64 = 0, MEFT_F32 = 1, MEFT_BF16 = 2 } meft_dtype;

/* Store precision. F64 mirrors the reference HostStore bit for bit (API-fidelity mode); MIXED keeps fp32
 * master weights / Adam moments / staging plus bf16 compute copies (the performance mode). COMPACT is MIXED with
 * the Adam moments m, v stored in bf16 (round to nearest even after every update; the update itself runs in fp32):
 * 20 bytes of tables per (pair, dim) instead of 28, so BASELINE config 3 (32 LLaMA-7B-width layers) fits one
 * B200. Opt-in; its Adam tolerance is stated in DESIGN.md §5 and pinned by tests/test_gpu_compact.py. */
typedef enum meft_precision { MEFT_STORE_F64 = 0, MEFT_STORE_MIXED = 1, MEFT_STORE_COMPACT = 2 } meft_precision;

/* Per-layer store tensors (HostLayer, memtier.hpp:90-106). Reference layouts for _host transfers:
 * W_A, M_A, V_A, STAGE_A are d x r; W_B, M_B, V_B, STAGE_B are r x d; W_G is N x d; PAIR_STEP is int64[r];
 * STAGED is int8[r]. On device every pair tensor is neuron-major [r x d]. *_COMPUTE are the bf16 copies the
 * kernels read in MIXED mode. */
typedef enum meft_tensor {
    MEFT_T_W_A = 0,
    MEFT_T_W_B = 1,
    MEFT_T_W_G = 2,
    MEFT_T_M_A = 3,
    MEFT_T_V_A = 4,
    MEFT_T_M_B = 5,
    MEFT_T_V_B = 6,
    MEFT_T_STAGE_A = 7,
    MEFT_T_STAGE_B = 8,
    MEFT_T_PAIR_STEP = 9,
    MEFT_T_STAGED = 10,
    MEFT_T_W_A_COMPUTE = 11,
    MEFT_T_W_B_COMPUTE = 12,
    MEFT_T_W_G_COMPUTE = 13,
    /* router training state (train_router; memtier.cpp:86-91): N x d moments, int64[N] step counters on the host
     * side (int32 on device); available after meft_store_enable_router, MEFT_E_LOGIC otherwise */
    MEFT_T_M_G = 14,
    MEFT_T_V_G = 15,
    MEFT_T_ROUTER_STEP = 16
} meft_tensor;

typedef struct meft_ctx meft_ctx;
typedef struct meft_store meft_store;

/* ------------------------------------------------------------------ context, errors, memory */

const char* meft_version(void);
/* device = CUDA ordinal; stream = a cudaStream_t, NULL for the legacy default stream, or MEFT_OWN_STREAM for a
 * private non-blocking stream owned by the context. */
#define MEFT_OWN_STREAM ((void*)(intptr_t)-1)
meft_status meft_ctx_create(int device, void* stream, meft_ctx** out);
void meft_ctx_destroy(meft_ctx* ctx);
void* meft_ctx_stream(meft_ctx* ctx);
const char* meft_last_error(const meft_ctx* ctx); /* ctx may be NULL: last error of this thread */
int64_t meft_last_error_index(const meft_ctx* ctx);
meft_status meft_synchronize(meft_ctx* ctx);
/* Number of kernels this library has launched from the calling thread (for launch accounting). */
int64_t meft_kernel_launches(void);

/* Per-phase device timing of meft_layer_step with CUDA events recorded on the context stream:
 * phase 0 selection (ke_select), 1 fetch (row gather), 2 FFN forward GEMMs, 3 FFN backward GEMMs (scatter
 * fused into their epilogues), 4 sparse Adam (staged compaction + update). read_timing synchronises, returns
 * the accumulated milliseconds and kernel launches per phase since the last read, and resets them. */
meft_status meft_ctx_set_timing(meft_ctx* ctx, int enable);

/* Selection algorithm for bf16 inputs. AUTO (default): certified tensor-core scoring with exact fp64 re-scoring
 * of the ambiguous candidates (select_tc.cuh); EXACT: fp64 SIMT scoring of every candidate. Both return the
 * reference's indices bit for bit; EXACT exists to cross-validate AUTO at full size. */
#define MEFT_SELECT_AUTO 0
#define MEFT_SELECT_EXACT 1
meft_status meft_ctx_set_selection(meft_ctx* ctx, int mode);

/* How the fused layer step's FFN GEMMs read the selected key/value rows (the reference's fetch,
 * memtier.cpp:117-126): KERNEL materialises them with a gather kernel; TMA has the GEMM producers load them
 * straight from the tables (contiguous runs of the union as plain TMA boxes, the rest with tile::gather4);
 * AUTO (default; environment MEFT_GATHER=kernel|tma overrides) takes TMA when the union is nearly one run.
 * Both give bit-identical results. */
#define MEFT_GATHER_AUTO 0
#define MEFT_GATHER_KERNEL 1
#define MEFT_GATHER_TMA 2
meft_status meft_ctx_set_gather(meft_ctx* ctx, int mode);
/* Where the fused layer step runs the lazy sparse Adam (memtier.cpp:187-210) when no scatter_grads are pending:
 * EPILOGUE (default; environment MEFT_ADAM_EPILOGUE=0 selects PASS) applies it inside the two weight-gradient
 * GEMMs' epilogues to the fp32 accumulator rows as they drain, overlapping the HBM-bound update with the
 * tensor-bound mainloop; PASS writes the gradients to a [|S| x d] block and runs a separate Adam kernel.
 * Both give bit-identical tables, moments and counters. */
#define MEFT_ADAM_EPILOGUE 0
#define MEFT_ADAM_PASS 1
meft_status meft_ctx_set_adam(meft_ctx* ctx, int mode);
/* The reference runs check_finite on every matmul output and the trainer turns the runtime_error into
 * DivergenceError (kernels.cpp:7-13, trainer.cpp:504-518). With enable != 0 the fused layer steps scan out and
 * grad_h once the step is done (one extra sync) and return MEFT_E_NONFINITE ("... non-finite ...") on NaN / Inf.
 * Default off: the scan costs a sync per step. */
meft_status meft_ctx_set_check_finite(meft_ctx* ctx, int enable);
/* Host synchronisation of the fused layer step. enable = 1: meft_layer_step reads the union size back once,
 * mid-step, and sizes the FFN GEMMs to it. enable = 0: the step never waits for the device -- the six FFN
 * GEMMs are launched for the capacity (M pairs) and read |S| from device memory before their first tile
 * (GemmEpilogue::extent), so consecutive layer steps enqueue back to back and a step can be captured into a CUDA
 * graph (meft_graph_*). Bit-identical results. It applies to the fused-Adam step (no pending scatter_grads, no base
 * FFN, no router training, check_finite off, M <= 65536, d % 32 == 0); any other step takes the synchronising
 * path (an error while capturing). A non-NULL info then costs one synchronisation at the END of the step.
 * MEFT_HOST_SYNC_AUTO (the default; environment MEFT_HOST_SYNC=0|1|auto for new contexts): the enqueue-only step
 * for a layer whose last read-back union was dense (one TMA run up to a hole per 12,800 rows and >= 3/4 of M: the
 * capacity launch is ~|S|; the LLaMA-shape layer), re-read every 64 steps; the read-back otherwise (a sparse union
 * would launch for far more than it selects). Capture needs 0 (or an AUTO layer already known dense). */
#define MEFT_HOST_SYNC_AUTO (-1)
meft_status meft_ctx_set_host_sync(meft_ctx* ctx, int enable);

/* CUDA graphs over the context stream. meft_graph_begin starts capturing the context stream; the calls that follow
 * must only enqueue work (e.g. meft_layer_step with host sync off, after one eager warm-up step so every scratch
 * buffer already exists -- an allocation while capturing fails the capture); meft_graph_end instantiates the
 * graph; meft_graph_launch replays it on the context stream (inputs and outputs are the captured buffers). */
typedef struct meft_graph meft_graph;
meft_status meft_graph_begin(meft_ctx* ctx);
meft_status meft_graph_end(meft_ctx* ctx, meft_graph** graph);
meft_status meft_graph_launch(meft_ctx* ctx, meft_graph* graph);
void meft_graph_destroy(meft_graph* graph);

/* Keep `sms` SMs free of the persistent tcgen05 GEMMs (process-wide; 0 = all SMs). The expert-sharded step sets it
 * while collectives are meant to overlap its FFN: NCCL's kernels need SMs of their own to make progress. */
meft_status meft_set_gemm_sm_reserve(int sms);
meft_status meft_ctx_read_timing(meft_ctx* ctx, double* ms5, int64_t* launches5);

meft_status meft_device_alloc(meft_ctx* ctx, size_t bytes, void** out);
meft_status meft_device_free(meft_ctx* ctx, void* ptr);
meft_status meft_host_alloc(meft_ctx* ctx, size_t bytes, void** out); /* pinned */
meft_status meft_host_free(meft_ctx* ctx, void* ptr);
meft_status meft_copy_to_device(meft_ctx* ctx, void* dst, const void* src, size_t bytes); /* stream-ordered */
meft_status meft_copy_to_host(meft_ctx* ctx, void* dst, const void* src, size_t bytes);   /* synchronises */
meft_status meft_memset(meft_ctx* ctx, void* dst, int value, size_t bytes);
meft_status meft_convert(meft_ctx* ctx, void* dst, meft_dtype dst_dt, const void* src, meft_dtype src_dt, int64_t n);

/* ------------------------------------------------------------------ selection */

/* Host-side clamp arithmetic of ke_select (experts.cpp:56-65) / topk_select (adapter.cpp:43-49):
 * kk_eff = min(kk, N); take = min(k, kk_eff*(M/N)); *warn = 1 when the reference would call warn().
 * Returns MEFT_E_INVALID for k < 1, kk < 1, N < 1 or N not dividing M (ExpertPartition::make). */
meft_status meft_selection_shape(int64_t M, int64_t N, int64_t kk, int64_t k, int64_t* take, int64_t* kk_eff,
                                 int* warn);

/* route_scores (experts.cpp:21-28) for T tokens: scores[T x N] fp64, each a strict left-to-right dot. */
meft_status meft_route_scores(meft_ctx* ctx, meft_dtype dt, const void* h, const void* w_g, int64_t T, int64_t d,
                              int64_t N, double* scores);

/* select_experts (experts.cpp:30-45) per row of scores[T x N]: tau[T x min(kk,N)] ascending. */
meft_status meft_select_experts(meft_ctx* ctx, const double* scores, int64_t T, int64_t N, int64_t kk,
                                int32_t* tau);

/* ke_select (experts.cpp:47-117). dt in {F64, BF16} for h [T x d], w_g [N x d], keys [M x d].
 * Outputs: per_token [T x take] (rows ascending), tau [T x kk_eff] (nullable), union_idx [M] ascending with
 * its length in *union_size_dev (device int32). Bit-exact with the reference on identical inputs. */
meft_status meft_ke_select(meft_ctx* ctx, meft_dtype dt, const void* h, const void* w_g, const void* keys,
                           int64_t T, int64_t d, int64_t M, int64_t N, int64_t kk, int64_t k, int32_t* per_token,
                           int32_t* tau, int32_t* union_idx, int32_t* union_size_dev);

/* topk_select (adapter.cpp:42-84): flat top-K over all M keys; take = min(k, M). */
meft_status meft_topk_select(meft_ctx* ctx, meft_dtype dt, const void* h, const void* keys, int64_t T, int64_t d,
                             int64_t M, int64_t k, int32_t* per_token, int32_t* union_idx, int32_t* union_size_dev);

/* ------------------------------------------------------------------ gather */

/* gather_adapter (adapter.cpp:86-110) on neuron-major tables: keys_s[i] = keys[S[i]], values_s[i] =
 * values[S[i]] (rows of d elements of dt). Validates S (synchronises): out of range -> MEFT_E_RANGE with the
 * index, not strictly ascending -> MEFT_E_INVALID. */
meft_status meft_gather_adapter(meft_ctx* ctx, meft_dtype dt, const void* keys, const void* values, int64_t M,
                                int64_t d, const int32_t* S, int64_t s, void* keys_s, void* values_s);

/* ------------------------------------------------------------------ sparse FFN (adapter half) */

/* sparse_ffn_pa adapter term (adapter.cpp:122-126) for every token against all s selected pairs.
 *   F64 : h [T x d] f64, keys_s/values_s [s x d] f64; z [T x ld_z] f64 receives h*w_a_k (the cache);
 *         out [T x d] f64 = (accumulate ? out : 0) + ReLU(z) * w_b_k.
 *   BF16: h, keys_s, values_s bf16; z receives bf16 ReLU(z) (a positive z never rounds to 0, so act > 0 is
 *         exactly z > 0); out f32. ld_z % 8 == 0, d % 8 == 0.
 */
meft_status meft_ffn_forward(meft_ctx* ctx, meft_dtype dt, const void* h, const void* keys_s, const void* values_s,
                             int64_t T, int64_t d, int64_t s, int64_t ld_z, void* z, void* out, int accumulate);

/* sparse_backward adapter term (adapter.cpp:166-175), given the forward cache z:
 *   masked = (grad_out * w_b_k^T) .* 1[z > 0]        (masked_ws [T x ld_z], dt)
 *   grad_values_s [s x d] = ReLU(z)^T grad_out       (w_b_k layout)
 *   grad_keys_s   [s x d] = masked^T h               (neuron-major, i.e. transpose of the reference d x s)
 *   grad_h [T x d] = (accumulate_grad_h ? grad_h : 0) + masked * w_a_k^T
 * F64: every buffer f64. BF16: grad_out/h/z/keys_s/values_s/masked bf16; grad_* f32. */
meft_status meft_ffn_backward(meft_ctx* ctx, meft_dtype dt, const void* grad_out, const void* h, const void* z,
                              const void* keys_s, const void* values_s, int64_t T, int64_t d, int64_t s,
                              int64_t ld_z, void* masked_ws, void* grad_keys_s, void* grad_values_s, void* grad_h,
                              int accumulate_grad_h);

/* Frozen base FFN half of sparse_ffn_pa / sparse_backward (adapter.cpp:119-120, 153-164), f64 only.
 * act: 0 SiLU, 1 ReLU. forward: base_pre [T x n] = h*w_in, out [T x d] = act(base_pre)*w_out.
 * backward: grad_h [T x d] = ((grad_out*w_out^T) .* act'(base_pre)) * w_in^T. */
meft_status meft_base_ffn_forward(meft_ctx* ctx, const double* h, const double* w_in, const double* w_out,
                                  int64_t T, int64_t d, int64_t n, int act, double* base_pre, double* out);
meft_status meft_base_ffn_backward(meft_ctx* ctx, const double* grad_out, const double* base_pre,
                                   const double* w_in, const double* w_out, int64_t T, int64_t d, int64_t n, int act,
                                   double* grad_h);

/* ---- Bookkeeping of the expert-sharded selection protocol (paper_2406_04984_b200/sharded.py) on the
 * device: deterministic stable bucketing instead of host-driven index manipulation between the exchanges.
 * world <= 64. Host-side count arrays are written after a stream synchronisation. */
/* Dispatch plan: row i = t*kk + s of tau goes to owner tau[i] / n_loc (experts per rank), rows bucketed by owner in
 * ascending i. send_rows [T*kk x d] bf16 (= h[t]; may be NULL: no row copy), send_exp (owner-local expert),
 * order[p] = i, inv[i] = p, counts[world] (host): rows per owner. */
meft_status meft_shard_dispatch(meft_ctx* ctx, const int32_t* tau, int64_t T, int64_t kk, int64_t n_loc, int world,
                                const uint16_t* h, int64_t d, uint16_t* send_rows, int32_t* send_exp, int32_t* order,
                                int32_t* inv, int64_t* counts);
/* dst[order[p]] = src[p] for n rows of `cols` fp32 (candidate scores back into (token, slot) order) */
meft_status meft_shard_unpermute_rows(meft_ctx* ctx, const float* src, const int32_t* order, int64_t n, int64_t cols,
                                      float* dst);
/* Exact re-scoring requests for the ambiguous candidates amb [T x C] (n_amb per token): key idx goes to owner
 * idx / M_loc as (receive row inv[t*kk + slot(idx)] + row_base[owner], local key idx - owner*M_loc), bucketed by owner
 * in (token, position) order; back[q] = t*C + a says where the answer goes. counts[world] and *total on the host. */
meft_status meft_shard_requests(meft_ctx* ctx, const int32_t* amb, const int32_t* n_amb, const int32_t* tau,
                                const int32_t* inv, int64_t T, int64_t C, int64_t kk, int64_t E, int64_t M_loc,
                                int world, const int64_t* row_base, int32_t* row, int32_t* key, int32_t* back,
                                int64_t* counts, int64_t* total);
/* dst[back[i]] = x[i] */
meft_status meft_shard_scatter_f64(meft_ctx* ctx, const double* x, const int32_t* back, int64_t n, double* dst);
/* dst[r] = src[idx[r]] for n rows of row_bytes (a multiple of 16, 16-byte aligned buffers): the owners of the
 * sharded selection gather their dispatched token rows from the all-gathered hidden states. */
meft_status meft_gather_rows(meft_ctx* ctx, const void* src, int64_t row_bytes, const int32_t* idx, int64_t n,
                             void* dst);

/* ---- The reference's frozen toy trunk (model.cpp:50-218), fp64 on the device: what the drop-in's model.hpp
 * functions call so that the reference trainer runs end to end on the B200. Arrays are device buffers (row-major,
 * T = batch * seq rows); reductions follow the reference's order (deterministic). Ids must be in range: the drop-in
 * validates them on the host with the reference's exceptions before calling. */
/* embed (model.cpp:50-68): h[b*seq + i] = emb[tokens[.]] + pos[i] */
meft_status meft_embed_f64(meft_ctx* ctx, const double* emb, int64_t vocab, const double* pos, int64_t max_seq,
                           int64_t d, const int32_t* tokens, int64_t batch, int64_t seq, double* h);
/* attention_forward (model.cpp:70-122): out = h + softmax(q k^T / sqrt(d), causal, same segment) v wo, q/k/v = h
 * wq/wk/wv; the cache (q, k, v [T x d], probs [T x seq]) is returned for the backward. */
meft_status meft_attention_forward_f64(meft_ctx* ctx, const double* h, const double* wq, const double* wk,
                                       const double* wv, const double* wo, const int32_t* segments, int64_t batch,
                                       int64_t seq, int64_t d, double* out, double* q, double* k, double* v,
                                       double* probs);
/* attention_backward (model.cpp:124-173): dh = dh_out + dq wq^T + dk wk^T + dv wv^T (weights frozen) */
meft_status meft_attention_backward_f64(meft_ctx* ctx, const double* wq, const double* wk, const double* wv,
                                        const double* wo, const int32_t* segments, int64_t batch, int64_t seq,
                                        int64_t d, const double* q, const double* k, const double* v,
                                        const double* probs, const double* dh_out, double* dh);
/* lm_loss_and_grad (model.cpp:175-203): tied logits h emb^T, scaled cross-entropy at loss_mask positions;
 * *loss_sum (host) and dh [T x d] (device). Synchronises. */
meft_status meft_lm_loss_f64(meft_ctx* ctx, const double* emb, int64_t vocab, int64_t d, const double* h, int64_t T,
                             const int32_t* targets, const uint8_t* loss_mask, double loss_scale, double* loss_sum,
                             double* dh);
/* argmax_logits (model.cpp:205-218): greedy token for one row, ties toward the lowest id; *token on the host. */
meft_status meft_argmax_logits_f64(meft_ctx* ctx, const double* emb, int64_t vocab, int64_t d, const double* h_row,
                                   int64_t* token);

/* Dense fp64 product C[m x n] = A[m x k] * B[k x n] (row-major), the reference matmul (kernels.cpp:57-76):
 * ascending-k fma chains that skip zero a-entries, bitwise equal to the compiled reference. Non-finite
 * results return MEFT_E_NONFINITE like check_finite (kernels.cpp:7-13); synchronises. */
meft_status meft_matmul_f64(meft_ctx* ctx, const double* A, const double* B, int64_t m, int64_t k, int64_t n,
                            double* C);

/* Layout/elementwise helpers of the fp64 API path: dst[cols x rows] = src[rows x cols]ᵀ (kernels.cpp:94-101);
 * y = act(x) with act 0 SiLU (x*sigmoid(x), kernels.cpp:15-17), 1 ReLU (kernels.cpp:78-84). */
meft_status meft_transpose_f64(meft_ctx* ctx, const double* src, double* dst, int64_t rows, int64_t cols);
meft_status meft_activation_f64(meft_ctx* ctx, int act, const double* x, double* y, int64_t n);

/* Row accumulation into an arbitrary row table (the drop-in's staging rows: scatter_grads memtier.cpp:139-149 on the
 * touched rows only, stage_router_grads memtier.cpp:157-172): for i in [0, n) in order, table[idx[i], :] +=
 * rows[i, :] and flags[idx[i]] = 1 (flags may be NULL). dt F64 or F32 for both. Repeated indices add in entry order
 * (segmented, atomic-free), so the result is bit-identical to the sequential loop. Indices must be in range. */
meft_status meft_rows_add(meft_ctx* ctx, meft_dtype dt, void* table, int64_t d, const int32_t* idx, int64_t n,
                          const void* rows, uint8_t* flags);
/* Lazy Adam over arbitrary fp64 row tables (the router rows of sparse_adam_update, memtier.cpp:211-227):
 * for each row r in rows[0..n): t = ++step[r]; Adam on w/m/v[r,:] with gradient stage[r,:]; stage[r,:] = 0;
 * staged[r] = 0. step is int64 [table rows]; staged uint8. */
meft_status meft_adam_rows_f64(meft_ctx* ctx, double* w, double* m, double* v, double* stage, int64_t* step,
                               uint8_t* staged, const int32_t* rows, int64_t n, int64_t d, double beta1, double beta2,
                               double eps, double lr);

/* ------------------------------------------------------------------ HBM-resident store */

/* HostStore for `layers` layers (memtier.hpp:108-133) resident in HBM. All tensors start at zero; use
 * meft_store_upload_host (or meft_store_init_reference) to set weights. */
meft_status meft_store_create(meft_ctx* ctx, int64_t layers, int64_t d, int64_t pairs, int64_t experts,
                              meft_precision precision, meft_store** out);
void meft_store_destroy(meft_store* store);
meft_status meft_store_info(const meft_store* store, int64_t* layers, int64_t* d, int64_t* pairs, int64_t* experts,
                            meft_precision* precision);
/* HostStore::init (memtier.cpp:60-96): W_A ~ U(+-1/sqrt(d)) from mix_seed(seed, 0x5000+2l), W_G from
 * 0x5001+2l, W_B = 0, moments/steps/staging zero. Generated on the host with the reference RNG (rng.hpp),
 * bit-identical to the reference tables; bf16 compute copies are rounded from them in MIXED mode. */
meft_status meft_store_init_reference(meft_ctx* ctx, meft_store* store, uint64_t seed);
/* The reference's seeded input streams (rng.hpp:13-21, 62-66): n draws of
 * SeededRng(mix_seed(seed, stream)).uniform(lo, hi) in storage order, i.e. uniform_matrix(rows, cols, lo, hi) for
 * n = rows * cols, into a host fp64 buffer; with round_bf16 != 0 each value is rounded to the nearest bf16 (ties to
 * even) and kept as a double. The synthetic inputs of BASELINE.md §3 (W_B 0x7001, h 0x7002, grad_out 0x7003) for
 * bench.py's two arms and the parity tests, so both arms see identical values. Host-only; no device work. */
meft_status meft_reference_uniform(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi, int round_bf16,
                                   double* host_out);
/* Host transfers in the reference layouts (see meft_tensor). host_dt F64 (or int64/int8 for counters). */
meft_status meft_store_upload_host(meft_ctx* ctx, meft_store* store, int64_t layer, meft_tensor t, const void* host,
                                   int64_t rows, int64_t cols);
meft_status meft_store_download_host(meft_ctx* ctx, meft_store* store, int64_t layer, meft_tensor t, void* host,
                                     int64_t rows, int64_t cols); /* synchronises */
/* Device view of a store tensor in its device layout. */
meft_status meft_store_tensor(meft_store* store, int64_t layer, meft_tensor t, void** dev, meft_dtype* dt,
                              int64_t* rows, int64_t* cols);
/* HostStore::init(..., train_router=true) (memtier.cpp:86-91): allocate zeroed router moments and step counters
 * for every layer (MEFT_T_M_G / V_G / ROUTER_STEP); idempotent. meft_store_train_router reports the flag. */
meft_status meft_store_enable_router(meft_ctx* ctx, meft_store* store);
/* The trainer's expert histogram (trainer.cpp:240): per layer, how often each expert was routed to (one count
 * per token and selected expert), accumulated on the device by every fused layer step. host_out: int64[N];
 * reset != 0 clears it after the read. Synchronises. */
meft_status meft_store_expert_histogram(meft_ctx* ctx, meft_store* store, int64_t layer, int64_t* host_out,
                                        int reset);
meft_status meft_store_train_router(const meft_store* store, int* on);

/* ------------------------------------------------------------------ MEFT1 checkpoints (memtier.cpp:288-396)
 * One JSON header line {extra, dim, experts, layers, magic "MEFT1", moment_precision "f64", pairs, step,
 * train_router, version 1, weight_precision "f32"} (keys sorted, as nlohmann::json dumps it), then per layer in
 * reference layouts: w_a f32 [d x r], w_b f32 [r x d], w_g f32 [N x d], m_a f64 [d x r], v_a f64 [d x r],
 * m_b f64 [r x d], v_b f64 [r x d], pair_step i64 [r], and with train_router m_g f64 [N x d], v_g f64 [N x d],
 * router_step i64 [N]. Staging is not saved (it is empty after every sparse_adam_update) and loads as zero.
 * Errors: extra not JSON -> MEFT_E_INVALID; cannot open / write failure -> MEFT_E_IO; missing or corrupt header,
 * bad magic, version != 1, missing field -> MEFT_E_CKPT_HEADER; non-positive shape, trailing bytes ->
 * MEFT_E_CKPT_SHAPE; short payload -> MEFT_E_CKPT_TRUNCATED (messages as the reference's). */
typedef struct meft_ckpt_header {
    int64_t layers, dim, pairs, experts, step;
    int train_router;
} meft_ckpt_header;
/* Device store <-> file: save_checkpoint / load_checkpoint for an HBM store (precision of the new store given).
 * `extra_json` NULL means "{}"; `extra_out` (may be NULL) receives the header's extra object, truncated to cap. */
meft_status meft_store_save(meft_ctx* ctx, meft_store* store, const char* path, int64_t step, const char* extra_json);
meft_status meft_store_load(meft_ctx* ctx, const char* path, meft_precision precision, meft_store** out,
                            meft_ckpt_header* header, char* extra_out, size_t extra_cap);
/* Host-resident stores (the C++ shim's HostStore): the same format through per-tensor callbacks. Values travel
 * as double (f32/f64 items) or int64 (counters) in the reference layout, n = rows * cols; a callback returns 0 on
 * success. The sink sees the parsed header before the first tensor of every layer. */
typedef int (*meft_ckpt_source)(void* user, int64_t layer, meft_tensor t, void* dst, int64_t n);
typedef int (*meft_ckpt_sink)(void* user, const meft_ckpt_header* h, int64_t layer, meft_tensor t, const void* src,
                              int64_t n);
meft_status meft_ckpt_save(const char* path, const meft_ckpt_header* header, const char* extra_json,
                           meft_ckpt_source source, void* user);
meft_status meft_ckpt_load(const char* path, meft_ckpt_header* header, char* extra_out, size_t extra_cap,
                           meft_ckpt_sink sink, void* user);

/* fetch (memtier.cpp:117-126): gather rows S of the layer's compute tables (validated like gather_adapter). */
meft_status meft_fetch(meft_ctx* ctx, meft_store* store, int64_t layer, const int32_t* S, int64_t s, void* keys_s,
                       void* values_s);
/* scatter_grads (memtier.cpp:128-155): stage[S_j] += grad (neuron-major rows, dtype gdt in {F64, F32}),
 * staged[S_j] = 1; repeated scatters sum. Validates S range (synchronises) -> MEFT_E_RANGE. */
meft_status meft_scatter_grads(meft_ctx* ctx, meft_store* store, int64_t layer, const int32_t* S, int64_t s,
                               const void* grad_keys_s, const void* grad_values_s, meft_dtype gdt);
/* sparse_adam_update (memtier.cpp:187-210): lazy Adam on every staged pair (per-pair step counter), then
 * clears staging. Untouched pairs stay bit-identical. No host synchronisation. */
meft_status meft_sparse_adam_update(meft_ctx* ctx, meft_store* store, int64_t layer, double beta1, double beta2,
                                    double eps, double lr);

/* ------------------------------------------------------------------ expert-sharded layer
 * Rank r owns experts [r*N/P, (r+1)*N/P) and their pairs; its store holds only those (pairs = M/P, experts = N/P).
 * The orchestration (paper_2406_04984_b200/sharded.py) moves rows between ranks with NCCL; these calls are the
 * per-rank compute. All selection pieces are the certified path of meft_ke_select split at the rank boundary, so
 * the sharded layer selects exactly the reference's indices. */

/* home rank: certified top-kk experts per token against the replicated router (experts.cpp:21-45). */
meft_status meft_route_select(meft_ctx* ctx, const uint16_t* h, const uint16_t* w_g, int64_t T, int64_t d, int64_t N,
                              int64_t kk, int32_t* tau);
/* norms (rounded up) and minimum LSB exponents of bf16 rows (inputs of the error bounds / exactness certificate). */
meft_status meft_row_stats(meft_ctx* ctx, const uint16_t* rows, int64_t n, int64_t d, float* norms, int32_t* minlsb);
/* owner rank: the same statistics for the layer's local keys (cached until the next update of the keys). */
meft_status meft_store_key_stats(meft_ctx* ctx, meft_store* store, int64_t layer, float* norms, int32_t* minlsb);
/* owner rank: approximate tcgen05 scores of R dispatched token rows against all E keys of their local expert
 * (expert_local[r] in [0, N/P)): cand [R x E] fp32 = float(fp64 sum of the K-chunk partial products) -- the
 * same approximation the fused selection classifies, and the one meft_topk_classify's bound is stated for. */
meft_status meft_score_candidates(meft_ctx* ctx, meft_store* store, int64_t layer, const uint16_t* rows,
                                  const int32_t* expert_local, int64_t R, float* cand);
/* owner rank: the reference's exact fp64 scores dot(rows[pair_row[q]], key[pair_key[q]]) of Q pairs. */
meft_status meft_exact_scores(meft_ctx* ctx, meft_store* store, int64_t layer, const uint16_t* rows, int64_t R,
                              const int32_t* pair_row, const int32_t* pair_key, int64_t Q, double* out);
/* home rank: certified classification of each token's C = kk*E approximate candidates (cand [T x C], slot order =
 * tau order; kn = norms of ALL M keys): certain members -> sure [T x take] / n_sure, ambiguous global indices ->
 * amb [T x C] / n_amb. Then, with the owners' exact scores x [T x C] (x[t][a] for amb[t][a]), finalize writes the
 * ascending per-token selection and marks union_flags [M]. */
meft_status meft_topk_classify(meft_ctx* ctx, const float* cand, const int32_t* tau, int64_t T, int64_t kk, int64_t E,
                               int64_t take, int64_t d, const float* hn, const float* kn, int32_t* sure,
                               int32_t* n_sure, int32_t* amb, int32_t* n_amb);
meft_status meft_topk_finalize(meft_ctx* ctx, const int32_t* sure, const int32_t* n_sure, const int32_t* amb,
                               const int32_t* n_amb, const double* x, int64_t T, int64_t C, int64_t take,
                               int32_t* per_token, uint8_t* union_flags);
/* Fused reduce-scatter over NVLink peer memory: with `peer` set, the out and grad_h GEMM epilogues store each
 * output row straight into its home rank's receive buffer, slot `rank`: row g of [world*rows x d] goes to
 * out_recv[g / rows][(rank * rows + g % rows) * d ...] (grad_h_recv likewise). Buffers are
 * [world x rows x d] fp32 on every home, mapped into this process (meft_ipc_*); out_partial / grad_h_partial are
 * then unused. Once every rank's stores are complete (a cross-rank barrier), each home folds its slots with
 * meft_peer_reduce -- the same data movement as a reduce-scatter, overlapped tile by tile with the GEMMs. */
typedef struct meft_peer_out {
    int world, rank;         /* world <= 8 */
    int64_t rows;            /* tokens per home rank */
    float* out_recv[8];      /* per home rank: its receive buffer for out */
    float* grad_h_recv[8];   /* per home rank: its receive buffer for grad_h */
} meft_peer_out;
/* out[i] = sum over slots s = 0..world-1 (in that order) of recv[s * rows * d + i], i < rows * d. */
meft_status meft_peer_reduce(meft_ctx* ctx, const float* recv, int world, int64_t rows, int64_t d, float* out);
/* CUDA IPC for the receive buffers (allocate them with meft_device_alloc): 64-byte handle out / mapped pointer. */
meft_status meft_ipc_handle(meft_ctx* ctx, void* dev_ptr, void* handle64);
meft_status meft_ipc_open(meft_ctx* ctx, const void* handle64, void** dev_ptr);
meft_status meft_ipc_close(meft_ctx* ctx, void* dev_ptr);
/* owner rank: the FFN of ALL T (all-gathered) tokens against its local part of the union (S_local: ascending local
 * pair ids), the fused scatter, and the lazy Adam of those pairs. out/grad_h are this shard's partial sums
 * [T x d] fp32 (to be reduce-scattered).
 * Overlap hooks (cudaEvent_t, each may be NULL): the backward waits for g_ready (e.g. the grad_out all-gather
 * on a communication stream); fwd_done is recorded once out_partial is final, grad_h_done once grad_h_partial
 * is, so their reduce-scatters can run while the rest of the step computes. */
meft_status meft_layer_ffn_local(meft_ctx* ctx, meft_store* store, int64_t layer, const uint16_t* h_all,
                                 const uint16_t* g_all, int64_t T, const int32_t* S_local, int64_t s, double beta1,
                                 double beta2, double eps, double lr, float* out_partial, float* grad_h_partial,
                                 void* g_ready, void* fwd_done, void* grad_h_done,
                                 const struct meft_peer_out* peer);

/* ------------------------------------------------------------------ whole layer step */

typedef struct meft_step_info {
    int64_t union_size; /* |S| */
    int64_t take;       /* per-token K after the clamp */
    int64_t kk_eff;
    int warned;         /* the reference would have called warn() */
    int gpu_launches;   /* kernels this step launched */
    int rescored;       /* ambiguous candidates re-scored exactly by the certified selection */
    int fallbacks;      /* of those, exact dots that needed the sequential fp64 chain */
    /* the reference's per-step bookkeeping for this layer, from the step's own selection (no extra sync):
     * CommMeter (memtier.cpp:56-58, 117-155): fetch 2*d*|S| host->device, scatter 2*d*|S| device->host,
     * push_hidden T*d; measure_beta (memtier.cpp:14-21) with batch*seq = T; cpu_flops (experts.cpp:119-129). */
    int64_t meter_h2d, meter_d2h, meter_hidden;
    double beta_paper, dedup_ratio, activated_fraction;
    int64_t router_flops, expert_scoring_flops;
} meft_step_info;

/* The frozen base FFN of the layer (BaseFfn, adapter.hpp:11-16) in bf16 on the device, reference layouts:
 * w_in [d x n], w_out [n x d] (row-major, n % 8 == 0); act 0 = SiLU (the default), 1 = ReLU. */
typedef struct meft_base_ffn {
    const uint16_t* w_in;
    const uint16_t* w_out;
    int64_t n;
    int act;
} meft_base_ffn;

/* One MEFT layer training step in MIXED precision, the trainer's per-layer sequence
 * (trainer.cpp:220,270,283,525): meft_ffn (ke_select -> fetch -> sparse_ffn_pa) -> sparse_backward ->
 * scatter_grads -> sparse_adam_update. h and grad_out are bf16 [T x d] on device; out and grad_h are f32
 * [T x d] (either may be NULL). Optional outputs per_token [T x take] / union_idx [M] (device int32) may be
 * NULL. With host sync on (meft_ctx_set_host_sync) it synchronises once, mid-step, to size the union; off, it does
 * not (the FFN GEMMs read the union size on the device) and a non-NULL info costs one sync at the end; the default
 * (MEFT_HOST_SYNC_AUTO) takes the second for dense unions.
 */
meft_status meft_layer_step(meft_ctx* ctx, meft_store* store, int64_t layer, const void* h, const void* grad_out,
                            int64_t T, int64_t kk, int64_t k, double beta1, double beta2, double eps, double lr,
                            float* out, float* grad_h, int32_t* per_token, int32_t* union_idx, meft_step_info* info);

/* Same step from HOST buffers (pinned or pageable): copies h/grad_out in and out/grad_h back inside the
 * call; returns when the results are on the host. */
/* meft_layer_step with the frozen base FFN (sparse_ffn_pa / sparse_backward with a real BaseFfn,
 * adapter.cpp:118-120, 153-164): out = act(h w_in) w_out + adapter; grad_h = ((G w_out^T) .* act'(pre)) w_in^T +
 * adapter part. The base weights receive no gradient (frozen). base == NULL or base->n == 0: meft_layer_step. */
meft_status meft_layer_step_base(meft_ctx* ctx, meft_store* store, int64_t layer, const void* h, const void* grad_out,
                                 int64_t T, int64_t kk, int64_t k, double beta1, double beta2, double eps, double lr,
                                 float* out, float* grad_h, int32_t* per_token, int32_t* union_idx,
                                 meft_step_info* info, const meft_base_ffn* base);
meft_status meft_layer_step_host(meft_ctx* ctx, meft_store* store, int64_t layer, const uint16_t* h_host,
                                 const uint16_t* grad_out_host, int64_t T, int64_t kk, int64_t k, double beta1,
                                 double beta2, double eps, double lr, float* out_host, float* grad_h_host,
                                 meft_step_info* info);

/* ---- The expert-sharded layer step behind the C ABI (one rank per GPU). The context carries a
 * communicator: NCCL (created from a unique id, or the caller's own ncclComm_t), or host callbacks (a process that
 * stands in for several ranks, e.g. the test suite's emulation on one GPU). NCCL is loaded at run time
 * (libnccl.so.2: the copy already in the process, e.g. torch's, else the system one); the sharded calls fail with
 * MEFT_E_NCCL when it is absent, nothing else needs it. */
/* ncclGetUniqueId into 128 bytes (rank 0 creates it; every rank passes the same bytes to meft_ctx_comm_init). */
meft_status meft_nccl_unique_id(void* id128);
/* A communicator owned by the context (ncclCommInitRank over `world` ranks). */
meft_status meft_ctx_comm_init(meft_ctx* ctx, const void* id128, int rank, int world);
/* The caller's ncclComm_t (not owned; must outlive its use by this context). */
meft_status meft_ctx_set_comm(meft_ctx* ctx, void* nccl_comm, int rank, int world);
/* Host-exchange communicator: every collective synchronises the context stream, copies its device payload to the
 * host and calls back. all_gather: each rank contributes `bytes`; recv holds world * bytes in rank order.
 * all_to_all_v: send holds world blocks (send_bytes[p] for rank p, consecutive); recv gets recv_bytes[p] from rank p,
 * consecutive in rank order. Callbacks return 0 on success. */
typedef struct meft_host_comm {
    void* user;
    int (*all_gather)(void* user, const void* send, size_t bytes, void* recv);
    int (*all_to_all_v)(void* user, const void* send, const size_t* send_bytes, void* recv, const size_t* recv_bytes);
} meft_host_comm;
meft_status meft_ctx_set_host_comm(meft_ctx* ctx, const meft_host_comm* comm, int rank, int world);
/* Releases the context's communicator (an owned NCCL communicator is destroyed). */
meft_status meft_ctx_clear_comm(meft_ctx* ctx);
/* One layer step of this rank's T tokens on its expert shard: `shard` holds experts [rank*N/P, (rank+1)*N/P) and
 * their M/P pairs (a MIXED/COMPACT store with experts = N/P, pairs = M/P); w_g is the replicated bf16 router
 * [N x d]. Every rank brings T tokens (h, grad_out bf16 [T x d]); the step covers all P*T tokens with the
 * reference's batch-union semantics: selection split at the rank boundary (indices == the single-GPU step's),
 * FFN + fused scatter + lazy Adam of the local part of the union on every owner, out / grad_h [T x d] fp32 summed
 * back to the token homes. Exchanges: all-gather of h and grad_out; all-to-all of (token id, expert) dispatch
 * entries (owners gather the token rows from the all-gathered h), of candidate scores, of exact-rescoring requests
 * and answers; all-gather of per-destination counts and key norms; MAX all-reduce of the M-byte union bitmap;
 * out / grad_h rows stored by the GEMM epilogues straight into their homes over peer memory and folded there
 * (meft_ctx_sharded_paths; else a reduce-scatter of out / grad_h). per_token [T x take] (global pair ids, ascending) may be NULL. At world 1 the
 * step equals meft_layer_step bit for bit. Replaces the reference trainer's per-layer calls (trainer.cpp:220, 270,
 * 283, 525) for a sharded layer. */
meft_status meft_layer_step_sharded(meft_ctx* ctx, meft_store* shard, int64_t layer, const uint16_t* w_g,
                                    const uint16_t* h, const uint16_t* grad_out, int64_t T, int64_t kk, int64_t k,
                                    double beta1, double beta2, double eps, double lr, float* out, float* grad_h,
                                    int32_t* per_token, meft_step_info* info);
/* Which data paths the last meft_layer_step_sharded on this context took. *peer = 1 when its out / grad_h GEMM
 * epilogues stored the partial sums straight into the token homes' receive buffers over peer memory (the
 * reduce-scatter fused into the GEMMs; the default whenever every rank can map every home's buffers -- CUDA IPC
 * across processes), 0 when it fell back to the communicator's reduce-scatters (MEFT_SHARDED_PEER=0, or a rank
 * could not allocate / map them). *overlap = 1 when grad_out's all-gather ran on a second NCCL communicator
 * (ncclCommSplit) and stream behind the selection and forward, 0 when it ran in stream order (host-callback
 * communicators, or no ncclCommSplit). Either pointer may be NULL. */
meft_status meft_ctx_sharded_paths(meft_ctx* ctx, int* peer, int* overlap);


#ifdef __cplusplus
}
#endif
#endif /* MEFT_CUDA_H */
