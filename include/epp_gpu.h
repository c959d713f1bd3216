/* epp-b200: C ABI of the B200 stage executor (libepp_gpu.so, sm_100a).
 *
 * The reference has no GPU code; this is the thin C ABI the
 * paper's runtime would sit on.  One `epp_stage` owns the
 * weights, gradients, optimizer state, per-sequence KV / dKV buffers (the
 * paper's "global buffer for KV intermediate activations")
 * and the saved activations of in-flight chunks for a contiguous range of
 * transformer layers on one device.  The caller (one host thread / process
 * per GPU) replays a plan document's per-stage op list: forward and backward
 * calls per chunk, in the order of the reference schedule
 * (proj/src/pipeline.cpp:96-297), moving the [T, hidden] activation /
 * gradient between adjacent stages.
 *
 * Conventions
 *   - return 0 on success, else EPP_GPU_E*; message in epp_gpu_last_error()
 *     (thread-local).
 *   - `stream` arguments are cudaStream_t passed as void*; all work is
 *     stream-ordered, nothing synchronises unless stated.
 *   - activations/gradients exchanged between stages: [T, hidden] row-major in
 *     the stage dtype (bf16 or fp32); the caller owns them.
 *   - a stage handle is single-threaded; distinct handles are independent.
 */
#ifndef EPP_GPU_H_
#define EPP_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { EPP_GPU_OK = 0, EPP_GPU_EARG = 1, EPP_GPU_ECUDA = 2, EPP_GPU_ESTATE = 3, EPP_GPU_EOTHER = 4 };
enum { EPP_ARCH_GPT = 0, EPP_ARCH_LLAMA = 1 };
enum { EPP_DTYPE_F32 = 0, EPP_DTYPE_BF16 = 1 };
/* chunk kinds, numbered as epp::ChunkKind (proj/include/epp/chunk.hpp:18) */
enum { EPP_CHUNK_BATCHED = 0, EPP_CHUNK_SPLIT = 1, EPP_CHUNK_HYBRID = 2 };

typedef struct epp_model_desc {
    int32_t arch;        /* EPP_ARCH_GPT: LayerNorm+GELU+MHA; EPP_ARCH_LLAMA: RMSNorm+SwiGLU+GQA */
    int32_t layers;      /* whole model */
    int32_t hidden;
    int32_t heads;
    int32_t kv_heads;
    int32_t head_dim;    /* 64 or 128 in bf16 mode */
    int32_t ffn;         /* GELU: hidden -> ffn -> hidden; SwiGLU: gate/up of width ffn */
    int32_t vocab;
    float rope_theta;
    float norm_eps;
} epp_model_desc;

/* One heterogeneous micro-batch, i.e. one epp::Chunk (chunk.hpp:32-46) plus
 * the executor-side facts the plan document implies. */
typedef struct epp_chunk_desc {
    int32_t id;
    int32_t seq;           /* owning long sequence of slices[0], -1 for Batched */
    int32_t kind;          /* EPP_CHUNK_* */
    int32_t tail;          /* no later slice of `seq` exists */
    int64_t context;       /* tokens of `seq` before slices[0] */
    int64_t seq_len;       /* total length of `seq` (sizes its KV buffer) */
    int32_t nslices;
    const int64_t* slices; /* host array, slices[0] primary */
    int32_t ckpt_layers;   /* plan ckpt[stage][pos]: recompute this many layers */
    float loss_scale;      /* last stage: d(loss)/d(sum of token losses) */
    const int32_t* token_ids;   /* device [T]; required on the embedding stage */
    const int32_t* target_ids;  /* device [T]; last stage; -1 = no target */
} epp_chunk_desc;

typedef struct epp_param_info {
    const char* name;
    int64_t numel;
    float* master;     /* fp32 master weights (device) */
    void* work;        /* working copy in the stage dtype (== master for fp32) */
    float* grad;       /* fp32 gradient accumulator (device) */
} epp_param_info;

typedef struct epp_stage epp_stage;

int epp_gpu_set_device(int device);

int epp_stage_create(const epp_model_desc* model, int first_layer, int num_layers,
                     int has_embed, int has_head, int dtype, epp_stage** out);
int epp_stage_destroy(epp_stage* st);

/* Deterministic N(0, 0.02) init (output projections scaled by 1/sqrt(2L)),
 * norm weights 1, biases 0. */
int epp_stage_init_weights(epp_stage* st, uint64_t seed, void* stream);
int epp_stage_num_params(epp_stage* st, int32_t* n);
int epp_stage_param(epp_stage* st, int32_t idx, epp_param_info* info);
/* Re-derive working copies after the caller wrote `master` buffers. */
int epp_stage_sync_weights(epp_stage* st, void* stream);

/* Forward of one chunk over this stage's layers.  act_in: [T, hidden]
 * (ignored on the embedding stage, which reads token_ids); act_out: [T,
 * hidden] (ignored on the last stage, which computes the loss and the
 * LM-head gradient instead).  Layers [0, ckpt_layers) of the stage keep only
 * their inputs and are recomputed by the backward. */
int epp_stage_forward(epp_stage* st, const epp_chunk_desc* chunk, const void* act_in,
                      void* act_out, void* stream);
/* Backward of one chunk: grad_in = d(loss)/d(act_out) (ignored on the last
 * stage), grad_out = d(loss)/d(act_in) (ignored on the embedding stage).
 * Accumulates parameter gradients; frees the chunk's saved activations, and
 * the sequence's KV/dKV buffers once its first slice (context 0) is done. */
int epp_stage_backward(epp_stage* st, const epp_chunk_desc* chunk, const void* grad_in,
                       void* grad_out, void* stream);
/* Explicit release of a sequence's KV / dKV buffers (normally automatic). */
int epp_seq_release(epp_stage* st, int32_t seq);

/* Last stage: accumulated (sum of token losses, #targets) since the last
 * reset.  Each chunk's losses are reduced in fp64 in a fixed order (no
 * atomics), then added to the fp64 accumulator in stream order: the result
 * is deterministic.  Synchronises `stream`. */
int epp_stage_loss(epp_stage* st, double out[2], int32_t reset, void* stream);
/* Same, stream-ordered and non-blocking: copies the two fp64 accumulators to
 * out2 (pinned host or device memory) when `stream` reaches this point. */
int epp_stage_loss_async(epp_stage* st, double* out2, int32_t reset, void* stream);
/* Per-micro-batch loss (SURVEY §8b `epp_stage_loss(stage, chunk_id, ...)`;
 * the unit is one epp::Chunk, proj/include/epp/chunk.hpp:32-46): (sum of the
 * chunk's token losses, #targets) of the latest forward of `chunk_id` since
 * the last loss reset.  EPP_GPU_EARG if the chunk was not forwarded on this
 * (last) stage.  Synchronises `stream`. */
int epp_stage_chunk_loss(epp_stage* st, int32_t chunk_id, double out[2], void* stream);
int epp_stage_zero_grads(epp_stage* st, void* stream);
/* Pre-reserve `bytes` in the device's stream-ordered pool that backs all
 * stage activations (kept reserved: later steps never wait on the driver to
 * map memory).  Synchronises `stream`. */
int epp_gpu_pool_reserve(uint64_t bytes, void* stream);
/* AdamW on fp32 masters (bias-corrected, step >= 1), one multi-tensor
 * launch over the stage (or its ZeRO-1 slice); zeroes the grads. */
int epp_stage_adamw_step(epp_stage* st, float lr, float beta1, float beta2, float eps,
                         float weight_decay, int32_t step, void* stream);
/* Device bytes held by this stage's in-flight chunks and sequences. */
int epp_stage_memory(epp_stage* st, int64_t* live_bytes, int64_t* peak_bytes);

/* ---- data parallelism (replicas of a stage) ------------------------------
 * Parameters live in per-kind arenas (fp32 masters, fp32 grads, working
 * copies in the stage dtype), in epp_stage_param order, split into BUCKETS:
 * [embedding] [layer first] ... [layer last] [final norm + LM head], each a
 * contiguous range padded to 4096 elements.  A replica group all-reduces (or
 * reduce-scatters) bucket by bucket as soon as the bucket's gradients are
 * final: with epp_stage_grad_events(st, 1) every backward records one event
 * per bucket after that bucket's last gradient update, and
 * epp_stage_bucket_wait makes another stream (the collective's) wait for it,
 * so the reduction of layer j overlaps the backward of layers < j.
 * epp_stage_opt_shard(st, r, R) (ZeRO-1): Adam state is kept only for slice r
 * of R of every bucket (*state_numel = elements held), epp_stage_adamw_step
 * then updates only those masters (and zeroes every gradient); the caller
 * all-gathers the masters and calls epp_stage_sync_weights.
 * offsets: nbuckets + 1 arena element offsets (cap entries written). */
int epp_stage_arena(epp_stage* st, float** master, void** work, float** grad, int64_t* numel);
int epp_stage_buckets(epp_stage* st, int64_t* offsets, int32_t cap, int32_t* nbuckets);
int epp_stage_grad_events(epp_stage* st, int32_t enable);
int epp_stage_bucket_wait(epp_stage* st, int32_t bucket, void* stream);
int epp_stage_opt_shard(epp_stage* st, int32_t rank, int32_t nranks, int64_t* state_numel);

/* Measured per-op trace of this stage (the measured counterpart of the
 * planner's simulated trace, proj/include/epp/pipeline.hpp:43-58 and the
 * trace document of proj/src/plan_io.cpp:169-209).  enable = 1 clears the
 * record and marks t = 0 on `stream`; every later forward / backward call is
 * bracketed by CUDA events (and each recompute layer inside a backward).
 * trace_read synchronises on the last event and writes up to `cap` events
 * (*n = the total): op 0 = F, 1 = B, 2 = R; an R event (the summed
 * recompute time) directly precedes its B event, as the simulator lays them
 * out; live_bytes = the stage's activation bytes after the op was enqueued. */
typedef struct epp_trace_event {
    int32_t chunk_id;
    int32_t op;
    double start_s;
    double end_s;
    int64_t live_bytes;
} epp_trace_event;
int epp_stage_trace(epp_stage* st, int32_t enable, void* stream);
int epp_stage_trace_read(epp_stage* st, epp_trace_event* out, int32_t cap, int32_t* n);

/* ---- stage-to-stage P2P over peer memory (NVLink) ------------------------
 * epp_p2p_init + epp_send / epp_recv between adjacent stages
 * (PAPER.md:726 uses NCCL; proj/src/pipeline.cpp:168-193 models the hand-off
 * as zero-latency).  One channel = one directed message stream (forward
 * activations p -> p+1 or backward gradients p+1 -> p) between two
 * endpoints, possibly in different processes / on different GPUs:
 *   1. each side: epp_p2p_create(role, arena_bytes, &ch, handle) on its own
 *      device (the receiver allocates the mailbox arena, >= the largest
 *      message); exchange the EPP_P2P_HANDLE_BYTES handles out of band (e.g.
 *      torch.distributed); each side: epp_p2p_open(ch, peer_handle).  Across
 *      processes the memory is mapped with CUDA IPC; in one process, call
 *      epp_p2p_init(ndev, devs) first (peer access).
 *   2. sender, per message: epp_p2p_send_reserve -> *dst (peer address; the
 *      stream waits until that region is free), write it (e.g. pass it as
 *      act_out / grad_out of epp_stage_forward / _backward: the last kernel
 *      stores over NVLink, no send buffer), epp_p2p_send_commit.
 *      receiver, per message: epp_p2p_recv_wait -> *src (the stream waits
 *      until the message has landed), read it, epp_p2p_recv_release.
 *   Messages must be consumed in the order they were sent and both sides
 *   must pass the same byte counts (both derive them from the plan).  All
 *   synchronisation is stream-ordered (flag stores + cuStreamWaitValue32); the
 *   host never blocks.  epp_p2p_send / epp_p2p_recv are the copying forms. */
#define EPP_P2P_HANDLE_BYTES 256
enum { EPP_P2P_SENDER = 0, EPP_P2P_RECEIVER = 1 };
typedef struct epp_p2p epp_p2p;
int epp_p2p_init(int ndev, const int* devs);
int epp_p2p_create(int role, uint64_t arena_bytes, epp_p2p** out, void* handle_out);
int epp_p2p_open(epp_p2p* ch, const void* peer_handle);
int epp_p2p_send_reserve(epp_p2p* ch, uint64_t bytes, void* stream, void** dst);
int epp_p2p_send_commit(epp_p2p* ch, void* stream);
int epp_p2p_recv_wait(epp_p2p* ch, uint64_t bytes, void* stream, const void** src);
int epp_p2p_recv_release(epp_p2p* ch, void* stream);
int epp_p2p_send(epp_p2p* ch, const void* src, uint64_t bytes, void* stream);
int epp_p2p_recv(epp_p2p* ch, void* dst, uint64_t bytes, void* stream);
/* messages and payload bytes this endpoint has sent / received */
int epp_p2p_stats(epp_p2p* ch, int64_t* messages, int64_t* bytes);
int epp_p2p_destroy(epp_p2p* ch);

/* ---- kernel-level entry points (unit tests, benchmarks) ------------------ */
/* C[M,N] = epi(A(m,k) B(n,k)); *_kmajor selects the operand layout
 * (kernels.h GemmArgs); epi: 0 store, 1 fp32 accumulate, 2 add residual R,
 * 3 store fp32. */
int epp_kernel_gemm(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda,
                    int32_t a_kmajor, const void* B, int64_t ldb, int32_t b_kmajor, void* C,
                    int64_t ldc, const void* R, int64_t ldr, int32_t epi, int32_t dtype,
                    void* stream);
/* Same with the fused MLP epilogues: epi 4 = StoreGelu (C = acc, C2 =
 * gelu_tanh(acc)), 5 = GeluBwd (C = acc * gelu_tanh'(R), and C2 =
 * gelu_tanh(R) when C2 is given), 7 = SwiGlu (N = 2F, B = [gate; up]
 * K-major: C = [g | u], C2 = silu(g) u), 8 = SwiGluBwd (acc = dA [M, F],
 * R = h = [g | u] with ldr >= 2F: C = dh = [dA u silu'(g) | dA silu(g)]
 * with ldc >= 2F, C2 = silu(g) u); outputs in the stage dtype.  7 / 8 run
 * on the CTA-pair kernel only (bf16, >= 60 pair tiles, F % 128 == 0 for 7). */
int epp_kernel_gemm_ex(int32_t M, int32_t N, int32_t K, const void* A, int64_t lda, int32_t a_kmajor,
                       const void* B, int64_t ldb, int32_t b_kmajor, void* C, int64_t ldc,
                       const void* R, int64_t ldr, void* C2, int64_t ldc2, int32_t epi, int32_t dtype,
                       void* stream);
/* Slice-causal attention over nseg segments (host arrays).  Segment i: query
 * rows [q_start[i], +q_len[i]) of q/o, keys at k[i]/v[i] (row stride
 * Hkv*hd), kv_ctx[i] context keys before the first query. lse: [H, T] log2. */
int epp_kernel_attention_fwd(int32_t T, int32_t H, int32_t Hkv, int32_t hd, float scale,
                             int32_t nseg, const int32_t* q_start, const int32_t* q_len,
                             const int32_t* kv_ctx, const void* const* k, const void* const* v,
                             const void* q, void* o, float* lse, int32_t dtype, void* stream);
/* Backward; dk/dv (fp32, per segment, same row layout as k/v) are ACCUMULATED
 * into, dq (fp32 [T,H,hd]) is written. */
int epp_kernel_attention_bwd(int32_t T, int32_t H, int32_t Hkv, int32_t hd, float scale,
                             int32_t nseg, const int32_t* q_start, const int32_t* q_len,
                             const int32_t* kv_ctx, const void* const* k, const void* const* v,
                             float* const* dk, float* const* dv, const void* q, const void* o,
                             const float* lse, const void* dout, float* dq, int32_t dtype,
                             void* stream);

/* Opt-in per-launch timing (CUDA events on the launching stream) of kernel
 * classes 0 = GEMM, 1 = attention forward, 2 = attention backward.
 * profile_read synchronises on the recorded events and returns total device
 * milliseconds, algorithmic FLOPs and launch count; reset drops the records. */
int epp_gpu_profile(int32_t enable);
int epp_gpu_profile_read(int32_t cls, double* ms, double* flops, int64_t* launches, int32_t reset);

/* Kernel launches of this library so far, per kernel (demangled name, sorted):
 * idx 0 takes a snapshot, idx 1.. read it; EPP_GPU_EARG past the end.  Shows
 * which kernel variants (e.g. the CTA-pair GEMM with the RopeScatter
 * epilogue) a test or benchmark really ran. */
int epp_gpu_kernel_stats(int32_t idx, const char** name, int64_t* count);

const char* epp_gpu_last_error(void);
/* Kernel launches issued by this library in this process (for bench claims). */
int64_t epp_gpu_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* EPP_GPU_H_ */
