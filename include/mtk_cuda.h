/*
 * mtk_cuda.h -- the C-ABI kernel seam of the B200 backend (libmtkcuda.so).
 *
 * The reference (mtk, /root/reference/proj) funnels every piece of training
 * arithmetic through "kernels writing into preallocated outputs"
 * (include/mtk/tensor.h:116-145) plus the fused-op bodies inside
 * src/graph.cpp, the Adam/EMA loops in src/train.cpp and the worker-ordered
 * gradient combine (train.cpp:254-269).  This header is that seam re-cut for
 * sm_100a: one extern "C" entry per reference kernel, plain device pointers,
 * sizes, strides and flags, a stream handle (a cudaStream_t passed as void*),
 * no C++ or torch types.  Each entry cites the reference interface it
 * replaces.
 *
 * Conventions
 *   - All tensors are dense fp32 unless stated; ids are int32.
 *   - "accumulate" flags: 1 = out += result (the reference's backward
 *     convention, tensor.cpp:589-596), 0 = out = result.
 *   - Functions never allocate device memory; workspaces come from the
 *     caller (the graph arena, tensor.cpp:30-59 semantics).
 *   - Return value: MTKC_OK or an error code; mtkc_last_error() gives the
 *     thread-local message.  Codes mirror the reference's error taxonomy
 *     (common.h:18-35) so the C++ host rethrows the same exception types.
 *   - Data-dependent errors that the reference raises mid-kernel (division
 *     by zero, tensor.cpp:161-165; fully-masked softmax row, :424-425;
 *     out-of-vocabulary ids, graph.cpp:602-606; non-finite gradients,
 *     train.cpp:51-53) set bits in a caller-provided device flag word
 *     instead of stopping the stream; the host checks the word at its next
 *     synchronisation point.
 */
#ifndef MTK_CUDA_H
#define MTK_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (common.h:18-35) ------------------------------------- */
enum {
  MTKC_OK = 0,
  MTKC_DIMENSION = 1, /* DimensionError */
  MTKC_NUMERIC = 2,   /* NumericError   */
  MTKC_CONTRACT = 3,  /* ContractError  */
  MTKC_DATA = 4,      /* DataError      */
  MTKC_CUDA = 7       /* CUDA runtime / launch failure */
};

/* ---- device flag bits (checked by the host at sync points) ------------- */
enum {
  MTKC_FLAG_DIV_ZERO = 1,     /* ewiseBinaryInto Div, tensor.cpp:161-165 */
  MTKC_FLAG_MASKED_ROW = 2,   /* softmaxInto fully-masked row, :424-425  */
  MTKC_FLAG_BAD_ID = 4,       /* embed/gather id range, graph.cpp:602-606 */
  MTKC_FLAG_NONFINITE = 8     /* allFinite, tensor.cpp:95-100            */
};

/* ---- elementwise op ids (tensor.h:100, EwiseOp) ------------------------ */
enum {
  MTKC_ADD = 0, MTKC_SUB = 1, MTKC_MUL = 2, MTKC_DIV = 3,
  MTKC_TANH = 4, MTKC_SIGMOID = 5, MTKC_RELU = 6, MTKC_EXP = 7,
  MTKC_LOG = 8, MTKC_NEG = 9
};
/* ---- reduce op ids (tensor.h:101, ReduceOp) ---------------------------- */
enum { MTKC_RSUM = 0, MTKC_RMAX = 1, MTKC_RMEAN = 2, MTKC_RARGMAX = 3 };

/* ======================================================================== */
/* runtime: device, memory, streams (replaces the host Arena backing store, */
/* tensor.cpp:30-59, and the implicit "everything is host memory" model)    */
/* ======================================================================== */
const char* mtkc_last_error(void);
int mtkc_init(int device);
int mtkc_device_count(int* count);
int mtkc_sm_count(int* count);
int mtkc_malloc(void** ptr, size_t bytes);
int mtkc_free(void* ptr);
int mtkc_host_alloc_pinned(void** ptr, size_t bytes);
int mtkc_host_free_pinned(void* ptr);
int mtkc_memcpy_h2d(void* dst, const void* src, size_t bytes, void* stream);
/* Host -> device copy from page-locked memory (mtkc_host_alloc_pinned) as a
 * kernel reading the mapped host buffer: stays inside the programmatic-
 * dependent-launch chain of the stream (Device::upload's staging ring under
 * MTK_UPLOAD_RING=1; the reference has no device, the seam is Tensor's
 * host->device sync, tensor.h:14-98).  MTK_COPY_ENGINE=1: cudaMemcpyAsync. */
int mtkc_upload_pinned(void* dst, const void* pinned_src, size_t bytes, void* stream);
int mtkc_memcpy_d2h(void* dst, const void* src, size_t bytes, void* stream);
int mtkc_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);
int mtkc_memset(void* dst, int value, size_t bytes, void* stream);
int mtkc_stream_create(void** stream);
int mtkc_stream_destroy(void* stream);
int mtkc_stream_sync(void* stream);
int mtkc_event_create(void** ev);
int mtkc_event_destroy(void* ev);
int mtkc_event_record(void* ev, void* stream);
int mtkc_stream_wait_event(void* stream, void* ev);
int mtkc_event_sync(void* ev);
int mtkc_event_elapsed_ms(void* start, void* stop, float* ms);
int mtkc_device_sync(void);
/* Kernel-launch counter (every mtkc_* kernel launch increments it). */
uint64_t mtkc_launch_count(void);
/* Host<->device byte counters of mtkc_memcpy_h2d / mtkc_memcpy_d2h. */
uint64_t mtkc_h2d_bytes(void);
uint64_t mtkc_d2h_bytes(void);
/* Per-kernel-class profiling with CUDA events on the launching stream.
 * While enabled, the GEMM, attention, layer-norm, cross-entropy, embedding
 * and Adam entry points bracket their launches with events and record the
 * algorithmic work (FLOPs for GEMM/attention, HBM bytes otherwise).
 * mtkc_prof_report synchronises and writes one line per class:
 *   "<class> <launches> <total_ms> <total_work>\n"  (then resets).
 * on = 2 (detail mode) appends the call's shape to the class name
 * ("gemm_tc:M8192_N512_K512_tA0_tB0"), for per-shape breakdowns. */
int mtkc_prof_enable(int on);
/* Keep the stream busy for `us` microseconds (profiling aid: lets the host
 * queue a whole step ahead so event timings measure device time only). */
int mtkc_gpu_sleep(int64_t us, void* stream);
int mtkc_prof_report(char* buf, size_t len);

/* ======================================================================== */
/* GEMM: matmulInto (tensor.cpp:258-306), matmulAccumInto (graph.cpp:273-   */
/* 291), affine (graph.cpp:334-336) and the GRU pre-activations (gruPre,    */
/* graph.cpp:633-645), with epilogues the reference runs as separate nodes. */
/* ======================================================================== */
enum { MTKC_GEMM_FP32 = 0, /* CUDA-core FP32, reference summation order   */
       MTKC_GEMM_TF32 = 1  /* tcgen05.mma kind::tf32, fp32 accumulate (TMEM) */ };
enum { MTKC_EPI_NONE = 0, MTKC_EPI_RELU = 1 };

typedef struct mtkc_gemm_args {
  int64_t M, N, K;      /* op(A) is M x K, op(B) is K x N, C is M x N        */
  int64_t batch;        /* >= 1; batch count of the product                  */
  const float* A;       /* row-major storage of A (or A^T when transA)       */
  int64_t lda;          /* row stride of the stored A                        */
  int64_t strideA;      /* batch stride of A, 0 = broadcast (tensor.cpp:246-256) */
  int transA;
  const float* B;
  int64_t ldb;
  int64_t strideB;
  int transB;
  float* C;
  int64_t ldc;
  int64_t strideC;      /* 0 with batch > 1 = sum the batch into one C (graph.cpp:281-290) */
  float alpha;          /* C = alpha*op(A)op(B) + beta*C                     */
  float beta;
  const float* bias;    /* optional [N] row-broadcast add (affine)           */
  int epilogue;         /* MTKC_EPI_NONE | MTKC_EPI_RELU                     */
  const float* gate;    /* optional [M x N], ldc-strided: out *= (gate > 0)  */
  int precision;        /* MTKC_GEMM_FP32 | MTKC_GEMM_TF32                   */
  float* workspace;     /* split-K scratch (may be NULL)                     */
  size_t workspace_bytes;
  const float* addend;  /* optional: the beta term reads addend (laid out like C)
                           instead of C -- a fused residual add, C write-only */
  float* colsum;        /* optional: the sums over k of one operand, written
                           (or added, colsum_accumulate) next to the product --
                           the bias gradient db = colsum(dY) of the dW GEMM
                           (affine backward), read from the tiles the product
                           already stages.  colsum_of = MTKC_COLSUM_B: [N],
                           colsum[n] = sum_k op(B)[k][n]; MTKC_COLSUM_A: [M],
                           colsum[m] = sum_k op(A)[m][k].  TF32 precision sums
                           the tf32-rounded operand in fp32 (deterministic,
                           fixed order); FP32 precision runs mtkc_colsum. */
  int colsum_of;
  int colsum_accumulate;
  uint32_t* relu_mask_out;   /* optional (batch 1): bit c%32 of word
                                [r * ceil(N/32) + c/32] = (C[r][c] > 0) after the
                                epilogue -- the ReLU gate of the consumer's
                                backward at 1/32 of the bytes of C */
  const uint32_t* gate_mask; /* optional (batch 1), instead of gate: C[r][c] is
                                zeroed where that bit of a relu_mask_out-style
                                mask (same N) is 0 */
} mtkc_gemm_args;

#define MTKC_COLSUM_A 1
#define MTKC_COLSUM_B 2

int mtkc_gemm(const mtkc_gemm_args* args, void* stream);
/* A group of products of one shape in one launch (the q/k/v projections of
 * MultiHeadAttention::apply, layers.cpp:100-108, share the input x):
 * kconcat = 0: C_p = alpha*op(A_p)op(B_p) + bias_p + beta*C_p for each p;
 * kconcat = 1: C_0 = alpha*sum_p op(A_p)op(B_p) + bias_0 + beta*C_0 (the
 * dX of the group: sum over the projections).  1 <= nprob <= 3; every
 * problem has the same M, N, K, leading dims, transposes, alpha, beta and
 * epilogue; no gate when nprob > 1.  Falls back to sequential mtkc_gemm. */
int mtkc_gemm_group(const mtkc_gemm_args* probs, int nprob, int kconcat, void* stream);
/* which path the last mtkc_gemm on this thread used: 0 simt, 1 tcgen05 */
int mtkc_gemm_last_path(void);
/* Cap the persistent tensor-core GEMM grid at `sms` CTAs (0 = every SM).
 * The data-parallel stepper leaves SMs to NCCL while overlapped gradient
 * buckets are in flight (a persistent GEMM holding all 148 SMs would queue
 * the all-reduce kernels behind it); host-side state, not stream-ordered. */
int mtkc_gemm_set_sm_limit(int sms);
/* Tuning switch: 1 (default) lets the tensor-core GEMM run 256-row tiles on
 * CTA pairs (cta_group::2), 0 keeps single-CTA 128-row tiles, 3 pairs only
 * the products without fused operand sums (colsum); host-side state, read
 * at each call (MTK_GEMM_NO_PAIR=1 sets 0 at load, MTK_GEMM_PAIR_NO_CS=1 3). */
int mtkc_gemm_set_pair(int enable);

/* ======================================================================== */
/* elementwise / broadcast (tensor.cpp:111-237, graph.cpp:139-268)          */
/* Shapes are passed right-aligned in 4 dims (tensor.cpp:102-108).          */
/* ======================================================================== */
/* out[od] = op(a, b), a/b broadcast to od (ewiseBinaryInto tensor.cpp:160-183) */
int mtkc_ewise_binary(int op, float* out, const int64_t od[4], const float* a,
                      const int64_t ad[4], const float* b, const int64_t bd[4], int* flags,
                      void* stream);
/* out = op(a) (ewiseUnaryInto tensor.cpp:185-190) */
int mtkc_ewise_unary(int op, float* out, const float* a, int64_t n, void* stream);
/* gx += dOp(go, y, x) (graph.cpp:193-221) */
int mtkc_unary_backward(int op, float* gx, const float* go, const float* y, const float* x,
                        int64_t n, void* stream);
/* binary backward for one operand: g_a += reduce_to(ad, f(go, other, y)) --
 * Add/Sub/Mul/Div rules of graph.cpp:149-180.  which = 0 for a, 1 for b. */
int mtkc_binary_backward(int op, int which, float* gtarget, const int64_t td[4],
                         const float* go, const int64_t od[4], const float* a,
                         const int64_t ad[4], const float* b, const int64_t bd[4],
                         const float* y, void* stream);
/* out = s*a + c (scale graph.cpp:236-252, addScalar :254-268) */
int mtkc_scale_shift(float* out, const float* a, float s, float c, int64_t n, void* stream);
/* out += alpha * a (axpy tensor.cpp:225-237) */
int mtkc_axpy(float* out, const float* a, float alpha, int64_t n, void* stream);
/* out[od] += sum of src[sd] down to od (accumulateReduced tensor.cpp:204-223) */
int mtkc_accumulate_reduced(float* out, const int64_t od[4], const float* src,
                            const int64_t sd[4], void* stream);
int mtkc_fill(float* out, float v, int64_t n, void* stream);
/* out[i] = s*x[i] + c[i % period]  (addPositionalEncoding layers.cpp:175-179:
 * scale(x, sqrt(e)) + PE broadcast over the batch) */
int mtkc_scale_add_periodic(float* out, const float* x, float s, const float* c, int64_t n,
                            int64_t period, void* stream);
/* gx = gx*(gate > 0): ReLU backward applied to an accumulated gradient */
int mtkc_relu_mask(float* gx, const float* gate, int64_t n, void* stream);
/* out = a*m + b*(1-m), m broadcast over cols: RNN padding blend
 * (models.cpp:170-172, 360-364) fused */
int mtkc_mask_blend(float* out, const float* a, const float* b, const float* m, int64_t rows,
                    int64_t cols, void* stream);
int mtkc_mask_blend_backward(float* ga, float* gb, const float* go, const float* m,
                             int64_t rows, int64_t cols, int accumulate_a, int accumulate_b,
                             void* stream);

/* Device dropout (throughput mode; graph.cpp:817-846 semantics with a
 * counter-based mask instead of host mt19937_64 draws): element idx of an
 * [outer x axis_len x inner] tensor uses mask index o*inner + j when
 * axis_len > 1 (variational dropout along that axis), else idx.  Mask value:
 * Philox4x32-10(key = seed, counter = mi/4) word mi%4, kept (1/(1-p)) iff its
 * high 24 bits >= ceil(p * 2^24).  addend != NULL: out = addend + x*m (the
 * pre-norm residual add(x, dropout(f)), layers.cpp:135). */
int mtkc_dropout(float* out, const float* x, const float* addend, int64_t n, int64_t inner,
                 int64_t axis_len, float p, uint64_t seed, void* stream);
/* gx (+)= go * m with the same mask */
int mtkc_dropout_backward(float* gx, const float* go, int64_t n, int64_t inner, int64_t axis_len,
                          float p, uint64_t seed, int accumulate, void* stream);
/* the mask itself (dropoutMask, graph.cpp:817-830) */
int mtkc_dropout_mask(float* out, int64_t n, float p, uint64_t seed, void* stream);

/* ======================================================================== */
/* reductions (reduceInto tensor.cpp:322-368, graph.cpp:463-524)            */
/* ======================================================================== */
int mtkc_reduce(int op, float* out, const float* in, int64_t outer, int64_t n, int64_t inner,
                void* stream);
int mtkc_reduce_backward(int op, float* gin, const float* gout, const float* in,
                         int64_t outer, int64_t n, int64_t inner, void* stream);
/* out[c] (+)= sum_r in[r*cols + c]; deterministic two-level (bias grads) */
int mtkc_colsum(float* out, const float* in, int64_t rows, int64_t cols, int accumulate,
                float* workspace, size_t workspace_bytes, void* stream);
/* n <= 3 column sums of one shape in one launch (bias gradients of grouped
 * projections / GRU gates); workspace >= n * ceil(rows/64) * cols floats. */
int mtkc_colsum_group(float* const* outs, const float* const* ins, const int* accumulate, int n,
                      int64_t rows, int64_t cols, float* workspace, size_t workspace_bytes,
                      void* stream);
/* Up to MTKC_COLSUM_MAX_JOBS column sums over the same `rows` in one
 * launch (the reference's per-parameter bias / layer-norm gain gradients,
 * graph.cpp:771, 801 and tensor.cpp:545-599, as the RNN scans' hoisted
 * sums): job z sums columns [0, cols) of in [rows x ld]; column c goes to
 * out[c / seg][c % seg] (accumulated when acc[c / seg]), dropped when that
 * out is NULL.  Sums are bit-identical to mtkc_colsum per job.  cols, ld,
 * seg multiples of 4, in 16-byte aligned; workspace >= ceil(rows/64) *
 * sum(cols) floats. */
#define MTKC_COLSUM_MAX_JOBS 4
#define MTKC_COLSUM_MAX_SEGS 6
typedef struct {
  const float* in;
  int64_t ld, cols, seg;
  int nseg;
  float* out[MTKC_COLSUM_MAX_SEGS];
  int acc[MTKC_COLSUM_MAX_SEGS];
} mtkc_colsum_job;
int mtkc_colsum_multi(const mtkc_colsum_job* jobs, int n, int64_t rows, float* workspace,
                      size_t workspace_bytes, void* stream);
/* flags |= MTKC_FLAG_NONFINITE if any in[i] is not finite (allFinite) */
int mtkc_check_finite(const float* in, int64_t n, int* flags, void* stream);
/* *dst |= *src on the device (stream-ordered): the step's device error bits
 * join the optimizer's skip word, so a step the reference would have thrown
 * in (graph.cpp:602-606, tensor.cpp:161-165, :424-425) never updates the
 * parameters (train.cpp:49-59 runs only after a clean forward/backward) */
int mtkc_flag_or(int* dst, const int* src, void* stream);

/* ======================================================================== */
/* softmax (softmaxInto tensor.cpp:393-440; graph softmax :526-555)          */
/* ======================================================================== */
/* x viewed as rows x cols (last axis).  mask (optional) broadcast against x
 * with right-aligned dims md[4]; xd[4] are x's dims. */
int mtkc_softmax(float* out, const float* x, const int64_t xd[4], const float* mask,
                 const int64_t md[4], int log_mode, int* flags, void* stream);
int mtkc_softmax_backward(float* gx, const float* y, const float* go, int64_t rows,
                          int64_t cols, void* stream);

/* ======================================================================== */
/* layout (transposeInto/concatInto/sliceInto tensor.cpp:480-541,           */
/* gatherRowsInto/scatterAddRows :456-476)                                  */
/* ======================================================================== */
int mtkc_transpose(float* out, const float* src, const int64_t sd[4], const int perm[4],
                   int accumulate, void* stream);
/* strided block copy: for o < outer: dst[o*dst_stride + dst_off .. +len] (+)=
 * src[o*src_stride + src_off .. +len]  (concat/slice and their backwards) */
/* up to MTKC_COPY_MAX_JOBS strided 2-d copies in one launch:
 * dst[r*ldd + c] (+)= src[r*lds + c] for r < rows, c < cols */
#define MTKC_COPY_MAX_JOBS 32
typedef struct mtkc_copy_job {
  const float* src;
  float* dst;
  int64_t rows, cols, lds, ldd;
  int accumulate;
} mtkc_copy_job;
int mtkc_copy_many(const mtkc_copy_job* jobs, int n, void* stream);
int mtkc_copy_blocks(float* dst, int64_t dst_stride, int64_t dst_off, const float* src,
                     int64_t src_stride, int64_t src_off, int64_t outer, int64_t len,
                     int accumulate, void* stream);
int mtkc_gather_rows(float* out, const float* src, const int32_t* rows, int64_t n,
                     int64_t cols, int64_t src_rows, int* flags, void* stream);
/* Deterministic scatter-add: out[ids[perm[k]]] += src[perm[k]] in segment
 * order.  perm sorts positions by id (stable), seg_start[u]..seg_start[u+1]
 * delimit the positions of unique id uniq[u]; each segment is summed in
 * original position order, matching the reference's sequential loop
 * (tensor.cpp:468-476) up to the rounding of one fp32 sum per row. */
int mtkc_scatter_add_rows(float* out, const float* src, const int32_t* perm,
                          const int32_t* seg_start, const int32_t* uniq, int64_t n_uniq,
                          int64_t cols, float scale, void* stream);
/* Same contract with long segments split into chunks of consecutive sorted
 * positions so one frequent id (e.g. </s> padding) does not serialise the
 * kernel.  chunk_start[c]..chunk_start[c+1] are chunk c's positions in perm,
 * chunk_row[c] its table row, chunk_slot[c] = -1 for a segment that is a
 * single chunk (added to out directly, in position order) or the partial
 * slot it writes.  Multi-chunk segment m owns slots multi_first[m] ..
 * multi_first[m+1]-1 and is added to row multi_row[m] in chunk order. */
int mtkc_scatter_add_rows_chunked(float* out, const float* src, const int32_t* perm,
                                  const int32_t* chunk_start, const int32_t* chunk_row,
                                  const int32_t* chunk_slot, int64_t n_chunks,
                                  const int32_t* multi_first, const int32_t* multi_row,
                                  int64_t n_multi, float* partial, int64_t cols, float scale,
                                  void* stream);

/* ======================================================================== */
/* layer norm (layerNormInto / layerNormBackward tensor.cpp:545-599)        */
/* ======================================================================== */
int mtkc_layernorm(float* out, const float* x, const float* gain, const float* bias,
                   float eps, float* inv_std, float* xhat, int64_t rows, int64_t d,
                   void* stream);
/* dx (+)= ..., dgain += ..., dbias += ... ; accumulate_dx selects dx mode.
 * dgain/dbias use a deterministic row-block partial sum (workspace). */
int mtkc_layernorm_backward(const float* dy, const float* gain, const float* inv_std,
                            const float* xhat, float* dx, float* dgain, float* dbias,
                            int64_t rows, int64_t d, int accumulate_dx, int accumulate_params,
                            float* workspace, size_t workspace_bytes, void* stream);

/* Vectorised variant (d % 4 == 0, d <= 1024, 16-byte aligned rows): the    */
/* forward caches only mean/inv_std per row (no xhat tensor); the backward  */
/* recomputes xhat from x and fuses the dgain/dbias column reductions into  */
/* the dx pass (deterministic; workspace >= ..._workspace_bytes).           */
int mtkc_layernorm_fast_supported(int64_t d);
int mtkc_layernorm_stats(float* out, const float* x, const float* gain, const float* bias,
                         float eps, float* mean, float* inv_std, int64_t rows, int64_t d,
                         void* stream);
size_t mtkc_layernorm_stats_workspace_bytes(int64_t rows, int64_t d);
int mtkc_layernorm_stats_backward(const float* dy, const float* x, const float* gain,
                                  const float* mean, const float* inv_std, float* dx,
                                  float* dgain, float* dbias, int64_t rows, int64_t d,
                                  int accumulate_dx, int accumulate_params, float* workspace,
                                  size_t workspace_bytes, void* stream);
/* Deferred parameter reduction: OR MTKC_LN_DEFER_PARAMS into              */
/* accumulate_params and the backward only writes its per-block partials   */
/* (mtkc_layernorm_stats_partial_blocks(rows) x 2 x d floats) into the      */
/* workspace; a later mtkc_layernorm_param_reduce_many sums many layers'   */
/* partials in one launch, bit-identical to the undeferred path.           */
#define MTKC_LN_DEFER_PARAMS 2
int64_t mtkc_layernorm_stats_partial_blocks(int64_t rows);
typedef struct mtkc_ln_param_job {
  float* dgain;
  float* dbias;
  const float* partials;
  int64_t blocks, d;
  int accumulate;
} mtkc_ln_param_job;
int mtkc_layernorm_param_reduce_many(const mtkc_ln_param_job* jobs, int n_jobs, void* stream);

/* ======================================================================== */
/* embedding (embed graph.cpp:595-622) fused with positional encoding       */
/* (addPositionalEncoding layers.cpp:175-179): out = E[id]*s + pe[pos]       */
/* pe may be NULL (plain gather); t = positions per sequence for pe lookup. */
/* ======================================================================== */
int mtkc_embed(float* out, const float* table, const int32_t* ids, int64_t n, int64_t e,
               int64_t vocab, float s, const float* pe, int64_t t, int* flags, void* stream);
/* packed rows: out[n,:] = table[ids[n],:]*s + pe[pos[n],:] (pos = position of
 * row n in its sentence; addPositionalEncoding over real tokens only) */
int mtkc_embed_pos(float* out, const float* table, const int32_t* ids, const int32_t* pos,
                   int64_t n, int64_t e, int64_t vocab, float s, const float* pe, int* flags,
                   void* stream);

/* ======================================================================== */
/* scaled dot-product multi-head attention core (MultiHeadAttention::apply,  */
/* layers.cpp:89-126: splitHeads, dot(q,k^T), scale, masked softmax, dot(w,v),*/
/* merge) fused.  q [b,tq,ldq], k/v [b,tk,ldk]; head h occupies columns      */
/* [h*dk, (h+1)*dk).  key_mask [b,tk] (NULL = all keys real); causal masks   */
/* j > tk - tq + i (layers.cpp:115-116).  probs [b,heads,tq,tk] is saved for */
/* the backward pass. out [b,tq,ldo].                                        */
/* ======================================================================== */
int mtkc_attention(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                   const float* k, const float* v, int64_t ldk, const float* key_mask,
                   int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                   int causal, int* flags, void* stream);
/* gq/gk/gv (+)= ...; dsbuf is a [b,heads,tq,tk] workspace */
int mtkc_attention_backward(const float* gout, int64_t ldo, const float* probs,
                            const float* q, int64_t ldq, const float* k, const float* v,
                            int64_t ldk, float* gq, float* gk, float* gv, float* dsbuf,
                            int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk,
                            float scale, int accumulate_q, int accumulate_k, int accumulate_v,
                            void* stream);
/* Same node on the tensor cores (mma.sync m16n8k8 tf32, fp32 accumulate):  */
/* the TF32-precision path for head dim 64 and tq, tk <= 64 (every BASELINE */
/* config); rows 16-byte aligned.  Arguments as above (no dsbuf).           */
int mtkc_attention_tc_supported(int64_t tq, int64_t tk, int64_t dk);
int mtkc_attention_tc(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                      const float* k, const float* v, int64_t ldk, const float* key_mask,
                      int64_t b, int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                      int causal, int* flags, void* stream);
/* colpart (optional, [3][b][heads*dk]): per sentence, the column sums of
 * this call's dq / dk / dv contributions -- the bias gradients of the q/k/v
 * projections after a [b]-row column sum, without re-reading dq/dk/dv. */
int mtkc_attention_tc_backward(const float* gout, int64_t ldo, const float* probs,
                               const float* q, int64_t ldq, const float* k, const float* v,
                               int64_t ldk, float* gq, float* gk, float* gv, int64_t b,
                               int64_t tq, int64_t tk, int heads, int64_t dk, float scale,
                               int accumulate_q, int accumulate_k, int accumulate_v,
                               float* colpart, void* stream);
/* Packed-row (varlen) form: the b sentences' query rows are qoff[i] ..
 * qoff[i+1]-1 of q / out, their key rows koff[i] .. koff[i+1]-1 of k / v
 * (device int32 [b+1]); every key within a sentence is real (no mask);
 * tq_max / tk_max bound the lengths and give probs its [b,heads,tq_max,
 * tk_max] layout.  Padding rows never exist, so position-wise work before
 * and after attention runs over real tokens only. */
int mtkc_attention_tc_varlen(float* out, int64_t ldo, float* probs, const float* q, int64_t ldq,
                             const float* k, const float* v, int64_t ldk, const int32_t* qoff,
                             const int32_t* koff, int64_t b, int64_t tq_max, int64_t tk_max,
                             int heads, int64_t dk, float scale, int causal, int* flags,
                             void* stream);
/* Length-bucketed launch of the packed form: only the n_sent sentences
 * sent_ids[0..n_sent) (device int32), all of length <= tile_len, with the
 * tile size of tile_len -- short sentences do not pay for the longest one. */
int mtkc_attention_tc_varlen_ids(float* out, int64_t ldo, float* probs, const float* q,
                                 int64_t ldq, const float* k, const float* v, int64_t ldk,
                                 const int32_t* qoff, const int32_t* koff,
                                 const int32_t* sent_ids, int64_t n_sent, int64_t tile_len,
                                 int64_t b, int64_t tq_max, int64_t tk_max, int heads, int64_t dk,
                                 float scale, int causal, int* flags, void* stream);
int mtkc_attention_tc_varlen_ids_backward(
    const float* gout, int64_t ldo, const float* probs, const float* q, int64_t ldq,
    const float* k, const float* v, int64_t ldk, float* gq, float* gk, float* gv,
    const int32_t* qoff, const int32_t* koff, const int32_t* sent_ids, int64_t n_sent,
    int64_t tile_len, int64_t b, int64_t tq_max, int64_t tk_max, int heads, int64_t dk,
    float scale, int accumulate_q, int accumulate_k, int accumulate_v, void* stream);
int mtkc_attention_tc_varlen_backward(const float* gout, int64_t ldo, const float* probs,
                                      const float* q, int64_t ldq, const float* k,
                                      const float* v, int64_t ldk, float* gq, float* gk,
                                      float* gv, const int32_t* qoff, const int32_t* koff,
                                      int64_t b, int64_t tq_max, int64_t tk_max, int heads,
                                      int64_t dk, float scale, int accumulate_q,
                                      int accumulate_k, int accumulate_v, void* stream);

/* ======================================================================== */
/* fused GRU block, pointwise part (gruCell graph.cpp:648-813, gruPre        */
/* :633-645).  The matrix products come from mtkc_gemm: hu = h[Uz|Ur|Uh]     */
/* and xw = x[Wz|Wr|Wx] ([b x 3d] each, ld 3d; xw NULL for transition-only   */
/* blocks).  Forward per row:                                                */
/*   z = sig(LNz(hu_z + xw_z + bz)), r = sig(LNr(hu_r + xw_r + br)),         */
/*   ac = LNx(xw_x) (0 without input) + (r*hu_h + bh), ht = tanh(ac),        */
/*   h' = (1-z)*ht + z*h.   LN is applied iff the ln pointers are non-NULL.  */
/* cache [b x 3d]: z | r | ht;  lnc [b x 3d] xhat_z | xhat_r | xhat_x and    */
/* lnrs [b x 3]: inverse std per gate (LN only).                             */
/* Backward per row from go = dL/dh': dpz, dpr = grads of the pre-LN gate    */
/* sums (U/W/bias products), duh = dL/d(h Uh), dac = dL/d(ac) (bh grad),      */
/* dax = dL/d(x Wx) (LN-inverted dac); gh (+)= go*z; lnparts [b x 6d] holds   */
/* per-row dgain/dbias terms (z, r, x) for a column reduction.               */
/* ======================================================================== */
typedef struct mtkc_gru_args {
  int64_t b, d;
  const float* h;      /* [b x d] state fed to the block */
  const float* hu;     /* [b x 3d] */
  const float* xw;     /* [b x 3d] or NULL */
  const float* bz;
  const float* br;
  const float* bh;
  const float* lnGz;   /* LN gains/biases or NULL (no layer norm) */
  const float* lnBz;
  const float* lnGr;
  const float* lnBr;
  const float* lnGx;
  const float* lnBx;
  float eps;
  float* hout;         /* [b x d] */
  float* cache;        /* [b x 3d] */
  float* lnc;          /* [b x 3d] (LN only) */
  float* lnrs;         /* [b x 3]  (LN only) */
  /* backward */
  const float* go;     /* [b x d] */
  float* gh;           /* [b x d] */
  int accumulate_h;
  float* dpz;          /* [b x d] each */
  float* dpr;
  float* duh;
  float* dac;
  float* dax;          /* may alias dac when there is no LN */
  float* lnparts;      /* [b x 6d] (LN only) */
  /* padding blend folded into the block (maskBlend, models.cpp:170-172 and
   * 362-363): with blend_mask [b] (0/1 per row) the forward writes
   * hout = h'*m + prev*(1-m); the backward feeds go*m to the block and
   * gprev (+)= go*(1-m) (gprev may be gh: the block's input is prev) */
  const float* blend_mask;
  const float* blend_prev;   /* [b x d] */
  float* gprev;              /* [b x d] or NULL (prev not differentiable) */
  int accumulate_prev;
} mtkc_gru_args;

int mtkc_gru_forward(const mtkc_gru_args* a, void* stream);
int mtkc_gru_backward(const mtkc_gru_args* a, void* stream);

/* Fused LSTM cell pointwise (north_star "fused GRU/LSTM cell ops"; the
 * reference has no LSTM -- pinned against a composition of its primitives).
 * pre [b x 4d] = h*U + x*W (gate blocks i, f, o, g), bias [4d], c [b x d];
 * out [b x 2d] = [h' | c'], cache [b x 5d] = [i | f | o | g | tanh(c')].
 * Backward: gout [b x 2d] -> dpre [b x 4d] (written), dc (+)= d(c) or NULL. */
int mtkc_lstm_forward(const float* pre, const float* bias, const float* c, float* out,
                      float* cache, int64_t b, int64_t d, void* stream);
int mtkc_lstm_backward(const float* gout, const float* cache, const float* c, float* dpre,
                       float* dc, int accumulate_c, int64_t b, int64_t d, void* stream);

/* ======================================================================== */
/* Persistent GRU scan (sequence-level recurrence of RnnEncoder::build and   */
/* RnnDecoder::step, models.cpp:146-187, 312-382; DeepTransitionCell         */
/* layers.cpp:183-244; gruCell graph.cpp:633-745; Bahdanau layers.cpp:59-79) */
/* as ONE cooperative launch over all T steps (both encoder directions in    */
/* one launch): per block and step the recurrent product h*[Uz|Ur|Uh] is a   */
/* K-split tcgen05 product over all SMs (fp32 partials, TMA-fed, TMEM        */
/* accumulators), then a row-wise pointwise phase sums the partials in a     */
/* fixed order and applies bias / layer norm / gates exactly like            */
/* mtkc_gru_forward; grid barriers separate the phases.  Outputs are the     */
/* same time-major buffers the per-step path writes, so the backward and     */
/* the hoisted weight-gradient products consume them unchanged.              */
/* ======================================================================== */
#define MTKC_RNN_MAX_BLOCKS 8
typedef struct mtkc_rnn_block {
  const float* U[3];     /* Uz, Ur, Uh [d x d] (reference layout, row-major) */
  const float* bias[3];  /* bz, br, bh [d] */
  const float* ln[6];    /* lnGz lnBz lnGr lnBr lnGx lnBx [d] or NULL */
  const float* W[3];     /* per-step input weights [kd x d] (decoder block 2), or NULL */
  float* hu;             /* [T*b x 3d] out: h*U per step */
  float* cache;          /* [T*b x 3d] out: z, r, h~ */
  float* lnc;            /* [T*b x 3d] out (LN only) */
  float* lnrs;           /* [T*b x 3]  out (LN only) */
  /* backward (mtkc_rnn_scan_backward) */
  float* dGx;            /* [T*b x 3d] out: dpz | dpr | dax (blocks with an input), or NULL */
  float* dac;            /* [T*b x d] out: candidate pre-activation gradient */
  float* lnp;            /* [T*b x 6d] out: LN gain/bias partials (LN only) */
} mtkc_rnn_block;

typedef struct mtkc_rnn_dir {
  int reverse;           /* 1: t = T-1 .. 0, state slots t+1 -> t */
  int nblocks;
  mtkc_rnn_block blk[MTKC_RNN_MAX_BLOCKS];
  float* HH;             /* [(T+1)*b x d]; the initial-state slot is pre-filled */
  float* sout;           /* [(nblocks-1)*T*b x d] outputs of blocks 1..K-1 (block k at k*T*b) */
  const float* xw1;      /* [T*b x 3d] hoisted input product of block 1, or NULL */
  float* xw2;            /* [T*b x 3d] out: per-step ctx*W of block 2 (attention) */
  /* backward */
  float* GH;             /* [(T+1)*b x d] state-slot gradients: pre-filled with the output
                            gradients (initial-state slot zero); the initial slot receives
                            the initial-state gradient */
  float* dG;             /* [nblocks*T*b x 3d] out: dpz | dpr | duh per block (block k at k*T*b) */
} mtkc_rnn_dir;

typedef struct mtkc_rnn_scan_args {
  int64_t b, T, d;
  int ndir;              /* 1 (decoder) or 2 (bidirectional encoder) */
  float eps;
  int lean_cache;        /* forward: store only what mtkc_rnn_scan_backward reads (the h-gate
                            third of hu, no xw2); 0 keeps the per-step path's full caches */
  const float* maskT;    /* [T x b] padding blend mask of the last block, or NULL */
  mtkc_rnn_dir dir[2];
  /* Bahdanau attention between blocks 1 and 2 (decoder, ndir == 1) */
  int has_att;
  int64_t S, a, kd;
  const float* attW;     /* [d x a] query projection */
  const float* attV;     /* [a] */
  const float* attLnG;   /* [a] or NULL */
  const float* attLnB;
  const float* keys;     /* [b x S x kd] */
  const float* uk;       /* [b x S x a] */
  const float* attMask;  /* [b x S] or NULL */
  float* wq;             /* [T*b x a] out */
  float* attT;           /* [T*b*S x a] out: tanh values */
  float* attWts;         /* [T*b x S] out: softmax weights */
  float* attLnx;         /* [T*b*S x a] out (LN only) */
  float* attLnrs;        /* [T*b x S] out (LN only) */
  float* ctx;            /* [T*b x kd] out */
  /* attention backward */
  const float* ctxGrad;  /* [T*b x kd] gradient reaching the contexts from the readout, or NULL */
  float* dctx;           /* [T*b x kd] out: total context gradient per step */
  float* dwq;            /* [T*b x a] out */
  float* guk;            /* [b x S x a] gradient of uk (written, or added when acc_uk) */
  int acc_uk;
  float* vpart;          /* [3][T*b x a] out: v, LN gain, LN bias partials per row */
  int* flags;
  float* workspace;
  size_t workspace_bytes;
} mtkc_rnn_scan_args;

/* 1 when the persistent path supports these dimensions (d % 32 == 0, ...) */
int mtkc_rnn_scan_supported(const mtkc_rnn_scan_args* a);
size_t mtkc_rnn_scan_workspace(const mtkc_rnn_scan_args* a);
int mtkc_rnn_scan_forward(const mtkc_rnn_scan_args* a, void* stream);
/* reverse sweep (gru_bwd_kernel / bahdanau backward arithmetic per block and
 * step; the state-gradient products dG*[Uz|Ur|Uh]^T, dGx*W^T and dwq*attW^T
 * as K-split tcgen05 phases).  Weight / bias / LN gradients are NOT formed:
 * the caller sums them over all b*T rows from dG, dGx, dac, lnp, dwq, vpart
 * (and the key gradient from attWts and dctx) after the sweep. */
/* keys gradient of the scan's attention: gkeys[r,s,:] (+)= sum_t attWts[t*b+r, s] *
 * dctx[t*b+r, :]  (T x (256 + S) floats of shared memory per CTA) */
int mtkc_rnn_key_grad(float* gkeys, const float* attW, const float* dctx, int64_t b, int64_t T,
                      int64_t S, int64_t kd, int accumulate, void* stream);
size_t mtkc_rnn_scan_bwd_workspace(const mtkc_rnn_scan_args* a);
int mtkc_rnn_scan_backward(const mtkc_rnn_scan_args* a, void* stream);

/* ======================================================================== */
/* Bahdanau MLP attention core (BahdanauAttention::apply layers.cpp:59-79),  */
/* fused: given wq = query*W [b x a] and uk = keys*U [b x s x a] (GEMMs, the */
/* latter computed once per batch), per row and source position j:           */
/*   t_j = tanh(LN(wq + uk_j)) (LN optional), e_j = t_j . v,                 */
/*   w = masked softmax_j(e), ctx = sum_j w_j keys_j.                        */
/* Backward produces d(wq), d(uk), d(keys) and per-row partials of d(v) and  */
/* the LN gain/bias gradients (column-summed over b by the caller).          */
/* ======================================================================== */
typedef struct mtkc_bahdanau_args {
  int64_t b, s, a, kd;
  const float* wq;     /* [b x a] */
  const float* uk;     /* [b x s x a] */
  const float* v;      /* [a] */
  const float* keys;   /* [b x s x kd] */
  const float* mask;   /* [b x s] or NULL */
  const float* lnG;    /* [a] or NULL (no layer norm) */
  const float* lnB;
  float eps;
  float* t;            /* [b x s x a] saved tanh */
  float* lnxh;         /* [b x s x a] (LN only) */
  float* lnrs;         /* [b x s]     (LN only) */
  float* w;            /* [b x s] attention weights */
  float* ctx;          /* [b x kd] */
  int* flags;
  /* backward */
  const float* gctx;   /* [b x kd] */
  float* gkeys;
  int acc_keys;
  float* gwq;
  int acc_wq;
  float* guk;
  int acc_uk;
  float* gv_part;      /* [b x a] */
  float* glnG_part;    /* [b x a] (LN only) */
  float* glnB_part;    /* [b x a] (LN only) */
  float* scratch;      /* [4 x b x s] workspace (scores; dw, de, LN row stats) */
} mtkc_bahdanau_args;

int mtkc_bahdanau_forward(const mtkc_bahdanau_args* a, void* stream);
int mtkc_bahdanau_backward(const mtkc_bahdanau_args* a, void* stream);

/* ======================================================================== */
/* cross-entropy over the vocabulary (crossEntropy graph.cpp:859-924)       */
/* fwd: per row lse = max + log(sum exp(x - max)); row_loss = m*(lse - x_y); */
/* loss = sum(row_loss)/count (deterministic single-block sum).              */
/* bwd: g (+)= (softmax(x) - onehot(y)) * m * go / count, go read on device. */
/* ======================================================================== */
int mtkc_xent_forward(const float* logits, const int32_t* targets, const float* mask,
                      int64_t rows, int64_t vocab, float* lse, float* row_loss, float* loss,
                      float count, void* stream);
/* Fused forward + backward (TF32 training path, vocab % 4 == 0, vocab <= 32768):
 * the loss as mtkc_xent_forward and, in place over `logits`, the gradient
 * (softmax - onehot) * m * scale / count for the loss seed `scale`. */
int mtkc_xent_fused_supported(int64_t vocab);
int mtkc_xent_fused(float* logits, const int32_t* targets, const float* mask, int64_t rows,
                    int64_t vocab, float scale, float* row_loss, float* loss, float count,
                    void* stream);
int mtkc_xent_backward(float* glogits, const float* logits, const float* lse,
                       const int32_t* targets, const float* mask, const float* gloss,
                       int64_t rows, int64_t vocab, float count, int accumulate,
                       void* stream);
/* TF32-precision variants: same outputs from one pass over each row (online
 * max / rescaled sum), exp via ex2.approx (relative error ~2^-21 per term);
 * the backward needs vocab % 4 == 0 and 16-byte aligned rows (else it runs
 * mtkc_xent_backward). */
int mtkc_xent_forward_fast(const float* logits, const int32_t* targets, const float* mask,
                           int64_t rows, int64_t vocab, float* lse, float* row_loss, float* loss,
                           float count, void* stream);
int mtkc_xent_backward_fast(float* glogits, const float* logits, const float* lse,
                            const int32_t* targets, const float* mask, const float* gloss,
                            int64_t rows, int64_t vocab, float count, int accumulate,
                            void* stream);

/* ======================================================================== */
/* optimizer (Adam::updateTensor train.cpp:30-47, Adam::update :49-59,      */
/* AveragedParameters::update :69-79) fused: one pass over the flat         */
/* parameter/gradient/moment/average buffers.  Skipped entirely (device-side)*/
/* when *flags has MTKC_FLAG_NONFINITE (all-or-nothing, train.cpp:51-53).    */
/* corr1/corr2 are the host's (Real)(1 - pow((double)beta, step)).           */
/* zero_grad: grad = 0 afterwards (train.cpp:57).                            */
/* ======================================================================== */
int mtkc_adam_ema(float* theta, float* grad, float* m, float* v, float* avg, int64_t n,
                  float lr, float beta1, float beta2, float eps, float corr1, float corr2,
                  float avg_beta, int do_avg, int zero_grad, const int* flags, void* stream);
/* avg = beta*avg + (1-beta)*theta (AveragedParameters::update train.cpp:69-79) */
int mtkc_ema(float* avg, const float* theta, int64_t n, float beta, void* stream);

/* ======================================================================== */
/* data-parallel gradient exchange (trainSync train.cpp:254-269): NCCL       */
/* all-reduce(sum) of grads pre-scaled by tokens_r/total.                    */
/* ======================================================================== */
int mtkc_nccl_unique_id(void* id_out_128);
int mtkc_nccl_comm_init(void** comm, int nranks, int rank, const void* id_128);
int mtkc_nccl_comm_destroy(void* comm);
/* number of ranks in the communicator (ncclCommCount) */
int mtkc_nccl_comm_count(void* comm, int* count);
int mtkc_allreduce_sum(void* comm, float* buf, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MTK_CUDA_H */
