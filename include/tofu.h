/* libtofu — C ABI of the B200-native Tofu hot path.
 *
 * Paper: "Supporting Very Large Models using Automatic Dataflow Graph Partitioning"
 * (Tofu, arXiv 1807.08887), /root/reference/PAPER.md, cited P:L<line>.
 *
 * Conventions for every call:
 *   - Return value: TOFU_OK (0) or a negative TOFU_ERR_*; on error tofu_last_error() returns a
 *     thread-local message.  No call aborts the process.
 *   - Pointers named *_dev are device pointers (cudaMalloc / torch CUDA tensors); all other pointers
 *     are host pointers.  Objects created by tofu_*_create are owned by the caller and released by the
 *     matching *_destroy.  Output text buffers are caller-owned: pass (buf, cap); the call writes a
 *     NUL-terminated string if it fits and always stores the required length (without NUL) in *len.
 *   - Streams are cudaStream_t passed as void*; NULL = the legacy default stream.  Device calls are
 *     asynchronous on that stream and never synchronise the host.
 *   - Tensors are dense row-major; dtype codes: TOFU_BF16 (2 bytes) / TOFU_F32 (4 bytes).
 */
#ifndef TOFU_H_
#define TOFU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOFU_OK 0
#define TOFU_ERR_ARG (-1)    /* invalid argument / shape */
#define TOFU_ERR_PARSE (-2)  /* TDL or graph JSON rejected */
#define TOFU_ERR_PLAN (-3)   /* no plan (e.g. no divisible dim) */
#define TOFU_ERR_CUDA (-4)   /* CUDA runtime / driver error */
#define TOFU_ERR_ALIGN (-5)  /* pointer / pitch alignment requirement violated */
#define TOFU_ERR_STATE (-6)  /* object used in the wrong state */
#define TOFU_ERR_SPACE (-7)  /* output buffer too small (len still reported) */

#define TOFU_BF16 0
#define TOFU_F32 1

const char* tofu_last_error(void);
const char* tofu_version(void);

/* ======================================================================================= a1
 * tofu_describe_op — analyse one TDL operator description (§4.1, §4.2).
 *   tdl   : text "def name(T1(r1), ...) -> lambda v1, ...: body" (grammar in DESIGN.md §R1).
 *   ways  : s >= 2, number of parts of a basic strategy.
 *   out   : JSON {"name","params":[[t,rank]],"out_vars","red_vars","reducer","class",
 *           "accesses":[{"tensor","index":[{"coef":{var:int},"const":int}|null]}],
 *           "strategies":[{"var","kind":"Concat"|"Reduce","regions":[[{"tensor",
 *             "dims":[{"lo":[num..],"c_lo":num,"hi":[num..],"c_hi":num}|null]}]]}]}
 *           where region j is worker j's symbolic interval (Eq. 1, closed, 𝒳 = largest index).
 * Errors: TOFU_ERR_PARSE (syntax, undeclared tensor, rank mismatch, non-affine index, nested reduce,
 *         Assumption #1 violation), TOFU_ERR_SPACE.
 */
int tofu_describe_op(const char* tdl, int ways, char* out, size_t cap, size_t* len);

/* ======================================================================================= graph
 * Graph JSON (same schema as oracle/graph.py): {"defs":{name:tdl}, "tensors":{name:{"shape",
 * "dtype":"bf16"|"f32","role","grad_of","merge"}}, "ops":[{"name","def","inputs","output",
 * "backward_of","merge","attrs"}], "alias":{new:old}}.  Ops are listed in execution order.
 */
typedef struct tofu_graph tofu_graph;
int tofu_graph_create(const char* graph_json, tofu_graph** out);
void tofu_graph_destroy(tofu_graph* g);

/* ======================================================================================= a2
 * tofu_plan_create — per-tensor partition plan for k workers minimising communicated elements
 * (§5), by the recursive 2-way (kᵢ-way) DP over the coarsened graph.
 * Cost model: DESIGN.md §R3 (direct transfer).  k = Πkᵢ, kᵢ non-increasing primes.
 *   opts may be NULL (defaults: frontier_cap 64, solution_cap 256, search = recursive).
 * Errors: TOFU_ERR_PLAN when some tensor/op has no divisible axis at a step.
 */
typedef struct {
  int frontier_cap;  /* co-optimal prefixes kept per step (>=1) */
  int solution_cap;  /* co-optimal step plans enumerated per prefix (>=1) */
  int search;        /* 0 = recursive (paper), 1 = flat exact (all steps jointly; small graphs) */
} tofu_plan_options;

typedef struct tofu_plan tofu_plan;
int tofu_plan_create(const tofu_graph* g, int k, const tofu_plan_options* opts, tofu_plan** out);
void tofu_plan_destroy(tofu_plan* p);
/* {"k","factors":[..],"tdims":{t:[d|null..]},"osplit":{op:[var..]},"cost":elements,"bytes":B,
 *  "deltas":[..],"frontier_truncated":bool,"search_ms":ms} */
int tofu_plan_json(const tofu_plan* p, char* out, size_t cap, size_t* len);
int tofu_plan_cost(const tofu_plan* p, int64_t* elements, int64_t* bytes);

/* ======================================================================================= a3/a8
 * Execution.  Each rank owns an arena (device memory, caller-allocated, 256-byte aligned) holding its
 * shards of every tensor and its staging buffers; tofu_exec_arena_bytes() gives the size.  A process
 * drives one or more ranks: n_local ranks listed in local_ranks; arena_dev[r] is rank r's arena base as
 * addressable from this process for ALL k ranks (local memory, or a peer mapping via CUDA IPC / NVLink).
 * With all k ranks local on one GPU ("virtual ranks") the same kernels run and peer pointers are local.
 * flags_dev: per-rank 64-byte-aligned signal words used for cross-process barriers (may be NULL when
 * all ranks are local).
 */
typedef struct tofu_exec tofu_exec;
int tofu_exec_arena_bytes(const tofu_graph* g, const tofu_plan* p, int rank, int64_t* bytes);
/* offset/shape of tensor t's shard inside rank's arena: box[2*d] = lo, box[2*d+1] = hi (closed). */
int tofu_exec_shard(const tofu_graph* g, const tofu_plan* p, int rank, const char* tensor, int64_t* offset,
                    int64_t* box, int* rank_out);
int tofu_exec_create(const tofu_graph* g, const tofu_plan* p, int n_local, const int* local_ranks,
                     void* const* arena_dev, void* const* flags_dev, tofu_exec** out);
void tofu_exec_destroy(tofu_exec* e);
/* One training step of the partitioned graph: for each op in order and each local rank: MultiFetch of
 * remote input regions (a5), sub-op (a4/a7), spread reduction / scatter of outputs to owners (a6). */
int tofu_execute(tofu_exec* e, void* stream);
/* Bytes moved between distinct ranks by the last tofu_execute, counted from the lowered pieces:
 * fetched (tensor dtype) and reduced/scattered (fp32 for partials).  elements likewise. */
int tofu_exec_ledger(const tofu_exec* e, int64_t* elements, int64_t* bytes);
/* Number of kernel launches issued by one tofu_execute (all local ranks). */
int tofu_exec_launch_count(const tofu_exec* e, int64_t* launches);
/* 1 = skip fetch/reduce kernels (compute-only time), 0 = normal. */
int tofu_exec_set_skip_comm(tofu_exec* e, int skip);
/* Launch list introspection (kernels, barriers and memsets of one step, in issue order). */
int tofu_exec_num_launches(const tofu_exec* e, int* n);
/* JSON {"index","kind":"fetch"|"compute"|"reduce"|"barrier"|"memset","op","def","rank","flops",
 *       "bytes"}: flops = 2·M·N·K for GEMM sub-ops; bytes = algorithmic bytes read + written. */
int tofu_exec_launch_desc(const tofu_exec* e, int index, char* out, size_t cap, size_t* len);
/* Issue launches [first, last) only (instrumented timing). */
int tofu_execute_range(tofu_exec* e, int first, int last, void* stream);
/* Record cudaEvent_t ev_start / ev_stop (on the execute stream) around launch `index` during every
 * subsequent tofu_execute; index < 0 disables. */
int tofu_exec_time_launch(tofu_exec* e, int index, void* ev_start, void* ev_stop);

/* ======================================================================================= kernels
 * Device entry points used by tofu_execute, exported for parity tests.
 */

/* a4 — C[m,n] (+)= Σ_k A[m,k]·B[k,n], bf16 operands, fp32 accumulation in TMEM (tcgen05).
 *   A K-major: A[m*lda+k]; MN-major: A[k*lda+m].  B K-major: B[n*ldb+k]; MN-major: B[k*ldb+n].
 *   c_mode 0: C bf16 = round(acc); 1: C f32 = acc; 2: C f32 += acc;
 *          3: fused momentum-SGD on a weight gradient (P:L674-678 optimizer chain folded into its
 *             producer): C f32 (momentum, in/out) = C*s0 + acc; D bf16 (weight, in/out) = D - C*s1.
 *   ldc/ldd in elements.  Requirements: lda, ldb, ldd multiples of 8, ldc*elem a multiple of 16 B;
 *   A, B, C, D 16-byte aligned.  bn: 0 = auto, 128 or 256.  max_ctas: 0 = #SMs (persistent grid).
 */
typedef struct {
  int M, N, K;
  const void* A;
  int lda, a_mn_major;
  const void* B;
  int ldb, b_mn_major;
  void* C;
  int ldc, c_mode;
  int bn, max_ctas;
  void* D;
  int ldd;
  float s0, s1;
  int splits;  /* split-K: 0 = auto (when the output tiles cannot fill the SMs), 1 = off, n = n splits;
                  tofu_gemm_plan_tmaps writes the chosen value back */
  void* ws;    /* split-K fp32 workspace (tofu_gemm_workspace_bytes); NULL = library-owned */
} tofu_gemm_args;
int tofu_gemm_bf16(const tofu_gemm_args* args, void* stream);
/* Split form used by the executor: encode the TMA descriptors (A, B, C, D, workspace) once into `tmaps`
 * (5 x 128 bytes, 64-byte aligned; args->splits/ws are updated), then launch with them.  Split-K results
 * are reduced in fixed split order (deterministic). */
int tofu_gemm_plan_tmaps(tofu_gemm_args* args, void* tmaps, int* bn_out);
int tofu_gemm_launch_planned(const tofu_gemm_args* args, const void* tmaps, int bn, void* stream);
int64_t tofu_gemm_workspace_bytes(const tofu_gemm_args* args);

/* a5/a6 — box copy / reduction pieces (rank <= 4, innermost dim last, strides in elements).
 * A piece copies (nsrc == 1) or sums in order (nsrc > 1, fp32 arithmetic) nsrc source boxes of the same
 * extent into one destination box, converting dtype.  Sources may be peer pointers. */
#define TOFU_MAX_SRC 8
typedef struct {
  int64_t extent[4];
  void* dst;
  int64_t dst_stride[4];
  int dst_dtype, nsrc;
  const void* src[TOFU_MAX_SRC];
  int64_t src_stride[4];
  int src_dtype, pad_;
} tofu_piece;
/* pieces_dev: device array of n pieces (caller-owned). */
int tofu_pieces_run(const tofu_piece* pieces_dev, int n, int64_t max_elems, void* stream);

/* a7 — element-wise kernels on contiguous n-element buffers.
 *   TOFU_EW_RELU      y = max(x0, 0)                      (bf16 -> bf16)
 *   TOFU_EW_RELU_GRAD y = x0 > 0 ? x1 : 0                 (bf16, bf16 -> bf16)
 *   TOFU_EW_MSE_GRAD  y = (x0 - x1) * s0                  (bf16, bf16 -> bf16)
 *   TOFU_EW_MOM       y = x0 * s0 + x1                    (f32, f32 -> f32)
 *   TOFU_EW_SGD       y = x0 - x1 * s0                    (bf16, f32 -> bf16)
 *   TOFU_EW_SGD_MOM   fused: m' = m*s0 + g; w' = w - m'*s1; x0 = m (f32, in/out), x1 = g (f32),
 *                     x2 = w (bf16, in/out); y unused
 *   TOFU_EW_SUMSQ     y[0] (f32, accumulated with atomicAdd) += Σ (x0 - x1)^2 * s0  (bf16, bf16)
 */
#define TOFU_EW_RELU 0
#define TOFU_EW_RELU_GRAD 1
#define TOFU_EW_MSE_GRAD 2
#define TOFU_EW_MOM 3
#define TOFU_EW_SGD 4
#define TOFU_EW_SGD_MOM 5
#define TOFU_EW_SUMSQ 6
int tofu_elementwise(int kind, int64_t n, void* y_dev, const void* x0_dev, const void* x1_dev, void* x2_dev,
                     float s0, float s1, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOFU_H_ */
