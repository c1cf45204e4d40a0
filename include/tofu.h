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
 *   opts may be NULL (defaults: frontier_cap 64, solution_cap 256, search = 2 auto).
 *   search = 2 (auto, reading R4 of DESIGN.md): the recursion, then — when the exact joint ("flat")
 *   search is small (Σ over op classes of its factor-table cells <= 2^20) — the flat search, whose plan
 *   replaces the recursion's only when strictly cheaper.  Under the direct-transfer cost model (R3) the
 *   recursion misses the optimum on a few small graphs (tests/test_oracle_optimality.py); auto returns the
 *   exhaustive optimum on every graph small enough to check it.
 * Errors: TOFU_ERR_PLAN when some tensor/op has no divisible axis at a step.
 */
typedef struct {
  int frontier_cap;  /* co-optimal prefixes kept per step (>=1) */
  int solution_cap;  /* co-optimal step plans enumerated per prefix (>=1) */
  int search;        /* 0 = recursive (paper), 1 = flat exact (all steps jointly; small graphs), 2 = auto */
} tofu_plan_options;

typedef struct tofu_plan tofu_plan;
int tofu_plan_create(const tofu_graph* g, int k, const tofu_plan_options* opts, tofu_plan** out);
void tofu_plan_destroy(tofu_plan* p);
/* {"k","factors":[..],"tdims":{t:[d|null..]},"osplit":{op:[var..]},"cost":elements,"bytes":B,
 *  "deltas":[..],"frontier_truncated":bool,"search":"recursive"|"flat","search_ms":ms} */
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
 * remote input regions (a5), sub-op (a4/a7), spread reduction / scatter of outputs to owners (a6).
 * Streams: compute launches go to `stream`; fetch / reduce / barrier launches go to an executor-owned comm
 * stream (always in multi-process mode; on virtual ranks by default, TOFU_STREAMS=1 keeps one stream), forked from `stream` at the start
 * and joined back at the end, each launch waiting (CUDA events) only for the launches it depends on (last
 * writer / readers of the tensors and of the two alternating staging buffers it touches).  Device barriers
 * (multi-process) are placed only before a launch that would otherwise race with a peer: reading peer memory
 * some rank wrote since the last barrier, or writing memory some rank read remotely since then; decided from
 * all ranks' lowering, so every process issues the same sequence.  `stream` may be capturing a CUDA graph. */
int tofu_execute(tofu_exec* e, void* stream);
/* Bytes moved between distinct ranks by the last tofu_execute, counted from the lowered pieces:
 * fetched (tensor dtype) and reduced/scattered (fp32 for partials).  elements likewise. */
int tofu_exec_ledger(const tofu_exec* e, int64_t* elements, int64_t* bytes);
/* Number of kernel launches issued by one tofu_execute (all local ranks). */
int tofu_exec_launch_count(const tofu_exec* e, int64_t* launches);
/* 1 = skip the fetch / reduce / barrier launches (compute-only time), 0 = normal.  A GEMM whose
 * operand is read in place from its owners (fused fetch, tofu_operand_pieces) still performs those reads inside
 * the compute launch: its time includes that transfer (it is not separable — the point of the fusion), so at
 * k > 1 the compute-only time is an upper bound for plans with fused operands. */
int tofu_exec_set_skip_comm(tofu_exec* e, int skip);
/* Launch list introspection (kernels, barriers and memsets of one step, in issue order). */
int tofu_exec_num_launches(const tofu_exec* e, int* n);
/* JSON {"index","kind":"fetch"|"compute"|"reduce"|"barrier"|"memset","op","def","rank","flops",
 *       "bytes"}: flops = 2·M·N·K for GEMM sub-ops; bytes = algorithmic bytes read + written. */
int tofu_exec_launch_desc(const tofu_exec* e, int index, char* out, size_t cap, size_t* len);
/* Per-rank share of the ledger (bytes per step): in_bytes = what `rank` reads from its peers (fetched input
 * regions, pulled partials), out_bytes = what its peers read from it.  Σ in = Σ out = the ledger bytes.
 * The step's NVLink bound is max over ranks of max(in, out) / per-direction bandwidth (bench.py).
 * Errors: TOFU_ERR_ARG (null exec, rank outside [0, k)). */
int tofu_exec_rank_bytes(const tofu_exec* e, int rank, int64_t* in_bytes, int64_t* out_bytes);
/* JSON list of the tensors the step never writes to HBM on some rank: intermediates of fused chains
 * (R8 / R13 — a weight gradient folded into the optimizer epilogue, a GEMM / convolution output
 * folded into its element-wise consumer).  Their storage holds no defined value after tofu_execute; parity
 * tests check them through their consumers.  Errors: TOFU_ERR_ARG (null exec) / TOFU_ERR_SPACE. */
int tofu_exec_unmaterialized(const tofu_exec* e, char* out, size_t cap, size_t* len);
/* Issue launches [first, last) only (instrumented timing). */
int tofu_execute_range(tofu_exec* e, int first, int last, void* stream);
/* Record cudaEvent_t ev_start / ev_stop (on the execute stream) around launch `index` during every
 * subsequent tofu_execute; index < 0 disables. */
int tofu_exec_time_launch(tofu_exec* e, int index, void* ev_start, void* ev_stop);

/* ======================================================================================= a8 (multi-process)
 * CUDA IPC for one process per GPU.  tofu_ipc_export: the 64-byte cudaIpcMemHandle of the
 * allocation holding dev_ptr (caller-allocated device memory, e.g. a torch tensor) and dev_ptr's byte offset
 * in it.  tofu_ipc_open: map a peer's exported allocation into THIS process on local_device (made current),
 * enabling peer access from local_device to peer_device first (peer_device < 0 or == local_device: same GPU,
 * nothing to enable); *ptr_out = mapped base + offset, an address this process's kernels on local_device
 * dereference over NVLink.  tofu_ipc_close(ptr, offset) unmaps it.  Errors: TOFU_ERR_ARG, TOFU_ERR_CUDA (no
 * peer access between the GPUs, an invalid handle). */
int tofu_ipc_export(const void* dev_ptr, void* handle_out, int64_t* offset_out);
int tofu_ipc_open(const void* handle, int64_t offset, int local_device, int peer_device, void** ptr_out);
int tofu_ipc_close(void* mapped_ptr, int64_t offset);
/* Test aid: a one-thread kernel that spins ns nanoseconds on the stream.  With TOFU_JITTER=<seed> in the
 * environment at tofu_exec_create, the executor inserts such spins (0-200 us, pseudo-random per rank, launch
 * and step) before a quarter of its launches, so cross-process synchronisation is exercised under skew. */
int tofu_spin(int64_t ns, void* stream);

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
/* An operand assembled from up to TOFU_MAX_PIECES 2-D strided views (the fused MultiFetch of a partitioned
 * sub-op, §6: the remote regions an operand needs are read by the GEMM's TMA producer straight
 * from their owners' shards — peer HBM over NVLink, or the rank's own shard — instead of being copied into
 * staging first).  The pieces tile the operand along one GEMM dimension: dim 0 = M (operand A) / N (B),
 * dim 1 = K.  Piece i covers [start[i], start[i+1]) (the last up to the operand's extent) of that
 * dimension and the whole operand in the other; its element (0, 0) is at ptr[i] with row pitch ld[i]
 * elements, in the operand's majorness.  Starts must be multiples of the tile (M 128, N the launch's BN,
 * K 64); start[0] = 0; pointers 16-byte aligned, pitches multiples of 8.  The memory must stay valid and
 * unchanged until the launch completes (the executor brackets such launches with device barriers). */
#define TOFU_MAX_PIECES 8
typedef struct {
  int n;    /* number of pieces, 1..TOFU_MAX_PIECES */
  int dim;  /* 0: M (A) / N (B); 1: K */
  int start[TOFU_MAX_PIECES];
  const void* ptr[TOFU_MAX_PIECES];
  int64_t ld[TOFU_MAX_PIECES];
} tofu_operand_pieces;

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
  int splits;  /* split-K: 0 = auto (when the output tiles cannot fill the SMs), 1 = off, n = n splits,
                  -1 = stream-K (needs sk_ws; not chosen automatically for the GEMM, see gemm_tcgen05.cu);
                  tofu_gemm_plan_tmaps writes the chosen value back */
  void* ws;    /* split-K fp32 workspace (tofu_gemm_workspace_bytes); NULL = library-owned */
  /* element-wise epilogue of a bf16 output (c_mode 0; the consumers' ops fused into their producer, DESIGN
   * R8/R13): ep bit 1 = add aux_add, bit 0 = relu, bit 2 = zero where aux_mask <= 0, applied in that order;
   * aux tensors bf16 with C's layout (pitch ldc).  ep != 0 disables split-K. */
  const void* aux_add;
  const void* aux_mask;
  int ep;
  /* stream-K workspace (tofu_sk_workspace_bytes, zero-filled once by its owner, left zeroed by every launch;
   * one launch at a time may use it): NULL = data-parallel tiles only.  With it (and splits = -1 for the
   * GEMM; automatic for compute-bound convolutions), shapes whose tile count leaves SMs idle in the last
   * wave split the k-loop of some tiles across CTAs and sum the fp32 partials in fixed CTA order before the
   * epilogue (common.cuh WorkList). */
  void* sk_ws;
  /* optional piecewise operands (NULL = A / B as given above): see tofu_operand_pieces */
  const tofu_operand_pieces* a_pieces;
  const tofu_operand_pieces* b_pieces;
  /* set by tofu_gemm_plan_tmaps: 1 = launched as clusters of 2 CTAs on vertically adjacent tiles that
   * share (TMA-multicast) the B tile; 3 = 2-CTA MMA pairs (tcgen05 cta_group::2, M = 256 over the pair, each
   * CTA staging its A rows and half of B).  On entry -1 forbids both, 2 requests the multicast pairs and 4 the
   * 2-CTA MMA where eligible (parity tests), 0 = automatic */
  int cl2;
  /* 1 = with split-K (splits > 1), leave the fp32 partial planes in ws ([splits][M][N], dense) and skip the
   * ordered reduction: the caller's next launch reduces them (the executor's gate GEMM + LSTM cell fusion).
   * 0 = C holds the result when the call returns (stream order). */
  int defer_reduce;
  /* 1 = every CTA walks its k-blocks from the last to the first (the same sums in reverse order): the executor
   * alternates it launch by launch over the same weight so that a pass starts on the rows the previous pass
   * read last, still in L2.  0 = ascending. */
  int k_reverse;
} tofu_gemm_args;
int tofu_gemm_bf16(const tofu_gemm_args* args, void* stream);
/* Split form used by the executor: encode the TMA descriptors (A, B, C, D, workspace, mask, then the
 * TOFU_MAX_PIECES piece maps of A and of B) once into `tmaps` (TOFU_GEMM_TMAPS x 128 bytes, 64-byte aligned;
 * args->splits/ws are updated), then launch with them.  Split-K results
 * are reduced in fixed split order (deterministic). */
#define TOFU_GEMM_TMAPS (6 + 2 * TOFU_MAX_PIECES)
int tofu_gemm_plan_tmaps(tofu_gemm_args* args, void* tmaps, int* bn_out);
int tofu_gemm_launch_planned(const tofu_gemm_args* args, const void* tmaps, int bn, void* stream);
int64_t tofu_gemm_workspace_bytes(const tofu_gemm_args* args);
/* Bytes of a stream-K workspace for the current device (one fp32 128x256 partial + 8 flags per SM). */
int64_t tofu_sk_workspace_bytes(void);

/* a4' — implicit-GEMM convolution sub-op (NHWC bf16 activations, weights [co][ky][kx][ci], fp32
 * accumulation in TMEM via tcgen05).  The convolution TDL defs (tofu_inputs.graphs.conv_defs; reading R11)
 * are executed as a GEMM one of whose operands is gathered pixel by pixel from an activation buffer S
 * (zero outside the buffer: zero padding) while the other is dense and loaded by TMA.
 *
 * Pixel grid: rows g = (gb, gy, gx) in [0,nb) x [0,ngy) x [0,ngx), flattened gb-major.  Tap t (< ntaps <=
 * TOFU_CONV_MAX_TAPS) reads S pixel (gb + sb0, ay*gy + cy + tap_dy[t], ax*gx + cx + tap_dx[t]) (buffer
 * coordinates; outside [0,sH) x [0,sW) the value is 0) at channels sc0 + [0, nch).
 *
 * kind 0 — forward / data gradient (P:L248-259 sub-op):  M = grid pixels, K = ntaps*nch (k = t*nch + c),
 *   N = n_out.  A[m,k] = S[...] gathered.  B dense in Bp (row pitch ldb, a box of rows x cols):
 *     b_mn_major 0 (forward, W[co][taps][ci]):   B[k,n] = Bp[n*ldb + tap_w[t]*b_tap + c]
 *     b_mn_major 1 (data grad, W[co][taps][ci]): B[k,n] = Bp[c*ldb + tap_w[t]*b_tap + n]
 *   (nch must be a multiple of 64, or — forward only — taps in natural order with b_tap == nch so the K
 *   columns are contiguous).  Output pixel of row (gb, gy, gx): C[gb*c_sb + (c_ys*gy + c_y0)*c_sy +
 *   (c_xs*gx + c_x0)*c_sx + n], c_mode 0 = bf16 store, 1 = f32 store (a Case-2 partial).
 * kind 1 — weight gradient:  M = m_out (output channels), N = ntaps*nch (n = t*nch + c), K = grid pixels.
 *   A[k,m] = Ap[k*lda + m] (the output gradient, pixel rows contiguous, MN-major), B[k,n] = S[...] gathered.
 *   C[m,n] f32 at Cp[m*ldc + n]: c_mode 1 store, 2 accumulate, 3 fused momentum-SGD (as tofu_gemm_args:
 *   C = momentum (in/out) = C*s0 + acc, D bf16 weight (in/out) = D - C*s1, row pitch ldd).  splits: split-K
 *   over pixels (0 = auto, 1 = off) with fp32 workspace ws (tofu_conv_workspace_bytes), reduced in fixed
 *   order (deterministic); the optimizer is applied by the reduction.
 * Tensor-core requirements: nch % 8 == 0, sc0 % 8 == 0, 16-byte aligned pointers, pitches multiples of 8
 * elements; shapes that miss them run on the direct path (field `direct`).
 */
#define TOFU_CONV_MAX_TAPS 64
typedef struct {
  int kind;
  int nb, ngy, ngx;
  int ay, ax, cy, cx, sb0;
  int ntaps, nch;
  short tap_dy[TOFU_CONV_MAX_TAPS], tap_dx[TOFU_CONV_MAX_TAPS], tap_w[TOFU_CONV_MAX_TAPS];
  const void* S;
  int64_t s_sb, s_sy, s_sx;
  int sH, sW, sc0;
  int n_out, m_out;         /* kind 0: N; kind 1: M */
  const void* Bp;           /* kind 0 dense operand */
  int64_t ldb;
  int b_mn_major, b_tap, b_rows, b_cols;   /* dense box extents (rows x cols of the Bp view) */
  const void* Ap;           /* kind 1 dense operand */
  int64_t lda;
  void* C;
  int64_t c_sb, c_sy, c_sx;
  int c_ys, c_y0, c_xs, c_x0;
  int64_t ldc;
  int c_mode;
  void* D;
  int64_t ldd;
  float s0, s1;
  int splits;
  void* ws;
  /* kind 0, c_mode 0: element-wise epilogue as tofu_gemm_args.ep (bit 1 add aux_add, bit 0 relu, bit 2 zero
   * where aux_mask <= 0); aux tensors bf16 with C's layout. */
  const void* aux_add;
  const void* aux_mask;
  int ep;
  void* sk_ws;  /* stream-K workspace, as tofu_gemm_args.sk_ws */
  /* set by tofu_conv_plan: 1 = the geometry misses the tensor-core kernel's 16-byte granules (a channel range
   * of fewer than 8 channels, unaligned pitches, e.g. an 8-way split of the 8-channel image); the same math
   * then runs on CUDA cores (fp32 accumulation, same epilogues).  Never chosen for aligned shapes. */
  int direct;
  /* set by tofu_conv_plan: 1 = the gathered operand is loaded by TMA in im2col mode (stride-1 grid; nch a
   * multiple of 64 (kind 0) / of the N tile (kind 1)), 0 = by the gather warps (cp.async); i2c_dy0/dx0: the
   * smallest tap offsets.
   * On entry, im2col = -1 keeps the gather warps (used by the parity tests). */
  int im2col, i2c_dy0, i2c_dx0;
  /* set by tofu_conv_plan (kind 1 with im2col): 1 = clusters of 2 CTAs on adjacent output-channel tiles share
   * (TMA-multicast) the gathered activations; on entry -1 forbids it, 2 requests it where eligible */
  int cl2;
} tofu_conv_args;
/* Encode TMA descriptors once (tmaps: 5 x 128 B, 64-byte aligned; args->splits / direct / im2col updated), then launch. */
int tofu_conv_plan(tofu_conv_args* args, void* tmaps);
int tofu_conv_launch_planned(const tofu_conv_args* args, const void* tmaps, void* stream);
int tofu_conv_bf16(const tofu_conv_args* args, void* stream);
int64_t tofu_conv_workspace_bytes(const tofu_conv_args* args);

/* Window ops of the WResNet stem and head (NHWC bf16, channel stride 1, C % 8 == 0; every pointer is the
 * element (first b, buffer row 0, buffer col 0, first channel) of its buffer, 16-byte aligned):
 *   tofu_maxpool:      out[b,oy,ox,c] = max_{ky,kx<3} X[b, 2oy+ky-1, 2ox+kx-1, c]   (0 outside X: R11; X >= 0)
 *                      iterates the Y-side box (nb, Ho, Wo) at global origin (oy0, ox0); X buffer (H, W) at
 *                      global origin (y0, x0).
 *   tofu_maxpool_grad: out[b,y,x,c] = Σ_{ty in [ty0,ty1], tx in [tx0,tx1]} select(X[b,y,x,c] == Y[b,oy,ox,c],
 *                      dY[b,oy,ox,c] * K[(y+1)%2 + 2ty, (x+1)%2 + 2tx, c], 0) with oy = (y+1-2ty)/2 (floor),
 *                      ox likewise, K = 0 past tap 2 and Y/dY = 0 outside their buffers (the maxpool_grad TDL
 *                      def); iterates the X-side box (nb, H, W) at (y0, x0); Y / dY buffers (Ho, Wo) at (oy0, ox0).
 *   tofu_gap:          out[b,c] (+partial) = Σ_{y<H, x<W} X[b,y,x,c] * s   (o_sb = row pitch of out)
 *   tofu_gap_grad:     out[b,y,x,c] = dY[b,c] * s over the (nb, H, W) box   (y_sb = row pitch of dY)
 * out_f32: 1 = f32 output (a Case-2 partial), 0 = bf16. */
typedef struct {
  int nb, C;
  int H, W, y0, x0;
  int Ho, Wo, oy0, ox0;
  int64_t x_sb, x_sy, x_sx;
  int64_t y_sb, y_sy, y_sx;
  int64_t d_sb, d_sy, d_sx;
  int64_t o_sb, o_sy, o_sx;
  int64_t k_sy, k_sx;
  const void* X;
  const void* Y;
  const void* dY;
  const void* K;
  void* out;
  int out_f32;
  int ty0, ty1, tx0, tx1;
  float s;
} tofu_window_args;
int tofu_maxpool(const tofu_window_args* a, void* stream);
int tofu_maxpool_grad(const tofu_window_args* a, void* stream);
int tofu_gap(const tofu_window_args* a, void* stream);
int tofu_gap_grad(const tofu_window_args* a, void* stream);

/* Weight re-layout for the convolution data gradient: WT[i][t][o] = W[o][t][i] (bf16, dense, co x taps x ci
 * -> ci x taps x co), so the data gradient reads its weight operand K-major (executor-owned copy, refreshed
 * before each data-gradient launch; DESIGN a10). */
int tofu_transpose_taps(const void* W, void* WT, int co, int taps, int ci, void* stream);

/* a5/a6 — box copy / reduction pieces (rank <= 4, innermost dim last, strides in elements).
 * A piece copies (nsrc == 1) or sums in order (nsrc > 1, fp32 arithmetic) nsrc source boxes of the same
 * extent into one destination box, converting dtype.  Sources may be peer pointers.
 * ep: the element-wise consumer of a reduced tensor applied to the sum v before the store (the
 * partition-n-reduce fused with the next coalesced element-wise op, P:L674-678 / DESIGN R8); aux0 is laid
 * out like dst (same strides):
 *   TOFU_PIECE_RELU      dst = max(v, 0)
 *   TOFU_PIECE_MASK      dst = aux0 (bf16) > 0 ? v : 0                       (relu gradient)
 *   TOFU_PIECE_MOM_SGD   dst (f32 momentum, in/out): m = dst * s0 + v; dst = m; aux0 (bf16 weight, in/out):
 *                        aux0 = aux0 - m * s1                                (momentum + SGD on a gradient)
 *   TOFU_PIECE_ADD       dst = v + aux0 (bf16)          TOFU_PIECE_ADDRELU  dst = max(v + aux0, 0) */
#define TOFU_MAX_SRC 8
#define TOFU_PIECE_COPY 0
#define TOFU_PIECE_RELU 1
#define TOFU_PIECE_MASK 2
#define TOFU_PIECE_MOM_SGD 3
#define TOFU_PIECE_ADD 4
#define TOFU_PIECE_ADDRELU 5
typedef struct {
  int64_t extent[4];
  void* dst;
  int64_t dst_stride[4];
  int dst_dtype, nsrc;
  const void* src[TOFU_MAX_SRC];
  int64_t src_stride[4];
  int src_dtype, pad_;
  int ep;          /* TOFU_PIECE_* */
  float s0, s1;
  int pad2_;
  void* aux0;
} tofu_piece;
/* A task: segments [q0, q0 + nq) of piece `piece` (a row — the normalised innermost dim — is cut into
 * segments of <= 256 vectors; segment q = row q / nseg, part q % nseg).  pad_ = 1 when the piece is a plain
 * copy (one source, same dtype, 16-byte vectors). */
typedef struct {
  int piece, pad_;
  int64_t q0, nq;
} tofu_piece_task;
/* Host: normalise the n pieces IN PLACE (dims contiguous in dst and src merged, unit dims dropped; pad_ =
 * the vector width V in {8,4,2,1} elements: V divides the row and keeps every row start and base pointer
 * V-element aligned) and cut them into tasks of whole segments (~4096 vectors, >= 8 segments).  tasks may be NULL (count only); *ntasks =
 * the number of tasks.  Errors: TOFU_ERR_ARG (nsrc outside [1, TOFU_MAX_SRC], a strided innermost dim in a
 * rank-4 piece, > 2^32 rows), TOFU_ERR_SPACE (cap < *ntasks; the first cap tasks are written). */
int tofu_pieces_tasks(tofu_piece* pieces, int n, tofu_piece_task* tasks, int64_t cap, int64_t* ntasks);
/* Device: run ntasks tasks over pieces (both device arrays, caller-owned, as tofu_pieces_tasks left them).
 * all_raw == 1 (every task's pad_ == 1) selects the plain-copy kernel (16-byte moves, high occupancy);
 * all_raw == 2 the many-source kernel (every source's vector in flight at once, one CTA per SM: for
 * reductions of >= 4 sources); 0 the general kernel.  Every kernel sums the sources in index order. */
int tofu_pieces_run(const tofu_piece* pieces_dev, const tofu_piece_task* tasks_dev, int64_t ntasks, int all_raw,
                    void* stream);

/* a7 — element-wise kernels on contiguous n-element buffers.
 *   TOFU_EW_RELU      y = max(x0, 0)                      (bf16 -> bf16)
 *   TOFU_EW_RELU_GRAD y = x0 > 0 ? x1 : 0                 (bf16, bf16 -> bf16)
 *   TOFU_EW_MSE_GRAD  y = (x0 - x1) * s0                  (bf16, bf16 -> bf16)
 *   TOFU_EW_MOM       y = x0 * s0 + x1                    (f32, f32 -> f32)
 *   TOFU_EW_SGD       y = x0 - x1 * s0                    (bf16, f32 -> bf16)
 *   TOFU_EW_SGD_MOM   fused: m' = m*s0 + g; w' = w - m'*s1; x0 = m (f32, in/out), x1 = g (f32),
 *                     x2 = w (bf16, in/out); y unused
 *   TOFU_EW_SUMSQ     y[0] (f32) += Σ (x0 - x1)^2 * s0  (bf16, bf16; per-block partials summed in block order
 *                     by the last block: deterministic; one such launch at a time per device)
 *   TOFU_EW_SUMSQ_MSE_GRAD  the loss and its gradient in one pass (P:L674-678 coalesced element-wise ops,
 *                     DESIGN R8): y[0] += Σ (x0 - x1)^2 * s0 as TOFU_EW_SUMSQ, and x2 (bf16) = (x0 - x1) * s1
 *   TOFU_EW_ADD       y = x0 + x1                         (bf16, bf16 -> bf16; gradient sums)
 *   TOFU_EW_ADDRELU   y = max(x0 + x1, 0)                 (bf16, bf16 -> bf16; residual join)
 */
#define TOFU_EW_RELU 0
#define TOFU_EW_RELU_GRAD 1
#define TOFU_EW_MSE_GRAD 2
#define TOFU_EW_MOM 3
#define TOFU_EW_SGD 4
#define TOFU_EW_SGD_MOM 5
#define TOFU_EW_SUMSQ 6
#define TOFU_EW_ADD 7
#define TOFU_EW_ADDRELU 8
#define TOFU_EW_SUMSQ_MSE_GRAD 9
int tofu_elementwise(int kind, int64_t n, void* y_dev, const void* x0_dev, const void* x1_dev, void* x2_dev,
                     float s0, float s1, void* stream);
/* The same with the loss reduction's workspace supplied by the caller (ws: tofu_sumsq_workspace_bytes() bytes
 * of device memory, zero-filled once, left zeroed by every launch): concurrent TOFU_EW_SUMSQ launches on
 * different streams / executors then cannot share the block partials and ticket (tofu_elementwise uses one
 * module-wide workspace: one such launch at a time per device).  The executor passes its own. */
int64_t tofu_sumsq_workspace_bytes(void);
int tofu_elementwise_ws(int kind, int64_t n, void* y_dev, const void* x0_dev, const void* x1_dev, void* x2_dev,
                        float s0, float s1, void* ws_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TOFU_H_ */
