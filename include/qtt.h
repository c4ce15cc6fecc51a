/*
 * qtt.h -- C ABI of the B200-native QTT apply library (libqtt_b200.so).
 *
 * The one operation: y = A x, where A is an N x N matrix (N = 2^d) stored in
 * Quantized Tensor-Train form and x, y are dense N x nrhs fp64 matrices.
 *
 *   Definition (PAPER.md Eq. (TTdeccores), with the product-tree
 *   tensorization of a matrix):
 *     A(overline{i_1..i_d}, overline{j_1..j_d})
 *         = G_1(:, i_1 j_1, :) G_2(:, i_2 j_2, :) ... G_d(:, i_d j_d, :)
 *   Method (Alg. 2 "QTT matrix by uncompressed vector product",
 *   P:1441-1532): contract one core per level, k = 1..d, an upward pass that
 *   costs 4 r_{k-1} r_k N flops per level per right-hand side.
 *
 * Conventions (readings R1, R2, R8):
 *   - cores[k-1] holds G_k as ranks[k-1] * 2 * 2 * ranks[k] doubles, row-major
 *     [alpha_{k-1}][i_k][j_k][alpha_k]; i_k is the ROW (target/output) digit,
 *     j_k the COLUMN (source/input) digit.
 *   - Digits are least-significant first: row index i = sum_k i_k 2^{k-1}
 *     (core 1 acts on bit 0, the finest level).  Vectors are in
 *     this hierarchical (Morton) order already.
 *   - x and y are column-major N x nrhs with leading dimension N.
 *
 * Semantics: y = A x up to fp64 rounding (IEEE binary64, FMA contraction,
 * no reduced precision).  NaN/Inf propagate per IEEE; nothing is checked.
 * Results are bitwise deterministic run to run, and each RHS column is
 * bitwise the same whatever nrhs it is applied with: there is no atomic
 * accumulation (the one atomic, the dynamic tile scheduler, decides only which
 * SM computes a tile, never the order of its arithmetic), and a split-K stage
 * (qtt_get_stage_split) sums its partial products in a fixed k-range order in
 * a separate launch, with the split fixed per plan.
 * No exceptions cross this boundary; every entry point returns a qtt_status_t.
 * Threading: a handle (its cached workspace, graphs and staging buffers) must
 * not be used by several host threads at once; separate handles are independent.
 */
#ifndef QTT_B200_H
#define QTT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque plan: packed (super-)cores in device memory + the stage schedule. */
typedef struct qtt_plan* qtt_handle_t;

/* A CUDA stream; layout-compatible with cudaStream_t / CUstream (NULL = the
 * legacy default stream).  Declared here so this header needs no CUDA include. */
typedef struct CUstream_st* qtt_stream_t;

typedef enum {
  QTT_SUCCESS = 0,
  QTT_ERROR_INVALID_VALUE = 1,  /* null pointer, bad d / ranks, nrhs < 1, x/y overlap, short workspace */
  QTT_ERROR_NOT_SUPPORTED = 2,  /* misaligned pointer, host pointer where device memory is required,
                                   no sm_100 device */
  QTT_ERROR_OUT_OF_MEMORY = 3,  /* device allocation failed */
  QTT_ERROR_CUDA = 4            /* a CUDA runtime call or kernel launch failed */
} qtt_status_t;

/* Human-readable name of a status code (static storage; never NULL). */
const char* qtt_status_string(qtt_status_t s);

/*
 * qtt_create -- build a plan from a core list and rank profile.
 *   out    : receives the handle (set to NULL on failure).
 *   d      : number of cores, 1 <= d <= 30 (N = 2^d).
 *   ranks  : host array of d+1 TT ranks; ranks[0] == ranks[d] == 1 and
 *            1 <= ranks[k] <= 4096 (PAPER P:531-534 dummy bonds r_0 = r_d = 1).
 *   cores  : host array of d HOST pointers; cores[k-1] points to
 *            ranks[k-1]*4*ranks[k] doubles in [a][i][j][b] order.
 * The library COPIES and repacks the cores into device memory it owns (on
 * the current CUDA device), so the caller may free its arrays on return.
 * Synchronous.  Plans the stages (see qtt_plan_stages) and uploads.
 */
qtt_status_t qtt_create(qtt_handle_t* out, int d, const int64_t* ranks,
                        const double* const* cores);

/*
 * qtt_create_ex -- qtt_create with the longest merged stage capped at
 * `max_stage_levels` levels (>= 1; 1 = one launch per level, i.e. PAPER
 * Alg. 2 executed level by level; qtt_create uses 10).  Otherwise identical.
 */
qtt_status_t qtt_create_ex(qtt_handle_t* out, int d, const int64_t* ranks,
                           const double* const* cores, int max_stage_levels);

/*
 * qtt_plan_stages -- the stage schedule qtt_create_ex would choose, computed
 * on the host without touching a GPU (pure function of the rank profile).
 * A stage is a run of consecutive levels [k_first, k_last] applied by one
 * kernel launch.  Alg. 2 applies one core per level; a stage of
 * L >= 2 levels applies instead the product of its L cores contracted over
 * the inner bonds (the super-core W[a][ii][jj][b], the QTT definition
 * P:519-523 restricted to the stage's L digits, built once at create time),
 * which is the same linear map, so the level intermediates never exist.  The
 * schedule minimises a cost model of FP64 tensor-core time, HBM bytes and
 * launch latency by dynamic programming over the levels.
 *   d, ranks          : as for qtt_create (validated the same way).
 *   smem_optin        : max dynamic shared memory per block (0 = B200's 232448).
 *   max_stage_levels  : >= 1, as for qtt_create_ex.
 *   n_stages          : receives the number of stages (<= d).
 *   k_first, k_last, variant : arrays of >= d ints (any may be NULL) receiving
 *                       per stage the 1-based level range and the variant
 *                       (0 generic, 1 DMMA one level, 2 DMMA merged stage,
 *                       3 merged stage with the super-core streamed from L2,
 *                       4 small latency-bound stage, warp tiles from L2).
 */
qtt_status_t qtt_plan_stages(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                             int* n_stages, int* k_first, int* k_last, int* variant);

/* qtt_plan_stages plus, per stage, the split-K factor (array of >= d ints,
 * may be NULL; 1 = unsplit; see qtt_get_stage_split).  Host only. */
qtt_status_t qtt_plan_stages_split(int d, const int64_t* ranks, size_t smem_optin, int max_stage_levels,
                                   int* n_stages, int* k_first, int* k_last, int* variant, int* ksplit);

/*
 * qtt_apply -- y = A x on `stream` (asynchronous, stream-ordered).
 *   x, y  : DEVICE pointers (on the handle's device) owned by the caller, column-major N x nrhs,
 *           16-byte aligned; the ranges [x, x+N*nrhs) and [y, y+N*nrhs)
 *           must not overlap (in-place is impossible, reading R13).
 *   nrhs  : number of right-hand sides, >= 1 (N * nrhs <= 2^60).  Every launch
 *           covers at most 2^31 GEMM rows (32-bit TMA row coordinates), so
 *           an apply with N * nrhs > 2^31 runs as consecutive groups of
 *           2^31 / N right-hand sides; qtt_apply also lowers the group while
 *           the group's workspace would not fit in the free device memory.
 *           Columns are independent, so results do not depend on the grouping.
 * Argument errors return synchronously and enqueue nothing.  The handle
 * keeps a cached workspace (at most qtt_workspace_size(h, nrhs) bytes),
 * allocated on first use with cudaMallocAsync on `stream`; it grows when a
 * later apply needs more, the old block being released stream-ordered after
 * its last user.  Applies on one handle from different streams are ordered one
 * after another through the workspace's event (no host sync); for
 * concurrent applies use qtt_apply_ws with one workspace per stream.
 * CUDA graph capture of `stream` is supported once the cached workspace
 * exists for this nrhs (apply once outside the capture, or use qtt_apply_ws);
 * otherwise QTT_ERROR_NOT_SUPPORTED.  Work captured into the caller's graph
 * is not tracked for the cross-stream ordering of later applies.
 */
qtt_status_t qtt_apply(qtt_handle_t h, const double* x, double* y, int64_t nrhs,
                       qtt_stream_t stream);

/*
 * qtt_stage_super_core -- HOST only (no GPU): the super-core a merged stage of
 * levels [k_first, k_last] applies (at most 12 levels), i.e. the QTT definition
 * restricted to those digits, contracted over the inner bonds:
 *   W[a][ii][jj][b] = sum G_k_first(a, i_1 j_1, :) ... G_k_last(:, i_L j_L, b),
 *   ii = sum_l i_l 2^{l-1}, jj = sum_l j_l 2^{l-1}   (l = 1 is level k_first)
 * written as ranks[k_first-1] * 2^L * 2^L * ranks[k_last] doubles, row-major.
 * cores/ranks as qtt_create (only levels k_first..k_last are read).
 */
qtt_status_t qtt_stage_super_core(int d, const int64_t* ranks, const double* const* cores, int k_first,
                                  int k_last, double* W);

/* Bytes of device workspace one apply with `nrhs` right-hand sides needs
 * (256 bytes of scheduler counters, two ping-pong buffers of max
 * stage-boundary rank * N * g doubles -- absent for a one-stage plan -- and
 * the split-K partials, where g = min(nrhs, 2^31 / N) is the launch group
 * of qtt_apply_ws, see qtt_apply).  Shard handles: g = nrhs. */
qtt_status_t qtt_workspace_size(qtt_handle_t h, int64_t nrhs, size_t* bytes);

/* qtt_apply with caller-owned DEVICE workspace `ws` of `ws_bytes` >= the
 * qtt_workspace_size(h, nrhs) (256-byte aligned).  Otherwise as qtt_apply. */
qtt_status_t qtt_apply_ws(qtt_handle_t h, const double* x, double* y, int64_t nrhs,
                          void* ws, size_t ws_bytes, qtt_stream_t stream);

/*
 * qtt_apply_host -- end-to-end convenience: x_host, y_host are HOST arrays
 * (pinned or pageable) of N*nrhs doubles.  Copies x to the device on
 * `stream`, applies, copies y back, and synchronizes `stream` before
 * returning.  Device staging buffers are cached in the handle.  Results are
 * bitwise those of qtt_apply on the same handle: large single-RHS applies
 * overlap the copies with the first / last stage (chunked launches of the
 * same stage kernels); latency-bound handles run H2D, their one-launch
 * apply, D2H.
 */
qtt_status_t qtt_apply_host(qtt_handle_t h, const double* x_host, double* y_host,
                            int64_t nrhs, qtt_stream_t stream);

/*
 * Morton ordering (grid points indexed by successive
 * bisection along each coordinate, "i.e., Morton ordered"; Remark
 * rem:interlace P:855-870).  A grid of n^dim points, n = 2^levels, dim in
 * {1,2,3}, d = dim*levels <= 30, stored in natural C order [z][y][x] (x
 * fastest), maps to the QTT-order vector x_qtt[q] whose index bit
 * dim*l + a is bit l of coordinate a (a = 0 x, 1 y, 2 z; l = 0 finest) --
 * DESIGN.md reading R18.
 *   qtt_morton_pack   : grid (natural) -> x (QTT order)
 *   qtt_morton_unpack : x (QTT order) -> grid (natural)
 * Both take DEVICE pointers to nrhs column-major blocks of N = 2^d doubles
 * (8-byte aligned, non-overlapping), are stream-ordered, and return
 * QTT_ERROR_INVALID_VALUE for bad dim/levels/nrhs or overlap,
 * QTT_ERROR_NOT_SUPPORTED for host pointers.
 */
qtt_status_t qtt_morton_pack(const double* grid, double* x, int dim, int levels, int64_t nrhs,
                             qtt_stream_t stream);
qtt_status_t qtt_morton_unpack(const double* x, double* grid, int dim, int levels, int64_t nrhs,
                               qtt_stream_t stream);

/*
 * qtt_apply_grid -- y = A x for vectors given as natural-order grids:
 * Morton pack, qtt_apply, Morton unpack on `stream` (dim must divide d).
 * grid_in / grid_out: DEVICE, nrhs blocks of N doubles, non-overlapping.  The
 * two QTT-order staging vectors are cached in the handle (cudaMallocAsync).
 */
qtt_status_t qtt_apply_grid(qtt_handle_t h, const double* grid_in, double* grid_out, int dim, int64_t nrhs,
                            qtt_stream_t stream);

/*
 * Products of QTT operators (NEXT-1): the paper applies its BIE
 * preconditioner as the product of two QTT matrices, X = M Y, because the
 * factors' ranks are smaller than the product's (P:1377-1402 Eq.
 * precond_mateq, Table TT-BIE-3).  A product handle
 * applies y = F_0 F_1 ... F_{n-1} x right to left on one stream (F_{n-1}
 * first), each factor through its own stage plan; the factors' costs add
 * (the composed QTT would have rank r_M r_Y per bond).
 *   qtt_product_create : factors = n_factors >= 1 handles with equal d on one
 *                        device; NOT owned (they must outlive the product).
 *   qtt_product_workspace_size / qtt_product_apply_ws : caller workspace =
 *                        the largest factor workspace + one (n = 2) or two
 *                        (n >= 3) N*nrhs intermediate vectors, 256-byte aligned.
 *   qtt_product_apply  : workspace cached in the product handle.
 * Argument rules and errors as qtt_apply / qtt_apply_ws.
 */
typedef struct qtt_product* qtt_product_t;
qtt_status_t qtt_product_create(qtt_product_t* out, int n_factors, const qtt_handle_t* factors);
qtt_status_t qtt_product_workspace_size(qtt_product_t p, int64_t nrhs, size_t* bytes);
qtt_status_t qtt_product_apply(qtt_product_t p, const double* x, double* y, int64_t nrhs,
                               qtt_stream_t stream);
qtt_status_t qtt_product_apply_ws(qtt_product_t p, const double* x, double* y, int64_t nrhs,
                                  void* ws, size_t ws_bytes, qtt_stream_t stream);
qtt_status_t qtt_product_destroy(qtt_product_t p);

/*
 * QTT-compressed matrix-vector product (NEXT-3; PAPER section 4.2
 * "QTT Compressed matrix-vector product"): for b given in QTT
 * form, the cores of c = A b are
 *   G^c_k((alpha beta), i_k, (alpha' beta')) = sum_j G^A_k(alpha, i_k j_k, alpha') G^b_k(beta, j_k, beta')
 * with ranks R_k = r^A_k * r^b_k (<= 4096, else QTT_ERROR_NOT_SUPPORTED).
 *   b_ranks : host, d+1 ranks of b (b_ranks[0] == b_ranks[d] == 1).
 *   b_cores : host array of d HOST pointers, core k of b as b_ranks[k-1]*2*b_ranks[k]
 *             doubles [beta][j][beta'] (copied; free on return).
 *   c_ranks : optional host array (d+1) receiving R_k.
 * qtt_compressed_matvec writes the DENSE c (N doubles, device, 16-byte aligned):
 * the product cores are densified on the GPU (Eq. TTdeccores for a vector,
 * split at level d/2 into two halves and one GEMM).
 * qtt_compressed_matvec_cores writes the product cores instead, concatenated
 * k = 1..d as [R_{k-1}][2][R_k] row-major into DEVICE memory of >= the sum of
 * their sizes in bytes (c_cores_bytes).  Both synchronize `stream` before
 * returning (the workspace is allocated and freed on it).
 */
qtt_status_t qtt_compressed_matvec(qtt_handle_t h, const int64_t* b_ranks, const double* const* b_cores,
                                   double* c, int64_t* c_ranks, qtt_stream_t stream);
qtt_status_t qtt_compressed_matvec_cores(qtt_handle_t h, const int64_t* b_ranks,
                                         const double* const* b_cores, double* c_cores,
                                         size_t c_cores_bytes, int64_t* c_ranks, qtt_stream_t stream);

/*
 * Top-bit sharding over P = 2^s GPUs (NEXT-4).  Split x and y
 * into P contiguous blocks of n = N/P entries by the top s index bits (in
 * Morton order: octree subdomains).  Levels 1..d-s pair only bits inside a
 * block (Alg. 2 level k touches digit k), so part g applies them
 * to its own block x_g, giving T_g[m][alpha] (n x r_{d-s}, natural row order);
 * then it projects onto every output block h with
 *   c_{h,g}[alpha] = G_{d-s+1}(alpha, h_1 g_1, :) ... G_d(:, h_s g_s, 0)
 * (the QTT definition P:519-523 on the top s digits), and
 *   y_h = sum_g T_g c_{h,g}         -- one ReduceScatter (sum) over the parts.
 *   qtt_create_shard   : plan part `part` (0 <= part < 2^log2_parts, 1 <= log2_parts < d)
 *                        of the operator; cores/ranks as qtt_create (all d cores).
 *                        The handle's qtt_get_info reports the LOCAL d - s and n.
 *   qtt_shard_apply[_ws]: x_local (DEVICE, n x nrhs column-major) -> send (DEVICE,
 *                        nrhs blocks of [P][n]: send[s][h][m] = (T_g c_{h,g})[m] of RHS s);
 *                        the caller reduce-scatters block h to part h (per RHS),
 *                        e.g. NCCL through torch.distributed.  Workspace as
 *                        qtt_workspace_size(h, nrhs).  qtt_apply on a shard handle
 *                        returns QTT_ERROR_INVALID_VALUE.
 *   qtt_shard_projection: HOST only (no GPU): writes W[h * r + alpha] = c_{h,part}[alpha],
 *                        P x r_{d-s} doubles.
 */
qtt_status_t qtt_create_shard(qtt_handle_t* out, int d, const int64_t* ranks, const double* const* cores,
                              int log2_parts, int part);
qtt_status_t qtt_shard_apply(qtt_handle_t h, const double* x_local, double* send, int64_t nrhs,
                             qtt_stream_t stream);
qtt_status_t qtt_shard_apply_ws(qtt_handle_t h, const double* x_local, double* send, int64_t nrhs,
                                void* ws, size_t ws_bytes, qtt_stream_t stream);
qtt_status_t qtt_shard_projection(int d, const int64_t* ranks, const double* const* cores, int log2_parts,
                                  int part, double* W);

/*
 * Fused exchange (the compute + collective step in one kernel): instead of a
 * send buffer and a ReduceScatter, the projection stage stores output block h
 * of part g straight into part h's receive buffer -- over NVLink when `recv`
 * holds peer mappings (cudaIpcOpenMemHandle) of the other GPUs' buffers.
 *   qtt_shard_set_peers  : recv[h] = part h's receive buffer as seen from this
 *                          device ([P][nrhs][n] doubles, 16-byte aligned), h = 0..P-1
 *                          (recv[part] is this part's own buffer).  Synchronous; must
 *                          not be called while a fused apply of this handle is in flight.
 *   qtt_shard_apply_fused: local stages + scatter projection; writes slot `part`
 *                          of every part's buffer.  The caller orders the P parts:
 *                          every part's fused apply complete before any part reduces,
 *                          and every reduction of the previous apply complete before
 *                          the next fused apply (parallel.py: interprocess CUDA events
 *                          behind host barriers; or stream sync + a process barrier).
 *   qtt_shard_reduce     : y_local[i] = sum_{g=0..P-1} recv[g * count + i] in that fixed
 *                          order (count = nrhs * n, even; deterministic).
 */
qtt_status_t qtt_shard_set_peers(qtt_handle_t h, double* const* recv, int parts);
qtt_status_t qtt_shard_apply_fused(qtt_handle_t h, const double* x_local, int64_t nrhs, qtt_stream_t stream);
qtt_status_t qtt_shard_reduce(const double* recv, double* y_local, int parts, int64_t count, qtt_stream_t stream);

/*
 * Receive buffers shared between the processes of a node (CUDA IPC): allocate
 * with qtt_ipc_alloc (a whole cudaMalloc allocation, so the IPC mapping starts
 * at the pointer), export its 64-byte handle, open the other processes'
 * handles (peer access enabled lazily), close / free at the end.
 */
qtt_status_t qtt_ipc_alloc(size_t bytes, void** ptr);
qtt_status_t qtt_ipc_free(void* ptr);
qtt_status_t qtt_ipc_get_handle(void* ptr, unsigned char* handle64);
qtt_status_t qtt_ipc_open(const unsigned char* handle64, void** ptr);
qtt_status_t qtt_ipc_close(void* ptr);

/* Plan facts: d, N, max rank, algorithmic flops per right-hand side
 * (4 * sum_k r_{k-1} r_k * N) and the number of stages one
 * apply runs (one kernel launch each; a split-K stage, see
 * qtt_get_stage_split, adds its reduce launch).  Any output pointer may be NULL. */
qtt_status_t qtt_get_info(qtt_handle_t h, int* d, int64_t* N, int64_t* max_rank,
                          double* flops_per_rhs, int* launches_per_apply);

/*
 * Per-stage description: stage s (0 <= s < launches_per_apply) covers levels
 * [*k_first, *k_last] (1-based) and runs kernel variant *variant (0 = generic,
 * 1 = fp64 tensor-core DMMA, one level; 2 = DMMA merged stage of several
 * levels with the super-core in shared memory; 3 = the same with the
 * super-core streamed from L2 in k-chunks; 4 = small latency-bound stage,
 * one warp per 16 x 32 output block; 5 = levels whose cores are all diagonal
 * in (i_k, j_k), i.e. A block-diagonal in those digits, applied as one
 * streaming batched GEMV whatever their number, see qtt_plan_stages).  The
 * diagonal levels are detected at qtt_create from exact zeros; the host-only
 * qtt_plan_stages knows ranks only and never plans variant 5.  Such zeros are
 * structural: a NaN/Inf in x then stays inside its block instead of spreading
 * through 0 * Inf products (reading R21).
 */
qtt_status_t qtt_get_stage(qtt_handle_t h, int s, int* k_first, int* k_last, int* variant);

/*
 * qtt_get_stage_split -- how many k-ranges stage s splits its GEMM into at
 * `nrhs` right-hand sides (1 = no split).  A variant-3 stage whose output
 * tiles alone would leave SMs idle (few GEMM rows, long K: the last stage of
 * a constant-rank profile, whose super-core has K = 2^L r) computes each
 * output tile as S partial sums over disjoint k-ranges, added in fixed order
 * k-range 0..S-1 by a second launch (bitwise reproducible).  The split
 * scratch is part of qtt_workspace_size.  Host-only query; no GPU work.
 */
qtt_status_t qtt_get_stage_split(qtt_handle_t h, int s, int64_t nrhs, int* ksplit);

/*
 * qtt_get_apply_plan -- what an apply with `nrhs` right-hand sides on this
 * handle launches (host-only query; no GPU work).
 *   launches : receives the number of kernel launches of the whole apply
 *              (stages, split-K reduce launches, RHS groups; 1 for a fused apply).
 *   n_stages, k_first, k_last, variant : the stages it runs (arrays of >= d
 *              ints, any may be NULL), as qtt_plan_stages; variant 6 = FUSED:
 *              every stage of the apply in ONE persistent launch (grid
 *              barriers between stages, intermediates in L2),
 *              chosen at create time for latency-bound sizes (small N * nrhs)
 *              when the cost model prefers it.  A handle with stage timing on
 *              (qtt_set_stage_timing) runs and reports the per-stage plan.
 */
qtt_status_t qtt_get_apply_plan(qtt_handle_t h, int64_t nrhs, int* launches, int* n_stages, int* k_first,
                                int* k_last, int* variant);

/* qtt_set_fused -- enable (1, the default) or disable (0) the fused one-launch
 * apply on this handle; disabled, every apply runs the per-stage plan.  Host
 * only; affects applies enqueued after the call.
 * The fused launch is NOT a cooperative launch (its grid is at most one CTA
 * per SM, which a whole device co-schedules).  On a device
 * partition with fewer SMs than the device reports (an SM-limited MPS client
 * or green context) its grid barrier could never complete: after 30 s it traps
 * and the apply's stream reports a CUDA error (QTT_ERROR_CUDA on the next
 * call that checks it).  There, disable the fused apply with this call, or
 * set QTT_FUSED_COOP=1 (cooperative launches, which fail cleanly and fall
 * back to the per-stage plan). */
qtt_status_t qtt_set_fused(qtt_handle_t h, int enable);

/*
 * Stage timing (for the bench's roofline): when enabled, each apply records
 * a CUDA event pair around every stage launch on the apply stream.
 * qtt_stage_times synchronizes those events, writes the summed milliseconds
 * per stage into ms[0..n_stages-1] and the number of timed applies into
 * *n_applies, and resets the accumulators.
 */
qtt_status_t qtt_set_stage_timing(qtt_handle_t h, int enable);
qtt_status_t qtt_stage_times(qtt_handle_t h, float* ms, int n_stages, int* n_applies);

/* Waits for the handle's last apply (event recorded on its stream), then
 * frees device memory.  NULL is a no-op. */
qtt_status_t qtt_destroy(qtt_handle_t h);

#ifdef __cplusplus
}
#endif

#endif /* QTT_B200_H */
