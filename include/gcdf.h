/* gcdf.h -- C ABI of libgcdf: the batched neural GCDF query and sparsity-aware
 * active-set detection of arXiv 2601.18548, on NVIDIA B200 (sm_100a).
 *
 * Citations are /root/reference/PAPER.md line numbers (the paper's LaTeX source);
 * "R<k>" refers to the readings listed in DESIGN.md §3.
 *
 * What is computed (the hot path):
 *   For every pair (waypoint configuration q_i of trajectory b, obstacle point p_j):
 *     x_in = [p_x - q_x, p_y - q_y, p_z, 0, 0, theta, j1..j6]
 *       base-frame bias of the obstacle point, PAPER.md:388 ("treat the robot base
 *       pose as the origin and bias all obstacle points"); R1, R2.
 *     f = MLP(x_in): the paper's "7-layer MLP" on the concatenation [p, q]
 *       (PAPER.md:284), ReLU hidden layers, signed scalar output; R7-R10.
 *     grad_q f in R^9 by the chain rule through the bias; R3.
 *   Constraint f - delta >= 0 over all i, j (Eq. 11d).
 *   Active set: f - delta <= tau (R12); per-waypoint min (union = min);
 *   records in step-major (waypoint, point id) order = c_gcdf of Eq. 14.
 *   Online point injection/removal without rebuilding.
 *
 * Conventions for every entry point:
 *   - Returns a gcdf_status (0 = OK, < 0 = error).  No C++ exception crosses the ABI.
 *   - Validation errors are atomic: the call changes nothing.  gcdf_last_error(ctx)
 *     returns the message of the last failing call (storage owned by ctx).
 *   - "_dev" pointers are CUDA device pointers (e.g. torch tensor data_ptr()),
 *     "_host" pointers are host memory.  The caller owns every argument buffer.
 *   - All device work is enqueued on the given stream (cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Only calls that return host results
 *     (update_scene's ids are computed on the host; detect with count_host_or_null
 *     != NULL) synchronize that stream.
 *   - A context is bound to one CUDA device and is NOT thread-safe.
 *   - After gcdf_bind_workspace no call allocates device memory.
 */
#ifndef GCDF_H
#define GCDF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gcdf_ctx gcdf_ctx;

enum gcdf_status {
  GCDF_OK = 0,
  GCDF_ERR_INVALID_ARG = -1,
  GCDF_ERR_IO = -2,
  GCDF_ERR_BAD_MAGIC = -3,     /* weights file does not start with "MLPW" */
  GCDF_ERR_VERSION = -4,       /* MLPW version != 1 */
  GCDF_ERR_DIM_MISMATCH = -5,  /* dims not [12, H x 6, 1] with H in {32, 128, 256}, or an activation / width
                                  the context's precision does not run */
  GCDF_ERR_NOT_LOADED = -6,    /* no weights loaded / no workspace bound */
  GCDF_ERR_CAPACITY = -7,      /* scene, waypoint, staging or output capacity exceeded */
  GCDF_ERR_UNKNOWN_ID = -8,    /* remove of an id that is not live (or duplicated in the call) */
  GCDF_ERR_NONFINITE = -9,     /* NaN / Inf in points or weights */
  GCDF_ERR_CUDA = -10,         /* CUDA runtime error (message has the CUDA string); sticky */
  GCDF_ERR_UNSUPPORTED = -11,  /* e.g. no sm_100 device */
  GCDF_ERR_NCCL = -12          /* NCCL (or the test exchange backend) failed; message has the NCCL string; sticky */
};

enum gcdf_precision {
  GCDF_FP32 = 0, /* fp32 SIMT path: parity path, tolerance 1e-4 rel / 1e-5 abs */
  GCDF_BF16 = 1, /* tcgen05 tensor-core path, bf16 operands, fp32 accumulate */
  GCDF_FP16 = 2, /* tcgen05 tensor-core path, fp16 operands, fp32 accumulate: same tensor peak as
                    bf16 with 3 more significand bits; meets the north-star tensor-path tolerance
                    (R17, §5); the default */
  GCDF_FP16X3 = 3, /* fp32-accurate tcgen05 path (NEXT-4): every hidden GEMM on 3-term split fp16
                    operands (a_hi w_hi + a_lo w_hi + a_hi w_lo), weights streamed from L2; meets
                    the fp32 tolerance of GCDF_FP32 (R25, §5 "K2c"); needs H = 128 */
  GCDF_BF16X3 = 4  /* the same 3-term split on bf16 operands (K2c with bf16 UMMAs): every product
                    to ~2^-16 relative, so the bf16 tensor path meets the north-star tensor
                    tolerance (2e-2 on f, 5e-2 on the gradient norm) that single-term bf16 misses
                    at the paper's gradient scale (R28, R29); needs H = 128 */
};

enum gcdf_tgrad {
  GCDF_TGRAD_CHAINRULE = 0, /* d f/d q_xy = -d F/d p'_xy; default, R3 */
  GCDF_TGRAD_QCHANNEL = 1   /* d f/d q_xy = d F/d x_in[3..4] (the network's q^t channels) */
};

enum gcdf_frame {
  GCDF_FRAME_TRANSLATE = 0, /* p' = p - [x, y, 0], theta fed to the network (R1) */
  GCDF_FRAME_SE2 = 1        /* NEXT-4 variant: p'_xy = R(-theta)(p_xy - [x, y]), theta channel fed 0
                               (R24; not with GCDF_TGRAD_QCHANNEL) */
};

typedef struct {
  int32_t precision;       /* gcdf_precision (default GCDF_FP16) */
  int32_t tgrad_mode;      /* gcdf_tgrad */
  int64_t scene_capacity;  /* global id space [0, scene_capacity) of obstacle points; < 2^31 */
  int32_t max_waypoints;   /* largest B*N accepted by query/detect; <= 65535 */
  int64_t max_active;      /* staging capacity (records) of detect on this rank */
  int32_t rank;            /* point sharding: this rank owns ids whose 128-id block */
  int32_t world;           /*   (id / 128) satisfies block % world == rank; world >= 1 */
  int64_t max_candidates;  /* range-partitioned detect: capacity of the per-step candidate
                              lists (sum over steps of |I_{M,i}|); 0 = partitioned detect off */
  int32_t frame;           /* gcdf_frame: base-frame transform of the points */
  int32_t exchange;        /* reserve the exchange buffers of the sharded detect (gcdf_dist_init*)
                              also at world == 1 (at world > 1 they are always reserved):
                              header 2 x (world + 1) x (2 max_waypoints + 1) x 8 B and records
                              (world + 1) x max_active x 48 B */
} gcdf_options;

/* One active constraint (48 B): f, grad_q f (9), wp = b*N + i, pt = global point id. */
typedef struct {
  float value;
  float grad[9];
  uint32_t wp;
  uint32_t pt;
} gcdf_active_t;

/* ------------------------------------------------------------------ lifecycle */
/* Fills *opt with defaults (precision FP16, chain rule, capacity 1<<20, 256 waypoints,
   max_active 1<<22, rank 0, world 1, max_candidates 0, frame TRANSLATE). */
void gcdf_default_options(gcdf_options *opt);

/* Creates a context on CUDA device cuda_device.  Fails with UNSUPPORTED unless the
   device is compute capability 10.0 (B200).  opt may be NULL (defaults).  INVALID_ARG for
   scene_capacity outside (0, 2^31), max_waypoints outside [1, 65535], max_active outside
   (0, 2^31), a bad rank / world pair or an unknown precision / tgrad / frame. */
int gcdf_create(int cuda_device, const gcdf_options *opt, gcdf_ctx **out);
int gcdf_destroy(gcdf_ctx *ctx);
const char *gcdf_last_error(const gcdf_ctx *ctx);
/* Returns 1 if the library was built with the tcgen05 kernels for sm_100a. */
int gcdf_has_tcgen05(void);

/* Device workspace: the caller allocates `bytes` (256-B aligned) and binds it.  It
   holds the scene slots, packed weights and detect scratch.  Rebinding resets the
   scene and requires reloading weights. */
int gcdf_workspace_bytes(const gcdf_ctx *ctx, int64_t *bytes);
int gcdf_bind_workspace(gcdf_ctx *ctx, void *dev_ptr, int64_t bytes);

/* ------------------------------------------------------------------ weights */
/* Loads an MLPW v1 file: "MLPW", u32 version = 1, u32 activation
   (1 = ReLU, R9; 2 = softplus log(1 + e^z), the NEXT-4 variant of R26 --
   GCDF_FP32 and GCDF_FP16 only), u32 L = 7, u32 dims[8] = [12, H, H, H, H, H, H, 1] with H in {32, 128, 256}
   (H = 32: GCDF_FP32; H = 256, the NEXT-4 width variant of DESIGN.md R27: GCDF_FP32, or GCDF_FP16
   with ReLU in the translation frame),
   then per layer f64 W[out][in] row-major and f64 b[out].  Packs fp32 and bf16
   (UMMA SWIZZLE_128B) copies into the workspace (enqueued on `stream`, host staging
   synchronized before return).  Errors: IO (missing/truncated), BAD_MAGIC, VERSION,
   DIM_MISMATCH, NONFINITE.  Atomic: a failed load keeps the previous weights. */
int gcdf_load_weights(gcdf_ctx *ctx, const char *mlpw_path, void *stream);

/* ------------------------------------------------------------------ scene (A0, A9) */
/* Incremental point injection / removal without problem reconstruction
   (PAPER.md:75 (c), :401 "both components can be modified online").
   add_xyz_host [n_add][3] fp32 metres; out_ids_host [n_add] receives the ids;
   remove_ids_host [n_remove].  Id rule (identical on every rank, so SPMD ranks
   agree without communication): removals are validated (live, not duplicated);
   each add takes the lowest id that is free at the start of the call (ids removed by
   this call become free for the NEXT call).  Each rank stores only the points whose
   128-id block it owns.  O(n_add + n_remove) device work: one scatter kernel.
   Errors: UNKNOWN_ID, NONFINITE, CAPACITY (atomic).  Synchronizes `stream` only to
   recycle its pinned staging buffer. */
int gcdf_update_scene(gcdf_ctx *ctx, const float *add_xyz_host, int64_t n_add, int64_t *out_ids_host,
                      const int64_t *remove_ids_host, int64_t n_remove, void *stream);

/* n_live: live points (global); id_bound: 1 + highest id ever assigned (ids < id_bound);
   local_bound: number of this rank's local slots covering ids < id_bound (a multiple of
   128; the stride of query outputs).  Local slot s holds global id
   ((s / 128) * world + rank) * 128 + s % 128. */
int gcdf_scene_info(const gcdf_ctx *ctx, int64_t *n_live, int64_t *id_bound, int64_t *local_bound);

/* ------------------------------------------------------------------ hot path */
/* A2 standalone: pair generation + base-frame transform.  out_dev [B*N][local_bound]
   float4 (p_x - q_x, p_y - q_y, p_z, live) for this rank's local slots. */
int gcdf_pairgen_transform(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, void *out_dev,
                           void *stream);

/* A2-A5 dense: values_dev [B*N][local_bound] fp32 and grads_dev [B*N][local_bound][9]
   fp32 for every pair of this rank's local slots; dead slots give +INF and a zero
   gradient.  q_dev [B][N][9] fp32 = [x, y, theta, j1..j6].
   grads_dev may be NULL (values only). */
int gcdf_query_values_grads(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, float *values_dev,
                            float *grads_dev, void *stream);

/* NEXT-3 (Theorem 1.2): batched single-step projection onto the zero
   level set, fused into the dense query: qz_dev [B*N][local_bound][9] receives
   q_z = q - f(p, q) M^{-1} grad_q f(p, q) for every pair (0 for dead slots), values_dev as
   in gcdf_query_values_grads; minv_host [9] = the diagonal of M^{-1} (finite, >= 0). */
int gcdf_project_dense(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, const float *minv_host,
                       float *values_dev, float *qz_dev, void *stream);

/* A2-A8 fused: query + threshold + per-waypoint min + stream compaction.
   out_dev [out_capacity] records in (wp, pt) order; wp_offsets_dev [B*N+1] (Eq. 14
   block structure); wp_min_dev [B*N] (+INF if no live point);
   wp_argmin_dev [B*N] (smallest id on ties, -1 if none); wp_key_dev [B*N] (may be
   NULL): int64 signed-order key (ordered(f) << 32 | pt) ^ INT64_MIN, INT64_MAX if
   none, for a cross-rank MIN reduction; count_dev [1] (total active).
   count_host_or_null: if non-NULL the stream is synchronized and the count written.
   CAPACITY is returned (count still exact, out content unspecified) when the count
   exceeds out_capacity or the staging capacity max_active; grow and retry.
   Sharded scene: once gcdf_dist_init / gcdf_dist_init_host ran, every rank
   calls with the same q, delta, tau and out_capacity (SPMD) and every rank receives the
   FULL, canonically ordered result over all ranks' points -- bit-identical to one GPU
   holding the whole scene.  On the stream, with no host synchronization (NCCL backend):
   the local fused detect writes this rank's records (at most S = min(max_active,
   ceil(out_capacity / world)); the ids of a rank are dealt round-robin by 128-id block, so
   the ranks' counts are balanced) and its header (wp_offsets + per-waypoint keys) into the
   exchange buffers; one NCCL group all-gathers the headers ((2 B*N + 1) x 8 B per rank) and
   the records (S x 48 B per rank); the merge kernel (K5) reduces the keys (MIN = global min
   / smallest-id argmin), sums the offsets and places every record by binary search.  A rank
   with more than S actives makes the call return CAPACITY (count_dev still the exact total;
   records unspecified).  Without a communicator, the result covers this rank's points
   only (gcdf_merge_active_sets merges such results). */
int gcdf_detect_active_set(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, float delta,
                           float tau, gcdf_active_t *out_dev, int64_t out_capacity, int64_t *wp_offsets_dev,
                           float *wp_min_dev, int64_t *wp_argmin_dev, int64_t *wp_key_dev,
                           int64_t *count_dev, int64_t *count_host_or_null, void *stream);

/* NEXT-1 range partition (R23): the fused detect over
   the pairs of each step i with the obstacle points of its partition
   I_{M,i} = { j : |p_j,xy - (x_i, y_i)| <= radius } only (radius > 0, metres, planar
   distance to the step's base position q_i[0:2]).  Outputs, order and errors as
   gcdf_detect_active_set, with wp_min / wp_argmin over I_{M,i}; part_sizes_dev [B*N]
   (may be NULL) receives m_i = |I_{M,i}| on this rank.  The planar grid (cell >= radius)
   over this rank's live points is rebuilt on the device when the scene or the radius
   changed since the last call; the partitions are built per call (bitmap + ordered
   compaction).  Needs max_candidates > 0 (INVALID_ARG otherwise); when sum_i m_i exceeds
   it the call evaluates nothing and returns CAPACITY (count 0). */
int gcdf_detect_active_set_partitioned(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, float radius,
                                       float delta, float tau, gcdf_active_t *out_dev, int64_t out_capacity,
                                       int64_t *wp_offsets_dev, float *wp_min_dev, int64_t *wp_argmin_dev,
                                       int64_t *wp_key_dev, int64_t *part_sizes_dev, int64_t *count_dev,
                                       int64_t *count_host_or_null, void *stream);

/* NEXT-2 (Eq. 14-19; R18): the consumer-side constraint
   vector and sparse Jacobian of an active set in (wp, pt) order (the output of a detect
   or merge): c_dev [n] (may be NULL) = f - delta; CSR with n = min(*count_dev, capacity)
   rows of 9 entries: row_ptr_dev [n+1] = 9 k, col_dev [9n] = 2*9*wp + t (the step's 9
   configuration columns in a decision vector of 2 n_dof = 18 entries per step, the
   trajectory blocks of 2*9*N columns back to back since wp = b*N + i), val_dev [9n] =
   the record's gradient.  Device memory only; the count stays on the device. */
int gcdf_sparse_jacobian(gcdf_ctx *ctx, const gcdf_active_t *recs_dev, const int64_t *count_dev,
                         int64_t capacity, float delta, float *c_dev, int64_t *row_ptr_dev, int32_t *col_dev,
                         float *val_dev, void *stream);

/* CUDA-graph form of the detect for launch-bound (small) workloads: the whole call chain of
   gcdf_detect_active_set (radius == 0) or gcdf_detect_active_set_partitioned (radius > 0)
   with exactly these arguments is captured once into a CUDA graph; gcdf_graph_launch
   replays it on `stream` (the contents of q_dev may change between launches, the pointers
   may not) and, with count_host non-NULL, synchronizes and returns the count / CAPACITY
   like the direct call.  After a scene update, gcdf_load_weights or gcdf_bind_workspace the
   next launch re-captures (the tile counts and the partition grid depend on the scene; the
   kernel nodes hold the output row, the bias and the kernel chosen for H / activation); a
   partitioned graph's grid is built outside the graph, at capture time and again at launch
   when a call at another radius rebuilt it meanwhile.  The graph owns a capture stream; it
   must be destroyed before its context. */
typedef struct gcdf_graph gcdf_graph;
int gcdf_graph_create_detect(gcdf_ctx *ctx, const float *q_dev, int32_t B, int32_t N, float radius, float delta,
                             float tau, gcdf_active_t *out_dev, int64_t out_capacity, int64_t *wp_offsets_dev,
                             float *wp_min_dev, int64_t *wp_argmin_dev, int64_t *wp_key_dev,
                             int64_t *part_sizes_dev, int64_t *count_dev, gcdf_graph **out);
int gcdf_graph_launch(gcdf_graph *graph, int64_t *count_host_or_null, void *stream);
int gcdf_graph_destroy(gcdf_graph *graph);

/* Host-buffer form of gcdf_detect_active_set (the end-to-end call): q_host [B][N][9] is
   copied to the device, the fused detect runs, and the results come back to host memory:
   count_host (total active, always written), out_host [out_capacity] (the first
   min(count, out_capacity) records), wp_offsets_host [B*N+1], wp_min_host [B*N] and
   wp_argmin_host [B*N] (each may be NULL except wp_offsets_host).  The device side lives
   in the bound workspace (sized by max_waypoints and max_active).  Host buffers may be
   pageable; page-locked ones get the full link bandwidth.  Synchronizes
   the stream.  CAPACITY when count > out_capacity or > max_active (records not copied in
   the latter case). */
int gcdf_detect_active_set_host(gcdf_ctx *ctx, const float *q_host, int32_t B, int32_t N, float delta,
                                float tau, gcdf_active_t *out_host, int64_t out_capacity,
                                int64_t *wp_offsets_host, float *wp_min_host, int64_t *wp_argmin_host,
                                int64_t *count_host, void *stream);

/* A6-A8 standalone over a dense value/gradient array (e.g. from
   gcdf_query_values_grads): same outputs as detect.  values_dev [n_wp][stride],
   grads_dev [n_wp][stride][9], column s = local slot s of this context's scene; stride
   >= local_bound and a multiple of 4 (16-B aligned rows); a value of +INF marks a dead
   slot (the query writes +INF there) and is never active nor the minimum.  Capacity: the
   records are written straight to out_dev in canonical order (no staging area), the first
   min(count, out_capacity) of them; count_dev always holds the full count; with
   count_host_or_null given, the call synchronizes and returns CAPACITY when count >
   out_capacity.  The scratch it uses lives in
   the bound workspace (sized by max_waypoints and the scene capacity). */
int gcdf_compact_dense(gcdf_ctx *ctx, const float *values_dev, const float *grads_dev, int32_t n_wp,
                       int64_t stride, float delta, float tau, gcdf_active_t *out_dev, int64_t out_capacity,
                       int64_t *wp_offsets_dev, float *wp_min_dev, int64_t *wp_argmin_dev,
                       int64_t *wp_key_dev, int64_t *count_dev, int64_t *count_host_or_null, void *stream);

/* Multi-GPU gather step: merge the per-rank active sets gathered from
   `world` ranks into one canonical (wp, pt) ordered set.
   recs_dev [world][rec_stride] (rank r's records at r*rec_stride, in its own order);
   offsets_dev [world][n_wp+1] (each rank's wp_offsets); wp_key_dev [n_wp] the MIN over
   ranks of wp_key.  Outputs as in detect.  Pure device work, no collective inside (the
   sharded detect runs the same merge kernel after its own NCCL exchange). */
int gcdf_merge_active_sets(gcdf_ctx *ctx, int32_t world, int32_t n_wp, const gcdf_active_t *recs_dev,
                           int64_t rec_stride, const int64_t *offsets_dev, const int64_t *wp_key_dev,
                           gcdf_active_t *out_dev, int64_t out_capacity, int64_t *wp_offsets_dev,
                           float *wp_min_dev, int64_t *wp_argmin_dev, int64_t *count_dev, void *stream);

/* ------------------------------------------------------------------ sharded scene */
/* NCCL unique id for gcdf_dist_init (call on one rank; the caller broadcasts the 128 bytes,
   e.g. through its torch.distributed process group).  NCCL is opened at run time
   (dlopen libnccl.so.2: the process's NCCL when torch loaded it); NCCL if that fails. */
int gcdf_nccl_unique_id(unsigned char out_id[128]);
/* Creates this context's NCCL communicator (ncclCommInitRank on the context's device):
   rank / world must equal gcdf_options.rank / world, and the exchange buffers must be
   reserved (world > 1 or gcdf_options.exchange).  Collective over the world: every rank
   calls it with the same id.  From then on detect / detect_partitioned / detect_host /
   the CUDA-graph detect return the gathered result (see gcdf_detect_active_set).  The
   communicator is destroyed with the context.  INVALID_ARG (mismatch, no buffers, already
   initialized), NCCL. */
int gcdf_dist_init(gcdf_ctx *ctx, const unsigned char id[128], int32_t rank, int32_t world);
/* TEST BACKEND of the same exchange: fn is a blocking host all-gather -- rank r's
   bytes_per_rank bytes of send_host land at recv_host + r * bytes_per_rank on every rank;
   it returns 0 on success.  The library synchronizes the stream and stages through pinned
   host memory, so several processes can share ONE GPU (no kernel waits on another rank).
   Not for production and not capturable into a CUDA graph. */
typedef int (*gcdf_host_allgather_fn)(const void *send_host, void *recv_host, int64_t bytes_per_rank, void *user);
int gcdf_dist_init_host(gcdf_ctx *ctx, gcdf_host_allgather_fn fn, void *user);
/* Broadcast of the waypoint batch q [B][N][9] fp32 (device, in place) from rank 0 to every
   rank, for drivers that are not SPMD: afterwards every rank's q equals rank
   0's, so a following detect sees identical waypoints on all ranks.  Enqueued on `stream`
   (NCCL: one ncclBroadcast; the host test backend synchronizes).  INVALID_ARG (no
   communicator, null q, B or N <= 0), NCCL, CUDA. */
int gcdf_broadcast_waypoints(gcdf_ctx *ctx, float *q, int32_t B, int32_t N, void *stream);
/* Communicator state: *kind 0 = none, 1 = NCCL, 2 = host test backend; *nccl_version (may be
   NULL) = ncclGetVersion of the opened library (0 if none). */
int gcdf_dist_info(const gcdf_ctx *ctx, int32_t *kind, int32_t *nccl_version);

/* Number of kernels this context launched since creation (for bench accounting). */
int64_t gcdf_launch_count(const gcdf_ctx *ctx);

/* Optional live timing of the fused MLP kernel (the dominant kernel): when enabled,
   query/detect record a CUDA event pair around that launch on the call's stream.
   gcdf_profile_read synchronizes on the last pair and returns the accumulated kernel
   milliseconds and launch count since the last reset.  gcdf_profile_read_exchange does the
   same for the exchange step of the sharded detect (the all-gather group + merge kernel). */
int gcdf_profile_enable(gcdf_ctx *ctx, int enable);
int gcdf_profile_read(gcdf_ctx *ctx, double *mlp_ms, int64_t *mlp_launches, int reset);
int gcdf_profile_read_exchange(gcdf_ctx *ctx, double *ms, int64_t *calls, int reset);

/* ------------------------------------------------------------------ diagnostics */
/* Runs one tcgen05 UMMA building block of the bf16 kernel on device `cuda_device`
   (unit test of descriptors and TMEM layout).  A_dev fp32 [128][128] (rounded to bf16,
   staged in TMEM), B_dev fp32 row-major (rounded to bf16, staged in smem, SWIZZLE_128B),
   D_dev fp32 [128][128] output.  mode 0: D = A B^T, B [128][128] (K-major B);
   mode 1: D = A B, B [128][128] (MN-major B); mode 2: D[:, 0:16] = A B^T, B [16][128];
   mode | 4: the same with fp16 operands instead of bf16.  Other modes: INVALID_ARG (the UMMA
   throughput probes live in tools/probes/umma_probes.cu, outside the library).
   Synchronizes the stream.  UNSUPPORTED without the tcgen05 build. */
int gcdf_selftest_umma(int cuda_device, int mode, const float *A_dev, const float *B_dev, float *D_dev,
                       void *stream);

/* Pipeline trace of the tensor-core kernel: when trace_dev (device, 3744 int64) is non-NULL,
   CTA 0 of every later query/detect records clock64 stamps [role 18][tile 4][phase 13][4]
   (role 0 = MMA issuer, 1 + w = epilogue warp w = 0..15 (warps 0-7 serve tile slot 0,
   8-15 slot 1), 17 = MMA issuer wait stamps).  NULL switches it off. */
int gcdf_debug_trace(gcdf_ctx *ctx, long long *trace_dev);

#ifdef __cplusplus
}
#endif
#endif /* GCDF_H */
