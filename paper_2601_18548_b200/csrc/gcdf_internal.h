// gcdf_internal.h -- private types shared by the host layer and the sm_100a kernels.
// Nothing here is visible through the C ABI (include/gcdf.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gcdf.h"

namespace gcdf {

constexpr int kNdof = 9;      // q = [x, y, theta, j1..j6]
constexpr int kNin = 12;      // MLP input 3 + n
constexpr int kTile = 128;    // pairs per tile = 1 waypoint x 128 consecutive local slots
constexpr int kHidden = 6;    // hidden (ReLU) layers of the 7-layer MLP (R7)

// fp32 weight block (SIMT path).  Hidden layer li = 0..4 is the paper's layer l = li + 2.
//   w1p[u]        = {W1[u][0], W1[u][1], W1[u][2], b1[u]}          (layer 1, point columns)
//   w1q[u][8]     = W1[u][5..11], 0                                 (layer 1, q^r columns)
//   w1full[u][12] = W1[u][0..11]                                    (layer-1 backward)
//   wt[li][k][tu][i] = W[tu + 16 i][k]   (forward  B operand, units interleaved by 16)
//   wb[li][k][tu][i] = W[k][tu + 16 i]   (backward B operand)
//   bias[li][u], w7[u], b7
struct WeightsF32 {
  const float4 *w1p;
  const float *w1q;
  const float *w1full;
  const float *wt[5];
  const float *wb[5];
  const float *bias[5];
  const float *w7;
  float b7;
};

// bf16 weight block (tcgen05 path): hidden W_l (l = 2..6) as [out][in] bf16 in the UMMA
// canonical SWIZZLE_128B layout: two 64-column chunks of [H rows][128 B], 16-B granule g
// of row r stored at granule g ^ (r % 8).  The same bytes serve as a K-major B operand
// (forward, N = out, K = in) and an MN-major B operand (backward, N = in, K = out).
// w1t: W1^T restricted to the 12 input columns, padded to N = 16 rows, K-major SW128.
// b1: layer 1 as a K = 32 GEMM on split hi/lo 16-bit operands (exact to ~fp32), and
// bext: per hidden layer a K = 16 block {b_hi, b_lo, 0...} multiplied by a constant
// "ones" A block -- both in the UMMA SWIZZLE_NONE K-major layout (gcdf_host.cpp).
// (H = 256, K2w: w_sw128 = the 40 streamed 32 KB chunks of a tile, w1t / b1 / bext at H = 256)
struct WeightsBF16 {
  const void *w_sw128;   // 5 * H * H * 2 bytes
  const void *w1t_sw128; // 16 * H * 2 bytes
  const void *b1_nosw;   // H * 32 * 2 bytes
  const void *bext_nosw; // 5 * H * 16 * 2 bytes
  const float *bh;       // [5][H] fp32 biases of layers 2..6 (epilogue-add variant)
  const void *w3_sw128;  // (GCDF_FP16X3) 5 x [hi | lo] SW128 images of W_2..W_6, 64 KB each
  const void *w1t3_sw128;  // (GCDF_FP16X3) W1^T [16][H] hi, lo (SW128), 4 KB each
  const float *w7;       // [H] fp32
  float b7;
  // (K2b, K2w: H = 128, 256) the output row in the kernel parameters (constant bank): w7 / 2
  // in fp32 and w7 as packed 16-bit pairs of the context's operand type; the layer-6
  // epilogue reads them as direct constant operands instead of shared-memory loads
  float w7half_p[256];
  uint32_t w7h_p[128];
};

struct SceneView {
  const float4 *pts;     // [local_cap] (x, y, z, live)
  int64_t local_bound;   // multiple of 128
  int32_t rank, world;
};

// Detect scratch (in the bound workspace).
struct DetectScratch {
  int2 *tile_meta;                 // [n_wp * tiles_per_wp] (staging base, count)
  gcdf_active_t *staging;          // [max_active]
  int64_t max_active;
  unsigned long long *counter;     // [2]: staging allocation counter, overflow flag
  unsigned long long *wp_key;      // [max_waypoints] unsigned order key, ~0 = none
};

// Range-partitioned tile map (NEXT-1): tile T of step w = tile_wp[T] covers candidates
// (T - tile_start[w]) * 128 + row of that step's list cand[cand_start[w] ...] (ascending
// local slots), cand_count[w] of them; *n_tiles tiles in all.  tile_wp == nullptr: the
// dense map (every step x every local slot).
struct PartView {
  const int32_t *tile_wp = nullptr;
  const int64_t *tile_start = nullptr;
  const int64_t *cand_start = nullptr;
  const int64_t *cand_count = nullptr;
  const int32_t *cand = nullptr;
  const int64_t *n_tiles = nullptr;
};

struct QueryArgs {
  SceneView scene;
  const float *q;                  // [n_wp][9]
  int32_t n_wp;
  int32_t tiles_per_wp;
  int32_t tgrad;                   // gcdf_tgrad
  int32_t frame;                   // gcdf_frame (1: SE(2), R24)
  int32_t act;                     // hidden activation (MLPW id): 1 ReLU (R9), 2 softplus (R26)
  // dense outputs (query) -- NULL in detect mode
  float *values;
  float *grads;                    // (project: the projected configurations q_z instead)
  // NEXT-3 single-step projection (Theorem 1.2): q_z = q - f M^{-1} grad_q f, M diagonal
  int32_t project;
  float minv[kNdof];
  // detect mode
  int32_t detect;
  float delta, tau;
  DetectScratch ds;
  // diagnostics (gcdf_debug_trace): CTA 0 records clock64 stamps, NULL in normal runs
  long long *trace;
  PartView part;                   // range partition (detect only), see PartView
};

// (step, local slot) of row `row` of tile T; valid = false for padding rows
__device__ __forceinline__ void tile_pair(const QueryArgs &a, int64_t T, int row, int &w, int64_t &slot,
                                          bool &valid) {
  if (a.part.tile_wp) {
    w = a.part.tile_wp[T];
    const int64_t k = (T - a.part.tile_start[w]) * kTile + row;
    valid = k < a.part.cand_count[w];
    slot = valid ? (int64_t)a.part.cand[a.part.cand_start[w] + k] : 0;
  } else {
    w = (int)(T / a.tiles_per_wp);
    slot = (T % a.tiles_per_wp) * kTile + row;
    valid = slot < a.scene.local_bound;
  }
}
// step (waypoint index) of tile T
__device__ __forceinline__ int tile_step(const QueryArgs &a, int64_t T) {
  return a.part.tile_wp ? a.part.tile_wp[T] : (int)(T / a.tiles_per_wp);
}
__device__ __forceinline__ int64_t query_tiles(const QueryArgs &a) {
  return a.part.tile_wp ? *a.part.n_tiles : (int64_t)a.n_wp * a.tiles_per_wp;
}
// trace layout: [role 0 = MMA thread (issue start / end per slot), 1 + w = epilogue warp w
// (lane 0), w = 0..15, 17 = MMA thread (wait start / wait done per slot)][tile 0..3][phase 0..12][4]
constexpr int kTraceTiles = 4, kTracePhases = 13, kTraceRoles = 18;
constexpr int kTraceLen = kTraceRoles * kTraceTiles * kTracePhases * 4;

__host__ __device__ inline int64_t local_to_global(int64_t slot, int rank, int world) {
  return ((slot / kTile) * world + rank) * kTile + slot % kTile;
}

// ---- launchers (return cudaError_t of the launch) ----
cudaError_t launch_scene_scatter(const float4 *payload, const int64_t *slots, int64_t n, float4 *pts,
                                 cudaStream_t s);
cudaError_t launch_fill(float4 *pts, int64_t n, cudaStream_t s);
cudaError_t launch_pairgen(const float4 *pts, int64_t local_bound, const float *q, int32_t n_wp, int frame,
                           float4 *out, cudaStream_t s);
cudaError_t launch_detect_init(DetectScratch ds, int32_t n_wp, cudaStream_t s);
cudaError_t launch_mlp_simt(int H, const WeightsF32 &w, const QueryArgs &a, int num_sms, cudaStream_t s);
cudaError_t launch_mlp_tc(int H, bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s);
// H = 256 variant of the tensor-core path (fp16, ReLU, translation frame; weights streamed; R27)
cudaError_t launch_mlp_tc_wide(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s);
// softplus variant of the tensor-core path (fp16 operands, translation frame; R26)
cudaError_t launch_mlp_tc_sp(const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s);
cudaError_t launch_mlp_tc3(bool f16, const WeightsBF16 &w, const QueryArgs &a, int num_sms, cudaStream_t s);
bool tc_compiled();
cudaError_t launch_selftest_umma(int mode, const float *A, const float *B, float *D, cudaStream_t s);
// standalone A6-A8 over dense values (two passes; writes the ordered output directly)
cudaError_t launch_compact_dense(const float *values, const float *grads, int64_t stride, int32_t n_wp,
                                 int32_t tiles_per_wp, SceneView scene, float delta, float tau,
                                 DetectScratch ds, gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets,
                                 float *wp_min, int64_t *wp_argmin, int64_t *wp_key, int64_t *count,
                                 int64_t *k3_scratch, cudaStream_t s, int *n_launches);
int64_t k3_scratch_elems(int64_t n_wp, int64_t tiles_per_wp);
cudaError_t launch_sparse_jacobian(const gcdf_active_t *recs, const int64_t *count, int64_t cap, float delta,
                                   float *c, int64_t *row_ptr, int32_t *col, float *val, int num_sms,
                                   cudaStream_t s);
// range partition (k_partition.cu).  Grid over this rank's live points, rebuilt on demand.
struct PartScratch {
  float *grid;            // [8]: ox, oy, inv_cs, cs, radius, nx, ny (as float bits), unused
  unsigned *bbox;         // [4] ordered-uint min x, min y, max x, max y
  int32_t *cell_count;    // [kPartMaxCells]
  int64_t *cell_start;    // [kPartMaxCells + 1]
  int32_t *cell_fill;     // [kPartMaxCells]
  int32_t *cell_items;    // [local_cap] slots sorted by cell
  float2 *cell_xy;        // [local_cap] their planar coordinates
  uint32_t *bitmap;       // [max_wp][words]
  int64_t words;          // local_cap / 32
  int32_t *chunk_cnt;     // [max_wp * nchunk]
  int64_t *chunk_off;     // [max_wp * nchunk + 1]
  int64_t nchunk;         // words / kPartChunkWords (rounded up)
  int64_t *scan_tmp;      // scan block sums
  int32_t *cand;          // [max_candidates]
  int64_t max_candidates;
  int64_t *cand_start;    // [max_wp + 1]
  int64_t *cand_count;    // [max_wp]
  int64_t *tile_start;    // [max_wp + 1]
  int32_t *tile_wp;       // [max_wp * tiles_cap]
  int64_t *n_tiles;       // [1]
};
constexpr int64_t kPartMaxCells = 1025 * 1025;  // grid cells (cell size >= extent / 1024)
constexpr int64_t kPartChunkWords = 1024;       // bitmap words per compaction chunk
int64_t part_scan_tmp_elems(int64_t n);          // block-sum scratch of an n-element scan
cudaError_t launch_part_grid(const float4 *pts, int64_t local_bound, float radius, PartScratch ps, cudaStream_t s,
                             int *n_launches);
cudaError_t launch_part_build(const float4 *pts, const float *q, int32_t n_wp, float radius, PartScratch ps,
                              unsigned long long *overflow_flag, cudaStream_t s, int *n_launches);
// finalize: tile counts -> wp_offsets, ordered copy staging -> out, wp_min/argmin/key, count
// (tile_start: per-step tile ranges of a partitioned detect with at most max_tiles_per_wp
// tiles per step; nullptr = tiles_per_wp per step).  fin_scratch: finalize_scratch_elems().
cudaError_t launch_finalize(DetectScratch ds, int32_t n_wp, int32_t tiles_per_wp, const int64_t *tile_start,
                            int64_t max_tiles_per_wp, gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets,
                            float *wp_min, int64_t *wp_argmin, int64_t *wp_key, int64_t *count, int64_t *fin_scratch,
                            cudaStream_t s, int *n_launches);
int64_t finalize_scratch_elems(int64_t max_wp, int64_t max_tiles_per_wp);
// Merge of gathered rank pieces (K5): rank r's wp_offsets at offsets[r * off_stride ..],
// its per-waypoint keys at keys[r * key_stride ..] (key_stride 0: keys already reduced),
// its records at recs[r * rec_stride ..]; a rank count above rec_stride sets *overflow.
cudaError_t launch_merge(int32_t world, int32_t n_wp, const gcdf_active_t *recs, int64_t rec_stride,
                         const int64_t *offsets, int64_t off_stride, const int64_t *keys, int64_t key_stride,
                         gcdf_active_t *out, int64_t out_capacity, int64_t *wp_offsets, float *wp_min,
                         int64_t *wp_argmin, int64_t *wp_key, int64_t *count, unsigned long long *overflow,
                         cudaStream_t s, int *n_launches);

}  // namespace gcdf
