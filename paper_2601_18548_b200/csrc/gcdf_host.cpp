// gcdf_host.cpp -- the C-ABI host layer of libgcdf (include/gcdf.h).
//
// Owns: argument validation (atomic failures), the MLPW v1 parser (its own
// implementation -- the oracle has a separate one), weight packing (fp32 SIMT layout and
// bf16 UMMA SWIZZLE_128B layout), the replicated scene-id allocator ("both
// components can be modified online"), the workspace carve-up, and kernel dispatch.
// No device memory is allocated after gcdf_bind_workspace; no CPU compute path exists
// for any hot-path step (every step runs in the kernels of this directory).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include <cstdlib>

#include "gcdf_comm.h"
#include "gcdf_internal.h"

using namespace gcdf;

namespace {

constexpr int64_t kUpdChunk = 65536;  // points per scene-update scatter chunk
constexpr int kMaxH = 256;   // fp32 block (SIMT layout, and w7 / biases for every path)
constexpr int kTcH = 128;    // the K2b / K2c / K2s 16-bit blocks (weights resident in smem)
constexpr int kEvPool = 64;

inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

struct Layout {
  int64_t pts, wf32, wbf16, wf16, wf16x3, wf16w, meta, cbits, staging, wp_key, wp_count, counter, upd_payload, upd_slots;
  int64_t h_q, h_out, h_offs, h_wmin, h_warg, h_count;
  // exchange buffers of the sharded detect (gcdf_comm.cpp): per-rank header
  // [wp_offsets (n_wp + 1) | wp_key (n_wp)] int64 and records, send + gathered
  int64_t x_hdr_send, x_hdr_recv, x_rec_send, x_rec_recv, x_count;
  int64_t p_grid, p_bbox, p_cell_count, p_cell_start, p_cell_fill, p_cell_items, p_cell_xy, p_bitmap, p_chunk_cnt, p_chunk_off,
      p_scan_tmp, p_cand, p_cand_start, p_cand_count, p_tile_start, p_tile_wp, p_n_tiles, p_words, p_nchunk;
  int64_t total;
  int64_t wf32_bytes, wbf16_bytes;
};

// fp32 block sizes (floats) for H = kMaxH
constexpr int64_t kF32W1p = kMaxH * 4, kF32W1q = kMaxH * 8, kF32W1full = kMaxH * 12;
constexpr int64_t kF32Mat = (int64_t)kMaxH * kMaxH;
constexpr int64_t kF32Total = kF32W1p + kF32W1q + kF32W1full + 10 * kF32Mat + 5 * kMaxH + kMaxH;
// bf16 block sizes (bytes)
constexpr int64_t kBfMat = (int64_t)kTcH * kTcH * 2;
constexpr int64_t kBfW1t = 16LL * kTcH * 2;
constexpr int64_t kBfB1 = 32LL * kTcH * 2;    // layer-1 split weights [128][K = 32], no swizzle
constexpr int64_t kBfBext = 16LL * kTcH * 2;  // per hidden layer bias block [128][K = 16], no swizzle
constexpr int64_t kBfTotal = 5 * kBfMat + kBfW1t + kBfB1 + 5 * kBfBext;
// GCDF_FP16X3 block: 5 x [W_l hi | W_l lo] SW128 images, then W1^T hi, lo
constexpr int64_t kX3Total = 5 * 2 * kBfMat + 2 * kBfW1t;
// H = 256 block (K2w, fp16): the 40 streamed 32 KB chunks of a tile in consumption order
// (W_2..W_6 forward, K-major [out][in]; then W_6^T..W_2^T, K-major [in][out]; 4 chunks of
// 64 K-columns each, SW128), then W1^T [16][256] SW128, layer-1 split [256][32] and the five
// bias blocks [256][16] (no swizzle)
constexpr int kWideH = 256;
constexpr int64_t kWideChunk = (int64_t)kWideH * 128;
constexpr int64_t kWideSeq = 40 * kWideChunk;
constexpr int64_t kWideW1t = 16LL * kWideH * 2, kWideB1 = 32LL * kWideH * 2;
constexpr int64_t kWideBext = 8LL * kWideH * 2;  // K-core 0 of [256][16] {b_hi, b_lo, 0..}; core 1 is zero
constexpr int64_t kWideTotal = kWideSeq + kWideW1t + kWideB1 + 5 * kWideBext;

}  // namespace

struct gcdf_ctx {
  int device = 0;
  int num_sms = 148;
  gcdf_options opt{};
  std::string err;
  bool cuda_failed = false;
  int64_t launches = 0;
  // workspace
  char *ws = nullptr;
  int64_t ws_bytes = 0;
  Layout L{};
  int64_t local_cap = 0;   // local slots (multiple of 128)
  int64_t tiles_cap = 0;   // local_cap / 128
  // weights
  bool loaded = false;
  int H = 0;
  int act = 1;  // MLPW activation: 1 ReLU (R9), 2 softplus (R26)
  std::vector<float> w7host;  // output row (fp32) for the kernel-parameter copy (bf16_view)
  float b7 = 0.f;
  // scene (replicated on every rank)
  std::vector<uint64_t> live;  // global id bitmap
  int64_t n_live = 0, id_bound = 0, cursor = 0;
  // pinned staging for scene updates
  float4 *h_payload = nullptr;
  int64_t *h_slots = nullptr;
  cudaEvent_t upd_done = nullptr;
  // optional MLP-kernel timing
  bool prof = false;
  std::vector<cudaEvent_t> ev;  // 2 * kEvPool
  int ev_used = 0;
  double prof_ms = 0.0;
  int64_t prof_n = 0;
  long long *trace = nullptr;  // diagnostics buffer (device), see gcdf_debug_trace
  // range partition: the planar grid is rebuilt when the scene or the radius changed
  bool part_dirty = true;
  float part_r = -1.f;
  int64_t scene_version = 0;   // bumped by every scene change (captured graphs re-capture)
  int64_t weights_version = 0; // bumped by gcdf_load_weights / gcdf_bind_workspace (same)
  bool exchange = false;       // exchange buffers reserved (world > 1 or opt.exchange)
  Comm comm;                   // gcdf_dist_init* (kind kCommNone until then)
  std::vector<cudaEvent_t> xev;  // exchange-step timing pairs (gcdf_profile_read_exchange)
  int xev_used = 0;
  double xprof_ms = 0.0;
  int64_t xprof_n = 0;
};

// A captured detect (gcdf_graph_create_detect): the arguments, the instantiated graph and
// the scene version it was captured at.
struct gcdf_graph {
  gcdf_ctx *ctx = nullptr;
  const float *q = nullptr;
  int32_t B = 0, N = 0;
  float radius = 0.f, delta = 0.f, tau = 0.f;
  gcdf_active_t *out = nullptr;
  int64_t cap = 0;
  int64_t *offs = nullptr, *warg = nullptr, *wkey = nullptr, *psizes = nullptr, *count = nullptr;
  float *wmin = nullptr;
  cudaStream_t cs = nullptr;   // capture stream
  cudaGraphExec_t exec = nullptr;
  int64_t version = -1;        // scene_version at capture
  int64_t wversion = -1;       // weights_version at capture (the kernel nodes hold the weights
                               // by value: output row, bias, and the kernel chosen for H / act)
};

namespace {

int fail(gcdf_ctx *c, int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

int cuda_fail(gcdf_ctx *c, cudaError_t e, const char *what) {
  if (c) c->cuda_failed = true;
  return fail(c, GCDF_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CK(c, expr, what)                               \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_fail(c, _e, what); \
  } while (0)

int precheck(gcdf_ctx *c, bool need_weights = true) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  if (c->cuda_failed) return fail(c, GCDF_ERR_CUDA, "context is in a failed CUDA state: %s", c->err.c_str());
  if (!c->ws) return fail(c, GCDF_ERR_NOT_LOADED, "no workspace bound");
  if (need_weights && !c->loaded) return fail(c, GCDF_ERR_NOT_LOADED, "no weights loaded");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaSetDevice");
  return GCDF_OK;
}

inline bool owned(const gcdf_ctx *c, int64_t id) {
  return ((id / kTile) % c->opt.world) == c->opt.rank;
}
inline int64_t local_slot(const gcdf_ctx *c, int64_t id) {
  return ((id / kTile) / c->opt.world) * kTile + id % kTile;
}
int64_t local_bound_of(const gcdf_ctx *c) {
  const int64_t nblk = (c->id_bound + kTile - 1) / kTile;
  const int64_t r = c->opt.rank, W = c->opt.world;
  const int64_t owned_blocks = nblk > r ? (nblk - r + W - 1) / W : 0;
  return owned_blocks * kTile;
}
inline bool is_live(const gcdf_ctx *c, int64_t id) { return (c->live[id >> 6] >> (id & 63)) & 1ull; }

WeightsF32 f32_view(const gcdf_ctx *c) {
  const int H = c->H;
  float *base = reinterpret_cast<float *>(c->ws + c->L.wf32);
  WeightsF32 w{};
  float *p = base;
  w.w1p = reinterpret_cast<const float4 *>(p); p += kF32W1p;
  w.w1q = p; p += kF32W1q;
  w.w1full = p; p += kF32W1full;
  for (int li = 0; li < 5; ++li) { w.wt[li] = p; p += (int64_t)H * H; }
  for (int li = 0; li < 5; ++li) { w.wb[li] = p; p += (int64_t)H * H; }
  for (int li = 0; li < 5; ++li) { w.bias[li] = p; p += H; }
  w.w7 = p;
  w.b7 = c->b7;
  return w;
}

uint16_t to_bf16_rne(float f);
uint16_t to_f16_rne(float f);

WeightsBF16 bf16_view(const gcdf_ctx *c) {
  WeightsF32 f = f32_view(c);
  WeightsBF16 w{};
  const bool bf = c->opt.precision == GCDF_BF16 || c->opt.precision == GCDF_BF16X3;
  const int64_t wo = bf ? c->L.wbf16 : c->L.wf16;
  w.w_sw128 = c->ws + wo;
  w.w1t_sw128 = c->ws + wo + 5 * kBfMat;
  w.b1_nosw = c->ws + wo + 5 * kBfMat + kBfW1t;
  w.bext_nosw = c->ws + wo + 5 * kBfMat + kBfW1t + kBfB1;
  if (c->H == kWideH) {  // K2w: streamed chunk sequence + resident small blocks
    const char *b = c->ws + c->L.wf16w;
    w.w_sw128 = b;
    w.w1t_sw128 = b + kWideSeq;
    w.b1_nosw = b + kWideSeq + kWideW1t;
    w.bext_nosw = b + kWideSeq + kWideW1t + kWideB1;
  }
  w.w3_sw128 = c->ws + c->L.wf16x3;
  w.w1t3_sw128 = c->ws + c->L.wf16x3 + 5 * 2 * kBfMat;
  if ((c->H == 128 || c->H == 256) && (int)c->w7host.size() == c->H) {
    const bool f16 = !bf;
    for (int i = 0; i < c->H; ++i) w.w7half_p[i] = 0.5f * c->w7host[i];
    for (int i = 0; i < c->H / 2; ++i) {
      const float a0 = c->w7host[2 * i], a1 = c->w7host[2 * i + 1];
      const uint32_t lo = f16 ? to_f16_rne(a0) : to_bf16_rne(a0);
      const uint32_t hi = f16 ? to_f16_rne(a1) : to_bf16_rne(a1);
      w.w7h_p[i] = lo | (hi << 16);
    }
  }
  w.bh = f.bias[0];  // the five fp32 bias rows are contiguous in the fp32 block
  w.w7 = f.w7;
  w.b7 = f.b7;
  return w;
}

PartScratch part_view(const gcdf_ctx *c) {
  const Layout &L = c->L;
  PartScratch p{};
  p.grid = reinterpret_cast<float *>(c->ws + L.p_grid);
  p.bbox = reinterpret_cast<unsigned *>(c->ws + L.p_bbox);
  p.cell_count = reinterpret_cast<int32_t *>(c->ws + L.p_cell_count);
  p.cell_start = reinterpret_cast<int64_t *>(c->ws + L.p_cell_start);
  p.cell_fill = reinterpret_cast<int32_t *>(c->ws + L.p_cell_fill);
  p.cell_items = reinterpret_cast<int32_t *>(c->ws + L.p_cell_items);
  p.cell_xy = reinterpret_cast<float2 *>(c->ws + L.p_cell_xy);
  p.bitmap = reinterpret_cast<uint32_t *>(c->ws + L.p_bitmap);
  p.words = L.p_words;
  p.chunk_cnt = reinterpret_cast<int32_t *>(c->ws + L.p_chunk_cnt);
  p.chunk_off = reinterpret_cast<int64_t *>(c->ws + L.p_chunk_off);
  p.nchunk = L.p_nchunk;
  p.scan_tmp = reinterpret_cast<int64_t *>(c->ws + L.p_scan_tmp);
  p.cand = reinterpret_cast<int32_t *>(c->ws + L.p_cand);
  p.max_candidates = c->opt.max_candidates;
  p.cand_start = reinterpret_cast<int64_t *>(c->ws + L.p_cand_start);
  p.cand_count = reinterpret_cast<int64_t *>(c->ws + L.p_cand_count);
  p.tile_start = reinterpret_cast<int64_t *>(c->ws + L.p_tile_start);
  p.tile_wp = reinterpret_cast<int32_t *>(c->ws + L.p_tile_wp);
  p.n_tiles = reinterpret_cast<int64_t *>(c->ws + L.p_n_tiles);
  return p;
}

DetectScratch scratch_view(const gcdf_ctx *c) {
  DetectScratch d{};
  d.tile_meta = reinterpret_cast<int2 *>(c->ws + c->L.meta);
  d.staging = reinterpret_cast<gcdf_active_t *>(c->ws + c->L.staging);
  d.max_active = c->opt.max_active;
  d.counter = reinterpret_cast<unsigned long long *>(c->ws + c->L.counter);
  d.wp_key = reinterpret_cast<unsigned long long *>(c->ws + c->L.wp_key);
  return d;
}

SceneView scene_view(const gcdf_ctx *c) {
  SceneView s{};
  s.pts = reinterpret_cast<const float4 *>(c->ws + c->L.pts);
  s.local_bound = local_bound_of(c);
  s.rank = c->opt.rank;
  s.world = c->opt.world;
  return s;
}

uint16_t to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

uint16_t to_f16_rne(float f) {
  const __half h = __float2half_rn(f);
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}

// UMMA canonical SWIZZLE_NONE, K-major: matrix [rows][K] 16-bit, rows % 8 == 0, K % 8 == 0:
// 8-row x 16-B core matrices; core (n / 8, k / 8) at (k / 8) * (rows * 16) + (n / 8) * 128,
// so one MMA K-step of 16 spans two K-cores LBO = rows * 16 bytes apart and the 8-row
// groups are SBO = 128 bytes apart.
void pack_nosw(const std::vector<float> &m, int rows, int K, uint16_t *dst, bool f16) {
  for (int r = 0; r < rows; ++r)
    for (int k = 0; k < K; ++k) {
      const int64_t byte = (int64_t)(k / 8) * rows * 16 + (r / 8) * 128 + (r % 8) * 16 + (k % 8) * 2;
      const float v = m[(size_t)r * K + k];
      dst[byte / 2] = f16 ? to_f16_rne(v) : to_bf16_rne(v);
    }
}

// hi/lo split of a value into two 16-bit operands (x ~= hi + lo to ~2^-22 relative for fp16)
void split16(double x, bool f16, float &hi, float &lo) {
  auto rnd = [&](float v) {
    uint16_t b = f16 ? to_f16_rne(v) : to_bf16_rne(v);
    if (f16) { __half_raw hr; hr.x = b; return __half2float(__half(hr)); }
    uint32_t u = (uint32_t)b << 16; float g; std::memcpy(&g, &u, 4); return g;
  };
  hi = rnd((float)x);
  lo = rnd((float)(x - (double)hi));
}

// UMMA canonical SWIZZLE_128B (K-major view): matrix [rows][cols] 16-bit, cols % 64 == 0.
// chunk = col / 64 -> [rows][128 B] block; 16-B granule g of row r at g ^ (r % 8).
void pack_sw128(const std::vector<float> &m, int rows, int cols, uint16_t *dst, bool f16) {
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) {
      const int chunk = c / 64, cb = (c % 64) * 2, g = cb / 16;
      const int64_t byte = (int64_t)chunk * rows * 128 + (int64_t)r * 128 + ((g ^ (r % 8)) * 16) + (cb % 16);
      const float v = m[(size_t)r * cols + c];
      dst[byte / 2] = f16 ? to_f16_rne(v) : to_bf16_rne(v);
    }
}

int count_launch(gcdf_ctx *c, cudaError_t e, const char *what, int n = 1) {
  c->launches += n;
  if (e != cudaSuccess) return cuda_fail(c, e, what);
  return GCDF_OK;
}

int prof_drain(gcdf_ctx *c) {
  for (int i = 0; i < c->ev_used; ++i) {
    CK(c, cudaEventSynchronize(c->ev[2 * i + 1]), "profile sync");
    float ms = 0.f;
    CK(c, cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]), "profile elapsed");
    c->prof_ms += ms;
    ++c->prof_n;
  }
  c->ev_used = 0;
  for (int i = 0; i < c->xev_used; ++i) {
    CK(c, cudaEventSynchronize(c->xev[2 * i + 1]), "profile sync");
    float ms = 0.f;
    CK(c, cudaEventElapsedTime(&ms, c->xev[2 * i], c->xev[2 * i + 1]), "profile elapsed");
    c->xprof_ms += ms;
    ++c->xprof_n;
  }
  c->xev_used = 0;
  return GCDF_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

void gcdf_default_options(gcdf_options *o) {
  if (!o) return;
  o->precision = GCDF_FP16;
  o->tgrad_mode = GCDF_TGRAD_CHAINRULE;
  o->scene_capacity = 1 << 20;
  o->max_waypoints = 256;
  o->max_active = 1 << 22;
  o->rank = 0;
  o->world = 1;
  o->max_candidates = 0;
  o->frame = GCDF_FRAME_TRANSLATE;
  o->exchange = 0;
}

int gcdf_has_tcgen05(void) { return tc_compiled() ? 1 : 0; }

int gcdf_create(int cuda_device, const gcdf_options *opt, gcdf_ctx **out) {
  if (!out) return GCDF_ERR_INVALID_ARG;
  *out = nullptr;
  gcdf_options o;
  gcdf_default_options(&o);
  if (opt) o = *opt;
  // scene_capacity < 2^31: local slots are int32 in the partition and ~0u is the dead-slot
  // sentinel of the tensor kernels; max_waypoints <= 65535: the finalize / compaction /
  // pair-generation kernels put the waypoint on gridDim.y
  if (o.scene_capacity <= 0 || o.scene_capacity >= (1LL << 31) || o.max_waypoints <= 0 ||
      o.max_waypoints > 65535 || o.max_active <= 0 ||
      o.max_active >= (1LL << 31) || o.world < 1 || o.rank < 0 || o.rank >= o.world ||
      (o.precision != GCDF_FP32 && o.precision != GCDF_BF16 && o.precision != GCDF_FP16 &&
       o.precision != GCDF_FP16X3 && o.precision != GCDF_BF16X3) ||
      (o.tgrad_mode != GCDF_TGRAD_CHAINRULE && o.tgrad_mode != GCDF_TGRAD_QCHANNEL) ||
      (o.frame != GCDF_FRAME_TRANSLATE && o.frame != GCDF_FRAME_SE2) ||
      (o.frame == GCDF_FRAME_SE2 && o.tgrad_mode == GCDF_TGRAD_QCHANNEL))  // R24: theta is not a channel in SE(2)
    return GCDF_ERR_INVALID_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return GCDF_ERR_UNSUPPORTED;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return GCDF_ERR_CUDA;
  if (prop.major != 10 || prop.minor != 0) return GCDF_ERR_UNSUPPORTED;  // sm_100a kernels only
  if (o.precision != GCDF_FP32 && !tc_compiled()) return GCDF_ERR_UNSUPPORTED;
  gcdf_ctx *c = new gcdf_ctx();
  c->device = cuda_device;
  c->num_sms = prop.multiProcessorCount;
  c->opt = o;
  const int64_t gblocks = (o.scene_capacity + kTile - 1) / kTile;
  const int64_t lblocks = (gblocks + o.world - 1) / o.world;
  c->local_cap = lblocks * kTile;
  c->tiles_cap = lblocks;
  c->live.assign((size_t)((o.scene_capacity + 63) / 64), 0ull);
  // workspace layout
  Layout &L = c->L;
  int64_t off = 0;
  L.pts = off; off = align256(off + c->local_cap * 16);
  L.wf32 = off; L.wf32_bytes = kF32Total * 4; off = align256(off + L.wf32_bytes);
  L.wbf16 = off; L.wbf16_bytes = kBfTotal; off = align256(off + kBfTotal);
  L.wf16 = off; off = align256(off + kBfTotal);
  L.wf16x3 = off; off = align256(off + kX3Total);
  L.wf16w = off; off = align256(off + kWideTotal);
  L.meta = off; off = align256(off + (int64_t)o.max_waypoints * c->tiles_cap * 8);
  L.cbits = off; off = align256(off + k3_scratch_elems(o.max_waypoints, c->tiles_cap) * 8);  // standalone K3
  L.staging = off; off = align256(off + o.max_active * (int64_t)sizeof(gcdf_active_t));
  L.wp_key = off; off = align256(off + (int64_t)o.max_waypoints * 8);
  L.wp_count = off; off = align256(off + finalize_scratch_elems(o.max_waypoints, c->tiles_cap) * 8);
  L.counter = off; off = align256(off + 16);
  L.upd_payload = off; off = align256(off + kUpdChunk * 16);
  L.upd_slots = off; off = align256(off + kUpdChunk * 8);
  // device side of gcdf_detect_active_set_host
  L.h_q = off; off = align256(off + (int64_t)o.max_waypoints * kNdof * 4);
  // (the gathered result of a sharded detect holds up to world x max_active records)
  L.h_out = off; off = align256(off + o.max_active * (int64_t)sizeof(gcdf_active_t) * o.world);
  L.h_offs = off; off = align256(off + ((int64_t)o.max_waypoints + 1) * 8);
  L.h_wmin = off; off = align256(off + (int64_t)o.max_waypoints * 4);
  L.h_warg = off; off = align256(off + (int64_t)o.max_waypoints * 8);
  L.h_count = off; off = align256(off + 8);
  c->exchange = o.world > 1 || o.exchange != 0;
  if (c->exchange) {
    const int64_t hdr = (2 * (int64_t)o.max_waypoints + 1) * 8;
    L.x_hdr_send = off; off = align256(off + hdr);
    L.x_hdr_recv = off; off = align256(off + hdr * o.world);
    L.x_rec_send = off; off = align256(off + o.max_active * (int64_t)sizeof(gcdf_active_t));
    L.x_rec_recv = off; off = align256(off + o.max_active * (int64_t)sizeof(gcdf_active_t) * o.world);
    L.x_count = off; off = align256(off + 8);
  }
  // range-partitioned detect (k_partition.cu), only with max_candidates > 0
  if (o.max_candidates > 0) {
    const int64_t W = o.max_waypoints;
    L.p_words = c->local_cap / 32;
    L.p_nchunk = (L.p_words + kPartChunkWords - 1) / kPartChunkWords;
    const int64_t max_tiles = std::min<int64_t>(W * c->tiles_cap, o.max_candidates / kTile + W);
    L.p_grid = off; off = align256(off + 64);
    L.p_bbox = off; off = align256(off + 64);
    L.p_cell_count = off; off = align256(off + kPartMaxCells * 4);
    L.p_cell_start = off; off = align256(off + (kPartMaxCells + 1) * 8);
    L.p_cell_fill = off; off = align256(off + kPartMaxCells * 4);
    L.p_cell_items = off; off = align256(off + c->local_cap * 4);
    L.p_cell_xy = off; off = align256(off + c->local_cap * 8);
    L.p_bitmap = off; off = align256(off + W * L.p_words * 4);
    L.p_chunk_cnt = off; off = align256(off + W * L.p_nchunk * 4);
    L.p_chunk_off = off; off = align256(off + (W * L.p_nchunk + 1) * 8);
    L.p_scan_tmp = off; off = align256(off + part_scan_tmp_elems(std::max<int64_t>(kPartMaxCells, W * L.p_nchunk)) * 8);
    L.p_cand = off; off = align256(off + o.max_candidates * 4);
    L.p_cand_start = off; off = align256(off + (W + 1) * 8);
    L.p_cand_count = off; off = align256(off + W * 8);
    L.p_tile_start = off; off = align256(off + (W + 1) * 8);
    L.p_tile_wp = off; off = align256(off + max_tiles * 4);
    L.p_n_tiles = off; off = align256(off + 8);
  }
  L.total = off;
  cudaSetDevice(cuda_device);
  if (cudaHostAlloc(&c->h_payload, kUpdChunk * 16, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&c->h_slots, kUpdChunk * 8, cudaHostAllocDefault) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->upd_done, cudaEventDisableTiming) != cudaSuccess) {
    gcdf_destroy(c);
    return GCDF_ERR_CUDA;
  }
  *out = c;
  return GCDF_OK;
}

int gcdf_destroy(gcdf_ctx *c) {
  if (!c) return GCDF_OK;
  cudaSetDevice(c->device);
  if (c->upd_done) { cudaEventSynchronize(c->upd_done); cudaEventDestroy(c->upd_done); }
  if (c->h_payload) cudaFreeHost(c->h_payload);
  if (c->h_slots) cudaFreeHost(c->h_slots);
  for (auto &e : c->ev) cudaEventDestroy(e);
  for (auto &e : c->xev) cudaEventDestroy(e);
  comm_destroy(c->comm);
  delete c;
  return GCDF_OK;
}

const char *gcdf_last_error(const gcdf_ctx *c) { return c ? c->err.c_str() : "null context"; }

int64_t gcdf_launch_count(const gcdf_ctx *c) { return c ? c->launches : 0; }

int gcdf_workspace_bytes(const gcdf_ctx *c, int64_t *bytes) {
  if (!c || !bytes) return GCDF_ERR_INVALID_ARG;
  *bytes = c->L.total;
  return GCDF_OK;
}

int gcdf_bind_workspace(gcdf_ctx *c, void *dev_ptr, int64_t bytes) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  if (!dev_ptr || bytes < c->L.total || ((uintptr_t)dev_ptr & 255))
    return fail(c, GCDF_ERR_INVALID_ARG, "workspace must be >= %lld bytes and 256-B aligned", (long long)c->L.total);
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, dev_ptr) != cudaSuccess || at.type != cudaMemoryTypeDevice || at.device != c->device)
    return fail(c, GCDF_ERR_INVALID_ARG, "workspace is not device memory of device %d", c->device);
  c->ws = static_cast<char *>(dev_ptr);
  c->ws_bytes = bytes;
  c->loaded = false;
  ++c->weights_version;
  ++c->scene_version;
  c->part_dirty = true;
  std::fill(c->live.begin(), c->live.end(), 0ull);
  c->n_live = c->id_bound = c->cursor = 0;
  cudaSetDevice(c->device);
  cudaError_t e = launch_fill(reinterpret_cast<float4 *>(c->ws + c->L.pts), c->local_cap, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return count_launch(c, e, "workspace init");
}

int gcdf_load_weights(gcdf_ctx *c, const char *path, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if (!path) return fail(c, GCDF_ERR_INVALID_ARG, "null path");
  std::ifstream fh(path, std::ios::binary);
  if (!fh) return fail(c, GCDF_ERR_IO, "cannot open %s", path);
  std::vector<char> buf((std::istreambuf_iterator<char>(fh)), std::istreambuf_iterator<char>());
  size_t pos = 0;
  auto rd = [&](void *d, size_t n) -> bool {
    if (pos + n > buf.size()) return false;
    std::memcpy(d, buf.data() + pos, n);
    pos += n;
    return true;
  };
  char magic[4];
  if (!rd(magic, 4)) return fail(c, GCDF_ERR_IO, "%s: truncated header", path);
  if (std::memcmp(magic, "MLPW", 4) != 0) return fail(c, GCDF_ERR_BAD_MAGIC, "%s: bad magic", path);
  uint32_t hdr[3];
  if (!rd(hdr, 12)) return fail(c, GCDF_ERR_IO, "%s: truncated header", path);
  if (hdr[0] != 1) return fail(c, GCDF_ERR_VERSION, "%s: version %u != 1", path, hdr[0]);
  const uint32_t act = hdr[1], L = hdr[2];
  if (L != 7) return fail(c, GCDF_ERR_DIM_MISMATCH, "%s: %u layers, expected 7 (R7)", path, L);
  uint32_t dims[8];
  if (!rd(dims, 32)) return fail(c, GCDF_ERR_IO, "%s: truncated dims", path);
  const int H = (int)dims[1];
  bool ok = dims[0] == (uint32_t)kNin && dims[7] == 1 && (H == 32 || H == 128 || H == kWideH);
  for (int l = 1; l <= 6; ++l) ok = ok && dims[l] == (uint32_t)H;
  if (!ok) return fail(c, GCDF_ERR_DIM_MISMATCH, "%s: dims must be [12, H x 6, 1], H in {32, 128, 256}", path);
  if (H == kWideH && c->opt.precision != GCDF_FP32 &&
      (c->opt.precision != GCDF_FP16 || act != 1 || c->opt.frame != GCDF_FRAME_TRANSLATE))
    return fail(c, GCDF_ERR_DIM_MISMATCH,
                "%s: H = 256 (NEXT-4) runs on GCDF_FP32, or on GCDF_FP16 with ReLU in the translation frame (K2w)",
                path);
  if (act != 1 && act != 2)
    return fail(c, GCDF_ERR_DIM_MISMATCH, "%s: activation %u (ReLU = 1, R9, or softplus = 2, R26)", path, act);
  if (act == 2 && c->opt.precision != GCDF_FP32 &&
      (c->opt.precision != GCDF_FP16 || c->opt.frame != GCDF_FRAME_TRANSLATE))
    return fail(c, GCDF_ERR_DIM_MISMATCH,
                "%s: softplus (R26) runs on GCDF_FP32, or on GCDF_FP16 in the translation frame", path);
  if (c->opt.precision != GCDF_FP32 && H == 32)
    return fail(c, GCDF_ERR_DIM_MISMATCH, "%s: the tensor-core path needs H = 128 or 256 (use GCDF_FP32 for H = %d)",
                path, H);
  std::vector<std::vector<double>> Wd(7), bd(7);
  for (int l = 0; l < 7; ++l) {
    Wd[l].resize((size_t)dims[l + 1] * dims[l]);
    bd[l].resize(dims[l + 1]);
    if (!rd(Wd[l].data(), Wd[l].size() * 8) || !rd(bd[l].data(), bd[l].size() * 8))
      return fail(c, GCDF_ERR_IO, "%s: truncated body (layer %d)", path, l + 1);
    for (double v : Wd[l]) if (!std::isfinite(v)) return fail(c, GCDF_ERR_NONFINITE, "%s: non-finite weight", path);
    for (double v : bd[l]) if (!std::isfinite(v)) return fail(c, GCDF_ERR_NONFINITE, "%s: non-finite bias", path);
  }
  if (pos != buf.size()) return fail(c, GCDF_ERR_DIM_MISMATCH, "%s: %zu trailing bytes", path, buf.size() - pos);

  // ---- pack fp32 (SIMT layout) ----
  std::vector<float> f32((size_t)kF32Total, 0.f);
  float *p = f32.data();
  auto W = [&](int l, int r, int col) { return (float)Wd[l][(size_t)r * dims[l] + col]; };
  for (int u = 0; u < H; ++u) {
    p[u * 4 + 0] = W(0, u, 0); p[u * 4 + 1] = W(0, u, 1); p[u * 4 + 2] = W(0, u, 2); p[u * 4 + 3] = (float)bd[0][u];
  }
  p += kF32W1p;
  for (int u = 0; u < H; ++u)
    for (int i = 0; i < 7; ++i) p[u * 8 + i] = W(0, u, 5 + i);
  p += kF32W1q;
  for (int u = 0; u < H; ++u)
    for (int i = 0; i < kNin; ++i) p[u * kNin + i] = W(0, u, i);
  p += kF32W1full;
  const int UPT = H / 16;
  for (int li = 0; li < 5; ++li, p += (int64_t)H * H)  // wt[k][tu][i] = W[tu + 16 i][k]
    for (int k = 0; k < H; ++k)
      for (int tu = 0; tu < 16; ++tu)
        for (int i = 0; i < UPT; ++i) p[(int64_t)k * H + tu * UPT + i] = W(li + 1, tu + 16 * i, k);
  for (int li = 0; li < 5; ++li, p += (int64_t)H * H)  // wb[k][tu][i] = W[k][tu + 16 i]
    for (int k = 0; k < H; ++k)
      for (int tu = 0; tu < 16; ++tu)
        for (int i = 0; i < UPT; ++i) p[(int64_t)k * H + tu * UPT + i] = W(li + 1, k, tu + 16 * i);
  for (int li = 0; li < 5; ++li, p += H)
    for (int u = 0; u < H; ++u) p[u] = (float)bd[li + 1][u];
  for (int u = 0; u < H; ++u) p[u] = W(6, 0, u);
  // ---- pack bf16 and fp16 (UMMA SW128); the weights are rounded f64 -> fp32 -> 16 bit ----
  std::vector<uint16_t> bf((size_t)kBfTotal / 2, 0), hf((size_t)kBfTotal / 2, 0);
  if (H == 128) {
    std::vector<float> m((size_t)H * H);
    for (int li = 0; li < 5; ++li) {
      for (int r = 0; r < H; ++r)
        for (int col = 0; col < H; ++col) m[(size_t)r * H + col] = W(li + 1, r, col);
      pack_sw128(m, H, H, bf.data() + (size_t)li * kBfMat / 2, false);
      pack_sw128(m, H, H, hf.data() + (size_t)li * kBfMat / 2, true);
    }
    std::vector<float> w1t((size_t)16 * H, 0.f);  // [n = input 0..15][k = unit]
    for (int n = 0; n < kNin; ++n)
      for (int k = 0; k < H; ++k) w1t[(size_t)n * H + k] = W(0, k, n);
    pack_sw128(w1t, 16, H, bf.data() + (size_t)5 * kBfMat / 2, false);
    pack_sw128(w1t, 16, H, hf.data() + (size_t)5 * kBfMat / 2, true);
    // layer 1 on the tensor cores, split in hi/lo 16-bit parts: K column 3 i + {0, 1, 2}
    // multiplies A = {x_hi, x_lo, x_hi} by B = {w_hi, w_hi, w_lo} for the ten inputs
    // i = [p'_x, p'_y, p_z, theta, j1..j6] (x_in columns 0, 1, 2, 5..11); columns 30, 31
    // multiply A = 1 by {b_hi, b_lo}.  Hidden-layer biases: K column 0, 1 = {b_hi, b_lo}.
    const int xin[10] = {0, 1, 2, 5, 6, 7, 8, 9, 10, 11};
    for (int f16 = 0; f16 < 2; ++f16) {
      uint16_t *dst = (f16 ? hf : bf).data();
      std::vector<float> b1((size_t)H * 32, 0.f);
      for (int u = 0; u < H; ++u) {
        float hi, lo;
        for (int i = 0; i < 10; ++i) {
          split16(Wd[0][(size_t)u * kNin + xin[i]], f16, hi, lo);
          b1[(size_t)u * 32 + 3 * i + 0] = hi;
          b1[(size_t)u * 32 + 3 * i + 1] = hi;
          b1[(size_t)u * 32 + 3 * i + 2] = lo;
        }
        split16(bd[0][u], f16, hi, lo);
        b1[(size_t)u * 32 + 30] = hi;
        b1[(size_t)u * 32 + 31] = lo;
      }
      pack_nosw(b1, H, 32, dst + (5 * kBfMat + kBfW1t) / 2, f16);
      for (int li = 0; li < 5; ++li) {
        std::vector<float> be((size_t)H * 16, 0.f);
        for (int u = 0; u < H; ++u) {
          float hi, lo;
          split16(bd[li + 1][u], f16, hi, lo);
          be[(size_t)u * 16 + 0] = hi;
          be[(size_t)u * 16 + 1] = lo;
        }
        pack_nosw(be, H, 16, dst + (5 * kBfMat + kBfW1t + kBfB1 + li * kBfBext) / 2, f16);
      }
    }
  }
  // ---- GCDF_FP16X3 / GCDF_BF16X3 (K2c): hi/lo split of the f64 weights in the context's
  // 16-bit type, [W_l hi | W_l lo] per layer ----
  std::vector<uint16_t> x3((size_t)kX3Total / 2, 0);
  const bool x3f16 = c->opt.precision != GCDF_BF16X3;
  if (H == 128) {
    std::vector<float> mh((size_t)H * H), ml((size_t)H * H);
    float hi, lo;
    for (int li = 0; li < 5; ++li) {
      for (size_t i = 0; i < mh.size(); ++i) {
        split16(Wd[li + 1][i], x3f16, hi, lo);
        mh[i] = hi;
        ml[i] = lo;
      }
      pack_sw128(mh, H, H, x3.data() + (size_t)(2 * li) * kBfMat / 2, x3f16);
      pack_sw128(ml, H, H, x3.data() + (size_t)(2 * li + 1) * kBfMat / 2, x3f16);
    }
    std::vector<float> th((size_t)16 * H, 0.f), tl((size_t)16 * H, 0.f);  // W1^T [n][k]
    for (int n = 0; n < kNin; ++n)
      for (int k = 0; k < H; ++k) {
        split16(Wd[0][(size_t)k * kNin + n], x3f16, hi, lo);
        th[(size_t)n * H + k] = hi;
        tl[(size_t)n * H + k] = lo;
      }
    pack_sw128(th, 16, H, x3.data() + (size_t)10 * kBfMat / 2, x3f16);
    pack_sw128(tl, 16, H, x3.data() + (size_t)(10 * kBfMat + kBfW1t) / 2, x3f16);
  }
  // ---- H = 256 (K2w) ----
  std::vector<uint16_t> wide;
  if (H == kWideH) {
    wide.assign((size_t)kWideTotal / 2, 0);
    std::vector<float> m((size_t)H * H), mt((size_t)H * H);
    const int64_t mat = 4 * kWideChunk;  // one layer image = 4 chunks
    for (int li = 0; li < 5; ++li) {
      for (int r = 0; r < H; ++r)
        for (int col = 0; col < H; ++col) {
          m[(size_t)r * H + col] = W(li + 1, r, col);   // [out][in]: forward B, K = in
          mt[(size_t)r * H + col] = W(li + 1, col, r);  // [in][out]: backward B, K = out
        }
      pack_sw128(m, H, H, wide.data() + (size_t)(li * mat) / 2, true);
      pack_sw128(mt, H, H, wide.data() + (size_t)((5 + (4 - li)) * mat) / 2, true);
    }
    std::vector<float> w1t((size_t)16 * H, 0.f);
    for (int n = 0; n < kNin; ++n)
      for (int k = 0; k < H; ++k) w1t[(size_t)n * H + k] = W(0, k, n);
    pack_sw128(w1t, 16, H, wide.data() + kWideSeq / 2, true);
    const int xin[10] = {0, 1, 2, 5, 6, 7, 8, 9, 10, 11};
    std::vector<float> b1((size_t)H * 32, 0.f);
    for (int u = 0; u < H; ++u) {
      float hi, lo;
      for (int i = 0; i < 10; ++i) {
        split16(Wd[0][(size_t)u * kNin + xin[i]], true, hi, lo);
        b1[(size_t)u * 32 + 3 * i + 0] = hi;
        b1[(size_t)u * 32 + 3 * i + 1] = hi;
        b1[(size_t)u * 32 + 3 * i + 2] = lo;
      }
      split16(bd[0][u], true, hi, lo);
      b1[(size_t)u * 32 + 30] = hi;
      b1[(size_t)u * 32 + 31] = lo;
    }
    pack_nosw(b1, H, 32, wide.data() + (kWideSeq + kWideW1t) / 2, true);
    for (int li = 0; li < 5; ++li) {
      std::vector<float> be((size_t)H * 8, 0.f);
      for (int u = 0; u < H; ++u) {
        float hi, lo;
        split16(bd[li + 1][u], true, hi, lo);
        be[(size_t)u * 8 + 0] = hi;
        be[(size_t)u * 8 + 1] = lo;
      }
      pack_nosw(be, H, 8, wide.data() + (kWideSeq + kWideW1t + kWideB1 + li * kWideBext) / 2, true);
    }
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!wide.empty())
    CK(c, cudaMemcpyAsync(c->ws + c->L.wf16w, wide.data(), wide.size() * 2, cudaMemcpyHostToDevice, s), "weights H2D");
  CK(c, cudaMemcpyAsync(c->ws + c->L.wf16x3, x3.data(), x3.size() * 2, cudaMemcpyHostToDevice, s), "weights H2D");
  CK(c, cudaMemcpyAsync(c->ws + c->L.wf32, f32.data(), f32.size() * 4, cudaMemcpyHostToDevice, s), "weights H2D");
  CK(c, cudaMemcpyAsync(c->ws + c->L.wbf16, bf.data(), bf.size() * 2, cudaMemcpyHostToDevice, s), "weights H2D");
  CK(c, cudaMemcpyAsync(c->ws + c->L.wf16, hf.data(), hf.size() * 2, cudaMemcpyHostToDevice, s), "weights H2D");
  CK(c, cudaStreamSynchronize(s), "weights sync");
  c->H = H;
  c->act = (int)act;
  c->w7host.assign(H, 0.f);
  for (int u = 0; u < H; ++u) c->w7host[u] = W(6, 0, u);
  c->b7 = (float)bd[6][0];
  c->loaded = true;
  ++c->weights_version;
  return GCDF_OK;
}

int gcdf_update_scene(gcdf_ctx *c, const float *add_xyz, int64_t n_add, int64_t *out_ids, const int64_t *rem,
                      int64_t n_rem, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if (n_add < 0 || n_rem < 0 || (n_add > 0 && (!add_xyz || !out_ids)) || (n_rem > 0 && !rem))
    return fail(c, GCDF_ERR_INVALID_ARG, "bad update arguments");
  // validate (atomic): removes live and unique, adds finite, capacity
  std::vector<int64_t> rs(rem, rem + n_rem);
  std::sort(rs.begin(), rs.end());
  for (int64_t i = 0; i < n_rem; ++i) {
    if (rs[i] < 0 || rs[i] >= c->opt.scene_capacity || !is_live(c, rs[i]))
      return fail(c, GCDF_ERR_UNKNOWN_ID, "remove id %lld is not live", (long long)rs[i]);
    if (i > 0 && rs[i] == rs[i - 1]) return fail(c, GCDF_ERR_UNKNOWN_ID, "remove id %lld repeated", (long long)rs[i]);
  }
  for (int64_t i = 0; i < 3 * n_add; ++i)
    if (!std::isfinite(add_xyz[i])) return fail(c, GCDF_ERR_NONFINITE, "non-finite point coordinate at %lld", (long long)i);
  if (c->opt.scene_capacity - c->n_live < n_add)
    return fail(c, GCDF_ERR_CAPACITY, "scene capacity %lld exceeded", (long long)c->opt.scene_capacity);
  // allocate: lowest ids free at the start of the call (removed ids stay live until after)
  int64_t cur = c->cursor;
  for (int64_t a = 0; a < n_add; ++a) {
    while (is_live(c, cur)) {
      // skip full words quickly
      if ((cur & 63) == 0 && c->live[cur >> 6] == ~0ull) cur += 64;
      else ++cur;
    }
    out_ids[a] = cur;
    c->live[cur >> 6] |= 1ull << (cur & 63);
    ++cur;
  }
  c->cursor = cur;
  for (int64_t i = 0; i < n_rem; ++i) c->live[rs[i] >> 6] &= ~(1ull << (rs[i] & 63));
  if (n_rem > 0) c->cursor = std::min(c->cursor, rs[0]);
  c->n_live += n_add - n_rem;
  for (int64_t a = 0; a < n_add; ++a) c->id_bound = std::max(c->id_bound, out_ids[a] + 1);
  if (n_add + n_rem > 0) {
    c->part_dirty = true;
    ++c->scene_version;
  }
  // device scatter of this rank's share, in pinned chunks
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float4 *d_pay = reinterpret_cast<float4 *>(c->ws + c->L.upd_payload);
  int64_t *d_slot = reinterpret_cast<int64_t *>(c->ws + c->L.upd_slots);
  float4 *pts = reinterpret_cast<float4 *>(c->ws + c->L.pts);
  int64_t n = 0;
  auto flush = [&]() -> int {
    if (n == 0) return GCDF_OK;
    CK(c, cudaMemcpyAsync(d_pay, c->h_payload, n * 16, cudaMemcpyHostToDevice, s), "scene H2D");
    CK(c, cudaMemcpyAsync(d_slot, c->h_slots, n * 8, cudaMemcpyHostToDevice, s), "scene H2D");
    int r = count_launch(c, launch_scene_scatter(d_pay, d_slot, n, pts, s), "scene scatter");
    if (r) return r;
    CK(c, cudaEventRecord(c->upd_done, s), "event");
    CK(c, cudaEventSynchronize(c->upd_done), "scene sync");  // pinned buffer reusable
    n = 0;
    return GCDF_OK;
  };
  for (int64_t i = 0; i < n_rem; ++i)
    if (owned(c, rs[i])) {
      c->h_payload[n] = make_float4(0.f, 0.f, 0.f, 0.f);
      c->h_slots[n] = local_slot(c, rs[i]);
      if (++n == kUpdChunk && (rc = flush())) return rc;
    }
  for (int64_t a = 0; a < n_add; ++a)
    if (owned(c, out_ids[a])) {
      c->h_payload[n] = make_float4(add_xyz[3 * a], add_xyz[3 * a + 1], add_xyz[3 * a + 2], 1.f);
      c->h_slots[n] = local_slot(c, out_ids[a]);
      if (++n == kUpdChunk && (rc = flush())) return rc;
    }
  return flush();
}

int gcdf_scene_info(const gcdf_ctx *c, int64_t *n_live, int64_t *id_bound, int64_t *local_bound) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  if (n_live) *n_live = c->n_live;
  if (id_bound) *id_bound = c->id_bound;
  if (local_bound) *local_bound = local_bound_of(c);
  return GCDF_OK;
}

static int check_wp(gcdf_ctx *c, const float *q, int32_t B, int32_t N) {
  if (!q || B <= 0 || N <= 0) return fail(c, GCDF_ERR_INVALID_ARG, "q must be non-null with B, N > 0");
  if ((int64_t)B * N > c->opt.max_waypoints)
    return fail(c, GCDF_ERR_CAPACITY, "B*N = %lld exceeds max_waypoints %d", (long long)B * N, c->opt.max_waypoints);
  return GCDF_OK;
}

static QueryArgs make_args(gcdf_ctx *c, const float *q, int32_t nwp) {
  QueryArgs a{};
  a.scene = scene_view(c);
  a.q = q;
  a.n_wp = nwp;
  a.tiles_per_wp = (int32_t)(a.scene.local_bound / kTile);
  a.tgrad = c->opt.tgrad_mode;
  a.frame = c->opt.frame;
  a.act = c->act;
  a.trace = c->trace;
  return a;
}

static cudaError_t run_mlp(gcdf_ctx *c, const QueryArgs &a, cudaStream_t s) {
  if ((int64_t)a.n_wp * a.tiles_per_wp == 0) return cudaSuccess;
  int slot = -1;
  if (c->prof) {
    if (c->ev_used == kEvPool && prof_drain(c)) return cudaErrorUnknown;
    slot = c->ev_used++;
    cudaEventRecord(c->ev[2 * slot], s);
  }
  cudaError_t e = c->opt.precision == GCDF_FP32
                      ? launch_mlp_simt(c->H, f32_view(c), a, c->num_sms, s)
                      : c->opt.precision == GCDF_FP16X3 || c->opt.precision == GCDF_BF16X3
                            ? launch_mlp_tc3(c->opt.precision == GCDF_FP16X3, bf16_view(c), a, c->num_sms, s)
                        : c->H == kWideH ? launch_mlp_tc_wide(bf16_view(c), a, c->num_sms, s)
                        : a.act == 2 ? launch_mlp_tc_sp(bf16_view(c), a, c->num_sms, s)
                            : launch_mlp_tc(c->H, c->opt.precision == GCDF_FP16, bf16_view(c), a, c->num_sms, s);
  if (slot >= 0) cudaEventRecord(c->ev[2 * slot + 1], s);
  return e;
}

int gcdf_profile_enable(gcdf_ctx *c, int enable) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  if (enable && c->ev.empty()) {
    c->ev.resize(2 * kEvPool);
    for (auto &e : c->ev) CK(c, cudaEventCreate(&e), "event create");
    c->xev.resize(2 * kEvPool);
    for (auto &e : c->xev) CK(c, cudaEventCreate(&e), "event create");
  }
  c->prof = enable != 0;
  return GCDF_OK;
}

int gcdf_profile_read_exchange(gcdf_ctx *c, double *ms, int64_t *n, int reset) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  int rc = prof_drain(c);
  if (rc) return rc;
  if (ms) *ms = c->xprof_ms;
  if (n) *n = c->xprof_n;
  if (reset) { c->xprof_ms = 0.0; c->xprof_n = 0; }
  return GCDF_OK;
}

int gcdf_profile_read(gcdf_ctx *c, double *ms, int64_t *n, int reset) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  cudaSetDevice(c->device);
  int rc = prof_drain(c);
  if (rc) return rc;
  if (ms) *ms = c->prof_ms;
  if (n) *n = c->prof_n;
  if (reset) { c->prof_ms = 0.0; c->prof_n = 0; }
  return GCDF_OK;
}

int gcdf_pairgen_transform(gcdf_ctx *c, const float *q, int32_t B, int32_t N, void *out, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if ((rc = check_wp(c, q, B, N))) return rc;
  if (!out) return fail(c, GCDF_ERR_INVALID_ARG, "null output");
  SceneView sv = scene_view(c);
  return count_launch(c, launch_pairgen(sv.pts, sv.local_bound, q, B * N, c->opt.frame, static_cast<float4 *>(out),
                                        static_cast<cudaStream_t>(stream)), "pairgen");
}

int gcdf_query_values_grads(gcdf_ctx *c, const float *q, int32_t B, int32_t N, float *values, float *grads,
                            void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if ((rc = check_wp(c, q, B, N))) return rc;
  if (!values) return fail(c, GCDF_ERR_INVALID_ARG, "null values output");
  QueryArgs a = make_args(c, q, B * N);
  a.values = values;
  a.grads = grads;
  a.detect = 0;
  return count_launch(c, run_mlp(c, a, static_cast<cudaStream_t>(stream)), "query kernel");
}

int gcdf_project_dense(gcdf_ctx *c, const float *q, int32_t B, int32_t N, const float *minv_host, float *values,
                       float *qz, void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if ((rc = check_wp(c, q, B, N))) return rc;
  if (!values || !qz || !minv_host) return fail(c, GCDF_ERR_INVALID_ARG, "project: null argument");
  for (int i = 0; i < kNdof; ++i)
    if (!std::isfinite(minv_host[i]) || minv_host[i] < 0.f)
      return fail(c, GCDF_ERR_INVALID_ARG, "project: M^-1 diagonal must be finite and >= 0");
  QueryArgs a = make_args(c, q, B * N);
  a.values = values;
  a.grads = qz;
  a.detect = 0;
  a.project = 1;
  for (int i = 0; i < kNdof; ++i) a.minv[i] = minv_host[i];
  return count_launch(c, run_mlp(c, a, static_cast<cudaStream_t>(stream)), "project kernel");
}

static int read_count(gcdf_ctx *c, int64_t cap, const int64_t *count_dev, int64_t *count_host, cudaStream_t s);

static int comm_rc(gcdf_ctx *c, int r, const std::string &msg) {
  if (r == kCommErrCuda) c->cuda_failed = true;
  return fail(c, r == kCommErrCuda ? GCDF_ERR_CUDA : GCDF_ERR_NCCL, "exchange: %s", msg.c_str());
}

// The sharded detect's exchange: the local finalize writes this rank's
// records and header into the send buffers, one all-gather group moves them, the merge
// kernel assembles the canonical result in the caller's buffers.  All on s.
static int exchange_detect(gcdf_ctx *c, int32_t nwp, int32_t tpw, gcdf_active_t *out, int64_t cap, int64_t *offs,
                           float *wmin, int64_t *warg, int64_t *wkey, int64_t *count_dev, int64_t *count_host,
                           cudaStream_t s, const int64_t *tile_start) {
  DetectScratch ds = scratch_view(c);
  const int W = c->comm.world;
  const int64_t S = std::max<int64_t>(1, std::min<int64_t>(c->opt.max_active, (cap + W - 1) / W));
  const int64_t hdr = 2 * (int64_t)nwp + 1;
  int64_t *hs = reinterpret_cast<int64_t *>(c->ws + c->L.x_hdr_send);
  int64_t *hr = reinterpret_cast<int64_t *>(c->ws + c->L.x_hdr_recv);
  gcdf_active_t *rs = reinterpret_cast<gcdf_active_t *>(c->ws + c->L.x_rec_send);
  gcdf_active_t *rr = reinterpret_cast<gcdf_active_t *>(c->ws + c->L.x_rec_recv);
  int64_t *lc = reinterpret_cast<int64_t *>(c->ws + c->L.x_count);
  int nl = 0;
  cudaError_t e = launch_finalize(ds, nwp, tpw, tile_start, c->tiles_cap, rs, S, hs, nullptr, nullptr, hs + nwp + 1,
                                  lc, reinterpret_cast<int64_t *>(c->ws + c->L.wp_count), s, &nl);
  int rc = count_launch(c, e, "detect finalize", nl);
  if (rc) return rc;
  int slot = -1;
  if (c->prof && c->comm.kind == kCommNccl) {
    if (c->xev_used == kEvPool && prof_drain(c)) return GCDF_ERR_CUDA;
    slot = c->xev_used++;
    CK(c, cudaEventRecord(c->xev[2 * slot], s), "profile event");
  }
  const void *send[2] = {hs, rs};
  void *recv[2] = {hr, rr};
  const int64_t bytes[2] = {hdr * 8, S * (int64_t)sizeof(gcdf_active_t)};
  std::string msg;
  const int r = comm_allgather(c->comm, 2, send, recv, bytes, s, &msg);
  if (r) return comm_rc(c, r, msg);
  nl = 0;
  e = launch_merge(W, nwp, rr, S, hr, hdr, hr + nwp + 1, hdr, out, cap, offs, wmin, warg, wkey, count_dev,
                   ds.counter + 1, s, &nl);
  if ((rc = count_launch(c, e, "exchange merge", nl))) return rc;
  if (slot >= 0) CK(c, cudaEventRecord(c->xev[2 * slot + 1], s), "profile event");
  return read_count(c, cap, count_dev, count_host, s);
}

static int finish_detect(gcdf_ctx *c, int32_t nwp, int32_t tpw, gcdf_active_t *out, int64_t cap, int64_t *offs,
                         float *wmin, int64_t *warg, int64_t *wkey, int64_t *count_dev, int64_t *count_host,
                         cudaStream_t s, const int64_t *tile_start = nullptr) {
  if (c->comm.kind != kCommNone)
    return exchange_detect(c, nwp, tpw, out, cap, offs, wmin, warg, wkey, count_dev, count_host, s, tile_start);
  DetectScratch ds = scratch_view(c);
  int nl = 0;
  cudaError_t e = launch_finalize(ds, nwp, tpw, tile_start, c->tiles_cap, out, cap, offs, wmin, warg, wkey,
                                  count_dev, reinterpret_cast<int64_t *>(c->ws + c->L.wp_count), s, &nl);
  int rc = count_launch(c, e, "detect finalize", nl);
  if (rc) return rc;
  return read_count(c, cap, count_dev, count_host, s);
}

// count_host (if non-NULL): synchronize, read the active count, CAPACITY if it exceeds the
// output capacity or the staging overflowed
static int read_count(gcdf_ctx *c, int64_t cap, const int64_t *count_dev, int64_t *count_host, cudaStream_t s) {
  DetectScratch ds = scratch_view(c);
  if (count_host) {
    unsigned long long hc[2];
    CK(c, cudaMemcpyAsync(hc, count_dev, 8, cudaMemcpyDeviceToHost, s), "count D2H");
    CK(c, cudaMemcpyAsync(hc + 1, ds.counter + 1, 8, cudaMemcpyDeviceToHost, s), "overflow D2H");
    CK(c, cudaStreamSynchronize(s), "detect sync");
    *count_host = (int64_t)hc[0];
    if (hc[1] || (int64_t)hc[0] > cap)
      return fail(c, GCDF_ERR_CAPACITY, "active count %lld exceeds output capacity %lld or staging %lld",
                  (long long)hc[0], (long long)cap, (long long)c->opt.max_active);
  }
  return GCDF_OK;
}

int gcdf_detect_active_set(gcdf_ctx *c, const float *q, int32_t B, int32_t N, float delta, float tau,
                           gcdf_active_t *out, int64_t cap, int64_t *offs, float *wmin, int64_t *warg,
                           int64_t *wkey, int64_t *count_dev, int64_t *count_host, void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if ((rc = check_wp(c, q, B, N))) return rc;
  if (!out || cap < 0 || !offs || !count_dev || !std::isfinite(delta) || !std::isfinite(tau))
    return fail(c, GCDF_ERR_INVALID_ARG, "detect: null output or non-finite delta/tau");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  QueryArgs a = make_args(c, q, B * N);
  a.detect = 1;
  a.delta = delta;
  a.tau = tau;
  a.ds = scratch_view(c);
  if ((rc = count_launch(c, launch_detect_init(a.ds, a.n_wp, s), "detect init"))) return rc;
  if ((rc = count_launch(c, run_mlp(c, a, s), "detect kernel"))) return rc;
  return finish_detect(c, a.n_wp, a.tiles_per_wp, out, cap, offs, wmin, warg, wkey, count_dev, count_host, s);
}

int gcdf_detect_active_set_partitioned(gcdf_ctx *c, const float *q, int32_t B, int32_t N, float radius, float delta,
                                       float tau, gcdf_active_t *out, int64_t cap, int64_t *offs, float *wmin,
                                       int64_t *warg, int64_t *wkey, int64_t *psizes, int64_t *count_dev,
                                       int64_t *count_host, void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if ((rc = check_wp(c, q, B, N))) return rc;
  if (!out || cap < 0 || !offs || !count_dev || !std::isfinite(delta) || !std::isfinite(tau))
    return fail(c, GCDF_ERR_INVALID_ARG, "detect: null output or non-finite delta/tau");
  if (!(radius > 0.f) || !std::isfinite(radius))
    return fail(c, GCDF_ERR_INVALID_ARG, "partition radius must be finite and > 0");
  if (c->opt.max_candidates <= 0)
    return fail(c, GCDF_ERR_INVALID_ARG, "partitioned detect needs gcdf_options.max_candidates > 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const PartScratch ps = part_view(c);
  const SceneView sv = scene_view(c);
  int nl = 0;
  if (c->part_dirty || c->part_r != radius) {
    if ((rc = count_launch(c, launch_part_grid(sv.pts, sv.local_bound, radius, ps, s, &nl), "partition grid", 0)))
      return rc;
    c->launches += nl;
    c->part_dirty = false;
    c->part_r = radius;
  }
  QueryArgs a = make_args(c, q, B * N);
  a.detect = 1;
  a.delta = delta;
  a.tau = tau;
  a.ds = scratch_view(c);
  if ((rc = count_launch(c, launch_detect_init(a.ds, a.n_wp, s), "detect init"))) return rc;
  nl = 0;
  if ((rc = count_launch(c, launch_part_build(sv.pts, q, a.n_wp, radius, ps, a.ds.counter + 1, s, &nl),
                         "partition build", 0)))
    return rc;
  c->launches += nl;
  a.part.tile_wp = ps.tile_wp;
  a.part.tile_start = ps.tile_start;
  a.part.cand_start = ps.cand_start;
  a.part.cand_count = ps.cand_count;
  a.part.cand = ps.cand;
  a.part.n_tiles = ps.n_tiles;
  if ((rc = count_launch(c, run_mlp(c, a, s), "detect kernel"))) return rc;
  if (psizes)
    CK(c, cudaMemcpyAsync(psizes, ps.cand_count, (int64_t)a.n_wp * 8, cudaMemcpyDeviceToDevice, s), "part sizes");
  return finish_detect(c, a.n_wp, a.tiles_per_wp, out, cap, offs, wmin, warg, wkey, count_dev, count_host, s,
                       ps.tile_start);
}

int gcdf_sparse_jacobian(gcdf_ctx *c, const gcdf_active_t *recs, const int64_t *count_dev, int64_t cap,
                         float delta, float *c_dev, int64_t *row_ptr, int32_t *col, float *val, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if (!recs || !count_dev || cap < 0 || !row_ptr || !col || !val || !std::isfinite(delta))
    return fail(c, GCDF_ERR_INVALID_ARG, "sparse_jacobian: bad arguments");
  return count_launch(c, launch_sparse_jacobian(recs, count_dev, cap, delta, c_dev, row_ptr, col, val, c->num_sms,
                                                static_cast<cudaStream_t>(stream)),
                      "sparse jacobian");
}

int gcdf_detect_active_set_host(gcdf_ctx *c, const float *q_host, int32_t B, int32_t N, float delta, float tau,
                                gcdf_active_t *out_host, int64_t cap, int64_t *offs_host, float *wmin_host,
                                int64_t *warg_host, int64_t *count_host, void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if ((rc = check_wp(c, q_host, B, N))) return rc;
  if (!out_host || cap < 0 || !offs_host || !count_host)
    return fail(c, GCDF_ERR_INVALID_ARG, "detect_host: null output");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nwp = (int64_t)B * N;
  float *q = reinterpret_cast<float *>(c->ws + c->L.h_q);
  gcdf_active_t *out = reinterpret_cast<gcdf_active_t *>(c->ws + c->L.h_out);
  int64_t *offs = reinterpret_cast<int64_t *>(c->ws + c->L.h_offs);
  float *wmin = reinterpret_cast<float *>(c->ws + c->L.h_wmin);
  int64_t *warg = reinterpret_cast<int64_t *>(c->ws + c->L.h_warg);
  int64_t *cnt = reinterpret_cast<int64_t *>(c->ws + c->L.h_count);
  CK(c, cudaMemcpyAsync(q, q_host, nwp * kNdof * 4, cudaMemcpyHostToDevice, s), "q H2D");
  int64_t n = -1;
  // device capacity: max_active (one rank), or with a communicator the caller's capacity
  // (which sets the exchange stride), at most world x max_active
  const int64_t icap = c->comm.kind == kCommNone ? c->opt.max_active
                                                 : std::min<int64_t>(std::max<int64_t>(cap, 1),
                                                                     c->opt.max_active * c->comm.world);
  rc = gcdf_detect_active_set(c, q, B, N, delta, tau, out, icap, offs, wmin, warg, nullptr, cnt, &n, stream);
  *count_host = n;
  if (rc && rc != GCDF_ERR_CAPACITY) return rc;
  const int64_t nc = rc ? 0 : std::min(n, cap);
  if (nc > 0)
    CK(c, cudaMemcpyAsync(out_host, out, nc * (int64_t)sizeof(gcdf_active_t), cudaMemcpyDeviceToHost, s),
       "records D2H");
  CK(c, cudaMemcpyAsync(offs_host, offs, (nwp + 1) * 8, cudaMemcpyDeviceToHost, s), "offsets D2H");
  if (wmin_host) CK(c, cudaMemcpyAsync(wmin_host, wmin, nwp * 4, cudaMemcpyDeviceToHost, s), "wp_min D2H");
  if (warg_host) CK(c, cudaMemcpyAsync(warg_host, warg, nwp * 8, cudaMemcpyDeviceToHost, s), "wp_argmin D2H");
  CK(c, cudaStreamSynchronize(s), "detect_host sync");
  if (rc) return rc;
  if (n > cap)
    return fail(c, GCDF_ERR_CAPACITY, "active count %lld exceeds host capacity %lld", (long long)n, (long long)cap);
  return GCDF_OK;
}

int gcdf_compact_dense(gcdf_ctx *c, const float *values, const float *grads, int32_t n_wp, int64_t stride,
                       float delta, float tau, gcdf_active_t *out, int64_t cap, int64_t *offs, float *wmin,
                       int64_t *warg, int64_t *wkey, int64_t *count_dev, int64_t *count_host, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  SceneView sv = scene_view(c);
  if (!values || !grads || n_wp <= 0 || n_wp > c->opt.max_waypoints || stride < sv.local_bound || (stride & 3) ||
      ((uintptr_t)values & 15) || !out || !offs ||
      !count_dev || !std::isfinite(delta) || !std::isfinite(tau))
    return fail(c, GCDF_ERR_INVALID_ARG, "compact_dense: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DetectScratch ds = scratch_view(c);
  const int32_t tpw = (int32_t)(sv.local_bound / kTile);
  if ((rc = count_launch(c, launch_detect_init(ds, n_wp, s), "compact init"))) return rc;
  int nl = 0;
  if ((rc = count_launch(c,
                         launch_compact_dense(values, grads, stride, n_wp, tpw, sv, delta, tau, ds, out, cap, offs,
                                              wmin, warg, wkey, count_dev,
                                              reinterpret_cast<int64_t *>(c->ws + c->L.cbits), s, &nl),
                         "compact kernels", 0)))
    return rc;
  c->launches += nl;
  return read_count(c, cap, count_dev, count_host, s);
}

int gcdf_merge_active_sets(gcdf_ctx *c, int32_t world, int32_t n_wp, const gcdf_active_t *recs, int64_t rec_stride,
                           const int64_t *offsets, const int64_t *wp_key, gcdf_active_t *out, int64_t cap,
                           int64_t *offs, float *wmin, int64_t *warg, int64_t *count, void *stream) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if (world < 1 || n_wp <= 0 || !recs || rec_stride < 0 || !offsets || !wp_key || !out || !offs || !count)
    return fail(c, GCDF_ERR_INVALID_ARG, "merge: bad arguments");
  int nl = 0;
  cudaError_t e = launch_merge(world, n_wp, recs, rec_stride, offsets, (int64_t)n_wp + 1, wp_key, 0, out, cap, offs,
                               wmin, warg, nullptr, count, nullptr, static_cast<cudaStream_t>(stream), &nl);
  return count_launch(c, e, "merge", nl);
}

// ---------------------------------------------------------------- CUDA graphs
static int graph_capture(gcdf_graph *g) {
  gcdf_ctx *c = g->ctx;
  if (g->exec) {
    cudaGraphExecDestroy(g->exec);
    g->exec = nullptr;
  }
  int rc = GCDF_OK;
  if (g->radius > 0.f && (c->part_dirty || c->part_r != g->radius)) {  // grid built eagerly, not in the graph
    const PartScratch ps = part_view(c);
    const SceneView sv = scene_view(c);
    int nl = 0;
    if ((rc = count_launch(c, launch_part_grid(sv.pts, sv.local_bound, g->radius, ps, g->cs, &nl), "grid", 0)))
      return rc;
    c->launches += nl;
    c->part_dirty = false;
    c->part_r = g->radius;
  }
  if (c->comm.kind == kCommHost)
    return fail(c, GCDF_ERR_INVALID_ARG, "graph: the host exchange backend (tests) cannot be captured");
  const bool prof = c->prof;
  c->prof = false;  // no profiling events inside a graph
  CK(c, cudaStreamBeginCapture(g->cs, cudaStreamCaptureModeRelaxed), "begin capture");
  if (g->radius > 0.f)
    rc = gcdf_detect_active_set_partitioned(c, g->q, g->B, g->N, g->radius, g->delta, g->tau, g->out, g->cap, g->offs,
                                            g->wmin, g->warg, g->wkey, g->psizes, g->count, nullptr, g->cs);
  else
    rc = gcdf_detect_active_set(c, g->q, g->B, g->N, g->delta, g->tau, g->out, g->cap, g->offs, g->wmin, g->warg,
                                g->wkey, g->count, nullptr, g->cs);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(g->cs, &graph);
  c->prof = prof;
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (e != cudaSuccess) return cuda_fail(c, e, "end capture");
  const cudaError_t e2 = cudaGraphInstantiate(&g->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e2 != cudaSuccess) return cuda_fail(c, e2, "graph instantiate");
  g->version = c->scene_version;
  g->wversion = c->weights_version;
  return GCDF_OK;
}

int gcdf_graph_create_detect(gcdf_ctx *c, const float *q, int32_t B, int32_t N, float radius, float delta, float tau,
                             gcdf_active_t *out, int64_t cap, int64_t *offs, float *wmin, int64_t *warg, int64_t *wkey,
                             int64_t *psizes, int64_t *count_dev, gcdf_graph **out_graph) {
  int rc = precheck(c);
  if (rc) return rc;
  if (!out_graph) return fail(c, GCDF_ERR_INVALID_ARG, "graph: null output handle");
  *out_graph = nullptr;
  if (!(radius >= 0.f) || !std::isfinite(radius)) return fail(c, GCDF_ERR_INVALID_ARG, "graph: radius must be >= 0");
  gcdf_graph *g = new gcdf_graph();
  g->ctx = c;
  g->q = q; g->B = B; g->N = N;
  g->radius = radius; g->delta = delta; g->tau = tau;
  g->out = out; g->cap = cap; g->offs = offs; g->wmin = wmin; g->warg = warg; g->wkey = wkey; g->psizes = psizes;
  g->count = count_dev;
  if (cudaStreamCreateWithFlags(&g->cs, cudaStreamNonBlocking) != cudaSuccess) {
    delete g;
    return fail(c, GCDF_ERR_CUDA, "graph: stream");
  }
  if ((rc = graph_capture(g)) || (rc = cudaStreamSynchronize(g->cs) == cudaSuccess ? GCDF_OK : GCDF_ERR_CUDA)) {
    gcdf_graph_destroy(g);
    return rc;
  }
  *out_graph = g;
  return GCDF_OK;
}

int gcdf_graph_launch(gcdf_graph *g, int64_t *count_host, void *stream) {
  if (!g) return GCDF_ERR_INVALID_ARG;
  gcdf_ctx *c = g->ctx;
  int rc = precheck(c);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (g->version != c->scene_version || g->wversion != c->weights_version) {
    // the scene changed (tile counts / grid differ) or the weights were reloaded (the kernel
    // nodes hold the output row, the bias and the kernel chosen for H / activation by value)
    CK(c, cudaStreamSynchronize(s), "graph: order before re-capture");
    if ((rc = graph_capture(g))) return rc;
    CK(c, cudaStreamSynchronize(g->cs), "graph: grid build");
  } else if (g->radius > 0.f && (c->part_dirty || c->part_r != g->radius)) {
    // a direct partitioned call at another radius rebuilt the grid (its parameters live on
    // the device and the graph reads them): rebuild it at this graph's radius, stream-ordered
    const PartScratch ps = part_view(c);
    const SceneView sv = scene_view(c);
    int nl = 0;
    if ((rc = count_launch(c, launch_part_grid(sv.pts, sv.local_bound, g->radius, ps, s, &nl), "grid", 0)))
      return rc;
    c->launches += nl;
    c->part_dirty = false;
    c->part_r = g->radius;
  }
  CK(c, cudaGraphLaunch(g->exec, s), "graph launch");
  return read_count(c, g->cap, g->count, count_host, s);
}

int gcdf_graph_destroy(gcdf_graph *g) {
  if (!g) return GCDF_OK;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->cs) cudaStreamDestroy(g->cs);
  delete g;
  return GCDF_OK;
}

int gcdf_nccl_unique_id(unsigned char out_id[128]) {
  if (!out_id) return GCDF_ERR_INVALID_ARG;
  std::string msg;
  return comm_unique_id(out_id, &msg) ? GCDF_ERR_NCCL : GCDF_OK;
}

static int dist_precheck(gcdf_ctx *c) {
  int rc = precheck(c, false);
  if (rc) return rc;
  if (!c->exchange)
    return fail(c, GCDF_ERR_INVALID_ARG, "dist_init: no exchange buffers (world == 1 needs gcdf_options.exchange)");
  if (c->comm.kind != kCommNone) return fail(c, GCDF_ERR_INVALID_ARG, "dist_init: communicator already initialized");
  return GCDF_OK;
}

int gcdf_dist_init(gcdf_ctx *c, const unsigned char id[128], int32_t rank, int32_t world) {
  int rc = dist_precheck(c);
  if (rc) return rc;
  if (!id || rank != c->opt.rank || world != c->opt.world)
    return fail(c, GCDF_ERR_INVALID_ARG, "dist_init: rank %d / world %d differ from the context's %d / %d", rank, world,
                c->opt.rank, c->opt.world);
  std::string msg;
  const int r = comm_init_nccl(c->comm, id, rank, world, &msg);
  if (r) return fail(c, GCDF_ERR_NCCL, "dist_init: %s", msg.c_str());
  return GCDF_OK;
}

int gcdf_dist_init_host(gcdf_ctx *c, gcdf_host_allgather_fn fn, void *user) {
  int rc = dist_precheck(c);
  if (rc) return rc;
  if (!fn) return fail(c, GCDF_ERR_INVALID_ARG, "dist_init_host: null all-gather");
  comm_init_host(c->comm, c->opt.rank, c->opt.world, fn, user);
  return GCDF_OK;
}

int gcdf_broadcast_waypoints(gcdf_ctx *c, float *q, int32_t B, int32_t N, void *stream) {
  int rc = precheck(c);
  if (rc) return rc;
  if (c->comm.kind == kCommNone) return fail(c, GCDF_ERR_INVALID_ARG, "broadcast_waypoints: no communicator");
  if (!q || B <= 0 || N <= 0) return fail(c, GCDF_ERR_INVALID_ARG, "broadcast_waypoints: bad arguments");
  std::string msg;
  const int r = comm_broadcast(c->comm, q, (int64_t)B * N * kNdof * (int64_t)sizeof(float),
                               static_cast<cudaStream_t>(stream), &msg);
  return r ? comm_rc(c, r, msg) : GCDF_OK;
}

int gcdf_dist_info(const gcdf_ctx *c, int32_t *kind, int32_t *nccl_version) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  if (kind) *kind = c->comm.kind;
  if (nccl_version) *nccl_version = c->comm.nccl_version;
  return GCDF_OK;
}

int gcdf_debug_trace(gcdf_ctx *c, long long *trace_dev) {
  if (!c) return GCDF_ERR_INVALID_ARG;
  c->trace = trace_dev;
  return GCDF_OK;
}

int gcdf_selftest_umma(int dev, int mode, const float *A, const float *B, float *D, void *stream) {
  if (!tc_compiled()) return GCDF_ERR_UNSUPPORTED;
  if (mode < 0 || mode > 6 || (mode & 3) > 2 || !A || !B || !D) return GCDF_ERR_INVALID_ARG;
  if (cudaSetDevice(dev) != cudaSuccess) return GCDF_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (launch_selftest_umma(mode, A, B, D, s) != cudaSuccess) return GCDF_ERR_CUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? GCDF_OK : GCDF_ERR_CUDA;
}

}  // extern "C"
