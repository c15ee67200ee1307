/* gcdf_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, float64 CPU oracle of the batched GCDF query and active-set
 * detection of arXiv 2601.18548.  It shares no code with the CUDA path
 * (paper_2601_18548_b200/csrc) and neither side includes or links the other.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load it.
 *
 * What it computes, step by step in the paper's order (citations are
 * /root/reference/PAPER.md line numbers):
 *   O1  MLPW v1 weights file, the "7-layer MLP" on [p, q]
 *       ("concatenation of p and q", input width 3+n).
 *   O3  base-frame bias of the obstacle point ("treat the robot
 *       base pose as the origin and bias all obstacle points"):
 *       x_in = [p_x - q_x, p_y - q_y, p_z, 0, 0, theta, j1..j6]  (R1, R2)
 *   O4  forward  z_l = W_l h_{l-1} + b_l, h_l = max(z_l, 0) (l < L), f = W_L h_{L-1} + b_L
 *       signed output, no output activation ("+-").
 *       kappa = min_{l,k} |z_{l,k}| (kink proximity, for test skips).
 *   O5  analytic backward of the same function; gradient w.r.t. q by the chain
 *       rule through the bias ("gradients with respect to
 *       translational degrees of freedom can be obtained through the chain rule
 *       by utilizing the gradients of obstacle point positions"):
 *       grad_q f = [-g0[0], -g0[1], g0[5], ..., g0[11]]   (TGRAD_QCHANNEL: g0[3], g0[4])
 *       ReLU'(0) = 0.
 *       Softplus variant (MLPW activation 2, NEXT-4, R26): h_l = log(1 + e^z_l),
 *       sigma'(z) = 1 / (1 + e^-z) (SPEC.md:281 picks softplus for smoothness; the paper
 *       names no activation).
 *       FRAME_SE2 (NEXT-4 variant, R24): p' = R(-theta)(p_xy - b) and the theta
 *       channel fed zero; grad by the chain rule through the rotation.
 *   O6  active <=> f - delta <= tau  (constraint f - delta >= 0, PAPER.md:362-363;
 *       tau: DESIGN.md R12); records appended in loop order (wp ascending, point id
 *       ascending) = the step-major order of c_gcdf (Eq. 14).
 *   O7  per-waypoint min / argmin (first = smallest id on ties; +inf / -1 if empty):
 *       union of obstacles = min of distance fields.
 *   O8  EMU_BF16 flags: same arithmetic in f64, but rounding to bf16 (via fp32,
 *       round-to-nearest-even) exactly where the tensor-core path rounds its MMA
 *       operands.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_INVALID (-1)
#define OR_ERR_IO (-2)
#define OR_ERR_BAD_MAGIC (-3)
#define OR_ERR_VERSION (-4)
#define OR_ERR_DIM (-5)
#define OR_ERR_NOMEM (-12)

#define OR_EMU_W 1           /* round hidden W_2..W_{L-1} and W_1 (as used by the gradient) to bf16 */
#define OR_EMU_A 2           /* round MMA A-operands h_1..h_{L-2}, e_{L-1}..e_1 to bf16 */
#define OR_TGRAD_QCHANNEL 4  /* translational gradient from the q^t input channels */
#define OR_FRAME_SE2 16      /* NEXT-4 variant (R24): rotate the points into the base frame too */
#define OR_EMU_FP16 8        /* with OR_EMU_W / OR_EMU_A: round to fp16 instead of bf16 */

#define OR_MAXL 16
#define OR_NDOF 9
#define OR_NIN 12

typedef struct {
  int act; /* 0 identity, 1 ReLU, 2 softplus (NEXT-4 variant, R26) */
  int L;   /* number of affine layers */
  int dims[OR_MAXL + 1];
  double *W[OR_MAXL]; /* [dims[l+1]][dims[l]] row-major */
  double *b[OR_MAXL];
  double *Wr[OR_MAXL]; /* bf16-rounded copies (O8) */
  double *Wh[OR_MAXL]; /* fp16-rounded copies (O8, OR_EMU_FP16) */
  int maxw;
} omlp_t;

/* ---------------------------------------------------------------- helpers */
static double bf16r(double v) {
  /* f64 -> fp32 (RN) -> bf16 (RN-even), as a CUDA kernel does with a float
     holding the value and cvt.rn.bf16.f32. */
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return v; /* inf/nan untouched */
  u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}

static double f16r(double v) {
  /* f64 -> fp32 (RN) -> fp16 (RN-even, with subnormals), as cvt.rn.f16x2.f32 does */
  float f = (float)v;
  _Float16 h = (_Float16)f;
  return (double)(float)h;
}

/* softplus(z) = log(1 + e^z), written as max(z, 0) + log1p(e^-|z|) so that neither
   exp overflows nor log1p loses the small tail (R26); its derivative is the
   logistic sigmoid 1 / (1 + e^-z). */
static double softplus(double z) { return (z > 0.0 ? z : 0.0) + log1p(exp(-fabs(z))); }
static double sigmoid(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double t = exp(z);
  return t / (1.0 + t);
}

static double act_fwd(int act, double z) {
  if (act == 1) return z > 0.0 ? z : 0.0;
  if (act == 2) return softplus(z);
  return z;
}

void or_free(omlp_t *m) {
  if (!m) return;
  for (int l = 0; l < m->L; ++l) {
    free(m->W[l]);
    free(m->b[l]);
    free(m->Wr[l]);
    free(m->Wh[l]);
  }
  free(m);
}

/* O1: parse MLPW v1. */
int or_load(const char *path, omlp_t **out) {
  *out = NULL;
  FILE *fh = fopen(path, "rb");
  if (!fh) return OR_ERR_IO;
  char magic[4];
  uint32_t hdr[3];
  if (fread(magic, 1, 4, fh) != 4) { fclose(fh); return OR_ERR_IO; }
  if (memcmp(magic, "MLPW", 4) != 0) { fclose(fh); return OR_ERR_BAD_MAGIC; }
  if (fread(hdr, 4, 3, fh) != 3) { fclose(fh); return OR_ERR_IO; }
  if (hdr[0] != 1) { fclose(fh); return OR_ERR_VERSION; }
  uint32_t L = hdr[2];
  if (L < 2 || L > OR_MAXL) { fclose(fh); return OR_ERR_DIM; }
  uint32_t dims[OR_MAXL + 1];
  if (fread(dims, 4, L + 1, fh) != L + 1) { fclose(fh); return OR_ERR_IO; }
  if (dims[0] != OR_NIN || dims[L] != 1) { fclose(fh); return OR_ERR_DIM; }
  for (uint32_t l = 0; l <= L; ++l)
    if (dims[l] == 0 || dims[l] > 4096) { fclose(fh); return OR_ERR_DIM; }
  if (hdr[1] > 2) { fclose(fh); return OR_ERR_DIM; } /* 0 identity, 1 ReLU, 2 softplus */
  omlp_t *m = (omlp_t *)calloc(1, sizeof(omlp_t));
  if (!m) { fclose(fh); return OR_ERR_NOMEM; }
  m->act = (int)hdr[1];
  m->L = (int)L;
  m->maxw = 0;
  for (uint32_t l = 0; l <= L; ++l) {
    m->dims[l] = (int)dims[l];
    if ((int)dims[l] > m->maxw) m->maxw = (int)dims[l];
  }
  for (int l = 0; l < m->L; ++l) {
    size_t nw = (size_t)m->dims[l + 1] * m->dims[l], nb = (size_t)m->dims[l + 1];
    m->W[l] = (double *)malloc(nw * sizeof(double));
    m->b[l] = (double *)malloc(nb * sizeof(double));
    m->Wr[l] = (double *)malloc(nw * sizeof(double));
    m->Wh[l] = (double *)malloc(nw * sizeof(double));
    if (!m->W[l] || !m->b[l] || !m->Wr[l] || !m->Wh[l]) { fclose(fh); or_free(m); return OR_ERR_NOMEM; }
    if (fread(m->W[l], 8, nw, fh) != nw || fread(m->b[l], 8, nb, fh) != nb) {
      fclose(fh); or_free(m); return OR_ERR_IO;
    }
    for (size_t i = 0; i < nw; ++i) {
      m->Wr[l][i] = bf16r(m->W[l][i]);
      m->Wh[l][i] = f16r(m->W[l][i]);
    }
  }
  /* trailing bytes mean the header does not describe the body */
  char extra;
  if (fread(&extra, 1, 1, fh) == 1) { fclose(fh); or_free(m); return OR_ERR_DIM; }
  fclose(fh);
  *out = m;
  return OR_OK;
}

int or_info(const omlp_t *m, int *act, int *L, int *dims) {
  *act = m->act;
  *L = m->L;
  for (int l = 0; l <= m->L; ++l) dims[l] = m->dims[l];
  return OR_OK;
}

/* ---------------------------------------------------------------- one pair (O3-O5) */
typedef struct {
  double *z;  /* [L-1][maxw] pre-activations of the hidden layers */
  double *h;  /* [L][maxw]  h_0 = x_in, h_l = act(z_l) */
  double *g;  /* [maxw] */
  double *e;  /* [maxw] */
} scratch_t;

static void eval_pair(const omlp_t *m, const double p[3], const double q[OR_NDOF], int flags,
                      scratch_t *s, double *f_out, double grad[OR_NDOF], double *kappa,
                      uint64_t *mhash) {
  const int L = m->L, MW = m->maxw;
  const int emu_w = flags & OR_EMU_W, emu_a = flags & OR_EMU_A;
  const int fp16 = flags & OR_EMU_FP16;
  double (*rnd)(double) = fp16 ? f16r : bf16r;
  double *const *Wround = fp16 ? m->Wh : m->Wr;
  double *h0 = s->h;
  /* O3: base-frame bias (translation only; q^t channels fed zero) */
  const double dx = p[0] - q[0], dy = p[1] - q[1];
  const double cth = cos(q[2]), sth = sin(q[2]);
  if (flags & OR_FRAME_SE2) {  /* R24: p' = R(-theta) (p_xy - b), the theta channel fed zero */
    h0[0] = cth * dx + sth * dy;
    h0[1] = -sth * dx + cth * dy;
  } else {
    h0[0] = dx;
    h0[1] = dy;
  }
  h0[2] = p[2];
  h0[3] = 0.0;
  h0[4] = 0.0;
  for (int k = 0; k < 7; ++k) h0[5 + k] = q[2 + k];
  if (flags & OR_FRAME_SE2) h0[5] = 0.0;
  /* O4: forward through the hidden layers l = 1..L-1 (array index l-1) */
  double kap = INFINITY;
  for (int l = 0; l < L - 1; ++l) {
    const int din = m->dims[l], dout = m->dims[l + 1];
    /* layer 1 (l == 0) runs in fp32/f64 on CUDA cores in every GPU path: never rounded */
    const double *Wl = (emu_w && l > 0) ? Wround[l] : m->W[l];
    const double *hin = s->h + (size_t)l * MW;
    double *zl = s->z + (size_t)l * MW;
    double *hout = s->h + (size_t)(l + 1) * MW;
    for (int k = 0; k < dout; ++k) {
      double acc = 0.0;
      for (int j = 0; j < din; ++j) {
        double a = hin[j];
        if (emu_a && l > 0) a = rnd(a); /* A operand h_{l} of layer l+1 rounded (O8) */
        acc += Wl[(size_t)k * din + j] * a;
      }
      zl[k] = acc + m->b[l][k];
      double az = fabs(zl[k]);
      if (az < kap) kap = az;
      hout[k] = act_fwd(m->act, zl[k]);
    }
  }
  /* output layer (no activation) */
  {
    const int din = m->dims[L - 1];
    const double *hin = s->h + (size_t)(L - 1) * MW;
    double acc = 0.0;
    for (int j = 0; j < din; ++j) acc += m->W[L - 1][j] * hin[j];
    *f_out = acc + m->b[L - 1][0];
  }
  /* mask signature (which ReLU units are active), for finite-difference skips */
  uint64_t hsh = 1469598103934665603ull;
  if (m->act == 1) {
    for (int l = 0; l < L - 1; ++l)
      for (int k = 0; k < m->dims[l + 1]; ++k) {
        hsh ^= (uint64_t)(s->z[(size_t)l * MW + k] > 0.0) + 0x9e37u * (uint64_t)(l * 4096 + k);
        hsh *= 1099511628211ull;
      }
  }
  /* O5: backward.  g = dF/dh_{L-1} = W_L^T (row vector), then e_l = g . sigma'(z_l),
     g_{l-1} = W_l^T e_l down to g_0 = dF/dx_in. */
  {
    const int dlast = m->dims[L - 1];
    for (int j = 0; j < dlast; ++j) s->g[j] = m->W[L - 1][j];
  }
  for (int l = L - 2; l >= 0; --l) {
    const int din = m->dims[l], dout = m->dims[l + 1];
    const double *zl = s->z + (size_t)l * MW;
    for (int k = 0; k < dout; ++k) {
      double d = (m->act == 1) ? (zl[k] > 0.0 ? 1.0 : 0.0) : 1.0;
      if (m->act == 2) {
        /* softplus'(z) = sigmoid(z).  EMU (tensor path, R26): the kernel keeps
           only the rounded activation h~ = rnd(softplus(z)) of layers 1..L-2 (its MMA A
           operand) and recovers sigmoid(z) = 1 - e^-softplus(z) from it; the last hidden
           layer's derivative is taken from the fp32 pre-activation. */
        if (emu_a && l < L - 2)
          d = -expm1(-rnd(s->h[(size_t)(l + 1) * MW + k]));
        else
          d = sigmoid(zl[k]);
      }
      double e = s->g[k] * d;
      if (emu_a) e = rnd(e); /* A operand of the backward GEMM (O8) */
      s->e[k] = e;
    }
    const double *Wl = emu_w ? Wround[l] : m->W[l];
    for (int j = 0; j < din; ++j) {
      double acc = 0.0;
      for (int k = 0; k < dout; ++k) acc += Wl[(size_t)k * din + j] * s->e[k];
      s->g[j] = acc;
    }
  }
  /* s->g now holds dF/dx_in[0..11]; map to dF/dq (chain rule through the bias) */
  if (flags & OR_FRAME_SE2) {
    /* p' = R(-theta) d, d = p_xy - b:  dp'/db = -R(-theta), dp'/dtheta = [p'_y, -p'_x];
       the theta channel is fed zero, so df/dtheta is the rotation term alone */
    const double gx = s->g[0], gy = s->g[1];
    grad[0] = -(cth * gx - sth * gy);
    grad[1] = -(sth * gx + cth * gy);
    grad[2] = gx * h0[1] - gy * h0[0];
    for (int k = 1; k < 7; ++k) grad[2 + k] = s->g[5 + k];
  } else {
    if (flags & OR_TGRAD_QCHANNEL) {
      grad[0] = s->g[3];
      grad[1] = s->g[4];
    } else {
      grad[0] = -s->g[0];
      grad[1] = -s->g[1];
    }
    for (int k = 0; k < 7; ++k) grad[2 + k] = s->g[5 + k];
  }
  if (kappa) *kappa = kap;
  if (mhash) *mhash = hsh;
}

/* ---------------------------------------------------------------- batched eval */
typedef struct {
  const omlp_t *m;
  const double *pts;
  int64_t M;
  const double *q;
  int64_t W;
  int flags;
  double *f, *g, *kappa;
  uint64_t *mhash;
  int tid, nthreads;
  int err;
} job_t;

static void *eval_rows(void *arg) {
  job_t *J = (job_t *)arg;
  const omlp_t *m = J->m;
  size_t MW = (size_t)m->maxw;
  scratch_t s;
  s.z = (double *)malloc(sizeof(double) * MW * (m->L));
  s.h = (double *)malloc(sizeof(double) * MW * (m->L + 1));
  s.g = (double *)malloc(sizeof(double) * MW);
  s.e = (double *)malloc(sizeof(double) * MW);
  if (!s.z || !s.h || !s.g || !s.e) { J->err = OR_ERR_NOMEM; goto done; }
  /* static round-robin over waypoint rows */
  for (int64_t w = J->tid; w < J->W; w += J->nthreads) {
    const double *qw = J->q + w * OR_NDOF;
    for (int64_t j = 0; j < J->M; ++j) {
      int64_t o = w * J->M + j;
      double grad[OR_NDOF];
      eval_pair(m, J->pts + 3 * j, qw, J->flags, &s, &J->f[o], grad,
                J->kappa ? &J->kappa[o] : NULL, J->mhash ? &J->mhash[o] : NULL);
      if (J->g) memcpy(J->g + o * OR_NDOF, grad, sizeof(grad));
    }
  }
done:
  free(s.z); free(s.h); free(s.g); free(s.e);
  return NULL;
}

/* f[W][M], g[W][M][9] (may be NULL), kappa[W][M] (may be NULL), mask_hash[W][M] (may be NULL). */
int or_eval(const omlp_t *m, const double *pts, int64_t M, const double *q, int64_t W, int flags,
            double *f, double *g, double *kappa, uint64_t *mask_hash, int nthreads) {
  if (!m || M < 0 || W < 0 || (M > 0 && W > 0 && (!pts || !q || !f))) return OR_ERR_INVALID;
  if ((flags & OR_FRAME_SE2) && (flags & OR_TGRAD_QCHANNEL)) return OR_ERR_INVALID;  /* no q^t channel in SE(2) */
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > W && W > 0) nthreads = (int)W;
  job_t jobs[256];
  pthread_t th[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = (job_t){m, pts, M, q, W, flags, f, g, kappa, mask_hash, t, nthreads, 0};
  }
  if (nthreads == 1) {
    eval_rows(&jobs[0]);
  } else {
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, eval_rows, &jobs[t]);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < nthreads; ++t)
    if (jobs[t].err) return jobs[t].err;
  return OR_OK;
}

/* ---------------------------------------------------------------- detect (O6, O7) */
/* pts[M][3] with ids[M] strictly ascending (the live scene, id -> xyz);
   q[W][9] with W = B*N rows, row index = wp = b*N + i.
   Records (value, grad[9], wp, pt) in (wp, pt) ascending order; at most cap are
   stored, *count receives the full count.  wp_offsets[W+1], wp_min[W], wp_argmin[W]. */
/* NEXT-1 range partition: "only considering obstacle points
   within a certain range of each reference base position" -- the partition of step i is
   I_{M,i} = { j : (p_{j,x} - x_i)^2 + (p_{j,y} - y_i)^2 <= radius^2 } (planar distance to
   the base position (x_i, y_i) = q_i[0:2], inclusive; reading R23).  radius <= 0
   (or +INF) = no partition: every live point of every step.  part_sizes[W] (may be NULL)
   receives m_i = |I_{M,i}|.  The value minimum and the records cover I_{M,i} only. */
int or_detect_part(const omlp_t *m, const double *pts, const int64_t *ids, int64_t M, const double *q,
                   int64_t W, int flags, double radius, double delta, double tau, double *rec_f, double *rec_g,
                   int64_t *rec_wp, int64_t *rec_pt, int64_t cap, int64_t *count, int64_t *wp_offsets,
                   double *wp_min, int64_t *wp_argmin, int64_t *part_sizes, int nthreads) {
  if (!m || M < 0 || W < 0) return OR_ERR_INVALID;
  const int partitioned = radius > 0.0 && isfinite(radius);
  for (int64_t j = 1; j < M; ++j)
    if (ids[j] <= ids[j - 1]) return OR_ERR_INVALID;
  int64_t rows_per_chunk = M > 0 ? (4 * 1024 * 1024) / M : W;
  if (rows_per_chunk < 1) rows_per_chunk = 1;
  if (rows_per_chunk > W) rows_per_chunk = W > 0 ? W : 1;
  double *f = (double *)malloc(sizeof(double) * (size_t)(rows_per_chunk * (M > 0 ? M : 1)));
  double *g = (double *)malloc(sizeof(double) * (size_t)(rows_per_chunk * (M > 0 ? M : 1)) * OR_NDOF);
  if (!f || !g) { free(f); free(g); return OR_ERR_NOMEM; }
  int64_t n = 0;
  for (int64_t w0 = 0; w0 < W; w0 += rows_per_chunk) {
    int64_t nr = (W - w0 < rows_per_chunk) ? (W - w0) : rows_per_chunk;
    int rc = or_eval(m, pts, M, q + w0 * OR_NDOF, nr, flags, f, g, NULL, NULL, nthreads);
    if (rc) { free(f); free(g); return rc; }
    for (int64_t r = 0; r < nr; ++r) {
      int64_t w = w0 + r;
      const double bx = q[w * OR_NDOF + 0], by = q[w * OR_NDOF + 1];
      wp_offsets[w] = n;
      double best = INFINITY;
      int64_t arg = -1, msize = 0;
      for (int64_t j = 0; j < M; ++j) {
        if (partitioned) {
          const double dx = pts[3 * j] - bx, dy = pts[3 * j + 1] - by;
          if (dx * dx + dy * dy > radius * radius) continue;  /* j not in I_{M,i} */
        }
        ++msize;
        double v = f[r * M + j];
        if (v < best) { best = v; arg = ids[j]; } /* strict: first (smallest id) wins ties */
        if (v - delta <= tau) {                   /* O6 */
          if (n < cap) {
            rec_f[n] = v;
            memcpy(rec_g + n * OR_NDOF, g + (r * M + j) * OR_NDOF, sizeof(double) * OR_NDOF);
            rec_wp[n] = w;
            rec_pt[n] = ids[j];
          }
          ++n;
        }
      }
      wp_min[w] = best;
      wp_argmin[w] = arg;
      if (part_sizes) part_sizes[w] = msize;
    }
  }
  wp_offsets[W] = n;
  *count = n;
  free(f);
  free(g);
  return OR_OK;
}

int or_detect(const omlp_t *m, const double *pts, const int64_t *ids, int64_t M, const double *q,
              int64_t W, int flags, double delta, double tau, double *rec_f, double *rec_g,
              int64_t *rec_wp, int64_t *rec_pt, int64_t cap, int64_t *count, int64_t *wp_offsets,
              double *wp_min, int64_t *wp_argmin, int nthreads) {
  return or_detect_part(m, pts, ids, M, q, W, flags, 0.0, delta, tau, rec_f, rec_g, rec_wp, rec_pt, cap, count,
                        wp_offsets, wp_min, wp_argmin, NULL, nthreads);
}

/* ---------------------------------------------------------------- NEXT-3 projection */
/* Theorem 1.2: single-step projection onto the zero level set,
   q_z = q_0 - lambda d with lambda = f(p, q_0) and d = M^{-1} grad_q f(p, q_0), M diagonal
   (minv[9] = its inverse diagonal).  f[W][M], g[W][M][9] (from or_eval), q[W][9] ->
   qz[W][M][9]. */
int or_project(const double *f, const double *g, const double *q, const double *minv, int64_t W, int64_t M,
               double *qz) {
  if (W < 0 || M < 0) return OR_ERR_INVALID;
  for (int64_t w = 0; w < W; ++w)
    for (int64_t j = 0; j < M; ++j) {
      const double lambda = f[w * M + j];
      for (int t = 0; t < OR_NDOF; ++t) {
        const double d = minv[t] * g[(w * M + j) * OR_NDOF + t];
        qz[(w * M + j) * OR_NDOF + t] = q[w * OR_NDOF + t] - lambda * d;
      }
    }
  return OR_OK;
}

/* ---------------------------------------------------------------- NEXT-2 sparse Jacobian */
/* Eq. 14-19 for the active constraints, in the records' (wp, pt) order
   (the step-major order of Eq. 14): c[k] = f_k - delta, and row k of the sparse Jacobian
   nabla_q c = [nabla_{q_i} c_{q_i} P_i] holds the n = 9 gradient entries of record k at
   columns 2 n wp_k + t, t = 0..n-1 (Eq. 19 with the reading of DESIGN.md R18: the
   identity I_n of P_i starts at column 2 n (i - 1) + 1, 1-based, of the 2 N n decision
   variables; trajectory b's block starts at 2 N n b, i.e. wp = b N + i).  CSR: row_ptr[k]
   = n k.  rec_wp[count], rec_f[count], rec_g[count][9]. */
int or_sparse_jacobian(const double *rec_f, const double *rec_g, const int64_t *rec_wp, int64_t count,
                       double delta, double *c, int64_t *row_ptr, int64_t *col, double *val) {
  if (count < 0) return OR_ERR_INVALID;
  for (int64_t k = 0; k < count; ++k) {
    c[k] = rec_f[k] - delta;
    row_ptr[k] = (int64_t)OR_NDOF * k;
    for (int t = 0; t < OR_NDOF; ++t) {
      col[OR_NDOF * k + t] = 2 * (int64_t)OR_NDOF * rec_wp[k] + t;
      val[OR_NDOF * k + t] = rec_g[OR_NDOF * k + t];
    }
  }
  row_ptr[count] = (int64_t)OR_NDOF * count;
  return OR_OK;
}

/* ---------------------------------------------------------------- scene (O2) */
/* The oracle's own replay of the id-assignment rule of gcdf_update_scene
   (include/gcdf.h): removals first; ids freed by this call are not reused by
   the adds of the same call; each add takes the lowest free id. */
typedef struct {
  int64_t cap;
  unsigned char *live;   /* [cap] */
  unsigned char *quar;   /* [cap] freed in the current call */
  double *xyz;           /* [cap][3] */
  int64_t n_live;
} oscene_t;

int or_scene_new(int64_t cap, oscene_t **out) {
  oscene_t *s = (oscene_t *)calloc(1, sizeof(oscene_t));
  if (!s) return OR_ERR_NOMEM;
  s->cap = cap;
  s->live = (unsigned char *)calloc((size_t)cap, 1);
  s->quar = (unsigned char *)calloc((size_t)cap, 1);
  s->xyz = (double *)calloc((size_t)cap * 3, sizeof(double));
  if (!s->live || !s->quar || !s->xyz) { free(s->live); free(s->quar); free(s->xyz); free(s); return OR_ERR_NOMEM; }
  *out = s;
  return OR_OK;
}

void or_scene_free(oscene_t *s) {
  if (!s) return;
  free(s->live); free(s->quar); free(s->xyz); free(s);
}

/* returns OR_ERR_INVALID (scene unchanged) on unknown/duplicate remove id, -7 on capacity. */
int or_scene_update(oscene_t *s, const float *add_xyz, int64_t n_add, int64_t *out_ids,
                    const int64_t *rem, int64_t n_rem) {
  for (int64_t i = 0; i < n_rem; ++i) {
    if (rem[i] < 0 || rem[i] >= s->cap || !s->live[rem[i]]) return OR_ERR_INVALID;
    for (int64_t k = 0; k < i; ++k)
      if (rem[k] == rem[i]) return OR_ERR_INVALID;
  }
  if (s->n_live - n_rem + n_add > s->cap) return -7;
  int64_t free_slots = 0;
  for (int64_t i = 0; i < s->cap; ++i) free_slots += !s->live[i];
  if (free_slots < n_add) return -7;
  for (int64_t i = 0; i < n_rem; ++i) { s->live[rem[i]] = 0; s->quar[rem[i]] = 1; }
  s->n_live -= n_rem;
  int64_t cur = 0;
  for (int64_t a = 0; a < n_add; ++a) {
    while (cur < s->cap && (s->live[cur] || s->quar[cur])) ++cur;
    if (cur >= s->cap) return -7; /* cannot happen for valid inputs when quarantine fits */
    s->live[cur] = 1;
    for (int k = 0; k < 3; ++k) s->xyz[cur * 3 + k] = (double)add_xyz[a * 3 + k];
    out_ids[a] = cur;
    ++s->n_live;
  }
  for (int64_t i = 0; i < n_rem; ++i) s->quar[rem[i]] = 0;
  return OR_OK;
}

/* live points in id order: ids[n_live], xyz[n_live][3] */
int64_t or_scene_export(const oscene_t *s, int64_t *ids, double *xyz) {
  int64_t n = 0;
  for (int64_t i = 0; i < s->cap; ++i)
    if (s->live[i]) {
      if (ids) ids[n] = i;
      if (xyz) memcpy(xyz + 3 * n, s->xyz + 3 * i, 3 * sizeof(double));
      ++n;
    }
  return n;
}
