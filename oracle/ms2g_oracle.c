/*
 * ms2g_oracle.c -- plain, slow, fp64 CPU oracle of the PnP-MS2G hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2203_07308_b200/csrc), and neither side includes the other.
 *
 * Citation keys: P:NN = /root/reference/PAPER.md line NN; S:NN = SPEC.md
 * line NN; SURVEY §8(c) O1..O13 = the readings adopted (listed in DESIGN.md).
 * Every routine follows its definition step by step, in the paper's order,
 * in double precision, with no blocking, fusion or reordering.
 *
 * Pins (tests/test_oracle_*.py): brute-force dense A (oracle/dense.py,
 * independent slab clipping), closed-form chords (uniform square, rectangles,
 * disks/ellipses), adjoint identity, A_s = A U_s, mass conservation of S_s /
 * U_s, finite differences of the LS objective, subset-partition identity,
 * SVD of the dense A, Gaussian closed-form weights, TV 2x2 closed form and
 * duality gap, TV at finite K (K = 1 by hand on a 3x3 impulse; mean,
 * translation / scale covariance, transposition, |u - f| <= 4 lam and the
 * non-increasing dual energy at K = 1, 2, 3, 10), SplitMix64 known answers,
 * CG normal-equation optimum.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t n;          /* image side N (fine grid)                       */
  double fov;         /* physical side W of the square FOV              */
  int32_t n_views;    /* V, views over [0, arc)                         */
  double arc;         /* angular range in radians                       */
  int32_t n_bins;     /* B detector bins                                */
  double sod, sdd;    /* source-to-centre, source-to-detector distances */
  double bin_pitch;   /* detector bin pitch; <= 0 -> (sdd/sod) * fov/n  */
} orc_geom;

/* ------------------------------------------------------------------ O1 --
 * Fan-beam geometry ("90 view equally space from [0,360)", P:152 for
 * a shorter arc; flat detector).
 *   theta_v = arc * v / V
 *   source  s_v = sod * (cos, sin)
 *   detector centre d_v = -(sdd - sod) * (cos, sin), axis e_v = (-sin, cos)
 *   bin t centre p = d_v + u_t e_v, u_t = (t - (B-1)/2) * pitch           */
static double orc_pitch(const orc_geom* g) {
  return g->bin_pitch > 0 ? g->bin_pitch : (g->sdd / g->sod) * g->fov / g->n;
}

void orc_ray_endpoints(const orc_geom* g, int v, int t, double src[2], double det[2]) {
  double th = g->arc * (double)v / (double)g->n_views;
  double c = cos(th), s = sin(th);
  double u = ((double)t - 0.5 * (double)(g->n_bins - 1)) * orc_pitch(g);
  src[0] = g->sod * c;
  src[1] = g->sod * s;
  det[0] = -(g->sdd - g->sod) * c + u * (-s);
  det[1] = -(g->sdd - g->sod) * s + u * c;
}

/* ------------------------------------------------------------------ O2 --
 * Siddon/Jacobs exact radiological path of ray (v,t) on the grid of factor
 * s (n_c = N/s pixels of side W/n_c over the same FOV).  Steps as in
 * parametric ray, slab clip, crossing sets, merge, drop zero
 * lengths, midpoint pixel, length (b-a)*|d|.  Returns the segment count
 * (<= cap written).                                                      */
static int merge_sorted(const double* a, int na, const double* b, int nb, double* out) {
  int i = 0, j = 0, k = 0;
  while (i < na && j < nb) out[k++] = (a[i] <= b[j]) ? a[i++] : b[j++];
  while (i < na) out[k++] = a[i++];
  while (j < nb) out[k++] = b[j++];
  return k;
}

typedef struct { double* ax; double* ay; double* all; } orc_scratch;

static int orc_scratch_init(orc_scratch* sc, int nc) {
  sc->ax = (double*)malloc(sizeof(double) * (nc + 2));
  sc->ay = (double*)malloc(sizeof(double) * (nc + 2));
  sc->all = (double*)malloc(sizeof(double) * (2 * nc + 6));
  return sc->ax && sc->ay && sc->all;
}
static void orc_scratch_free(orc_scratch* sc) { free(sc->ax); free(sc->ay); free(sc->all); }

/* crossing parameters of one plane family, in ascending order, strictly inside (amin, amax) */
static int plane_crossings(double s0, double d0, double origin, double h, int nc,
                           double amin, double amax, double* out) {
  int m = 0;
  if (d0 == 0.0) return 0;          /* plane family skipped when the component is exactly 0 (Z14) */
  for (int k = 0; k <= nc; ++k) {
    double a = (origin + k * h - s0) / d0;
    if (a > amin && a < amax) out[m++] = a;
  }
  if (d0 < 0) {                      /* generated in descending order: reverse */
    for (int i = 0; i < m / 2; ++i) { double tmp = out[i]; out[i] = out[m - 1 - i]; out[m - 1 - i] = tmp; }
  }
  return m;
}

static int orc_siddon(const orc_geom* g, int factor, int v, int t, orc_scratch* sc,
                      int* pix, double* len) {
  int nc = g->n / factor;
  double h = g->fov / nc, lo = -0.5 * g->fov, hi = 0.5 * g->fov;
  double src[2], det[2];
  orc_ray_endpoints(g, v, t, src, det);
  double d[2] = {det[0] - src[0], det[1] - src[1]};
  double dl = sqrt(d[0] * d[0] + d[1] * d[1]);
  /* 2. slab clip to the FOV, alpha in [0,1] */
  double amin = 0.0, amax = 1.0;
  for (int a = 0; a < 2; ++a) {
    if (d[a] == 0.0) {
      if (src[a] < lo || src[a] > hi) return 0;
      continue;
    }
    double a1 = (lo - src[a]) / d[a], a2 = (hi - src[a]) / d[a];
    double mn = a1 < a2 ? a1 : a2, mx = a1 < a2 ? a2 : a1;
    if (mn > amin) amin = mn;
    if (mx < amax) amax = mx;
  }
  if (amin >= amax) return 0;
  /* 3. crossing sets; 4. merge with {amin, amax}, sorted */
  int nx = plane_crossings(src[0], d[0], lo, h, nc, amin, amax, sc->ax);
  int ny = plane_crossings(src[1], d[1], lo, h, nc, amin, amax, sc->ay);
  sc->all[0] = amin;
  int na = 1 + merge_sorted(sc->ax, nx, sc->ay, ny, sc->all + 1);
  sc->all[na++] = amax;
  /* 5. consecutive pairs -> midpoint pixel, length; zero-length dropped */
  int m = 0;
  for (int k = 0; k + 1 < na; ++k) {
    double a0 = sc->all[k], a1 = sc->all[k + 1];
    if (!(a1 - a0 > 0.0)) continue;
    double mid = 0.5 * (a0 + a1);
    double px = src[0] + mid * d[0], py = src[1] + mid * d[1];
    int j = (int)floor((px - lo) / h), i = (int)floor((py - lo) / h);
    if (j < 0) j = 0;
    if (j > nc - 1) j = nc - 1;
    if (i < 0) i = 0;
    if (i > nc - 1) i = nc - 1;
    pix[m] = i * nc + j;
    len[m] = (a1 - a0) * dl;
    ++m;
  }
  return m;
}

/* public: segments of one ray (pix = i*n_c + j, physical lengths) */
int orc_ray_segments(const orc_geom* g, int factor, int v, int t, int* pix, double* len, int cap) {
  int nc = g->n / factor;
  orc_scratch sc;
  if (!orc_scratch_init(&sc, nc)) return -1;
  int* p = (int*)malloc(sizeof(int) * (2 * nc + 6));
  double* l = (double*)malloc(sizeof(double) * (2 * nc + 6));
  int m = orc_siddon(g, factor, v, t, &sc, p, l);
  for (int k = 0; k < m && k < cap; ++k) { pix[k] = p[k]; len[k] = l[k]; }
  free(p); free(l); orc_scratch_free(&sc);
  return m;
}

/* public: one ray sum, O2 step 6 (fp64, ray order) */
double orc_ray_sum(const orc_geom* g, int factor, const double* x, int v, int t) {
  int nc = g->n / factor;
  orc_scratch sc;
  orc_scratch_init(&sc, nc);
  int* p = (int*)malloc(sizeof(int) * (2 * nc + 6));
  double* l = (double*)malloc(sizeof(double) * (2 * nc + 6));
  int m = orc_siddon(g, factor, v, t, &sc, p, l);
  double acc = 0.0;
  for (int k = 0; k < m; ++k) acc += l[k] * x[p[k]];
  free(p); free(l); orc_scratch_free(&sc);
  return acc;
}

/* ----------------------------------------------------- threading helper --
 * Threads own disjoint contiguous ranges of the selected views.   */
typedef struct {
  const orc_geom* g; int factor; const double* x; const double* b; double* out;
  const int* views; int k0, k1; double* img; double scale; long long nnz;
} orc_job;

static void* fwd_worker(void* arg) {
  orc_job* jb = (orc_job*)arg;
  int nc = jb->g->n / jb->factor, B = jb->g->n_bins;
  orc_scratch sc; orc_scratch_init(&sc, nc);
  int* p = (int*)malloc(sizeof(int) * (2 * nc + 6));
  double* l = (double*)malloc(sizeof(double) * (2 * nc + 6));
  for (int k = jb->k0; k < jb->k1; ++k) {
    int v = jb->views ? jb->views[k] : k;
    for (int t = 0; t < B; ++t) {
      int m = orc_siddon(jb->g, jb->factor, v, t, &sc, p, l);
      double acc = 0.0;
      for (int q = 0; q < m; ++q) acc += l[q] * jb->x[p[q]];
      jb->nnz += m;
      /* residual form r = A_s x - b on the selected rows (Eq. 7) */
      if (jb->b) acc -= jb->b[(size_t)v * B + t];
      if (jb->out) jb->out[(size_t)k * B + t] = acc;
    }
  }
  free(p); free(l); orc_scratch_free(&sc);
  return NULL;
}

static void* bwd_worker(void* arg) {
  orc_job* jb = (orc_job*)arg;
  int nc = jb->g->n / jb->factor, B = jb->g->n_bins;
  orc_scratch sc; orc_scratch_init(&sc, nc);
  int* p = (int*)malloc(sizeof(int) * (2 * nc + 6));
  double* l = (double*)malloc(sizeof(double) * (2 * nc + 6));
  for (int k = jb->k0; k < jb->k1; ++k) {
    int v = jb->views ? jb->views[k] : k;
    for (int t = 0; t < B; ++t) {
      double r = jb->x[(size_t)k * B + t];   /* sinogram is compacted [n_sel][B] */
      int m = orc_siddon(jb->g, jb->factor, v, t, &sc, p, l);
      for (int q = 0; q < m; ++q) jb->img[p[q]] += l[q] * r;
    }
  }
  free(p); free(l); orc_scratch_free(&sc);
  return NULL;
}

static int run_jobs(orc_job* proto, int n_sel, int nthreads, void* (*fn)(void*), orc_job** jobs_out) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n_sel) nthreads = n_sel > 0 ? n_sel : 1;
  orc_job* jobs = (orc_job*)calloc(nthreads, sizeof(orc_job));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  for (int r = 0; r < nthreads; ++r) {
    jobs[r] = *proto;
    jobs[r].k0 = (int)((long long)n_sel * r / nthreads);
    jobs[r].k1 = (int)((long long)n_sel * (r + 1) / nthreads);
    jobs[r].nnz = 0;
  }
  for (int r = 0; r < nthreads; ++r) pthread_create(&th[r], NULL, fn, &jobs[r]);
  for (int r = 0; r < nthreads; ++r) pthread_join(th[r], NULL);
  free(th);
  *jobs_out = jobs;
  return nthreads;
}

/* public O2: out[k][t] = (A_s x)[views[k]][t] - b[views[k]][t]  (b may be NULL).
 * views == NULL means all V views (n_sel = V).  Returns nnz visited.      */
long long orc_forward(const orc_geom* g, int factor, const double* x, const double* b,
                      double* out, const int* views, int n_sel, int nthreads) {
  orc_job proto = {g, factor, x, b, out, views, 0, 0, NULL, 1.0, 0};
  orc_job* jobs;
  int nt = run_jobs(&proto, n_sel, nthreads, fwd_worker, &jobs);
  long long nnz = 0;
  for (int r = 0; r < nt; ++r) nnz += jobs[r].nnz;
  free(jobs);
  return nnz;
}

/* public O3: img = scale * A_s^T sino, sino compacted [n_sel][B].
 * Per-thread fp64 images summed in thread-index order.            */
void orc_backward(const orc_geom* g, int factor, const double* sino, double* img, double scale,
                  const int* views, int n_sel, int nthreads) {
  int nc = g->n / factor;
  size_t np = (size_t)nc * nc;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n_sel) nthreads = n_sel > 0 ? n_sel : 1;
  double* part = (double*)calloc(np * nthreads, sizeof(double));
  orc_job* jobs = (orc_job*)calloc(nthreads, sizeof(orc_job));
  pthread_t* th = (pthread_t*)calloc(nthreads, sizeof(pthread_t));
  for (int r = 0; r < nthreads; ++r) {
    orc_job jb = {g, factor, sino, NULL, NULL, views,
                  (int)((long long)n_sel * r / nthreads), (int)((long long)n_sel * (r + 1) / nthreads),
                  part + np * r, 1.0, 0};
    jobs[r] = jb;
  }
  for (int r = 0; r < nthreads; ++r) pthread_create(&th[r], NULL, bwd_worker, &jobs[r]);
  for (int r = 0; r < nthreads; ++r) pthread_join(th[r], NULL);
  for (size_t p = 0; p < np; ++p) {
    double acc = 0.0;
    for (int r = 0; r < nthreads; ++r) acc += part[np * r + p];
    img[p] = scale * acc;
  }
  free(part); free(jobs); free(th);
}

/* public: backprojection at ONE pixel by the plain definition of A^T:
 * (A_s^T r)_j = sum_rays len(R cap pixel_j) r_ray, the length taken by
 * clipping the ray segment against the closed pixel square (slab method).
 * Used for sampled parity at full size.  Same geometry O1.               */
double orc_backward_pixel(const orc_geom* g, int factor, const double* sino, const int* views,
                          int n_sel, int pi, int pj) {
  int nc = g->n / factor, B = g->n_bins;
  double h = g->fov / nc, lo = -0.5 * g->fov;
  double box_lo[2] = {lo + pj * h, lo + pi * h}, box_hi[2] = {lo + (pj + 1) * h, lo + (pi + 1) * h};
  double acc = 0.0;
  for (int k = 0; k < n_sel; ++k) {
    int v = views ? views[k] : k;
    for (int t = 0; t < B; ++t) {
      double src[2], det[2];
      orc_ray_endpoints(g, v, t, src, det);
      double d[2] = {det[0] - src[0], det[1] - src[1]};
      double amin = 0.0, amax = 1.0;
      int miss = 0;
      for (int a = 0; a < 2; ++a) {
        if (d[a] == 0.0) {
          if (src[a] < box_lo[a] || src[a] > box_hi[a]) miss = 1;
          continue;
        }
        double a1 = (box_lo[a] - src[a]) / d[a], a2 = (box_hi[a] - src[a]) / d[a];
        double mn = a1 < a2 ? a1 : a2, mx = a1 < a2 ? a2 : a1;
        if (mn > amin) amin = mn;
        if (mx < amax) amax = mx;
      }
      if (miss || !(amax > amin)) continue;
      acc += (amax - amin) * sqrt(d[0] * d[0] + d[1] * d[1]) * sino[(size_t)k * B + t];
    }
  }
  return acc;
}

/* ------------------------------------------------------------ O4 / O5 --
 * S_s: s x s average pool (north-star D, BASELINE configs "2x2 average
 * pool"); U_s: nearest replication (north-star U^T, Z2).               */
void orc_sketch_down(int n, int s, const double* x, double* v) {
  int nc = n / s;
  for (int I = 0; I < nc; ++I)
    for (int J = 0; J < nc; ++J) {
      double acc = 0.0;
      for (int a = 0; a < s; ++a)
        for (int b = 0; b < s; ++b) acc += x[(size_t)(s * I + a) * n + (s * J + b)];
      v[(size_t)I * nc + J] = acc / ((double)s * s);
    }
}

void orc_sketch_up(int n, int s, const double* gc, double* out) {
  int nc = n / s;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = gc[(size_t)(i / s) * nc + (j / s)];
}

/* --------------------------------------------------------- NEXT-1 bicubic --
 * The paper's own S and U: "MATLAB imresize function with bicubic
 * interpolation" ("bi-cubic interpolation suffice").  Reading
 * (SPEC S:126): Keys cubic convolution, a = -0.5; sample
 * centres aligned (u = (i + 0.5)/scale - 0.5); on downscale the kernel is
 * widened by the factor (antialiasing) and each output's weights are
 * renormalised to sum 1; replicate (clamp) boundary; separable, rows then
 * columns.  scale = 1/s for down, s for up.                                */
double orc_keys(double x) {
  const double a = -0.5;
  double t = fabs(x);
  if (t <= 1.0) return (a + 2.0) * t * t * t - (a + 3.0) * t * t + 1.0;
  if (t < 2.0) return a * t * t * t - 5.0 * a * t * t + 8.0 * a * t - 4.0 * a;
  return 0.0;
}

/* 1-D resample of n_in samples to n_out samples (step `in` apart in memory) */
static void resample_1d(const double* in, int n_in, int in_stride, double* out, int n_out, int out_stride,
                        double scale) {
  double kscale = scale < 1.0 ? scale : 1.0;      /* antialias on downscale */
  double support = 2.0 / kscale;
  for (int i = 0; i < n_out; ++i) {
    double u = (i + 0.5) / scale - 0.5;
    int j0 = (int)floor(u - support), j1 = (int)ceil(u + support);
    double acc = 0.0, wsum = 0.0;
    for (int j = j0; j <= j1; ++j) {
      double w = kscale * orc_keys(kscale * (u - j));
      if (w == 0.0) continue;
      int jc = j < 0 ? 0 : (j > n_in - 1 ? n_in - 1 : j);
      acc += w * in[(size_t)jc * in_stride];
      wsum += w;
    }
    out[(size_t)i * out_stride] = acc / wsum;
  }
}

/* 2-D: rows (along j) then columns (along i) */
static void resample_2d(const double* x, int n_in, double* out, int n_out, double scale) {
  double* tmp = (double*)malloc(sizeof(double) * (size_t)n_in * n_out);
  for (int i = 0; i < n_in; ++i) resample_1d(x + (size_t)i * n_in, n_in, 1, tmp + (size_t)i * n_out, n_out, 1, scale);
  for (int j = 0; j < n_out; ++j) resample_1d(tmp + j, n_in, n_out, out + j, n_out, n_out, scale);
  free(tmp);
}

void orc_bicubic_down(int n, int s, const double* x, double* v) {
  if (s == 1) { memcpy(v, x, sizeof(double) * (size_t)n * n); return; }
  resample_2d(x, n, v, n / s, 1.0 / s);
}

void orc_bicubic_up(int n, int s, const double* gc, double* out) {
  if (s == 1) { memcpy(out, gc, sizeof(double) * (size_t)n * n); return; }
  resample_2d(gc, n / s, out, n, (double)s);
}

/* ------------------------------------------------------------ O6 / O7 --
 * g = c * U_s A_s^T (A_s S_s x - b_M),  c = V/|M|  (Eq. 6,
 * P:95-97 Eq. 7, S:284/S:302 for the V/|M| reading Z7).  views == NULL
 * means all views (Option 1, c = 1).  g is full resolution N^2.          */
/* kind 0: average pool / replication (O4/O5); kind 1: bicubic (NEXT-1) */
void orc_sketched_grad_kind(const orc_geom* g, int factor, int kind, const double* x, const double* b,
                            double* grad, const int* views, int n_sel, int nthreads) {
  int n = g->n, nc = n / factor, V = g->n_views, B = g->n_bins;
  if (!views) n_sel = V;
  double* v = (double*)malloc(sizeof(double) * nc * nc);
  double* r = (double*)malloc(sizeof(double) * (size_t)n_sel * B);
  double* G = (double*)malloc(sizeof(double) * nc * nc);
  if (kind == 1) orc_bicubic_down(n, factor, x, v);        /* v = S(y) */
  else orc_sketch_down(n, factor, x, v);
  orc_forward(g, factor, v, b, r, views, n_sel, nthreads); /* r = A_s v - b */
  orc_backward(g, factor, r, G, (double)V / n_sel, views, n_sel, nthreads); /* G = c A_s^T r */
  if (kind == 1) orc_bicubic_up(n, factor, G, grad);       /* U G */
  else orc_sketch_up(n, factor, G, grad);
  free(v); free(r); free(G);
}

void orc_sketched_grad(const orc_geom* g, int factor, const double* x, const double* b, double* grad,
                       const int* views, int n_sel, int nthreads) {
  orc_sketched_grad_kind(g, factor, 0, x, b, grad, views, n_sel, nthreads);
}

/* ------------------------------------------------------------------ O8 --
 * Step size eta = 1/L ("eta = O(1/L)"; BASELINE configs[0] "L from 20
 * power iterations").  v0 = 1/||1||; w = A_s^T A_s v; L = <v,w>; v = w/||w||.
 * Full view set (Z7).                                                     */
double orc_power_iteration(const orc_geom* g, int factor, int iters, int nthreads) {
  int nc = g->n / factor, V = g->n_views, B = g->n_bins;
  size_t np = (size_t)nc * nc;
  double* v = (double*)malloc(sizeof(double) * np);
  double* w = (double*)malloc(sizeof(double) * np);
  double* s = (double*)malloc(sizeof(double) * (size_t)V * B);
  for (size_t p = 0; p < np; ++p) v[p] = 1.0 / sqrt((double)np);
  double L = 0.0;
  for (int k = 0; k < iters; ++k) {
    orc_forward(g, factor, v, NULL, s, NULL, V, nthreads);
    orc_backward(g, factor, s, w, 1.0, NULL, V, nthreads);
    double dot = 0.0, nrm = 0.0;
    for (size_t p = 0; p < np; ++p) { dot += v[p] * w[p]; nrm += w[p] * w[p]; }
    L = dot;
    nrm = sqrt(nrm);
    for (size_t p = 0; p < np; ++p) v[p] = w[p] / nrm;
  }
  free(v); free(w); free(s);
  return L;
}

/* ------------------------------------------------------------------ O9 --
 * Gaussian denoiser (BASELINE configs[0] "3x3 Gaussian (sigma=0.8)"):
 * separable [w1,w0,w1], w_k ∝ exp(-k^2/(2 sigma^2)) normalised; replicate
 * boundary; rows then columns.                                   */
static int clampi(int a, int lo, int hi) { return a < lo ? lo : (a > hi ? hi : a); }

void orc_gauss3_weights(double sigma, double w[3]) {
  double e = exp(-1.0 / (2.0 * sigma * sigma));
  double z = 1.0 + 2.0 * e;
  w[0] = e / z; w[1] = 1.0 / z; w[2] = e / z;
}

void orc_gauss3(int n, double sigma, const double* z, double* out) {
  double w[3];
  orc_gauss3_weights(sigma, w);
  double* tmp = (double*)malloc(sizeof(double) * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int b = -1; b <= 1; ++b) acc += w[b + 1] * z[(size_t)i * n + clampi(j + b, 0, n - 1)];
      tmp[(size_t)i * n + j] = acc;
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int a = -1; a <= 1; ++a) acc += w[a + 1] * tmp[(size_t)clampi(i + a, 0, n - 1) * n + j];
      out[(size_t)i * n + j] = acc;
    }
  free(tmp);
}

/* TV-prox by Chambolle's 2004 dual fixed point ("TV-prox"; north star
 * "Chambolle TV-prox iterations"; reading Z18).  Forward differences with
 * zero last row/column (Neumann); div = -grad^T.  p^0 = 0,
 *   q = grad(div p^n - f/lambda),  p^{n+1} = (p^n + tau q)/(1 + tau |q|),
 *   u = f - lambda div p^K.
 * p layout: p[0..n^2) = x-component (along columns j), p[n^2..2n^2) = y.  */
void orc_grad(int n, const double* u, double* gx, double* gy) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      size_t q = (size_t)i * n + j;
      gx[q] = (j < n - 1) ? u[q + 1] - u[q] : 0.0;
      gy[q] = (i < n - 1) ? u[q + n] - u[q] : 0.0;
    }
}

void orc_div(int n, const double* px, const double* py, double* d) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      size_t q = (size_t)i * n + j;
      double a = (j < n - 1 ? px[q] : 0.0) - (j > 0 ? px[q - 1] : 0.0);
      double b = (i < n - 1 ? py[q] : 0.0) - (i > 0 ? py[q - n] : 0.0);
      d[q] = a + b;
    }
}

void orc_tv_chambolle(int n, double lambda, double tau, int iters, const double* f, double* u,
                      double* p_out) {
  size_t np = (size_t)n * n;
  if (lambda == 0.0) {             /* prox of the zero function: identity */
    memcpy(u, f, sizeof(double) * np);
    if (p_out) memset(p_out, 0, sizeof(double) * 2 * np);
    return;
  }
  double* px = (double*)calloc(np, sizeof(double));
  double* py = (double*)calloc(np, sizeof(double));
  double* d = (double*)malloc(sizeof(double) * np);
  double* qx = (double*)malloc(sizeof(double) * np);
  double* qy = (double*)malloc(sizeof(double) * np);
  for (int it = 0; it < iters; ++it) {
    orc_div(n, px, py, d);
    for (size_t q = 0; q < np; ++q) d[q] -= f[q] / lambda;
    orc_grad(n, d, qx, qy);
    for (size_t q = 0; q < np; ++q) {
      double nq = sqrt(qx[q] * qx[q] + qy[q] * qy[q]);
      px[q] = (px[q] + tau * qx[q]) / (1.0 + tau * nq);
      py[q] = (py[q] + tau * qy[q]) / (1.0 + tau * nq);
    }
  }
  orc_div(n, px, py, d);
  for (size_t q = 0; q < np; ++q) u[q] = f[q] - lambda * d[q];
  if (p_out) { memcpy(p_out, px, sizeof(double) * np); memcpy(p_out + np, py, sizeof(double) * np); }
  free(px); free(py); free(d); free(qx); free(qy);
}

/* ------------------------------------------------------------------ O13 --
 * Schedule: SplitMix64 stream (one per solve, seeded with `seed`), and a
 * Fisher-Yates shuffle of [0..n_subsets-1] per epoch ("randomly
 * sampled minibatch", "uniformly sampled"; readings Z8, Z9).        */
uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z;
  *state += 0x9E3779B97F4A7C15ULL;
  z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

typedef struct { int32_t factor, n_iters, n_epochs; } orc_stage;
typedef struct { int32_t i, stage, factor, subset; double eta, a; } orc_sched_entry;

/* momentum a_i = (i-1)/(i+3) ("convergent FISTA"); i is the global
 * 1-based counter of the iterate just produced (reading Z4).       */
double orc_momentum(int i) { return (double)(i - 1) / (double)(i + 3); }

/* Fills entries (eta left 0); returns the number of steps, or -1 on a bad
 * description.  Option 1: N_k steps of the full view set (subset -1).
 * Option 2: n_epochs_k epochs of n_subsets steps, subset order per epoch a
 * Fisher-Yates shuffle of the identity [0..n_subsets-1].                  */
int orc_schedule(const orc_stage* st, int n_stages, int option, int n_subsets, uint64_t seed,
                 orc_sched_entry* out, int cap) {
  uint64_t state = seed;
  int i = 0;
  int* perm = (int*)malloc(sizeof(int) * (n_subsets > 0 ? n_subsets : 1));
  for (int k = 0; k < n_stages; ++k) {
    if (option == 1 || option == 4) {
      for (int j = 0; j < st[k].n_iters; ++j) {
        ++i;
        if (i <= cap) {
          orc_sched_entry e = {i, k, st[k].factor, option == 4 ? i - 1 : -1, 0.0, orc_momentum(i)};
          out[i - 1] = e;
        }
      }
    } else if (option == 2 || option == 3 || option == 5) {   /* 3 SVRG, 5 SAGA: same subset schedule */
      if (n_subsets < 1) { free(perm); return -1; }
      for (int ep = 0; ep < st[k].n_epochs; ++ep) {
        for (int q = 0; q < n_subsets; ++q) perm[q] = q;
        for (int q = n_subsets - 1; q >= 1; --q) {
          int j = (int)(orc_splitmix64(&state) % (uint64_t)(q + 1));
          int tmp = perm[q]; perm[q] = perm[j]; perm[j] = tmp;
        }
        for (int q = 0; q < n_subsets; ++q) {
          ++i;
          if (i <= cap) {
            orc_sched_entry e = {i, k, st[k].factor, perm[q], 0.0, orc_momentum(i)};
            out[i - 1] = e;
          }
        }
      }
    } else {
      free(perm);
      return -1;
    }
  }
  free(perm);
  return i;
}

/* Option 4 (NEXT-4; "M_i is a randomly sampled minibatch", P:98
 * "uniformly sampled minibatch"): every step draws m distinct
 * views uniformly without replacement -- a partial Fisher-Yates shuffle of
 * [0..V-1] (for q < m: j = q + next() mod (V - q), swap) driven by one
 * SplitMix64 stream seeded with `seed` -- and uses them in ascending order.
 * out receives n_steps * m view indices, step-major.                       */
static int cmp_int(const void* a, const void* b) { return (*(const int*)a > *(const int*)b) - (*(const int*)a < *(const int*)b); }

int orc_minibatch_views(int V, int m, uint64_t seed, int n_steps, int* out) {
  if (m < 1 || m > V) return -1;
  uint64_t state = seed;
  int* arr = (int*)malloc(sizeof(int) * V);
  for (int st = 0; st < n_steps; ++st) {
    for (int q = 0; q < V; ++q) arr[q] = q;
    for (int q = 0; q < m; ++q) {
      int j = q + (int)(orc_splitmix64(&state) % (uint64_t)(V - q));
      int tmp = arr[q]; arr[q] = arr[j]; arr[j] = tmp;
    }
    qsort(arr, m, sizeof(int), cmp_int);
    memcpy(out + (size_t)st * m, arr, sizeof(int) * m);
  }
  free(arr);
  return 0;
}

/* subset k = { v : v mod n_subsets == k }  ("8 interleaved subsets") */
int orc_subset_views(int n_views, int n_subsets, int k, int* out) {
  int m = 0;
  for (int v = 0; v < n_views; ++v)
    if (v % n_subsets == k) out[m++] = v;
  return m;
}

/* ------------------------------------------------------------------ O11 --
 * Algorithm 1 with the readings of SURVEY O11:
 *   x0 = y0 (given), x_prev = x0, i = 0
 *   for stage k: eta_k = 1/L_20(A_{s_k});  repeat N_k:
 *     i += 1; v = S(y); G = grad (Opt. 1 / Opt. 2); z = y - eta U G;
 *     x = (1-alpha) z + alpha D(z); y = x + a_i (x - x_prev); x_prev = x
 * den_kind: 0 identity, 1 gauss3 (sigma), 2 TV-Chambolle (lambda, tau, iters).
 * Returns 0, or 3 with *bad_i set when an iterate is non-finite.  */
static int g_resampler = 0;
void orc_set_resampler(int kind) { g_resampler = kind; }

int orc_pnp_ms2g(const orc_geom* g, const orc_stage* st, int n_stages, int option, int n_subsets,
                 uint64_t seed, int den_kind, double sigma, double lambda, double tau, int den_iters,
                 double alpha, int power_iters, const double* b, const double* x0, double* x_out,
                 orc_sched_entry* trace, double* etas, int nthreads, int* bad_i) {
  int n = g->n, V = g->n_views;
  size_t np = (size_t)n * n;
  int total = orc_schedule(st, n_stages, option, n_subsets, seed, NULL, 0);
  if (total < 0) return 2;
  orc_sched_entry* sch = (orc_sched_entry*)malloc(sizeof(orc_sched_entry) * (total > 0 ? total : 1));
  orc_schedule(st, n_stages, option, n_subsets, seed, sch, total);
  double* x = (double*)malloc(sizeof(double) * np);
  double* xp = (double*)malloc(sizeof(double) * np);
  double* y = (double*)malloc(sizeof(double) * np);
  double* gr = (double*)malloc(sizeof(double) * np);
  double* z = (double*)malloc(sizeof(double) * np);
  double* dz = (double*)malloc(sizeof(double) * np);
  int* views = (int*)malloc(sizeof(int) * V);
  /* Option 3 (NEXT-4, "stochastic variance-reduced gradient estimator",
   * SVRG): at the start of every epoch the snapshot xs = y and its full
   * sketched gradient mu = g_s(xs) are taken; a step on subset M uses
   *   G = (V/|M|) U A_{s,M}^T A_{s,M} S (y - xs) + mu
   * (= the SVRG estimator g_M(y) - g_M(xs) + g(xs) of the quadratic). */
  double* xs = (option == 3) ? (double*)malloc(sizeof(double) * np) : NULL;
  double* mu = (option == 3) ? (double*)malloc(sizeof(double) * np) : NULL;
  double* dd = (option == 3) ? (double*)malloc(sizeof(double) * np) : NULL;
  double* zero = (option == 3) ? (double*)calloc((size_t)V * g->n_bins, sizeof(double)) : NULL;
  /* Option 5 (NEXT-4, "SAGA"): table phi_k of the scaled subset
   * gradients g_k = (V/|M_k|) U A_{s,M_k}^T (A_{s,M_k} S y - b_{M_k}), filled
   * at every stage start with all K subsets at the current y; a step on
   * subset j with new = g_j(y) uses G = new - phi_j + mean_k phi_k and then
   * stores phi_j = new.                                                    */
  double* phi = (option == 5) ? (double*)malloc(sizeof(double) * np * (size_t)n_subsets) : NULL;
  double* pavg = (option == 5) ? (double*)malloc(sizeof(double) * np) : NULL;
  /* Option 4: n_subsets carries the minibatch size m (views per step) */
  int* mb = NULL;
  if (option == 4) {
    mb = (int*)malloc(sizeof(int) * (size_t)(total > 0 ? total : 1) * n_subsets);
    if (orc_minibatch_views(V, n_subsets, seed, total, mb) != 0) { free(mb); free(sch); return 2; }
  }
  memcpy(x, x0, sizeof(double) * np);
  memcpy(xp, x0, sizeof(double) * np);
  memcpy(y, x0, sizeof(double) * np);
  int rc = 0, step = 0;
  for (int k = 0; k < n_stages && rc == 0; ++k) {
    double L = orc_power_iteration(g, st[k].factor, power_iters, nthreads);
    double eta = 1.0 / L;
    if (etas) etas[k] = eta;
    int nk = (option == 1 || option == 4) ? st[k].n_iters : st[k].n_epochs * n_subsets;
    if (option == 5 && nk > 0) {              /* SAGA table at the stage start */
      for (size_t p = 0; p < np; ++p) pavg[p] = 0.0;
      for (int q = 0; q < n_subsets; ++q) {
        int m = orc_subset_views(V, n_subsets, q, views);
        double* ph = phi + np * (size_t)q;
        orc_sketched_grad_kind(g, st[k].factor, g_resampler, y, b, ph, views, m, nthreads);
        for (size_t p = 0; p < np; ++p) pavg[p] += ph[p] / n_subsets;
      }
    }
    for (int j = 0; j < nk; ++j, ++step) {
      orc_sched_entry e = sch[step];
      int i = e.i;
      if (e.subset < 0) {
        orc_sketched_grad_kind(g, e.factor, g_resampler, y, b, gr, NULL, V, nthreads);
      } else if (option == 4) {
        orc_sketched_grad_kind(g, e.factor, g_resampler, y, b, gr, mb + (size_t)step * n_subsets, n_subsets,
                               nthreads);
      } else if (option == 5) {
        int m = orc_subset_views(V, n_subsets, e.subset, views);
        double* ph = phi + np * (size_t)e.subset;
        orc_sketched_grad_kind(g, e.factor, g_resampler, y, b, gr, views, m, nthreads);   /* new */
        for (size_t p = 0; p < np; ++p) {
          double d = gr[p] - ph[p];
          ph[p] = gr[p];
          gr[p] = d + pavg[p];
          pavg[p] += d / n_subsets;
        }
      } else if (option == 3) {
        if (j % n_subsets == 0) {                    /* epoch start: snapshot */
          memcpy(xs, y, sizeof(double) * np);
          orc_sketched_grad_kind(g, e.factor, g_resampler, xs, b, mu, NULL, V, nthreads);
        }
        for (size_t p = 0; p < np; ++p) dd[p] = y[p] - xs[p];
        int m = orc_subset_views(V, n_subsets, e.subset, views);
        orc_sketched_grad_kind(g, e.factor, g_resampler, dd, zero, gr, views, m, nthreads);
        for (size_t p = 0; p < np; ++p) gr[p] += mu[p];
      } else {
        int m = orc_subset_views(V, n_subsets, e.subset, views);
        orc_sketched_grad_kind(g, e.factor, g_resampler, y, b, gr, views, m, nthreads);
      }
      for (size_t p = 0; p < np; ++p) z[p] = y[p] - eta * gr[p];
      if (den_kind == 1) orc_gauss3(n, sigma, z, dz);
      else if (den_kind == 2) orc_tv_chambolle(n, lambda, tau, den_iters, z, dz, NULL);
      else memcpy(dz, z, sizeof(double) * np);
      double a = orc_momentum(i);
      int finite = 1;
      for (size_t p = 0; p < np; ++p) {
        double xn = (1.0 - alpha) * z[p] + alpha * dz[p];
        y[p] = xn + a * (xn - xp[p]);
        x[p] = xn;
        if (!isfinite(xn) || !isfinite(y[p])) finite = 0;
      }
      memcpy(xp, x, sizeof(double) * np);
      e.eta = eta;
      if (trace) trace[step] = e;
      if (!finite) { rc = 3; if (bad_i) *bad_i = i; break; }
    }
  }
  memcpy(x_out, x, sizeof(double) * np);
  free(sch); free(x); free(xp); free(y); free(gr); free(z); free(dz); free(views);
  free(xs); free(mu); free(dd); free(zero); free(mb); free(phi); free(pavg);
  return rc;
}
