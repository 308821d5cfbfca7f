// image_ops.cu -- streaming kernels of the PnP-MS2G step (sm_100a):
//   sketch S_s (+ transposed copy for the projector), upsample+step,
//   Gaussian / TV-prox denoisers fused with the RED-PRO mix and the FISTA
//   momentum, and the fp64 reductions of the power iteration.
// These are HBM/L2-streaming kernels; one thread per
// output pixel, coalesced along rows, 32x32 shared tiles for transposes.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace ms2g {

// Pixel kernels run on a (32 x 8)-thread block over a (columns, rows, batch)
// grid: the pixel comes from the block/thread indices, no index division
// (64-bit / and % of a flat index cost more than the pixel's arithmetic).
static inline dim3 px_grid(int cols, int rows, int batch) {
  return dim3((unsigned)((cols + 31) / 32), (unsigned)((rows + 7) / 8), (unsigned)batch);
}
static const dim3 kPxBlock(32, 8);
#define PIXEL_IJB(rows, cols)                              \
  const int j = blockIdx.x * 32 + threadIdx.x;             \
  const int i = blockIdx.y * 8 + threadIdx.y;              \
  const size_t b = blockIdx.z;                             \
  if (i >= (rows) || j >= (cols)) return

static inline int grid1d(size_t total, int block = 256, int cap = 148 * 32) {
  size_t g = (total + block - 1) / block;
  if (g > (size_t)cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

// -------------------------------------------------------------- sketch --
// S_s: s x s average pool (north-star D; BASELINE configs "2x2 average pool").
__global__ void k_sketch_down(const float* __restrict__ x, float* __restrict__ v, int n, int s, int nc) {
  PIXEL_IJB(nc, nc);
  const float inv = 1.0f / (float)(s * s);
  const float* xb = x + b * n * n;
  float acc = 0.f;
  for (int a = 0; a < s; ++a) {
    const float* row = xb + (size_t)(s * i + a) * n + (size_t)s * j;
    for (int c = 0; c < s; ++c) acc += row[c];
  }
  v[(b * nc + i) * nc + j] = (s == 1) ? acc : acc * inv;
}

int launch_sketch_down(int n, int s, int batch, const float* x, float* v, cudaStream_t st) {
  const int nc = n / s;
  k_sketch_down<<<px_grid(nc, nc, batch), kPxBlock, 0, st>>>(x, v, n, s, nc);
  return check_launch("k_sketch_down");
}

// ---------------------------------------------------------- upsample+step --
// z = y - eta * U_s g, U_s = nearest replication (reading Z2).
__global__ void k_up_step(const float* __restrict__ g, const float* __restrict__ y,
                          const float* __restrict__ eta_dev, float eta, float* __restrict__ z, int n, int s,
                          int nc) {
  PIXEL_IJB(n, n);
  const float e = eta_dev ? *eta_dev : eta;
  const size_t idx = (b * n + i) * n + j;
  const float gv = g[(b * nc + i / s) * nc + (j / s)];
  z[idx] = y ? fmaf(-e, gv, y[idx]) : gv;   // y - eta G with one rounding (as k_reduce_up_step)
}

int launch_up_step(int n, int s, int batch, const float* g, const float* y, const float* eta_dev, float eta,
                   float* z, cudaStream_t st) {
  k_up_step<<<px_grid(n, n, batch), kPxBlock, 0, st>>>(g, y, eta_dev, eta, z, n, s, n / s);
  return check_launch("k_up_step");
}

// ------------------------------------------------------ bicubic (NEXT-1) --
// The paper's S and U: MATLAB imresize, bicubic.  Keys cubic
// convolution a = -0.5, centre-aligned samples u = (i + 0.5)/scale - 0.5,
// kernel widened by the factor on downscale (antialiasing) with per-output
// renormalisation, clamped boundary; separable (rows then columns).  The
// per-output taps are tabulated on the host in fp64 once per plan.
static double keys_cubic(double x) {
  const double a = -0.5;
  const double t = std::fabs(x);
  if (t <= 1.0) return (a + 2.0) * t * t * t - (a + 3.0) * t * t + 1.0;
  if (t < 2.0) return a * t * t * t - 5.0 * a * t * t + 8.0 * a * t - 4.0 * a;
  return 0.0;
}

static void bicubic_table(int n_in, int n_out, double scale, int& taps, std::vector<int>& idx,
                          std::vector<float>& w) {
  const double ks = scale < 1.0 ? scale : 1.0;
  const double support = 2.0 / ks;
  taps = (int)std::ceil(2.0 * support) + 2;
  idx.assign((size_t)n_out * taps, 0);
  w.assign((size_t)n_out * taps, 0.f);
  for (int o = 0; o < n_out; ++o) {
    const double u = (o + 0.5) / scale - 0.5;
    const int j0 = (int)std::floor(u - support);
    std::vector<double> ww(taps, 0.0);
    double sum = 0.0;
    for (int k = 0; k < taps; ++k) {
      const int j = j0 + k;
      ww[k] = ks * keys_cubic(ks * (u - j));
      sum += ww[k];
      idx[(size_t)o * taps + k] = j < 0 ? 0 : (j > n_in - 1 ? n_in - 1 : j);
    }
    for (int k = 0; k < taps; ++k) w[(size_t)o * taps + k] = (float)(ww[k] / sum);
  }
}

int build_bicubic_tables(FactorTables& f, int n) {
  if (f.factor == 1) return MS2G_OK;
  std::vector<int> idx;
  std::vector<float> w;
  bicubic_table(n, f.nc, 1.0 / f.factor, f.taps_down, idx, w);
  MS2G_CUDA(cudaMalloc(&f.d_idx_down, sizeof(int) * idx.size()));
  MS2G_CUDA(cudaMalloc(&f.d_w_down, sizeof(float) * w.size()));
  MS2G_CUDA(cudaMemcpy(f.d_idx_down, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
  MS2G_CUDA(cudaMemcpy(f.d_w_down, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice));
  bicubic_table(f.nc, n, (double)f.factor, f.taps_up, idx, w);
  MS2G_CUDA(cudaMalloc(&f.d_idx_up, sizeof(int) * idx.size()));
  MS2G_CUDA(cudaMalloc(&f.d_w_up, sizeof(float) * w.size()));
  MS2G_CUDA(cudaMemcpy(f.d_idx_up, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice));
  MS2G_CUDA(cudaMemcpy(f.d_w_up, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice));
  return MS2G_OK;
}

// rows pass: out[b][r][o] = sum_t w[o][t] in[b][r][idx[o][t]]   (rows x n_in -> rows x n_out)
__global__ void k_rs_rows(const float* __restrict__ in, float* __restrict__ out, int rows, int n_in, int n_out,
                          int taps, const int* __restrict__ idx, const float* __restrict__ w) {
  PIXEL_IJB(rows, n_out);                      // i = input row r, j = output sample o
  const float* row = in + (b * rows + i) * n_in;
  float acc = 0.f;
  for (int t = 0; t < taps; ++t) acc = fmaf(__ldg(w + j * taps + t), row[__ldg(idx + j * taps + t)], acc);
  out[(b * rows + i) * n_out + j] = acc;
}

// columns pass: val = sum_t w[o][t] in[b][idx[o][t]][c]; z = y - eta val (y != NULL) or val
__global__ void k_rs_cols(const float* __restrict__ in, float* __restrict__ out, int cols, int n_in, int n_out,
                          int taps, const int* __restrict__ idx, const float* __restrict__ w,
                          const float* __restrict__ y, const float* __restrict__ eta_dev, float eta) {
  PIXEL_IJB(n_out, cols);                      // i = output row o, j = column c
  const float e_ = eta_dev ? *eta_dev : eta;
  const float* base = in + b * (size_t)n_in * cols + j;
  float acc = 0.f;
  for (int t = 0; t < taps; ++t)
    acc = fmaf(__ldg(w + i * taps + t), base[(size_t)__ldg(idx + i * taps + t) * cols], acc);
  const size_t e = (b * n_out + i) * cols + j;
  out[e] = y ? y[e] - e_ * acc : acc;
}

int launch_resample_down(ms2g_plan* p, const FactorTables& f, int kind, int batch, const float* x, float* v,
                         cudaStream_t st) {
  const int n = p->d.n;
  if (kind == 0 || f.factor == 1) return launch_sketch_down(n, f.factor, batch, x, v, st);
  k_rs_rows<<<px_grid(f.nc, n, batch), kPxBlock, 0, st>>>(x, p->w_rs, n, n, f.nc, f.taps_down, f.d_idx_down,
                                                          f.d_w_down);
  MS2G_TRY(check_launch("k_rs_rows"));
  k_rs_cols<<<px_grid(f.nc, f.nc, batch), kPxBlock, 0, st>>>(p->w_rs, v, f.nc, n, f.nc, f.taps_down, f.d_idx_down,
                                                             f.d_w_down, nullptr, nullptr, 0.f);
  return check_launch("k_rs_cols");
}

int launch_resample_up_step(ms2g_plan* p, const FactorTables& f, int kind, int batch, const float* g,
                            const float* y, const float* eta_dev, float eta, float* z, cudaStream_t st) {
  const int n = p->d.n;
  if (kind == 0 || f.factor == 1) return launch_up_step(n, f.factor, batch, g, y, eta_dev, eta, z, st);
  k_rs_rows<<<px_grid(n, f.nc, batch), kPxBlock, 0, st>>>(g, p->w_rs, f.nc, f.nc, n, f.taps_up, f.d_idx_up,
                                                          f.d_w_up);
  MS2G_TRY(check_launch("k_rs_rows"));
  k_rs_cols<<<px_grid(n, n, batch), kPxBlock, 0, st>>>(p->w_rs, z, n, f.nc, n, f.taps_up, f.d_idx_up, f.d_w_up, y,
                                                       eta_dev, eta);
  return check_launch("k_rs_cols");
}

// --------------------------------------------------- mix + momentum core --
// x = (1-alpha) z + alpha D(z);  y = x + a (x - x_prev);
// a non-finite x or y records the global iteration in *flag.
__device__ __forceinline__ void mix_momentum(size_t idx, float zv, float dv, const float* __restrict__ xprev,
                                             float* __restrict__ xout, float* __restrict__ yout, float alpha,
                                             float a, int mode, int* flag, int iter) {
  if (mode == 0) {  // plain denoiser output
    xout[idx] = dv;
    return;
  }
  const float xv = (1.f - alpha) * zv + alpha * dv;
  const float yv = xv + a * (xv - xprev[idx]);
  xout[idx] = xv;
  yout[idx] = yv;
  if (!isfinite(xv) || !isfinite(yv)) atomicMin(flag, iter);
}

// Gaussian 3x3 (BASELINE configs[0], sigma = 0.8): separable [w1, w0, w1],
// replicate boundary, rows then columns.
__global__ void k_gauss_mm(const float* __restrict__ z, const float* __restrict__ xprev, float* __restrict__ xout,
                           float* __restrict__ yout, int n, float w0, float w1, float alpha, float a, int mode,
                           int* flag, int iter) {
  pdl_wait();
  pdl_release();
  PIXEL_IJB(n, n);
  const size_t np = (size_t)n * n;
  const float* zb = z + b * np;
  const int jl = max(j - 1, 0), jr = min(j + 1, n - 1);
  float t[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int r = min(max(i + q - 1, 0), n - 1);
    const float* row = zb + (size_t)r * n;
    t[q] = w1 * row[jl] + w0 * row[j] + w1 * row[jr];
  }
  const float dv = w1 * t[0] + w0 * t[1] + w1 * t[2];
  const size_t p = (size_t)i * n + j;
  mix_momentum(b * np + p, zb[p], dv, xprev, xout, yout, alpha, a, mode, flag, iter);
}

int launch_gauss_mix_mom(int n, int batch, float sigma, const float* z, const float* xprev, float* xout,
                         float* yout, float alpha, float a, int mode, int* flag, int iter, cudaStream_t st) {
  const double e = exp(-1.0 / (2.0 * (double)sigma * (double)sigma));
  const float w1 = (float)(e / (1.0 + 2.0 * e)), w0 = (float)(1.0 / (1.0 + 2.0 * e));
  MS2G_CUDA(launch_k(k_gauss_mm, px_grid(n, n, batch), kPxBlock, 0, st, z, xprev, xout, yout, n, w0, w1, alpha, a,
                     mode, flag, iter));
  return check_launch("k_gauss_mm");
}

__global__ void k_copy_mm(const float* __restrict__ z, const float* __restrict__ xprev, float* __restrict__ xout,
                          float* __restrict__ yout, float a, int mode, int* flag, int iter, size_t total) {
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const float zv = z[idx];
    mix_momentum(idx, zv, zv, xprev, xout, yout, 1.f, a, mode, flag, iter);
  }
}

int launch_copy_mix_mom(int n, int batch, const float* z, const float* xprev, float* xout, float* yout, float a,
                        int mode, int* flag, int iter, cudaStream_t st) {
  const size_t total = (size_t)n * n * batch;
  k_copy_mm<<<grid1d(total), 256, 0, st>>>(z, xprev, xout, yout, a, mode, flag, iter, total);
  return check_launch("k_copy_mm");
}

// ------------------------------------------------------------- TV-prox --
// Chambolle 2004 dual fixed point ("TV-prox"; reading Z18):
//   w = div p - f/lambda,  q = grad w,  p <- (p + tau q) / (1 + tau |q|),
//   u = f - lambda div p.  Forward differences, zero last row/column.
// p layout: [batch][2][n][n] (x-component, then y-component).
__device__ __forceinline__ float tv_div(const float* __restrict__ px, const float* __restrict__ py, int n, int i,
                                        int j) {
  const size_t q = (size_t)i * n + j;
  const float a = (j < n - 1 ? px[q] : 0.f) - (j > 0 ? px[q - 1] : 0.f);
  const float b = (i < n - 1 ? py[q] : 0.f) - (i > 0 ? py[q - n] : 0.f);
  return a + b;
}

// The per-point arithmetic of every TV-prox form, in one explicit order (no
// compiler contraction choices), so that all forms produce the same bits:
//   w = d - f / lambda  (d = div p, 0 at p^0 = 0)
//   p' = (p + tau q) / (1 + tau |q|)  with the MUFU square root / reciprocal
//   u = f - lambda div p
__device__ __forceinline__ float tv_w(float d, float f, float inv_lambda) { return fmaf(-f, inv_lambda, d); }
__device__ __forceinline__ float tv_rden(float qx, float qy, float tau) {
  float sq, rden;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(sq) : "f"(fmaf(qy, qy, qx * qx)));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rden) : "f"(fmaf(tau, sq, 1.f)));
  return rden;
}
__device__ __forceinline__ float tv_p(float p, float q, float tau, float rden) { return fmaf(tau, q, p) * rden; }
__device__ __forceinline__ float tv_u(float f, float div, float lambda) { return fmaf(-lambda, div, f); }

// One dual iteration.  The block's 32 x 8 pixels need w = div p - f / lambda
// on themselves and one column / row beyond: w is formed once per point into
// a (8+1) x (32+1) shared tile (instead of three times per pixel), then
// q = grad w and the p update.  first != 0: p^0 = 0 (no warm start, pin not
// read), so w = -f / lambda.
// The TV chain is launched with programmatic dependent launch (launch_k,
// internal.cuh): each of the K + 1 kernels reads what does not depend on its
// predecessor (f = z, written before the chain) before griddepcontrol.wait.
bool pdl_enabled() {
  static const bool on = !(getenv("MS2G_PDL") && atoi(getenv("MS2G_PDL")) == 0);   // experiment switch
  return on;
}

__global__ void __launch_bounds__(256) k_tv_iter(const float* __restrict__ f, const float* __restrict__ pin,
                                                 float* __restrict__ pout, int n, float inv_lambda, float tau,
                                                 int first) {
  __shared__ float sw[9][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 8;
  const size_t b = blockIdx.z, np = (size_t)n * n;
  const float* fb = f + b * np;
  const float* px = pin + b * 2 * np;
  const float* py = px + np;
  // the <= 2 tile entries of this thread: f first (unless this is the first
  // iteration, whose predecessor produced f)
  float fe[2] = {0.f, 0.f};
  if (!first) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int e = ty * 32 + tx + 256 * k;
      if (e >= 9 * 33) break;
      const int gi = i0 + e / 33, gj = j0 + e % 33;
      if (gi < n && gj < n) fe[k] = fb[(size_t)gi * n + gj];
    }
  }
  pdl_wait();
  pdl_release();
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = ty * 32 + tx + 256 * k;
    if (e >= 9 * 33) break;
    const int li = e / 33, lj = e % 33, gi = i0 + li, gj = j0 + lj;
    float w = 0.f;
    if (gi < n && gj < n) {
      const size_t q = (size_t)gi * n + gj;
      const float fq = first ? fb[q] : fe[k];
      w = tv_w(first ? 0.f : tv_div(px, py, n, gi, gj), fq, inv_lambda);
    }
    sw[li][lj] = w;
  }
  __syncthreads();
  const int i = i0 + ty, j = j0 + tx;
  if (i >= n || j >= n) return;
  const size_t p = (size_t)i * n + j;
  const float wc = sw[ty][tx];
  const float qx = (j < n - 1) ? sw[ty][tx + 1] - wc : 0.f;
  const float qy = (i < n - 1) ? sw[ty + 1][tx] - wc : 0.f;
  // 1 / (1 + tau |q|) with the MUFU square root and reciprocal (relative error
  // ~1e-7 per call, far inside the 1e-5 operator gate; the geometry is exact)
  const float rden = tv_rden(qx, qy, tau);
  float* ox = pout + b * 2 * np;
  ox[p] = tv_p(first ? 0.f : px[p], qx, tau, rden);
  ox[np + p] = tv_p(first ? 0.f : py[p], qy, tau, rden);
}
__global__ void k_tv_final(const float* __restrict__ f, const float* __restrict__ pin,
                           const float* __restrict__ xprev, float* __restrict__ xout, float* __restrict__ yout,
                           int n, float lambda, float alpha, float a, int mode, int* flag, int iter) {
  const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
  const size_t b = blockIdx.z;
  const bool in = i < n && j < n;
  const size_t np = (size_t)n * n, idx = b * np + (size_t)i * n + j;
  const float* px = pin + b * 2 * np;
  const float fv = in ? f[idx] : 0.f;     // f precedes the TV chain (PDL: read before the wait)
  pdl_wait();
  pdl_release();
  if (!in) return;
  const float u = tv_u(fv, tv_div(px, px + np, n, i, j), lambda);
  mix_momentum(idx, fv, u, xprev, xout, yout, alpha, a, mode, flag, iter);
}

// out = a x + b y  (SVRG difference / correction, NEXT-4)
__global__ void k_axpby(float* __restrict__ out, const float* __restrict__ x, const float* __restrict__ y, float a,
                        float b, size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    out[i] = a * x[i] + b * y[i];
}

int launch_axpby(float* out, const float* x, const float* y, float a, float b, size_t count, cudaStream_t st) {
  k_axpby<<<grid1d(count), 256, 0, st>>>(out, x, y, a, b, count);
  return check_launch("k_axpby");
}

// SAGA update (NEXT-4, Option 5): d = new - phi_j; phi_j = new;
// G = d + avg (into `nw`); avg += d / K
__global__ void k_saga(float* __restrict__ nw, float* __restrict__ phi, float* __restrict__ avg, float invK,
                       size_t count) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const float n_ = nw[i], d = n_ - phi[i];
    phi[i] = n_;
    nw[i] = d + avg[i];
    avg[i] += d * invK;
  }
}

int launch_saga(float* nw, float* phi, float* avg, int K, size_t count, cudaStream_t st) {
  k_saga<<<grid1d(count), 256, 0, st>>>(nw, phi, avg, 1.f / (float)K, count);
  return check_launch("k_saga");
}

__global__ void k_fill(float* __restrict__ x, size_t count, float value) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    x[i] = value;
}

int launch_fill(float* x, size_t count, float value, cudaStream_t st) {
  k_fill<<<grid1d(count), 256, 0, st>>>(x, count, value);
  return check_launch("k_fill");
}

// ---------------------------------------------- TV-prox, persistent form --
// All K dual iterations and the output step in ONE cooperative launch,
// temporally blocked in row strips.  The batch's image rows form one list;
// CTA c owns rows [R0, R1) = [c R, (c+1) R) and keeps p = (px, py), w =
// div p - f / lambda (and f when it fits) for rows [R0 - k - 1, R1 + k) in
// shared memory: p_new at a row needs p of the rows above and below only, so
// k iterations computed on that halo'd strip, the valid region shrinking by
// one row per side per iteration, leave p^{+k} exact on [R0 - 1, R1) without
// any exchange.  The K iterations run in rounds of k; since p^0 = 0 (no warm
// start) the first round needs no neighbour data at all, and when K fits one
// round (k = K: 512^2 batch 1 and smaller) the kernel never synchronises with
// another CTA.  Between rounds each CTA stores its own rows of p to global
// memory (the plan's dual buffers, double-buffered by round parity), raises
// its 64-bit flag (launch generation << 32 | round, st.release.gpu after one
// fence by thread 0) and loads its halo rows after the flags of the CTAs
// owning them (and of every CTA that reads its rows) reached the round
// (ld.acquire.gpu).  A buffer is rewritten two rounds later, after every CTA
// reading it has published the round in between.  The generation (one device
// word, bumped by the last CTA to finish) keeps flags monotonic across
// launches and graph replays.  Halo rows are computed redundantly with the
// same arithmetic as their owner, term by term as k_tv_iter / k_tv_final
// (same order, MUFU sqrt / rcp): results are bitwise equal to the K + 1-launch
// form.  Waits are bounded by 2 s of %globaltimer (then *err is raised and
// the kernel finishes instead of hanging the device).
struct TvSync {
  unsigned long long* flags;   // [CTAs]
  unsigned* gen_ticket;        // {generation, finished-CTA ticket}
  int* err;
  float* pg[2];                // global p by round parity, layout [batch][2][n][n]
};

__device__ __forceinline__ unsigned long long tv_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tv_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long tv_clock_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// global px / py of row R (global row index b n + i) in a [batch][2][n][n] buffer
__device__ __forceinline__ float* tv_row(float* base, int R, int n, int comp) {
  const int b = R / n, i = R - b * n;
  return base + ((size_t)b * 2 + comp) * n * n + (size_t)i * n;
}

__global__ void __launch_bounds__(1024, 1) k_tv_persist(const float* __restrict__ f, int n, int total_rows,
                                                        int rows_per, int kround, int f_in_smem, float lambda,
                                                        float inv_lambda, float tau, int iters, TvSync sy,
                                                        const float* __restrict__ xprev, float* __restrict__ xout,
                                                        float* __restrict__ yout, float alpha, float a, int mode,
                                                        int* flag, int iter) {
  extern __shared__ float sm[];
  const int c = blockIdx.x, C = gridDim.x;
  const int R0 = c * rows_per, R1 = min(total_rows, R0 + rows_per);
  const int A = max(0, R0 - kround - 1), E = min(total_rows, R1 + kround);   // strip with halos [A, E)
  const int W = rows_per + 2 * kround + 1;          // allocated rows per array
  float* px = sm;                                    // local row r <-> global row A + r
  float* py = px + (size_t)W * n;
  float* w = py + (size_t)W * n;
  float* fs = w + (size_t)W * n;                     // f (only when f_in_smem)
  const int tx = threadIdx.x, ty = threadIdx.y, TX = blockDim.x, TY = blockDim.y;
  const unsigned long long gen = (unsigned long long)*(volatile unsigned*)sy.gen_ticket << 32;
  // f rows of the strip: shared memory (loaded once) or global (L2)
  if (f_in_smem) {
    for (int r = ty; r < E - A; r += TY)
      for (int j = tx; j < n; j += TX) fs[(size_t)r * n + j] = f[(size_t)(A + r) * n + j];
    __syncthreads();
  }
  const float* frow_base = f_in_smem ? fs : f + (size_t)A * n;
  // CTAs whose rows this one reads or whose readers include it (symmetric range)
  const int c_lo = max(0, (R0 - kround - 1) / rows_per), c_hi = min(C - 1, (R1 + kround) / rows_per);

  int it = 0, round = 0;
  while (it < iters) {
    const int kr = min(kround, iters - it);
    if (round > 0) {   // halo rows of p^it from the owners' published rows
      if (tx == 0 && ty == 0) {
        const unsigned long long target = gen | (unsigned long long)round;
        const unsigned long long t0 = tv_clock_ns();
        for (int q = c_lo; q <= c_hi; ++q) {
          if (q == c) continue;
          while (tv_ld_acquire(sy.flags + q) < target) {
            if (*(volatile int*)sy.err || tv_clock_ns() - t0 > 2000000000ull) {
              atomicExch(sy.err, 1);
              break;
            }
          }
        }
      }
      __syncthreads();
      float* pg = (round & 1) ? sy.pg[1] : sy.pg[0];
      for (int r = ty; r < E - A; r += TY) {
        const int R = A + r;
        if (R >= R0 && R < R1) continue;            // own rows: already in shared memory
        const float* gx = tv_row(pg, R, n, 0);
        const float* gy = tv_row(pg, R, n, 1);
        for (int j = tx; j < n; j += TX) {
          px[(size_t)r * n + j] = __ldcg(gx + j);
          py[(size_t)r * n + j] = __ldcg(gy + j);
        }
      }
      __syncthreads();
    }
    for (int jj = 0; jj < kr; ++jj, ++it) {
      const bool first = it == 0;
      // p_new on [lo, hi): the valid region shrinks by one row per side per
      // iteration, except at the ends of the row list (no rows beyond)
      const int lo = (A == 0) ? 0 : A + jj + 1;
      const int hi = (E == total_rows) ? total_rows : E - jj - 1;
      const int whi = min(hi + 1, total_rows);       // w on [lo, whi)
      for (int r = lo - A + ty; r < whi - A; r += TY) {
        const int R = A + r, i = R % n;
        const float* fr = frow_base + (size_t)r * n;
        const float* pxr = px + (size_t)r * n;
        const float* pyr = py + (size_t)r * n;
        for (int j = tx; j < n; j += TX) {
          float d = 0.f;
          if (!first) {
            const float ax = (j < n - 1 ? pxr[j] : 0.f) - (j > 0 ? pxr[j - 1] : 0.f);
            const float by = (i < n - 1 ? pyr[j] : 0.f) - (i > 0 ? pyr[j - n] : 0.f);
            d = ax + by;
          }
          w[(size_t)r * n + j] = tv_w(d, fr[j], inv_lambda);
        }
      }
      __syncthreads();
      for (int r = lo - A + ty; r < hi - A; r += TY) {
        const int i = (A + r) % n;
        const float* wr = w + (size_t)r * n;
        float* pxr = px + (size_t)r * n;
        float* pyr = py + (size_t)r * n;
        for (int j = tx; j < n; j += TX) {
          const float wc = wr[j];
          const float qx = (j < n - 1) ? wr[j + 1] - wc : 0.f;
          const float qy = (i < n - 1) ? wr[j + n] - wc : 0.f;
          const float rden = tv_rden(qx, qy, tau);
          pxr[j] = tv_p(first ? 0.f : pxr[j], qx, tau, rden);
          pyr[j] = tv_p(first ? 0.f : pyr[j], qy, tau, rden);
        }
      }
      __syncthreads();
    }
    ++round;
    if (it < iters) {   // publish own rows of p^it for the next round's halos
      float* pg = (round & 1) ? sy.pg[1] : sy.pg[0];
      for (int r = R0 - A + ty; r < R1 - A; r += TY) {
        float* gx = tv_row(pg, A + r, n, 0);
        float* gy = tv_row(pg, A + r, n, 1);
        for (int j = tx; j < n; j += TX) {
          __stcg(gx + j, px[(size_t)r * n + j]);
          __stcg(gy + j, py[(size_t)r * n + j]);
        }
      }
      // one thread releases for the block: bar.sync orders the block's stores
      // before thread 0's gpu-scope fence + release (cumulativity)
      __syncthreads();
      if (tx == 0 && ty == 0) {
        __threadfence();
        tv_st_release(sy.flags + c, gen | (unsigned long long)round);
      }
    }
  }
  // u = f - lambda div p^K on the own rows (row R0 - 1 of p is valid in the
  // strip), then the mix + momentum epilogue
  for (int r = R0 - A + ty; r < R1 - A; r += TY) {
    const int R = A + r, i = R % n;
    const float* pxr = px + (size_t)r * n;
    const float* pyr = py + (size_t)r * n;
    for (int j = tx; j < n; j += TX) {
      float dv = 0.f;
      if (iters > 0) {
        const float ax = (j < n - 1 ? pxr[j] : 0.f) - (j > 0 ? pxr[j - 1] : 0.f);
        const float by = (i < n - 1 ? pyr[j] : 0.f) - (i > 0 ? pyr[j - n] : 0.f);
        dv = ax + by;
      }
      const size_t idx = (size_t)R * n + j;
      const float fv = f[idx];
      mix_momentum(idx, fv, tv_u(fv, dv, lambda), xprev, xout, yout, alpha, a, mode, flag, iter);
    }
  }
  // the last CTA to finish advances the generation for the next launch
  __syncthreads();
  if (tx == 0 && ty == 0) {
    __threadfence();
    if (atomicAdd(sy.gen_ticket + 1, 1u) == (unsigned)C - 1) {
      sy.gen_ticket[1] = 0u;
      atomicAdd(sy.gen_ticket, 1u);
    }
  }
}

// shared memory of a strip with k-row halos: px, py, w (+ f)
static size_t tv_persist_smem(int n, int rows_per, int k, bool with_f) {
  return sizeof(float) * (size_t)(rows_per + 2 * k + 1) * n * (with_f ? 4 : 3);
}

// Persistent TV workspace (TvWs in internal.cuh): usable when a strip with a
// halo of at least one row fits one CTA's shared memory; the round length k
// is the largest that fits (k = K: no exchange at all).
int launch_tv_persist(const TvWs& ws, int n, int batch, float lambda, float tau, int iters, const float* f,
                      float* p0, float* p1, const float* xprev, float* xout, float* yout, float alpha, float a,
                      int mode, int* flag, int iter, cudaStream_t st, bool* used) {
  *used = false;
  static const bool off = getenv("MS2G_TV_PERSIST") && atoi(getenv("MS2G_TV_PERSIST")) == 0;   // experiment switch
  static const int kmax_env = getenv("MS2G_TV_KROUND") ? atoi(getenv("MS2G_TV_KROUND")) : 0;    // experiment switch
  if (off || !ws.flags || iters < 1) return MS2G_OK;
  // Rounds of at most 5 iterations (measured on B200, scripts/tv_probe.py,
  // profiles/r02_tv_probe.log, K = 10, us per call vs the K + 1 launches:
  // 512^2 x 8 126.6 vs 167.1, 1024^2 81.7 vs 106.5; longer rounds recompute
  // more halo rows than the exchanges they save).  A single image of at most
  // 512^2 keeps the K + 1 launches: inside a solve graph they run back to
  // back, and the C3 solve measured 1 ms slower with the persistent form
  // (cached-step solve 6.54 vs 5.58 ms, profiles/r02_launches_solve_c3.md);
  // MS2G_TV_PERSIST=1 forces it.
  static const bool force = getenv("MS2G_TV_PERSIST") && atoi(getenv("MS2G_TV_PERSIST")) == 1;
  if (!force && batch == 1 && n <= 512) return MS2G_OK;
  const int total_rows = n * batch;
  int C = std::min(ws.max_ctas, total_rows);
  const int rows_per = (total_rows + C - 1) / C;
  C = (total_rows + rows_per - 1) / rows_per;
  if (C > ws.max_ctas) return MS2G_OK;
  // the longest round that fits, with f in shared memory or (if that allows
  // fewer rounds) read from L2
  const int kcap = std::min(iters, kmax_env > 0 ? kmax_env : 5);
  auto kfit = [&](bool wf) {
    int kk = kcap;
    while (kk >= 1 && tv_persist_smem(n, rows_per, kk, wf) > (size_t)ws.smem_optin) --kk;
    return kk;
  };
  const int k1 = kfit(true), k0 = kfit(false);
  if (k0 < 1) return MS2G_OK;                      // not even a one-row halo fits
  auto rounds = [&](int kk) { return (iters + kk - 1) / kk; };
  const bool with_f = k1 >= 1 && rounds(k1) <= rounds(k0);
  const int k = with_f ? k1 : k0;
  const size_t smem = tv_persist_smem(n, rows_per, k, with_f);
  static std::atomic<uint64_t> attr_devices{0};
  int dev = 0;
  MS2G_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_devices.load() & bit)) {
    MS2G_CUDA(cudaFuncSetAttribute(k_tv_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, ws.smem_optin));
    attr_devices.fetch_or(bit);
  }
  TvSync sy{ws.flags, ws.gen_ticket, ws.err, {p0, p1}};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C);
  cfg.blockDim = dim3(256, 4);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: the round waits cannot deadlock
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MS2G_CUDA(cudaLaunchKernelEx(&cfg, k_tv_persist, f, n, total_rows, rows_per, k, with_f ? 1 : 0, lambda,
                               1.f / lambda, tau, iters, sy, xprev, xout, yout, alpha, a, mode, flag, iter));
  MS2G_TRY(check_launch("k_tv_persist"));
  *used = true;
  return MS2G_OK;
}

int launch_tv(int n, int batch, float lambda, float tau, int iters, const float* f, float* p0, float* p1,
              const float* xprev, float* xout, float* yout, float alpha, float a, int mode, int* flag, int iter,
              cudaStream_t st, const TvWs* ws) {
  const size_t total = (size_t)n * n * batch;
  if (lambda == 0.f) {  // prox of the zero function: identity
    return launch_copy_mix_mom(n, batch, f, xprev, xout, yout, a, mode, flag, iter, st);
  }
  if (ws) {
    bool used = false;
    MS2G_TRY(launch_tv_persist(*ws, n, batch, lambda, tau, iters, f, p0, p1, xprev, xout, yout, alpha, a, mode,
                               flag, iter, st, &used));
    if (used) return MS2G_OK;
  }
  // p^0 = 0 at every call (no warm start): the first iteration does not read p
  if (iters < 1) MS2G_TRY(launch_fill(p0, 2 * total, 0.f, st));
  float* pin = p0;
  float* pout = p1;
  for (int k = 0; k < iters; ++k) {
    MS2G_CUDA(launch_k_pdl(k_tv_iter, px_grid(n, n, batch), kPxBlock, 0, st, f, (const float*)pin, pout, n,
                           1.f / lambda, tau, (int)(k == 0)));
    MS2G_TRY(check_launch("k_tv_iter"));
    float* tmp = pin;
    pin = pout;
    pout = tmp;
  }
  MS2G_CUDA(launch_k_pdl(k_tv_final, px_grid(n, n, batch), kPxBlock, 0, st, f, (const float*)pin, xprev, xout, yout, n,
                     lambda, alpha, a, mode, flag, iter));
  return check_launch("k_tv_final");
}

// ------------------------------------------------------ power iteration --
// (the step itself, O8 / Z6, is k_reduce_power in projector.cu: fused with
// the backprojection's chunk sum, last-block fp64 finalisation)
// {L, eta, (float) eta} from a factor's cache into a stage's slots (each may be NULL)
__global__ void k_cached_step(const double* __restrict__ cache, double* L_out, double* eta_out, float* etaf_out) {
  if (L_out) *L_out = cache[0];
  if (eta_out) *eta_out = cache[1];
  if (etaf_out) *etaf_out = reinterpret_cast<const float*>(cache + 2)[0];
}

int launch_cached_step(const double* cache, double* L_out, double* eta_out, float* etaf_out, cudaStream_t st) {
  if (!L_out && !eta_out && !etaf_out) return MS2G_OK;
  k_cached_step<<<1, 1, 0, st>>>(cache, L_out, eta_out, etaf_out);
  return check_launch("k_cached_step");
}

// flag[0]: first non-finite global iteration (INT_MAX = none); flag[1]: a
// non-finite INPUT (b or x0) was seen by k_check_finite
__global__ void k_init_flag(int* flag) {
  flag[0] = INT_MAX;
  flag[1] = 0;
}

// Non-finite input check at the start of a solve (SURVEY §8(b):
// "non-finite input ... -> MS2G_ERR_INPUT"): any NaN / Inf in b or x0 raises
// flag[1].  One streaming pass over the inputs (C4: 13 MB).
__global__ void k_check_finite(const float* __restrict__ a, size_t na, const float* __restrict__ c, size_t nc_,
                               int* flag) {
  bool bad = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < na + nc_; i += (size_t)gridDim.x * blockDim.x) {
    const float v = i < na ? a[i] : c[i - na];
    bad |= !isfinite(v);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag + 1, 1);
}

int launch_check_finite(const float* a, size_t na, const float* c, size_t nc_, int* flag, cudaStream_t st) {
  k_check_finite<<<grid1d(na + nc_, 256, 148 * 8), 256, 0, st>>>(a, na, c, nc_, flag);
  return check_launch("k_check_finite");
}

int launch_init_flag(int* flag, cudaStream_t st) {
  k_init_flag<<<1, 1, 0, st>>>(flag);
  return check_launch("k_init_flag");
}

}  // namespace ms2g
