// projector.cu -- fan-beam Siddon projector A_s and its exact adjoint A_s^T
// for sm_100a (north-star subsystems (1) and (2); Eqs. 5-7).
//
// Both kernels evaluate the SAME segment weights from the same 32-byte ray
// record (RayEntry, built on the host in fp64).  The ray is marched along its
// major axis (x when |dx| >= |dy|, else y) one pixel column at a time; within
// column c the minor coordinate goes from F(c) = F0 + c S to F(c) + S, with
// F in 64-bit fixed point (32 fractional bits).  Integer arithmetic is exact,
// so F(c) is bit-identical whether reached incrementally (forward) or
// directly (adjoint), and no crossing parameter is ever accumulated in fp32
// (DESIGN.md "precision").  Since the slope S is in [0, 1], each column holds
// one segment or two split at the grid line m0 + 1:
//   w0 = min((2^32 - lo(F)) * Ly32, Lc),  w1 = Lc - w0.
// Lengths are physical (the oracle's (alpha_b - alpha_a) |d|).
#include <climits>

#include "internal.cuh"

namespace ms2g {

__device__ __forceinline__ void seg_weights(long long F, unsigned long long S, float Lc, float Ly32, int& m0,
                                            int& m1, float& w0, float& w1) {
  const long long F1 = F + (long long)S;
  m0 = (int)(F >> 32);
  m1 = (int)(F1 >> 32);
  w0 = Lc;
  w1 = 0.f;
  if (m1 != m0) {
    const unsigned lo = (unsigned)(unsigned long long)F;
    const float rem = lo ? (float)(0u - lo) : 4294967296.0f;
    w0 = fminf(rem * Ly32, Lc);
    w1 = Lc - w0;
  }
}

// ---------------------------------------------------------------- forward --
// One thread per ray; a warp holds 32 consecutive bins of one view, so at a
// given column the lanes read adjacent minor indices: contiguous addresses in
// x (major-y rays) or in its transpose xT (major-x rays).  The 8 warps of a
// block are 8 consecutive views over the same bins, which trace nearly the
// same image lines: L1 reuse.  Residual epilogue fused ("A_s v - b").
constexpr int kFwdWarps = 8;

__global__ void __launch_bounds__(256) k_forward(const RayEntry* __restrict__ rays, int B, int V_r,
                                                 const int* __restrict__ sel, int n_sel,
                                                 const float* __restrict__ x, const float* __restrict__ xT,
                                                 int nc, const float* __restrict__ bsino,
                                                 float* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = blockIdx.y * kFwdWarps + warp;
  if (k >= n_sel) return;
  const int t = blockIdx.x * 32 + lane;
  const int bz = blockIdx.z;
  const size_t np = (size_t)nc * nc;
  const int g = sel ? __ldg(sel + k) : k;
  const bool valid = t < B;
  long long F0 = 0;
  unsigned long long S = 0;
  float Lc = 0.f, Ly32 = 0.f;
  int flags = 0, cl = INT_MAX, ch = INT_MIN;
  if (valid) {
    const RayEntry R = rays[(size_t)g * B + t];
    F0 = R.F0; S = R.S; Lc = R.Lc; Ly32 = R.Ly32; flags = R.flags;
    if (R.c_lo < R.c_hi) { cl = R.c_lo; ch = R.c_hi; }
  }
  const int wcl = __reduce_min_sync(0xffffffffu, cl);
  const int wch = __reduce_max_sync(0xffffffffu, ch);
  float acc = 0.f;
  if (wcl < wch) {
    const float* img = ((flags & kMajorY) ? x : xT) + (size_t)bz * np;
    const bool mir = flags & kMirror;
    const int msign = mir ? -1 : 1;
    const float* rowp = img + (size_t)wcl * nc + (mir ? nc - 1 : 0);
    long long F = F0 + (long long)wcl * (long long)S;
#pragma unroll 2
    for (int c = wcl; c < wch; ++c) {
      int m0, m1;
      float w0, w1;
      seg_weights(F, S, Lc, Ly32, m0, m1, w0, w1);
      const bool inr = (c >= cl) && (c < ch);
      if (inr && (unsigned)m0 < (unsigned)nc) acc = fmaf(w0, __ldg(rowp + msign * m0), acc);
      if (inr && m1 != m0 && (unsigned)m1 < (unsigned)nc) acc = fmaf(w1, __ldg(rowp + msign * m1), acc);
      F += (long long)S;
      rowp += nc;
    }
  }
  if (valid) {
    float r = acc;
    if (bsino) r -= __ldg(bsino + ((size_t)bz * V_r + g) * B + t);
    out[((size_t)bz * n_sel + k) * B + t] = r;
  }
}

int launch_forward(ms2g_plan* p, const FactorTables& f, const float* x, const float* xT, const float* b,
                   float* out, const int* d_sel, int n_sel, int batch, cudaStream_t s) {
  if (n_sel <= 0) return MS2G_OK;
  dim3 grid((p->B + 31) / 32, (n_sel + kFwdWarps - 1) / kFwdWarps, batch);
  k_forward<<<grid, 256, 0, s>>>(f.d_rays, p->B, p->V_r, d_sel, n_sel, x, xT, f.nc, b, out);
  return check_launch("k_forward");
}

// --------------------------------------------------------------- adjoint --
// Tile-driven ray scatter: a block owns a 32x32 pixel tile and a chunk of
// views; each warp takes one view at a time, finds the bins whose rays meet
// the tile (detector coordinate of the tile corners), and walks those rays one
// per step with LANE = major index inside the tile.  A lane therefore only
// touches its own column (major-x rays) or row (major-y rays) of the warp's
// private shared-memory accumulator: no atomics, deterministic order.  The 8
// warp tiles are summed in fixed order at the end.
constexpr int kBT = 32;
constexpr int kBW = 8;

__global__ void __launch_bounds__(256) k_backward(const RayEntry* __restrict__ rays,
                                                  const ViewEntry* __restrict__ views, int B,
                                                  const int* __restrict__ sel, int n_sel, int vpc,
                                                  const float* __restrict__ sino, float* __restrict__ out,
                                                  int nc, int tiles_x, float scale, int accumulate,
                                                  int partial) {
  __shared__ float acc[kBW][kBT][kBT + 1];
  __shared__ RayEntry stg[kBW][32];
  __shared__ float rstg[kBW][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tile = blockIdx.x, chunk = blockIdx.y, bz = blockIdx.z;
  const int tx = tile % tiles_x, ty = tile / tiles_x;
  const int x0 = tx * kBT, y0 = ty * kBT;
  const int x1 = min(x0 + kBT, nc), y1 = min(y0 + kBT, nc);
  float(*A)[kBT + 1] = acc[warp];
#pragma unroll 4
  for (int r = 0; r < kBT; ++r) A[r][lane] = 0.f;
  __syncwarp();
  const int kb = chunk * vpc, ke = min(n_sel, kb + vpc);
  const float* sb = sino + (size_t)bz * n_sel * B;
  for (int k = kb + warp; k < ke; k += kBW) {
    const int g = sel ? __ldg(sel + k) : k;
    const ViewEntry V = views[g];
    // detector coordinate of the tile's 4 corners (lanes 0..3)
    const float px = (lane & 1) ? (float)x1 : (float)x0;
    const float py = (lane & 2) ? (float)y1 : (float)y0;
    const float dx = px - V.Sx, dy = py - V.Sy;
    const float tau = V.off + V.scale * (dx * V.ex + dy * V.ey) / (dx * V.nx + dy * V.ny);
    float tmin = (lane < 4) ? tau : INFINITY, tmax = (lane < 4) ? tau : -INFINITY;
#pragma unroll
    for (int o = 2; o; o >>= 1) {
      tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    }
    tmin = __shfl_sync(0xffffffffu, tmin, 0);
    tmax = __shfl_sync(0xffffffffu, tmax, 0);
    const int t_lo = max(0, (int)floorf(tmin - 0.01f));
    const int t_hi = min(B - 1, (int)ceilf(tmax + 0.01f));
    for (int tb = t_lo; tb <= t_hi; tb += 32) {
      const int t = tb + lane;
      if (t <= t_hi) {
        stg[warp][lane] = rays[(size_t)g * B + t];
        rstg[warp][lane] = __ldg(sb + (size_t)k * B + t);
      }
      __syncwarp();
      const int nr = min(32, t_hi - tb + 1);
      int prev_major = -1;
      for (int q = 0; q < nr; ++q) {
        const float r = rstg[warp][q];
        if (r == 0.f) continue;
        const RayEntry R = stg[warp][q];
        const int majY = R.flags & kMajorY;
        if (majY != prev_major) {  // lanes switch between column and row ownership
          __syncwarp();
          prev_major = majY;
        }
        const int c = (majY ? y0 : x0) + lane;
        const int ce = majY ? y1 : x1;
        if (c < ce && c >= R.c_lo && c < R.c_hi) {
          const long long F = R.F0 + (long long)c * (long long)R.S;
          int m0, m1;
          float w0, w1;
          seg_weights(F, R.S, R.Lc, R.Ly32, m0, m1, w0, w1);
          const bool mir = R.flags & kMirror;
          const int p0 = mir ? nc - 1 - m0 : m0;
          const int p1 = mir ? p0 - 1 : p0 + 1;
          const int mb = majY ? x0 : y0, me = majY ? x1 : y1;
          if ((unsigned)m0 < (unsigned)nc && p0 >= mb && p0 < me) {
            float* cell = majY ? &A[lane][p0 - mb] : &A[p0 - mb][lane];
            *cell = fmaf(w0, r, *cell);
          }
          if (m1 != m0 && (unsigned)m1 < (unsigned)nc && p1 >= mb && p1 < me) {
            float* cell = majY ? &A[lane][p1 - mb] : &A[p1 - mb][lane];
            *cell = fmaf(w1, r, *cell);
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  const size_t np = (size_t)nc * nc;
  for (int idx = threadIdx.x; idx < kBT * kBT; idx += blockDim.x) {
    const int ly = idx / kBT, lx = idx % kBT;
    const int yy = y0 + ly, xx = x0 + lx;
    if (yy < nc && xx < nc) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kBW; ++w) s += acc[w][ly][lx];
      const size_t o = (size_t)yy * nc + xx;
      if (partial) {
        out[((size_t)bz * gridDim.y + chunk) * np + o] = s;
      } else {
        float* dst = out + (size_t)bz * np + o;
        float v = scale * s;
        if (accumulate) v += *dst;
        *dst = v;
      }
    }
  }
}

__global__ void k_chunk_reduce(const float* __restrict__ part, int nchunks, size_t np, size_t total,
                               float* __restrict__ out, float scale, int accumulate) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / np, p = i % np;
    const float* src = part + b * nchunks * np + p;
    float s = 0.f;
    for (int c = 0; c < nchunks; ++c) s += src[(size_t)c * np];
    float v = scale * s;
    if (accumulate) v += out[i];
    out[i] = v;
  }
}

int launch_backward(ms2g_plan* p, const FactorTables& f, const float* sino, float* img, float scale,
                    int accumulate, const int* d_sel, int n_sel, int batch, cudaStream_t s) {
  const int tiles_x = (f.nc + kBT - 1) / kBT;
  int nchunks = f.bp_chunks;
  const int max_chunks = (n_sel + kBW - 1) / kBW;
  if (nchunks > max_chunks) nchunks = max_chunks;
  if (nchunks < 1) nchunks = 1;
  const int vpc = (n_sel + nchunks - 1) / nchunks;
  const int partial = nchunks > 1;
  dim3 grid(tiles_x * tiles_x, nchunks, batch);
  k_backward<<<grid, kBT * kBW, 0, s>>>(f.d_rays, f.d_views, p->B, d_sel, n_sel, vpc, sino,
                                        partial ? p->w_part : img, f.nc, tiles_x, scale, accumulate, partial);
  MS2G_TRY(check_launch("k_backward"));
  if (partial) {
    const size_t np = (size_t)f.nc * f.nc, total = np * batch;
    const int blocks = (int)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
    k_chunk_reduce<<<blocks, 256, 0, s>>>(p->w_part, nchunks, np, total, img, scale, accumulate);
    MS2G_TRY(check_launch("k_chunk_reduce"));
  }
  return MS2G_OK;
}

}  // namespace ms2g
