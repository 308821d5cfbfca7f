// projector.cu -- fan-beam Siddon projector A_s and its exact adjoint A_s^T
// for sm_100a (north-star subsystems (1) and (2); Eqs. 5-7).
//
// Both kernels evaluate the SAME segment weights from the same 32-byte ray
// record (RayEntry, built on the host in fp64).  A ray is marched along its
// major axis (x when |dx| >= |dy|, else y) one pixel column at a time; in
// column c its minor coordinate runs from F(c) = F0 + c S to F(c) + S, with F
// in 64-bit fixed point (32 fractional bits).  Integer arithmetic is exact, so
// F(c) is bit-identical whether reached incrementally (forward) or directly
// (adjoint), and no crossing parameter is ever accumulated in fp32 (DESIGN.md
// "precision").  Since the slope is in [0, 1), a column holds one segment or
// two split at the grid line m0 + 1 (seg_weights).  Lengths are physical
// (the oracle's (alpha_b - alpha_a) |d|).
#include <algorithm>
#include <climits>
#include <cstring>

#include "internal.cuh"

namespace ms2g {

// Hide a value from the optimizer so that 32-bit compares of the high word of
// a 64-bit fixed-point coordinate stay 32-bit.
__device__ __forceinline__ int opaque_i32(int v) {
  int r;
  asm("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Weights of the (up to) two segments of one column.  lo = low word of F.
//   no crossing: w0 = Lc, w1 = 0
//   crossing   : w0 = (2^32 - lo) * Ly32 (clamped to Lc), w1 = Lc - w0
__device__ __forceinline__ void seg_weights(unsigned lo, bool cross, float Lc, float Ly32, float& w0, float& w1) {
  const float wc = fminf(fmaf((float)(~lo), Ly32, Ly32), Lc);
  w0 = cross ? wc : Lc;
  w1 = Lc - w0;
}

// ------------------------------------------------------------ pair prep --
// The forward projector gathers the two pixels (m0, m0+1) of a column with
// ONE 8-byte load from "pair images": for every line of the minor-contiguous
// layout, element kPairPad + k + 2 (k = -2 .. n_c) holds (v[k], v[k+1] - v[k])
// with zeros outside the grid (the difference the forward's end-coordinate
// weights need, formed once here in the same fp32 subtraction), and kPairPad
// zero elements pad each end of a line.  Four images, indexed by the ray class (flags & 3):
//   0 major-x      : lines = columns j of x, pairs along rows     (x^T)
//   1 major-y      : lines = rows i of x,    pairs along columns
//   2 major-x, mirrored: as 0 with each pair reversed (v[k+1], v[k] - v[k+1]) and
//      each line stored back to front (element nc - k holds it), so that the
//      forward indexes every class the same way
//   3 major-y, mirrored: as 1, reversed likewise
//
// The kernel also forms its input on the fly (fused producers, one launch
// instead of two): with s > 1 the coarse value is the s x s mean of the
// full-resolution image (S_s, the same summation order as k_sketch_down);
// with scale_dev != NULL it is w * (float)scale_dev[0] (the power iteration's
// v = w / ||w||, as k_scale did).  v_out != NULL also stores the coarse values
// (each block stores the rows it owns).
__device__ __forceinline__ float pair_src(const float* __restrict__ xb, int k, int j, int nc, int s, int nsrc,
                                          float inv_s2, float scale) {
  if (s == 1) return xb[(size_t)k * nc + j] * scale;
  float acc = 0.f;
  for (int a = 0; a < s; ++a) {
    const float* row = xb + (size_t)(s * k + a) * nsrc + (size_t)s * j;
    if (s == 4) {            // one 16-byte load per row (same summation order)
      const float4 v = *reinterpret_cast<const float4*>(row);
      acc += v.x; acc += v.y; acc += v.z; acc += v.w;
    } else if (s == 2) {
      const float2 v = *reinterpret_cast<const float2*>(row);
      acc += v.x; acc += v.y;
    } else {
      for (int c = 0; c < s; ++c) acc += row[c];
    }
  }
  return acc * inv_s2 * scale;
}

//
// Batches with il = NB > 1 (experiment switch MS2G_FWD_INTERLEAVE; measured
// slower, see fwd_launch_batch): the NB images of a group INTERLEAVED,
// element (line, pos) holding NB consecutive pairs.
__global__ void k_pair_prep(const float* __restrict__ x, float2* __restrict__ pairs, size_t pair_stride, int nc,
                            int s, const double* __restrict__ scale_dev, float* __restrict__ v_out, int class_mask,
                            int il, unsigned* __restrict__ rmaxv, int V_r) {
  // T[r][c] = v[O0-2+r][L0+c] (column pairs, classes 0/2); with s > 1 also
  // T2[r][c] = v[L0+r][O0-2+c] (row pairs, classes 1/3), so each s x s mean
  // is formed once per tile (s = 1 reads the row pairs directly)
  __shared__ float T[33][33], T2[32][34];
  pdl_wait();
  pdl_release();
  const int bz = blockIdx.z;
  if (rmaxv && blockIdx.x == 0 && blockIdx.y == 0)   // the next forward's per-view maxima start at 0
    for (int i = threadIdx.y * 32 + threadIdx.x; i < V_r; i += 256) rmaxv[(size_t)bz * V_r + i] = 0u;
  const int nsrc = nc * s;
  const float* xb = x + (size_t)bz * nsrc * nsrc;
  const float inv_s2 = 1.0f / (float)(s * s);
  const float scale = scale_dev ? (float)scale_dev[0] : 1.f;
  const int L = (int)pair_line(nc);
  const int mul = il > 1 ? il : 1, grp = bz / mul, sub = bz - grp * mul;   // interleaving group / slot
  const size_t ib = (size_t)grp * nc * L + kPairPad;                       // + the leading pad of a line
  // output positions o = -kPairPad .. nc + 2 + kPairPad (outside 0 .. nc + 2: the zero pads), lines
  const int O0 = blockIdx.x * 32 - kPairPad, L0 = blockIdx.y * 32;
  // rows k = O0-2 .. O0+30 for the column-pair images (this block owns O0-2 .. O0+29)
  for (int r = threadIdx.y; r < 33; r += 8) {
    const int k = O0 - 2 + r, j = L0 + threadIdx.x;
    const bool in = k >= 0 && k < nc && j < nc;
    const float val = in ? pair_src(xb, k, j, nc, s, nsrc, inv_s2, scale) : 0.f;
    T[r][threadIdx.x] = val;
    if (v_out && in && r < 32) v_out[((size_t)bz * nc + k) * nc + j] = val;
  }
  const bool rows2 = s > 1 && (class_mask & 10);
  if (rows2)
    for (int r = threadIdx.y; r < 32; r += 8)
      for (int c = threadIdx.x; c < 33; c += 32) {
        const int i = L0 + r, k = O0 - 2 + c;
        T2[r][c] = (i < nc && k >= 0 && k < nc) ? pair_src(xb, i, k, nc, s, nsrc, inv_s2, scale) : 0.f;
      }
  __syncthreads();
  const int o = O0 + threadIdx.x;
  if (o > nc + 2 + kPairPad) return;
  for (int jj = threadIdx.y; jj < 32; jj += 8) {
    const int line = L0 + jj;
    if (line >= nc) break;
    const size_t e = (ib + (size_t)line * L + o) * mul + sub;
    const float a = T[threadIdx.x][jj], b = T[threadIdx.x + 1][jj];   // v[o-2][line], v[o-1][line]
    const size_t er = (ib + (size_t)line * L + (nc + 2 - o)) * mul + sub;   // back-to-front line
    // only the ray classes this plan's views contain (a view shard of 45
    // degrees has one or two): the others are never read by the forward
    if (class_mask & 1) pairs[e] = make_float2(a, b - a);
    if (class_mask & 4) pairs[2 * pair_stride + er] = make_float2(b, a - b);
    if (!(class_mask & 10)) continue;
    const int k = o - 2;
    float c, d;
    if (rows2) {
      c = T2[jj][threadIdx.x];
      d = T2[jj][threadIdx.x + 1];
    } else {
      c = (k >= 0 && k < nc) ? pair_src(xb, line, k, nc, s, nsrc, inv_s2, scale) : 0.f;
      d = (k + 1 >= 0 && k + 1 < nc) ? pair_src(xb, line, k + 1, nc, s, nsrc, inv_s2, scale) : 0.f;
    }
    if (class_mask & 2) pairs[pair_stride + e] = make_float2(c, d - c);
    if (class_mask & 8) pairs[3 * pair_stride + er] = make_float2(d, c - d);
  }
}

// group size of the batched forward (and of the pair interleaving) for a batch
static int batch_group(int batch) { return (batch % 8 == 0) ? 8 : (batch % 4 == 0) ? 4 : (batch % 2 == 0) ? 2 : 1; }

int launch_pair_prep(ms2g_plan* p, int nc, int batch, const float* x, cudaStream_t s, int factor,
                     const double* scale_dev, float* v_out) {
  dim3 grid(((int)pair_line(nc) + 31) / 32, (nc + 31) / 32, batch), block(32, 8);
  static const bool il_on = getenv("MS2G_FWD_INTERLEAVE") != nullptr;   // experiment switch
  const int il = il_on ? batch_group(batch) : 1;
  MS2G_CUDA(launch_k(k_pair_prep, grid, block, 0, s, x, p->w_pair, p->pair_stride, nc, factor, scale_dev, v_out,
                     p->class_mask, il, p->w_rmaxv, p->V_r));
  return check_launch("k_pair_prep");
}

// ---------------------------------------------------------------- forward --
// One thread per ray; a warp holds 32 consecutive bins of one view, so at a
// given column the lanes read adjacent minor indices of the same pair-image
// line (coalesced).  The 4 warps of a block are 4 consecutive views over the
// same bins, tracing nearly the same lines: L1 reuse.  Residual epilogue fused
// ("A_s v - b").
//
// End-coordinate weights.  In column c the ray's minor coordinate runs from
// F(c) to E(c) = F(c) + S.  With u = floor(E) + 1 (the pair index of the
// (lower, upper) rows floor(E) - 1, floor(E), shifted by the pair images'
// 2-element pad) and m = min(frac32(E), S) (the part of the step above the
// grid line floor(E); m = S when the column crosses no line),
//   upper row: m Ly32,   lower row: Lc - m Ly32   (Ly32 = Lc / S),
// so  sum_c w.x = Lc sum_c x_lower + Ly32 sum_c m (x_upper - x_lower): the
// per-ray constants leave the column loop.  Without a crossing the lower-row
// weight is a rounding residual (|.| <= 2^-23 Lc), not an exact zero.
#ifndef MS2G_FWD_WARPS
#define MS2G_FWD_WARPS 4
#endif
constexpr int kFwdWarps = MS2G_FWD_WARPS;
// column-loop unroll of the single-image forward (16) and of the batched one (4)
#ifndef MS2G_FWD_UNROLL
#define MS2G_FWD_UNROLL 16
#endif
constexpr int kFwdUnroll = MS2G_FWD_UNROLL;
#ifndef MS2G_FWD_UNROLL_B
#define MS2G_FWD_UNROLL_B 4
#endif
constexpr int kFwdUnrollB = MS2G_FWD_UNROLL_B;


// max |r| of the warp's rays into the view's word (float bits: for r >= 0 the
// unsigned order is the float order, NaN above +inf) -- the bound of the
// fixed-point adjoint's scale.  The words are zeroed by the pair prep.
__device__ __forceinline__ void fwd_view_max(unsigned* rmaxv, size_t idx, bool vk, bool valid, float r) {
#ifndef MS2G_NO_RMAXV
  const unsigned bits = __reduce_max_sync(0xffffffffu, valid ? __float_as_uint(fabsf(r)) : 0u);
  if (rmaxv && vk && (threadIdx.x & 31) == 0) atomicMax(rmaxv + idx, bits);
#endif
}

// the same for several views per warp (the TILE forward): groups of G lanes
template <int G>
__device__ __forceinline__ void fwd_view_max_g(unsigned* rmaxv, size_t idx, bool vk, bool valid, float r) {
  unsigned bits = valid ? __float_as_uint(fabsf(r)) : 0u;
#pragma unroll
  for (int o = 1; o < G; o <<= 1) bits = max(bits, __shfl_xor_sync(0xffffffffu, bits, o));
  if (rmaxv && vk && (threadIdx.x & (G - 1)) == 0) atomicMax(rmaxv + idx, bits);
}

// (pl, pu) = pair element e of a pair image (one 8-byte non-coherent load)
__device__ __forceinline__ void fwd_ld_pair(const float2* base, unsigned e, float& pl, float& pu) {
  asm("{\n\t.reg .u64 ad;\n\tmad.wide.u32 ad, %2, 8, %3;\n\tld.global.nc.v2.f32 {%0, %1}, [ad];\n\t}"
      : "=f"(pl), "=f"(pu) : "r"(e), "l"(base));
}

// A lane whose ray misses the grid reads the zero element u = 0 throughout
// (F0 = -1, S = 0).  The warp may skip the clamp when every lane's pair index
// u stays within kPairPad of 0 .. nc + 2 over the warp's columns [wcl, wch)
// (u is monotone in c: the ends decide).  99 % of the warps of the C3 / C4
// geometries stay within ~60 rows; the others are mostly warps whose rays
// change ray class (frame) inside the warp.
__device__ __forceinline__ bool fwd_fast_warp(bool valid, int cl, int ch, int wcl, int wch, int nc, long long& F0,
                                              unsigned& S) {
  bool fit = true;
  if (valid && cl > ch) {
    F0 = -(1LL << 32);
    S = 0;
  } else if (valid && wcl < wch) {
    const long long e0 = F0 + (long long)(wcl + 1) * (long long)S;   // E at the first column
    const long long e1 = F0 + (long long)wch * (long long)S;         // E at the last column
    fit = (e0 >> 32) + 1 >= -kPairPad && (e1 >> 32) + 1 <= nc + 2 + kPairPad;
  }
  return __all_sync(0xffffffffu, fit);
}

// Single images (NB = 1 here; batches use k_forward_batch below).
// Each warp's column range is cut into SEG equal segments whose partial sums
// are combined in fixed order through shared memory; SPLIT warps of the block
// (the same 32 rays) take SEG / SPLIT segments each.  More, shorter work
// units help launches with few views (a view shard, a minibatch) whose single
// wave would otherwise wait on its longest rays; the summation order depends
// on SEG only, not on SPLIT.
template <int NB, int SPLIT, int SEG, int TILE = 1>
// resident blocks the single-image forward is compiled for: 8 (64 registers)
// -- with the 4-view warps and a 16-column unroll it outruns the 32-register
// build at full occupancy (C4 s=1 0.640 -> 0.545 ms)
#ifndef MS2G_FWD_MINB
#define MS2G_FWD_MINB 8
#endif
__global__ void __launch_bounds__(32 * kFwdWarps, SPLIT == 1 ? MS2G_FWD_MINB : 64 / kFwdWarps) k_forward(const RayEntry* __restrict__ rays, int B, int V_r,
                                                 const int* __restrict__ sel, int n_sel,
                                                 const float2* __restrict__ pairs, size_t pair_stride, int nc,
                                                 const float* __restrict__ bsino, float* __restrict__ out,
                                                 const int* __restrict__ order, int allow_fast,
                                                 unsigned* __restrict__ rmaxv) {
  constexpr int VPB = kFwdWarps / SPLIT;             // views per block
  constexpr int SPW = SEG / SPLIT;                   // segments per warp

  __shared__ float2 red[VPB][SEG][NB][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int vw = warp / SPLIT, q = warp % SPLIT;
  // block -> (bin block, view block): the plan's longest-first order for
  // full-view launches, else the grid position
  int bxi = blockIdx.x, byi = blockIdx.y;
  if (order) {
    const int item = __ldg(order + blockIdx.y * gridDim.x + blockIdx.x);
    MS2G_DASSERT(item >= 0 && item < (int)(gridDim.x * gridDim.y));
    bxi = item % gridDim.x;
    byi = item / gridDim.x;
  }
  // TILE = views per warp (SPLIT = 1): a warp takes 32 / TILE adjacent bins
  // of TILE of the block's 4 views instead of 32 bins of one view -- rays of
  // neighbouring views at the same bins cross a column within a few rows of
  // each other, so a warp's gathers span fewer pair-image sectors
  constexpr int BPW = 32 / TILE;                     // bins per warp and view
  // (warp w: view group w / TILE of TILE views, bin group w % TILE of BPW bins)
  const int k = byi * VPB + (TILE > 1 ? (warp / TILE) * TILE + lane / BPW : vw);
  const bool vk = k < n_sel;
  const int t = bxi * 32 + (TILE > 1 ? (warp % TILE) * BPW + lane % BPW : lane);
  const int bz0 = blockIdx.z * NB;
  const int g = (sel && vk) ? __ldg(sel + k) : k;
  const bool valid = vk && t < B;
  long long F0 = 0;
  unsigned S = 1;
  float Lc = 0.f, Ly32 = 0.f;
  int cls = 0, cl = INT_MAX, ch = INT_MIN;
  if (valid) {
    const RayEntry R = rays[(size_t)g * B + t];
    F0 = R.F0; S = R.S; Lc = R.Lc; Ly32 = R.Ly32; cls = R.flags & 3;
    if (R.c_lo < R.c_hi) { cl = R.c_lo; ch = R.c_hi; }
  }
  pdl_wait();      // the ray table is static; the pair images and b come from the predecessors
  pdl_release();
  const int wcl = __reduce_min_sync(0xffffffffu, cl);
  const int wch = __reduce_max_sync(0xffffffffu, ch);
  const int len = wch > wcl ? wch - wcl : 0;
  const int L = (int)pair_line(nc);
  const size_t istride = (size_t)nc * L;            // pair-image stride between batch images
  const float2* base = pairs + cls * pair_stride + (size_t)bz0 * istride;
  const bool fast = fwd_fast_warp(valid, cl, ch, wcl, wch, nc, F0, S) && allow_fast;
  // element of pair index u on line c: c L + kPairPad + u for every class
  // (the mirrored images are stored back to front).  Fast warps (all rays
  // within kPairPad rows of the grid over the warp's columns) advance
  // (u + c L, frac) as ONE 64-bit fixed-point number: one add.cc/addc pair
  // per column gives both the element and the weight.  Other warps clamp u
  // to the zero pads (unsigned: negatives clamp too).
  const unsigned umax = (unsigned)(nc + 2);
#pragma unroll 1
  for (int j = 0; j < SPW; ++j) {
    const int sg = q * SPW + j;
    const int c0 = wcl + (sg * len) / SEG, c1 = wcl + ((sg + 1) * len) / SEG;
    float sa[NB], sb[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) { sa[i] = 0.f; sb[i] = 0.f; }
    if (c0 < c1) {
      const long long Es = F0 + (long long)c0 * (long long)S + (long long)S + (1LL << 32);
      unsigned elo = (unsigned)Es, ehi = (unsigned)(Es >> 32);
      if (fast) {
        unsigned qhi = ehi + (unsigned)(c0 * L + kPairPad);
#pragma unroll(SPLIT == 1 ? kFwdUnroll : kFwdUnrollB)
        for (int c = c0; c < c1; ++c) {
          unsigned lo1, hi1;
          asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, %5;" : "=r"(lo1), "=r"(hi1)
              : "r"(elo), "r"(qhi), "r"(S), "r"(L));
          const float mf = (float)min(elo, S);
          MS2G_DASSERT(qhi < (unsigned)(nc * L));
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            float pl, pu;
            fwd_ld_pair(base + i * istride, qhi, pl, pu);
            sa[i] += pl;
            sb[i] = fmaf(mf, pu, sb[i]);
          }
          elo = lo1;
          qhi = hi1;
        }
      } else {
        unsigned offk = (unsigned)(c0 * L + kPairPad);
#pragma unroll(SPLIT == 1 ? kFwdUnroll : kFwdUnrollB)
        for (int c = c0; c < c1; ++c) {
          unsigned lo1, hi1;
          asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, 0;" : "=r"(lo1), "=r"(hi1) : "r"(elo), "r"(ehi), "r"(S));
          const float mf = (float)min(elo, S);
          const unsigned e = offk + min(ehi, umax);
          MS2G_DASSERT(e < (unsigned)(nc * L));
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            float pl, pu;
            fwd_ld_pair(base + i * istride, e, pl, pu);
            sa[i] += pl;
            sb[i] = fmaf(mf, pu, sb[i]);
          }
          elo = lo1;
          ehi = hi1;
          offk += L;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) red[TILE > 1 ? warp : vw][sg][i][lane] = make_float2(sa[i], sb[i]);
  }
  __syncthreads();
  if (q != 0) return;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    float r = 0.f;
    if (valid) {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int sg = 0; sg < SEG; ++sg) {
        const float2 v = red[TILE > 1 ? warp : vw][sg][i][lane];
        a += v.x;
        b += v.y;
      }
      r = fmaf(Lc, a, Ly32 * b);
      if (bsino) r -= __ldg(bsino + ((size_t)(bz0 + i) * V_r + g) * B + t);
      out[((size_t)(bz0 + i) * n_sel + k) * B + t] = r;
    }
    if (TILE > 1) fwd_view_max_g<32 / TILE>(rmaxv, (size_t)(bz0 + i) * V_r + k, vk, valid, r);
    else fwd_view_max(rmaxv, (size_t)(bz0 + i) * V_r + k, vk, valid, r);
  }
}

// Batched traversal (NB >= 2 images share the weights): each view's rays are
// split into 2 column halves taken by 2 warps; partial sums combined in fixed
// order.  Kept separate from the single-image kernel: with the segment loop
// ptxas needs 72 instead of 56 registers at NB = 8 and the launch is 1.5x
// slower (C5 batch 8, s=1: 0.73 vs 1.11 ms).
template <int NB, bool IL>
__global__ void __launch_bounds__(32 * kFwdWarps) k_forward_batch(const RayEntry* __restrict__ rays, int B, int V_r,
                                                                 const int* __restrict__ sel, int n_sel,
                                                                 const float2* __restrict__ pairs, size_t pair_stride,
                                                                 int nc, const float* __restrict__ bsino,
                                                                 float* __restrict__ out, unsigned* __restrict__ rmaxv) {
  constexpr int SPLIT = 2, VPB = kFwdWarps / SPLIT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = warp % SPLIT;
  const int k = blockIdx.y * VPB + warp / SPLIT;
  const bool vk = k < n_sel;
  const int t = blockIdx.x * 32 + lane;
  const int bz0 = blockIdx.z * NB;
  const int g = (sel && vk) ? __ldg(sel + k) : k;
  const bool valid = vk && t < B;
  long long F0 = 0;
  unsigned S = 1;
  float Lc = 0.f, Ly32 = 0.f;
  int cls = 0, cl = INT_MAX, ch = INT_MIN;
  if (valid) {
    const RayEntry R = rays[(size_t)g * B + t];
    F0 = R.F0; S = R.S; Lc = R.Lc; Ly32 = R.Ly32; cls = R.flags & 3;
    if (R.c_lo < R.c_hi) { cl = R.c_lo; ch = R.c_hi; }
  }
  pdl_wait();      // the ray table is static; the pair images and b come from the predecessors
  pdl_release();
  int wcl = __reduce_min_sync(0xffffffffu, cl);
  int wch = __reduce_max_sync(0xffffffffu, ch);
  if (wcl < wch) {
    const int len = wch - wcl;
    const int c0 = wcl + (q * len) / SPLIT, c1 = wcl + ((q + 1) * len) / SPLIT;
    wcl = c0;
    wch = c1;
  }
  float sa[NB], sb[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) { sa[i] = 0.f; sb[i] = 0.f; }
  if (wcl < wch) {
    const int L = (int)pair_line(nc);
    const size_t istride = (size_t)nc * L;
    // separate layout: image i's pair image at base + i istride; interleaved
    // (IL): the group's NB pairs of element e at base + e NB
    const float2* base = pairs + cls * pair_stride + (size_t)bz0 * istride;
    const unsigned umax = (unsigned)(nc + 2);
    const long long Es = F0 + (long long)wcl * (long long)S + (long long)S + (1LL << 32);
    unsigned elo = (unsigned)Es, ehi = (unsigned)(Es >> 32);
    // u clamped to the zero pads (the carry-chained form of k_forward saves
    // 2 of ~5 NB instructions per column here and costs 6 registers at NB = 8)
    unsigned offk = (unsigned)(wcl * L + kPairPad);
#pragma unroll kFwdUnrollB
    for (int c = wcl; c < wch; ++c) {
      unsigned lo1, hi1;
      asm("add.cc.u32 %0, %2, %4;\n\taddc.u32 %1, %3, 0;" : "=r"(lo1), "=r"(hi1) : "r"(elo), "r"(ehi), "r"(S));
      const float mf = (float)min(elo, S);
      const unsigned e = offk + min(ehi, umax);
      MS2G_DASSERT(e < (unsigned)(nc * L));
      if (IL) {
        const float4* q = reinterpret_cast<const float4*>(base + (size_t)e * NB);
#pragma unroll
        for (int i = 0; i < NB; i += 2) {
          float4 v;
          asm("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];"
              : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(q + i / 2));
          sa[i] += v.x;
          sb[i] = fmaf(mf, v.y, sb[i]);
          sa[i + 1] += v.z;
          sb[i + 1] = fmaf(mf, v.w, sb[i + 1]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          float pl, pu;
          asm("{\n\t.reg .u64 ad;\n\tmad.wide.u32 ad, %2, 8, %3;\n\tld.global.nc.v2.f32 {%0, %1}, [ad];\n\t}"
              : "=f"(pl), "=f"(pu) : "r"(e), "l"(base + i * istride));
          sa[i] += pl;
          sb[i] = fmaf(mf, pu, sb[i]);
        }
      }
      elo = lo1;
      ehi = hi1;
      offk += L;
    }
  }
  __shared__ float2 red[kFwdWarps][NB][32];
#pragma unroll
  for (int i = 0; i < NB; ++i) red[warp][i][lane] = make_float2(sa[i], sb[i]);
  __syncthreads();
  if (q != 0) return;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    float r = 0.f;
    if (valid) {
      float a = 0.f, b = 0.f;
#pragma unroll
      for (int j = 0; j < SPLIT; ++j) {
        const float2 v = red[warp + j][i][lane];
        a += v.x;
        b += v.y;
      }
      r = fmaf(Lc, a, Ly32 * b);
      if (bsino) r -= __ldg(bsino + ((size_t)(bz0 + i) * V_r + g) * B + t);
      out[((size_t)(bz0 + i) * n_sel + k) * B + t] = r;
    }
    fwd_view_max(rmaxv, (size_t)(bz0 + i) * V_r + k, vk, valid, r);
  }
}

template <int NB>
static void fwd_launch_batch(int n_sel, int batch, cudaStream_t s, ms2g_plan* p, const FactorTables& f,
                             const int* d_sel, const float* b, float* out) {
  dim3 grid((p->B + 31) / 32, (n_sel + kFwdWarps / 2 - 1) / (kFwdWarps / 2), batch / NB);
  // Interleaved pairs (MS2G_FWD_INTERLEAVE, as the pair prep) measured 2x
  // SLOWER (C5 batch 8, s=1: 1.53 vs 0.735 ms): a lane's 64 B come in four
  // 16-B loads whose warp addresses are 64 B apart, so each load spans 16
  // cache lines -- 4 x 16 L1 wavefronts per column against 8 x 2 for the
  // separate layout (profiles/r02_fwd_batch_probe.log).  Kept as the switch.
  static const bool il_on = getenv("MS2G_FWD_INTERLEAVE") != nullptr;
  if (!il_on)
    (void)launch_k(k_forward_batch<NB, false>, grid, dim3(32 * kFwdWarps), 0, s, f.d_rays, p->B, p->V_r, d_sel, n_sel,
                   (const float2*)p->w_pair, p->pair_stride, f.nc, b, out, p->w_rmaxv);
  else
    (void)launch_k(k_forward_batch<NB, true>, grid, dim3(32 * kFwdWarps), 0, s, f.d_rays, p->B, p->V_r, d_sel, n_sel,
                   (const float2*)p->w_pair, p->pair_stride, f.nc, b, out, p->w_rmaxv);
}

template <int NB, int SPLIT, int SEG, int TILE = 1>
static void fwd_launch2(int n_sel, int batch, cudaStream_t s, ms2g_plan* p, const FactorTables& f,
                        const int* d_sel, const float* b, float* out, const int* order_sel) {
  constexpr int VPB = kFwdWarps / SPLIT;
  dim3 grid((p->B + 31) / 32, (n_sel + VPB - 1) / VPB, batch / NB);
  // longest-first block order: the plan's for full-view launches, the
  // caller's (built for this view list with fwd_views_per_block) for subsets
  static const bool no_order = getenv("MS2G_FWD_NO_ORDER") != nullptr;   // experiment switch
  const int* order = no_order ? nullptr
                              : (d_sel ? order_sel
                                       : ((n_sel == p->V_r && f.fwd_order_vpb == VPB) ? f.d_fwd_order : nullptr));
  // experiment / test switch: every warp on the clamped path (bitwise equal)
  static const int allow_fast = getenv("MS2G_FWD_NO_FAST") ? 0 : 1;
  (void)launch_k(k_forward<NB, SPLIT, SEG, TILE>, grid, dim3(32 * kFwdWarps), 0, s, f.d_rays, p->B, p->V_r, d_sel, n_sel,
                 (const float2*)p->w_pair, p->pair_stride, f.nc, b, out, order, allow_fast, p->w_rmaxv);
}

// views per block of the single-image forward kernel for a launch of n_sel
// views x batch images (4 segments per ray: one warp per view, or 4 warps per
// view when the launch is under ~1.5 waves of warps)
int fwd_views_per_block(const ms2g_plan* p, int n_sel, int batch) {
  const long long units = (long long)((p->B + 31) / 32) * n_sel * batch;
  const long long wave = (long long)p->sm_count * 64;
  return (2 * units < 3 * wave) ? kFwdWarps / 4 : kFwdWarps;
}

int launch_forward(ms2g_plan* p, const FactorTables& f, const float* b, float* out, const int* d_sel, int n_sel,
                   int batch, cudaStream_t s, const int* order_sel) {
  if (n_sel <= 0) return MS2G_OK;
  // batches share one traversal (k_forward_batch) on coarse grids; at
  // n_c >= 512 the single-image kernel (4-view warps, 64 registers) run over
  // the batch is faster per image (C5 s=1: 0.0893 ms per image against 0.741
  // / 8 = 0.0926 ms; s=2 keeps the shared traversal, 0.26 against 0.41 ms)
  static const bool nb_env = getenv("MS2G_FWD_BATCH_SHARED") != nullptr;   // experiment switch
  const int nb = (f.nc >= 512 && !nb_env) ? 1 : batch_group(batch);
  const int slot = timing_begin(p, 0, f.factor, s);
  // Work-unit shape (measured on B200, CUDA events):
  //  * single images: 4 segments per ray; one warp takes all four (SPLIT 1:
  //    C4 s=1 0.78 -> 0.73 ms, C3 0.126 -> 0.123 ms) unless the launch is
  //    under ~1.5 waves of warps, where 4 warps share them (SPLIT 4: C4's
  //    180-view shard 0.157 -> 0.138 ms);
  //  * batches: k_forward_batch, 2 column halves on 2 warps (C5 batch 8, s=1:
  //    0.73 ms against 0.84-1.1 ms for the segmented kernel).
  if (nb == 8) fwd_launch_batch<8>(n_sel, batch, s, p, f, d_sel, b, out);
  else if (nb == 4) fwd_launch_batch<4>(n_sel, batch, s, p, f, d_sel, b, out);
  else if (nb == 2) fwd_launch_batch<2>(n_sel, batch, s, p, f, d_sel, b, out);
  else if (fwd_views_per_block(p, n_sel, batch) != kFwdWarps) {
    // short launches (view shards, registered subsets): 4 warps per view,
    // 4 segments per ray; SPLIT x SEG = 2 x 4, 4 x 8, 2 x 8 measured slower
    // ("tried and measured")
    fwd_launch2<1, 4, 4>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
  } else {
    static const int tile = getenv("MS2G_FWD_TILE") ? atoi(getenv("MS2G_FWD_TILE")) : (kFwdWarps == 8 ? 8 : 4);   // experiment switch
    if (tile == kFwdWarps && tile == 8) fwd_launch2<1, 1, 4, (kFwdWarps == 8 ? 8 : 4)>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
    else if (tile == 4) {
      // column segments per ray: each about <= 256 columns long (the fp32
      // summation error of a segment grows with its length; C4 forward parity
      // 1.9e-6 with 4 segments of 256 at 1024^2, 2.8e-6 with 2 of 512), so 4
      // at n_c >= 1024 and 2 below (C4 s=2: 0.297 -> 0.280 ms)
      static const int seg_env = getenv("MS2G_FWD_SEG") ? atoi(getenv("MS2G_FWD_SEG")) : 0;   // experiment switch
      const int seg = seg_env ? seg_env : (f.nc >= 1024 ? 4 : 2);
      if (seg == 2) fwd_launch2<1, 1, 2, 4>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
      else if (seg == 1) fwd_launch2<1, 1, 1, 4>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
      else if (seg == 8) fwd_launch2<1, 1, 8, 4>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
      else fwd_launch2<1, 1, 4, 4>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
    }
    else if (tile == 2) fwd_launch2<1, 1, 4, 2>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
    else fwd_launch2<1, 1, 4, 1>(n_sel, batch, s, p, f, d_sel, b, out, order_sel);
  }
  const int rc = check_launch("k_forward");
  timing_end(p, slot, s);
  return rc;
}

// --------------------------------------------------------------- adjoint --
// Tile-driven ray scatter.  Two tile families cover the image: X-tiles
// (32 columns x H rows) take only the major-x rays, Y-tiles (32 rows x H
// columns) only the major-y rays, so every block uses one accumulator layout
// T[minor][major] whose long side is the MINOR axis: a ray of slope <= 1 then
// crosses most of the 32 major lanes inside the tile (modelled lane
// utilisation 0.84 at H = 64, 0.88 at H = 96, against 0.73 for 32x32 tiles).
// A block owns one tile and a chunk of views (blocks start longest first, from
// the plan's cost table); each warp takes one view at a time and walks the rays that
// meet the tile, one per step, with LANE = major index inside the tile.  A
// lane only touches its own major line of the warp's private accumulator (no
// atomics, fixed order, deterministic) and the lane is the fastest-varying
// coordinate, so every access of a step hits 32 distinct banks.  The bins
// that meet each (tile, view) are precomputed per plan (k_bp_ranges), split
// into <= 2 runs of one ray class, so the addressing constants are
// loop-invariant.  The ray records of the next 32-ray round are fetched from
// global memory while the current round is processed (software pipeline).
//
// Step (the forward's weights): the lane's end coordinate E = Et + lane*S
// gives u = floor(E) + 1 (tile-relative; upper row u - 1, lower row u - 2) and
// m = min(frac32(E), S):   T[u - 1] += m (Ly32 r),   T[u - 2] += (S - m)(Ly32 r)
// (Lc = S Ly32 up to rounding).  u is clamped to H + 2 (unsigned, so
// negatives clamp too) and every warp window has two pad rows on each side
// (shared between neighbouring windows), so no predicate is needed.  Record
// per ray: {lo(Et), hi(Et), S, Ly32 r}, one broadcast LDS.128 per step.  The
// kernel is bound by the L1/shared data pipe (91-95 % of the peak): ~4.2
// shared-memory wavefronts per step (each 32-bit LDS / STS 1, the broadcast
// record almost free; ncu at C4 s=1) plus the ray-record / residual loads.
//
// The X- and Y-families write separate partial planes (per view chunk too);
// k_chunk_reduce sums them in fixed order.
constexpr int kBT = 32;                          // major extent (lanes)
#ifndef MS2G_BW
#define MS2G_BW 4
#endif
constexpr int kBW = MS2G_BW;                     // warps per block
constexpr int kPadR = 2;
// minor extent H of the tiles: 64 (6 blocks of 36 KB per SM) or, for n_c >=
// 1024, 96 (4 blocks of 51 KB; lane utilisation 0.88, measured 10 % faster
// at 1024^2 and slower on coarser grids)
#ifndef MS2G_BH96_MIN_NC
#define MS2G_BH96_MIN_NC 1024
#endif
// The minor extent of the fixed-point form's tiles for full view sets:
// taller tiles cover more of each ray per visit (fewer rays clipped by the
// tile's minor edges, fewer record loads per segment) and, with the windows
// shared by the block's warps, cost no more shared memory.  View shards and
// small plans keep the shorter tiles (more blocks per launch).  Measured at
// C4 (CUDA events, C4 adjoint s=1 / s=2): 96 -> 256 at 1024^2 1.13 -> 1.02 ms
// (320 no better), 64 -> 128 at 512^2 0.58 -> 0.52 ms (192 / 256 no better,
// one shared window each); the 180-view shard prefers 128 at 1024^2 (0.169
// against 0.188 ms at 96, 0.201 at 256) and 128 at 512^2 (0.101 against 0.105).
int bp_height(int nc, int V_r) {
  static const int h1 = getenv("MS2G_BP_H1024") ? atoi(getenv("MS2G_BP_H1024")) : 0;   // experiment switches
  static const int h2 = getenv("MS2G_BP_H512") ? atoi(getenv("MS2G_BP_H512")) : 0;
  const bool full = V_r >= 720 && !getenv("MS2G_BP_FP32");
  if (nc >= MS2G_BH96_MIN_NC) return h1 ? h1 : (full ? 256 : 128);
  if (nc >= 512) return h2 ? h2 : 128;
  return 64;
}
// Warps per block and accumulator windows: the fp32 form needs one window
// per warp (plain read-modify-writes); the fixed-point form's integer adds
// are atomic, so at H = 96 two warps share a window -- twice the warps
// (latency hiding: the step is a chain of dependent integer / FMA
// operations) in the same shared memory: C4 s=1 1.17 -> 1.13 ms.  At H = 64
// 8 warps (or 2 windows) measured slower (0.60 against 0.58 ms at C4 s=2).
#ifndef MS2G_FX96_W
#define MS2G_FX96_W 8
#endif
#ifndef MS2G_FX96_WIN
#define MS2G_FX96_WIN 4
#endif
#ifndef MS2G_FX64_W
#define MS2G_FX64_W 4
#endif
#ifndef MS2G_FX64_WIN
#define MS2G_FX64_WIN 4
#endif
template <bool FX, int H>
struct BpWarps {
  static constexpr int kW = FX ? (H >= 96 ? MS2G_FX96_W : MS2G_FX64_W) : kBW;        // warps per block
  // accumulator windows: 4 at H <= 96, 2 at H = 128 .. 192, 1 from H = 256
#ifndef MS2G_FX_ONEWIN_H
#define MS2G_FX_ONEWIN_H 128
#endif
  static constexpr int kWin = FX ? (H >= MS2G_FX_ONEWIN_H ? 1 : H >= 128 ? 2 : H >= 96 ? MS2G_FX96_WIN : MS2G_FX64_WIN) : kBW;
};
template <int H, bool FX = false>
struct BpShape {
  // one shared window (H >= 256): 36 pad rows per side hold every row a ray
  // of the tile's range can reach over the tile's 32 columns (slope <= 1, the
  // range table's margin), so the step needs no clamp; otherwise 2 rows and
  // the row index clamped into them
  static constexpr bool kNoClamp = FX && BpWarps<FX, H>::kWin == 1;
  static constexpr int kPad = kNoClamp ? 36 : kPadR;
  static constexpr int kWinR = H + kPad;                 // rows per window (+ shared pads)
  static constexpr int kAccRows = kPad + BpWarps<FX, H>::kWin * kWinR;
  static constexpr size_t kSmem = sizeof(float) * kAccRows * kBT;
  // resident blocks per SM: 24 (H = 64) / 16 (H = 96) warps of the fp32 form; the
  // fixed-point form keeps the block count (shared memory) at twice the warps
#ifndef MS2G_FX_WARPS_SM
#define MS2G_FX_WARPS_SM 32
#endif
  static constexpr int kMinBlocks = (FX && H >= 96) ? MS2G_FX_WARPS_SM / BpWarps<FX, H>::kW : (H <= 64 ? 24 : 16) / kBW;
};

struct BpTiling {
  int maj, mnr, per;   // tiles along the major axis, along the minor axis, per family
};
static inline BpTiling bp_tiling(int nc, int H) {
  BpTiling t;
  t.maj = (nc + kBT - 1) / kBT;
  t.mnr = (nc + H - 1) / H;
  t.per = t.maj * t.mnr;
  return t;
}
int bp_tile_count(int nc, int H) { return 2 * bp_tiling(nc, H).per; }

// Per (tile, view): bins [ta_r, te_r] of run r (r < n) of the tile family's
// major axis, class cls_r.
__global__ void k_bp_ranges(const ViewEntry* __restrict__ views, int V_r, int B, int nc, int H, int tmaj, int per,
                            int4* __restrict__ out, int* __restrict__ err) {
  const size_t n = (size_t)2 * per * V_r;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int g = (int)(i % V_r);
    const int tile = (int)(i / V_r);
    const int fam = tile >= per;
    const int ti = tile - fam * per;
    const int c0 = (ti % tmaj) * kBT, m0 = (ti / tmaj) * H;
    const int c1 = min(c0 + kBT, nc), m1 = min(m0 + H, nc);
    const float x0 = fam ? m0 : c0, x1 = fam ? m1 : c1, y0 = fam ? c0 : m0, y1 = fam ? c1 : m1;
    const ViewEntry V = views[g];
    float tmin = INFINITY, tmax = -INFINITY;
    for (int c = 0; c < 4; ++c) {
      const float px = (c & 1) ? x1 : x0, py = (c & 2) ? y1 : y0;
      const float dx = px - V.Sx, dy = py - V.Sy;
      const float tau = V.off + V.scale * (dx * V.ex + dy * V.ey) / (dx * V.nx + dy * V.ny);
      tmin = fminf(tmin, tau);
      tmax = fmaxf(tmax, tau);
    }
    const int t_lo = max(0, (int)floorf(tmin - 0.01f));
    const int t_hi = min(B - 1, (int)ceilf(tmax + 0.01f));
    int nr = 0, ta[2] = {0, 0}, te[2] = {-1, -1}, cl[2] = {0, 0};
    for (int sg = 0; sg < V.nseg; ++sg) {
      if (((V.seg_cls[sg] & kMajorY) != 0) != (fam != 0)) continue;
      const int a = max(t_lo, (int)V.seg_t[sg]), e = min(t_hi, (int)V.seg_t[sg + 1] - 1);
      if (a > e) continue;
      if (nr == 2) { atomicExch(err, 1); break; }
      ta[nr] = a; te[nr] = e; cl[nr] = V.seg_cls[sg]; ++nr;
    }
    out[i] = make_int4((ta[0] & 0xffff) | (te[0] << 16), (ta[1] & 0xffff) | (te[1] << 16),
                       cl[0] | (cl[1] << 8) | (nr << 16), 0);
  }
}

int launch_bp_ranges(const FactorTables& f, int V_r, int B, int4* out, int* err, cudaStream_t s) {
  const int H = f.bp_h;
  const BpTiling t = bp_tiling(f.nc, H);
  const size_t n = (size_t)2 * t.per * V_r;
  const int blocks = (int)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
  k_bp_ranges<<<blocks, 256, 0, s>>>(f.d_views, V_r, B, f.nc, H, t.maj, t.per, out, err);
  return check_launch("k_bp_ranges");
}

// The adjoint's steps over one round of <= 32 ray records (one broadcast
// LDS.128 each): per step the lane's end coordinate, the two weights and two
// shared read-modify-writes, the lower row at a compile-time offset.
#ifndef MS2G_BP_UNROLL
#define MS2G_BP_UNROLL 8
#endif
constexpr int kBpUnroll = MS2G_BP_UNROLL;
template <bool MIR, int H, bool FX = false, bool NOCLAMP = false>
__device__ __forceinline__ void bp_steps(const float4* __restrict__ p4, const int* __restrict__ p1, int nrays,
                                         int lane, unsigned sbase, unsigned acc0, unsigned acc1) {
  constexpr int kStride = MIR ? -4 * kBT : 4 * kBT;   // bytes per row step of u
  (void)acc0;
  (void)acc1;
  float4 a = p4[0];
#pragma unroll kBpUnroll
  for (int q = 0; q < nrays; ++q) {
    const float4 an = p4[q + 1];
    const unsigned S = __float_as_uint(a.z);
    unsigned lo, u;
    asm("mad.lo.cc.u32 %0, %2, %3, %4;\n\tmadc.hi.u32 %1, %2, %3, %5;"
        : "=r"(lo), "=r"(u)
        : "r"((unsigned)lane), "r"(S), "r"(__float_as_uint(a.x)), "r"(__float_as_uint(a.y)));
    const unsigned m = min(lo, S);
    const float mu = (float)m, ml = FX ? 0.f : (float)(S - m);
    const unsigned adu = sbase + (NOCLAMP ? u : min(u, (unsigned)(H + 2))) * (unsigned)kStride;   // mod 2^32
    MS2G_DASSERT(adu >= acc0 && adu < acc1 && adu - (unsigned)kStride >= acc0 && adu - (unsigned)kStride < acc1);
    if (FX) {
      // up = round(m K); dn = round(S K) - round(m K), with round(S K) + M
      // precomputed per ray (p1): one FFMA and two IADDs for both weights
      const int ub = __float_as_int(fmaf(mu, a.w, 12582912.f));
      const int up = ub - 0x4B400000;
      const int dn = p1[q] - ub;
      if (MIR) asm volatile("red.shared.add.u32 [%0], %1;\n\tred.shared.add.u32 [%0+128], %2;" :: "r"(adu), "r"(up), "r"(dn) : "memory");
      else asm volatile("red.shared.add.u32 [%0], %1;\n\tred.shared.add.u32 [%0+-128], %2;" :: "r"(adu), "r"(up), "r"(dn) : "memory");
    } else
    if (MIR)
      asm volatile("{\n\t.reg .f32 c0, c1;\n\t"
                   "ld.shared.f32 c0, [%0];\n\t"
                   "ld.shared.f32 c1, [%0+128];\n\t"
                   "fma.rn.f32 c0, %1, %3, c0;\n\t"
                   "fma.rn.f32 c1, %2, %3, c1;\n\t"
                   "st.shared.f32 [%0], c0;\n\t"
                   "st.shared.f32 [%0+128], c1;\n\t}"
                   :: "r"(adu), "f"(mu), "f"(ml), "f"(a.w) : "memory");
    else
      asm volatile("{\n\t.reg .f32 c0, c1;\n\t"
                   "ld.shared.f32 c0, [%0];\n\t"
                   "ld.shared.f32 c1, [%0+-128];\n\t"
                   "fma.rn.f32 c0, %1, %3, c0;\n\t"
                   "fma.rn.f32 c1, %2, %3, c1;\n\t"
                   "st.shared.f32 [%0], c0;\n\t"
                   "st.shared.f32 [%0+-128], c1;\n\t}"
                   :: "r"(adu), "f"(mu), "f"(ml), "f"(a.w) : "memory");
    a = an;
  }
}

template <int H, bool FX>
__global__ void __launch_bounds__(32 * BpWarps<FX, H>::kW, BpShape<H, FX>::kMinBlocks) k_backward(const RayBp* __restrict__ rays,
                                                          const int4* __restrict__ ranges, int V_r, int B,
                                                          const int* __restrict__ sel, int n_sel,
                                                          const float* __restrict__ sino, float* __restrict__ part,
                                                          int nc, int tmaj, int per, int chx, int vpcx, int vpcy,
                                                          const int* __restrict__ order,
                                                          const float* __restrict__ bpw, float lc_max,
                                                          const unsigned* __restrict__ rmaxv) {
  extern __shared__ float4 dyn_smem[];
  float* acc = reinterpret_cast<float*>(dyn_smem);   // kAccRows x kBT (dynamic: may exceed 48 KB)
  constexpr int kBH = H, kWinR = BpShape<H, FX>::kWinR, kAccRows = BpShape<H, FX>::kAccRows;
  constexpr int NW = BpWarps<FX, H>::kW, NWIN = BpWarps<FX, H>::kWin;   // warps, windows (warp w -> window w % NWIN)
  __shared__ float4 st4[NW][33];   // entry 32 is a pipeline pad
  __shared__ int st1[NW][33];      // FX: round(S K) + 1.5 * 2^23 (as float bits) per ray
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // blockIdx.x = (family, view chunk, tile): X-family blocks first
  const int bx = order ? __ldg(order + blockIdx.x) : (int)blockIdx.x, bz = blockIdx.z;
  const int fam = bx >= per * chx;                 // 0: X-tile (major x), 1: Y-tile (major y)
  const int bi = bx - fam * per * chx;
  const int ti = bi % per, chunk = bi / per;
  const int tile = fam * per + ti;                 // index into the range table
  MS2G_DASSERT(bx >= 0 && bx < (int)gridDim.x && ti < per);
  const int vpc = fam ? vpcy : vpcx;
  const int plane = fam ? chx + chunk : chunk;
  const int c0 = (ti % tmaj) * kBT, m0 = (ti / tmaj) * kBH;   // major / minor origin
  const int win = warp % NWIN;
  constexpr int kPad = BpShape<H, FX>::kPad;
  float* T = acc + (kPad + win * kWinR) * kBT;
  for (int i = threadIdx.x; i < kAccRows * kBT; i += 32 * NW) acc[i] = 0.f;
  __syncthreads();
  pdl_wait();      // the residual sinogram comes from the forward
  pdl_release();
  const int kb = chunk * vpc, ke = min(n_sel, kb + vpc);
  const float* sb = sino + (size_t)bz * n_sel * B;
  const int4* trange = ranges + (size_t)tile * V_r;

  // ---- round iterator: (view k, run, [tb, te]) of this warp ----
  int vbase = kb + warp - 32 * NW;      // first view of the current 32-view batch
  int g_lane = 0;                       // rank-local view held by this lane for the batch
  int4 rr_lane = make_int4(0, 0, 0, 0); // its range record
  int j = 31;                           // index of the current view within the batch
  int k = -1, g = 0, nr = 0, run = 0, tb = 0, te = -1, cls = 0;
  int ra0 = 0, re0 = -1, ra1 = 0, re1 = -1, cls0 = 0, cls1 = 0;
  auto next_round = [&]() -> bool {
    tb += 32;
    while (tb > te) {
      ++run;
      if (run >= nr) {
        ++j;
        if (j == 32) {                    // load the next batch of 32 views (lane j <-> view)
          vbase += 32 * NW;
          if (vbase >= ke) return false;
          const int kk = vbase + lane * NW;
          g_lane = (kk < ke) ? (sel ? __ldg(sel + kk) : kk) : 0;
          rr_lane = (kk < ke) ? __ldg(trange + g_lane) : make_int4(0, 0, 0, 0);
          j = 0;
        }
        k = vbase + j * NW;
        if (k >= ke) return false;
        g = __shfl_sync(0xffffffffu, g_lane, j);
        const int rx = __shfl_sync(0xffffffffu, rr_lane.x, j);
        const int ry = __shfl_sync(0xffffffffu, rr_lane.y, j);
        const int rz = __shfl_sync(0xffffffffu, rr_lane.z, j);
        ra0 = rx & 0xffff; re0 = (short)(rx >> 16); ra1 = ry & 0xffff; re1 = (short)(ry >> 16);
        cls0 = rz & 0xff; cls1 = (rz >> 8) & 0xff; nr = (rz >> 16) & 0xff;
        run = -1;
        continue;
      }
      tb = run ? ra1 : ra0;
      te = run ? re1 : re0;
      cls = run ? cls1 : cls0;
    }
    return true;
  };

  // Fixed-point accumulation (FX): each warp window accumulates integers
  // round(w r sigma) with the native shared-memory integer add (ATOMS.ADD:
  // one instead of two shared wavefronts per update, and order-independent).
  // sigma = 2^e per warp, the largest power of two with
  //   sum over the warp's views of W_v * max|r|  < 2^31  (no overflow: W_v
  //     bounds the weight a pixel receives from one view, plan_bp_bounds)
  //   Lc_max * max|r|                            < 2^22  (every contribution
  //     fits the FFMA-against-1.5*2^23 rounding trick)
  // from the per-view bounds of the warp's views.  A non-finite residual
  // makes the warp's window NaN (the solve's divergence check).
  __shared__ float s_inv[NWIN];
  __shared__ int s_bad[NWIN];
  __shared__ float s_w[NW];
  __shared__ unsigned s_r[NW];
  float sig = 1.f;
  if (FX) {
    // the warp's views are kb + warp + NW j: W and max |r| per view (the
    // forward's epilogue wrote rmaxv; a caller's sinogram got launch_view_absmax),
    // combined over the warps sharing the window
    unsigned rbits = 0;
    float wsum = 0.f;
    for (int kk = kb + warp + NW * lane; kk < ke; kk += 32 * NW) {
      const int gg = sel ? __ldg(sel + kk) : kk;
      wsum += __ldg(bpw + (size_t)fam * V_r + gg);
      rbits = max(rbits, __ldcg(rmaxv + (size_t)bz * V_r + kk));
    }
    rbits = __reduce_max_sync(0xffffffffu, rbits);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if (lane == 0) {
      s_w[warp] = wsum;
      s_r[warp] = rbits;
    }
    __syncthreads();
    wsum = 0.f;
    rbits = 0;
    for (int w = win; w < NW; w += NWIN) {     // fixed order
      wsum += s_w[w];
      rbits = max(rbits, s_r[w]);
    }
    int e = 0;
    const bool bad = rbits >= 0x7f800000u;   // inf / nan
    if (!bad && rbits != 0u) {
      const double rm = (double)__uint_as_float(rbits);
      const double t = fmin(2.1e9 / ((double)wsum * rm), 4.19e6 / ((double)lc_max * rm));   // < 2^31, < 2^22
      e = min(126, max(-126, ilogb(t)));
    }
    sig = ldexpf(1.f, e);      // a power of two: the conversion back is exact
    if (lane == 0 && warp < NWIN) {
      s_inv[win] = ldexpf(1.f, -e);
      s_bad[win] = bad ? 1 : 0;
    }
  }
  run = 0; nr = 0; te = -1; tb = 0;
  bool have = next_round();
  RayBp Rn;
  float rn = 0.f;
  int tn = tb + lane;
  if (have && tn <= te) {
    Rn = rays[(size_t)g * B + tn];
    rn = __ldg(sb + (size_t)k * B + tn);
  }
  const unsigned tbase = (unsigned)__cvta_generic_to_shared(T) + 4u * (unsigned)lane;
  const unsigned acc0 = (unsigned)__cvta_generic_to_shared(acc), acc1 = acc0 + 4u * kAccRows * kBT;
  (void)acc0;
  (void)acc1;
  while (have) {
    // commit the prefetched round to shared memory (tile-relative end coordinate, +1 row)
    const int cte = te, ctb = tb;
    const bool mir = cls & kMirror;
    if (tn <= cte) {
      const int mb = mir ? nc - m0 - kBH : m0;
      const long long Et = Rn.F0 + (long long)c0 * (long long)Rn.S + (long long)Rn.S - ((long long)(mb - 1) << 32);
      const float K = FX ? Rn.Ly32 * (rn * sig) : Rn.Ly32 * rn;
      st4[warp][lane] = make_float4(__uint_as_float((unsigned)Et), __uint_as_float((unsigned)(Et >> 32)),
                                    __uint_as_float(Rn.S), K);
      if (FX) st1[warp][lane] = __float_as_int(fmaf((float)Rn.S, K, 12582912.f));
    }
    __syncwarp();
    // fetch the next round while this one is processed
    have = next_round();
    tn = tb + lane;
    if (have && tn <= te) {
      Rn = rays[(size_t)g * B + tn];
      rn = __ldg(sb + (size_t)k * B + tn);
    }
    // upper row u - 1 -> byte address sbase + u * stride, the lower row one
    // stride back (an immediate offset: the loop is instantiated per sign)
    //   plain:  phys row = u - 1      (sbase at row -1)
    //   mirror: phys row = kBH - u    (sbase at row kBH, negative stride)
    const int nrays = min(32, cte - ctb + 1);
    constexpr bool kNC = BpShape<H, FX>::kNoClamp;
    if (mir) bp_steps<true, kBH, FX, kNC>(st4[warp], st1[warp], nrays, lane, tbase + 4u * kBT * kBH, acc0, acc1);
    else bp_steps<false, kBH, FX, kNC>(st4[warp], st1[warp], nrays, lane, tbase - 4u * kBT, acc0, acc1);
    __syncwarp();
  }
  __syncthreads();
  // Sum the warp windows in fixed order: element (row l, lane) of the tile.
  constexpr int kPer = kBT * kBH / (32 * NW);
  float sum[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int idx = threadIdx.x + i * 32 * NW;    // row idx / 32, lane idx % 32
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < NWIN; ++w) {
      const float v = acc[(kPad + w * kWinR) * kBT + idx];
      if (FX) s += s_bad[w] ? __int_as_float(0x7fc00000) : (float)__float_as_int(v) * s_inv[w];
      else s += v;
    }
    sum[i] = s;
  }
  const size_t np = (size_t)nc * nc;
  const int nplanes = chx + (int)((gridDim.x - per * chx) / per);   // X chunks + Y chunks
  MS2G_DASSERT(plane < nplanes);
  float* dst = part + ((size_t)bz * nplanes + plane) * np;
  if (!fam) {       // X-tile: row l = y - m0, lane = x - c0 (coalesced)
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int idx = threadIdx.x + i * 32 * NW;
      const int yy = m0 + (idx >> 5), xx = c0 + (idx & 31);
      if (yy < nc && xx < nc) dst[(size_t)yy * nc + xx] = sum[i];
    }
  } else {          // Y-tile: row l = x - m0, lane = y - c0; transpose through a (kBH+1)-stride scratch
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int idx = threadIdx.x + i * 32 * NW;
      acc[(idx & 31) * (kBH + 1) + (idx >> 5)] = sum[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int idx = threadIdx.x + i * 32 * NW;    // y = idx / kBH, x = idx % kBH (tile-relative)
      const int ly = idx / kBH, lx = idx % kBH;
      const int yy = c0 + ly, xx = m0 + lx;
      if (yy < nc && xx < nc) dst[(size_t)yy * nc + xx] = acc[ly * (kBH + 1) + lx];
    }
  }
}

// ------------------------------------------------ adjoint, gather variant --
// Pixel-driven gather (north-star subsystem (2), first alternative): one
// thread per pixel accumulates in a register over the views of its chunk;
// per (pixel, view) the candidate bins are the detector interval of the
// pixel's four corners (the fan projection of a convex pixel), and each
// candidate ray's weight is evaluated with the SAME fixed-point end
// coordinate as the forward and the scatter: with E = F0 + (c + 1) S at the
// pixel's major column c, the pixel (frame row k) receives m Ly32 when
// floor(E) = k and (S - m) Ly32 when floor(E) - 1 = k, m = min(frac32(E), S)
// (zero otherwise).  No shared memory, no atomics, deterministic; partial
// planes per view chunk as the scatter (k_chunk_reduce and the fused
// epilogues sum them).  Kept as the measured alternative (MS2G_BP_VARIANT=
// gather): its per-segment instruction count is ~3x the scatter's (DESIGN.md
// "adjoint design", profiles/r02_adjoint_variants.md).
__global__ void __launch_bounds__(256) k_backward_gather(const RayEntry* __restrict__ rays,
                                                         const ViewEntry* __restrict__ views, int B,
                                                         const int* __restrict__ sel, int n_sel,
                                                         const float* __restrict__ sino, float* __restrict__ part,
                                                         int nc, int vpc, int nplanes) {
  const int tiles_x = (nc + 31) / 32, per = tiles_x * ((nc + 7) / 8);
  const int chunk = blockIdx.x / per, ti = blockIdx.x - chunk * per;
  const int j = (ti % tiles_x) * 32 + threadIdx.x, i = (ti / tiles_x) * 8 + threadIdx.y;
  if (i >= nc || j >= nc) return;
  const size_t bz = blockIdx.z, np = (size_t)nc * nc;
  const int kb = chunk * vpc, ke = min(n_sel, kb + vpc);
  const float* sb = sino + bz * n_sel * B;
  float acc = 0.f;
  for (int k = kb; k < ke; ++k) {
    const int g = sel ? __ldg(sel + k) : k;
    const ViewEntry V = views[g];
    float tmin = INFINITY, tmax = -INFINITY;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float dx = (float)(j + (q & 1)) - V.Sx, dy = (float)(i + (q >> 1)) - V.Sy;
      const float tau = fmaf(V.scale, __fdividef(dx * V.ex + dy * V.ey, dx * V.nx + dy * V.ny), V.off);
      tmin = fminf(tmin, tau);
      tmax = fmaxf(tmax, tau);
    }
    const int t0 = max(0, (int)ceilf(tmin - 0.01f)), t1 = min(B - 1, (int)floorf(tmax + 0.01f));
    const RayEntry* rv = rays + (size_t)g * B;
    const float* rr = sb + (size_t)k * B;
    for (int t = t0; t <= t1; ++t) {
      const RayEntry R = rv[t];
      const int cls = R.flags & 3;
      const int c = (cls & kMajorY) ? i : j;
      const int mn = (cls & kMajorY) ? j : i;
      const int kf = (cls & kMirror) ? nc - 1 - mn : mn;
      const long long E = R.F0 + (long long)(c + 1) * (long long)R.S;
      const int fl = (int)(E >> 32);
      const unsigned m = min((unsigned)E, R.S);
      float w = 0.f;
      if (fl == kf) w = (float)m * R.Ly32;
      else if (fl - 1 == kf) w = (float)(R.S - m) * R.Ly32;
      acc = fmaf(w, __ldg(rr + t), acc);
    }
  }
  part[(bz * nplanes + chunk) * np + (size_t)i * nc + j] = acc;
}

// out = scale * sum of the nplanes partial planes (+ out if accumulate), fixed
// order.  grid.y = batch image (no index division).
__global__ void __launch_bounds__(256) k_chunk_reduce(const float* __restrict__ part, int nplanes, size_t np,
                                                      float* __restrict__ out, float scale, int accumulate, int G) {
  pdl_wait();
  pdl_release();
  __shared__ PlaneSmem sm;
  const size_t b = blockIdx.y;
  const float* src = part + b * nplanes * np;
  float* ob = out + b * np;
  const int tid = threadIdx.y * 32 + threadIdx.x, tile = plane_tile(G);
  for (size_t p0 = (size_t)blockIdx.x * tile; p0 < np; p0 += (size_t)gridDim.x * tile) {
    sum_planes(src, nplanes, np, p0, G, sm);
    const size_t p = p0 + tid;
    if (tid < tile && p < np) {
      float v = scale * sm.tot[tid];
      if (accumulate) v += ob[p];
      ob[p] = v;
    }
    if (G != 1) __syncthreads();   // tot is rewritten by the next tile
  }
}

// Fused epilogues of the backprojection (the chunk sum feeds its consumer in
// the same pass; no G round trip, one launch instead of two or four).
//
// G = c * sum of the planes (fixed order, as k_chunk_reduce), then the step
// z = y - eta U_s G (as k_up_step) for the s x s fine pixels of each
// coarse pixel (y == NULL: z = U_s G); grid = coarse pixels (x: columns,
// y: rows, z: batch).
// The G = 1 rule of sum_planes (one thread per coarse pixel adding its planes
// in order) on a (columns, rows, batch) grid of (32 x 8) blocks: no index
// division, each thread writes its s x s fine pixels.
__global__ void __launch_bounds__(256) k_reduce_up_step_px(const float* __restrict__ part, int nplanes, int nc,
                                                           float c, const float* __restrict__ y,
                                                           const float* __restrict__ eta_dev, float* __restrict__ z,
                                                           int s) {
  pdl_wait();
  pdl_release();
  const int J = blockIdx.x * 32 + threadIdx.x, I = blockIdx.y * 8 + threadIdx.y;
  if (I >= nc || J >= nc) return;
  const size_t b = blockIdx.z, np = (size_t)nc * nc;
  const float* src = part + b * nplanes * np + (size_t)I * nc + J;
  float acc = 0.f;
  for (int q = 0; q < nplanes; ++q) acc += src[(size_t)q * np];
  const float G = c * acc;
  const float e = eta_dev ? *eta_dev : 0.f;
  const int n = nc * s;
  for (int a = 0; a < s; ++a) {
    const size_t row = (b * n + (size_t)(s * I + a)) * n + (size_t)s * J;
    for (int q = 0; q < s; ++q) z[row + q] = y ? fmaf(-e, G, y[row + q]) : G;   // one rounding, as k_up_step
  }
}

__global__ void __launch_bounds__(256) k_reduce_up_step(const float* __restrict__ part, int nplanes, int nc, float c,
                                                        const float* __restrict__ y,
                                                        const float* __restrict__ eta_dev, float* __restrict__ z,
                                                        int s, int G) {
  pdl_wait();
  pdl_release();
  __shared__ PlaneSmem sm;
  const size_t b = blockIdx.y, np = (size_t)nc * nc;
  const float* src = part + b * nplanes * np;
  const float e = eta_dev ? *eta_dev : 0.f;
  const int n = nc * s, tid = threadIdx.y * 32 + threadIdx.x, tile = plane_tile(G);
  for (size_t p0 = (size_t)blockIdx.x * tile; p0 < np; p0 += (size_t)gridDim.x * tile) {
    sum_planes(src, nplanes, np, p0, G, sm);
    // the s x s fine pixels of the tile's 32 coarse pixels, spread over all
    // 256 threads: consecutive threads write consecutive fine columns of a row
    const unsigned I0 = (unsigned)(p0 / (unsigned)nc), J0 = (unsigned)(p0 - (size_t)I0 * nc);
    for (int q = tid; q < tile * s * s; q += 256) {
      const int a = q / (tile * s), r = q - a * tile * s, x = r / s, u = r - x * s;
      if (p0 + x >= np) continue;
      unsigned I = I0, J = J0 + x;              // coarse pixel p0 + x (the tile may wrap a row)
      while (J >= (unsigned)nc) { J -= nc; ++I; }
      const size_t idx = (b * n + (size_t)(s * I + a)) * n + (size_t)(s * J + u);
      const float G_ = c * sm.tot[x];
      z[idx] = y ? fmaf(-e, G_, y[idx]) : G_;   // one rounding, as k_up_step
    }
    __syncthreads();   // tot is rewritten by the next tile
  }
}

// Power-iteration step (O8) fused with the chunk sum: w = sum of the planes
// (written to w_out), fp64 block partials of <v, w> and <w, w>; the last
// block to finish (atomic ticket) reduces the partials in fixed block order
// (deterministic) into pw = {L = <v,w>, 1/||w||} and, if given, the step
// L_out, eta_out = 1/L, etaf_out.  The next pair prep scales by pw[1].
__global__ void __launch_bounds__(256) k_reduce_power(const float* __restrict__ part, int nplanes, size_t np,
                                                      float* __restrict__ w_out, const float* __restrict__ v,
                                                      double* __restrict__ red, unsigned* __restrict__ ticket,
                                                      double* __restrict__ pw, double* L_out, double* eta_out,
                                                      float* etaf_out, int G) {
  pdl_wait();
  pdl_release();
  __shared__ double sd[256], sn[256];
  __shared__ PlaneSmem sm;
  __shared__ bool last;
  const int tid = threadIdx.y * 32 + threadIdx.x, tile = plane_tile(G);
  double d = 0.0, q = 0.0;
  for (size_t p0 = (size_t)blockIdx.x * tile; p0 < np; p0 += (size_t)gridDim.x * tile) {
    sum_planes(part, nplanes, np, p0, G, sm);
    const size_t i = p0 + tid;
    if (tid < tile && i < np) {
      const float w = sm.tot[tid];
      w_out[i] = w;
      const double wd = w;
      d += (double)v[i] * wd;
      q += wd * wd;
    }
    if (G != 1) __syncthreads();   // tot is rewritten by the next tile
  }
  sd[tid] = d;
  sn[tid] = q;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      sd[tid] += sd[tid + o];
      sn[tid] += sn[tid + o];
    }
    __syncthreads();
  }
  if (tid == 0) {
    red[2 * blockIdx.x] = sd[0];
    red[2 * blockIdx.x + 1] = sn[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  d = 0.0;
  q = 0.0;
  for (int b = tid; b < (int)gridDim.x; b += 256) {
    d += __ldcg(red + 2 * b);
    q += __ldcg(red + 2 * b + 1);
  }
  sd[tid] = d;
  sn[tid] = q;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) {
      sd[tid] += sd[tid + o];
      sn[tid] += sn[tid + o];
    }
    __syncthreads();
  }
  if (tid != 0) return;
  d = sd[0];
  q = sn[0];
  pw[0] = d;
  pw[1] = q > 0.0 ? 1.0 / sqrt(q) : 0.0;
  if (L_out) *L_out = d;
  if (eta_out) *eta_out = 1.0 / d;
  if (etaf_out) *etaf_out = (float)(1.0 / d);
  *ticket = 0u;                        // ready for the next launch (graph replays)
}

int launch_reduce_up_step(const float* part, int nplanes, int nc, int batch, float c, const float* y,
                          const float* eta_dev, float* z, int s, cudaStream_t st) {
  const size_t np = (size_t)nc * nc;
  const int G = plane_groups(np, nplanes);
  if (G == 1) {
    dim3 grid((nc + 31) / 32, (nc + 7) / 8, batch);
    MS2G_CUDA(launch_k(k_reduce_up_step_px, grid, dim3(32, 8), 0, st, part, nplanes, nc, c, y, eta_dev, z, s));
    return check_launch("k_reduce_up_step_px");
  }
  dim3 grid(plane_blocks(np, G, 4096), batch);
  MS2G_CUDA(launch_k(k_reduce_up_step, grid, dim3(32, kPlaneGroups), 0, st, part, nplanes, nc, c, y, eta_dev, z, s,
                     G));
  return check_launch("k_reduce_up_step");
}

// max |sino| of each view (float bits), one block per (view, image): the
// fixed-point adjoint's scale for a sinogram that did not come from
// launch_forward (ms2g_back_project)
__global__ void __launch_bounds__(256) k_view_absmax(const float* __restrict__ sino, int n_sel, int B, int V_r,
                                                     unsigned* __restrict__ rmaxv) {
  __shared__ unsigned wm[8];
  const int k = blockIdx.x, bz = blockIdx.y;
  const float* row = sino + ((size_t)bz * n_sel + k) * B;
  unsigned m = 0;
  for (int t = threadIdx.x; t < B; t += 256) m = max(m, __float_as_uint(fabsf(row[t])));
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = max(m, wm[w]);
    rmaxv[(size_t)bz * V_r + k] = max(m, wm[0]);
  }
}

int launch_view_absmax(ms2g_plan* p, const float* sino, int n_sel, int batch, cudaStream_t s) {
  if (n_sel <= 0) return MS2G_OK;
  MS2G_CUDA(launch_k(k_view_absmax, dim3(n_sel, batch), dim3(256), 0, s, sino, n_sel, p->B, p->V_r, p->w_rmaxv));
  return check_launch("k_view_absmax");
}

int launch_reduce_power(ms2g_plan* p, const float* part, int nplanes, size_t np, float* w_out, const float* v,
                        double* red, int red_blocks, unsigned* ticket, double* pw, double* L_out, double* eta_out,
                        float* etaf_out, cudaStream_t st, int tile_planes) {
  // one pass over nplanes x np floats: as many blocks as the buffer allows
  // (the fixed-order last-block reduction handles any grid size)
  // the plane rule (and with it the tiling, hence the fp64 dot order) of the
  // backprojection's plane count: an exchange path passes its one summed
  // plane with the count it came from, so every path gives the same bits
  const int G = plane_groups(np, std::max(nplanes, tile_planes));
  const int blocks = plane_blocks(np, G, red_blocks);
  MS2G_CUDA(launch_k(k_reduce_power, dim3(blocks), dim3(32, kPlaneGroups), 0, st, part, nplanes, np, w_out, v, red,
                     ticket, pw, L_out, eta_out, etaf_out, G));
  return check_launch("k_reduce_power");
}

template <int H>
static int bwd_launch(dim3 grid, cudaStream_t s, ms2g_plan* p, const FactorTables& f, const float* sino,
                      const int* d_sel, int n_sel, const int* ch, const int* vpc, const BpTiling& t,
                      const int* order) {
  constexpr size_t smem = BpShape<H, false>::kSmem, smem_fx = BpShape<H, true>::kSmem;
  // several blocks of 36-51 KB per SM need the maximum shared-memory carveout;
  // function attributes are per device, so remember which devices have them
  static std::atomic<uint64_t> attr_devices{0};
  int dev = 0;
  MS2G_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_devices.load() & bit)) {
    MS2G_CUDA(cudaFuncSetAttribute(k_backward<H, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fx));
    MS2G_CUDA(cudaFuncSetAttribute(k_backward<H, true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    MS2G_CUDA(cudaFuncSetAttribute(k_backward<H, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    MS2G_CUDA(cudaFuncSetAttribute(k_backward<H, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr_devices.fetch_or(bit);
  }
  // experiment / test switch: the fp32 read-modify-write accumulation
  static const bool fp32 = getenv("MS2G_BP_FP32") != nullptr;
  if (fp32)
    MS2G_CUDA(launch_k(k_backward<H, false>, grid, dim3(32 * kBW), smem, s, f.d_rays_bp, (const int4*)f.d_bpr, p->V_r,
                       p->B, d_sel, n_sel, sino, p->w_part, f.nc, t.maj, t.per, ch[0], vpc[0], vpc[1], order,
                       (const float*)f.d_bpw, f.lc_max, (const unsigned*)p->w_rmaxv));
  else
    MS2G_CUDA(launch_k(k_backward<H, true>, grid, dim3(32 * BpWarps<true, H>::kW), smem_fx, s, f.d_rays_bp,
                       (const int4*)f.d_bpr, p->V_r,
                       p->B, d_sel, n_sel, sino, p->w_part, f.nc, t.maj, t.per, ch[0], vpc[0], vpc[1], order,
                       (const float*)f.d_bpw, f.lc_max, (const unsigned*)p->w_rmaxv));
  return MS2G_OK;
}

// View chunks per tile family of a backprojection over n_sel views.  The
// plan's chunking is for all V_r views; a view subset (Option 2, a minibatch)
// keeps the views per chunk, not the chunk count: otherwise a 90-view subset
// would be cut into 4-view chunks whose fixed cost (accumulator zeroing,
// partial planes, their reduction) dominates.
void bp_launch_chunks(const ms2g_plan* p, const FactorTables& f, int n_sel, int* ch) {
  for (int fam = 0; fam < 2; ++fam) {
    ch[fam] = (int)(((long long)f.bp_chunks[fam] * n_sel + p->V_r - 1) / p->V_r);
    const int max_chunks = (n_sel + kBW - 1) / kBW;
    if (ch[fam] > max_chunks) ch[fam] = max_chunks;
    if (ch[fam] < 1) ch[fam] = 1;
  }
}

int launch_backward(ms2g_plan* p, const FactorTables& f, const float* sino, float* img, float scale,
                    int accumulate, const int* d_sel, int n_sel, int batch, cudaStream_t s, int publish,
                    const int* order_sel, int* nplanes_out) {
  const size_t np = (size_t)f.nc * f.nc, total = np * batch;
  static const bool gather = getenv("MS2G_BP_VARIANT") && !strcmp(getenv("MS2G_BP_VARIANT"), "gather");
  if (gather) {   // experiment switch: the pixel-driven gather variant
    const int per = ((f.nc + 31) / 32) * ((f.nc + 7) / 8);
    const int planes_alloc = f.bp_chunks[0] + f.bp_chunks[1];
    const long long target = 24LL * p->sm_count;
    int nch = (int)std::min<long long>(planes_alloc, std::max<long long>(1, (target + (long long)per * batch - 1) /
                                                                              ((long long)per * batch)));
    nch = std::max(1, std::min(nch, n_sel));
    const int vpc = (n_sel + nch - 1) / nch;
    nch = (n_sel + vpc - 1) / vpc;
    const int slot = timing_begin(p, 1, f.factor, s);
    k_backward_gather<<<dim3(per * nch, 1, batch), dim3(32, 8), 0, s>>>(f.d_rays, f.d_views, p->B, d_sel, n_sel, sino,
                                                                       p->w_part, f.nc, vpc, nch);
    MS2G_TRY(check_launch("k_backward_gather"));
    timing_end(p, slot, s);
    if (nplanes_out) *nplanes_out = nch;
    if (publish == 2) return MS2G_OK;
    if (publish == 3) return launch_mc_publish(p, p->w_part, nch, np, total, scale, s);
    if (publish) return launch_chunk_reduce_publish(p, p->w_part, nch, np, total, scale, s);
    const int G = plane_groups(np, nch);
    k_chunk_reduce<<<dim3(plane_blocks(np, G, 4096), batch), dim3(32, kPlaneGroups), 0, s>>>(p->w_part, nch, np, img,
                                                                                             scale, accumulate, G);
    return check_launch("k_chunk_reduce");
  }
  const int H = f.bp_h;
  const BpTiling t = bp_tiling(f.nc, H);
  int ch[2], vpc[2];
  bp_launch_chunks(p, f, n_sel, ch);
  for (int fam = 0; fam < 2; ++fam) vpc[fam] = (n_sel + ch[fam] - 1) / ch[fam];
  dim3 grid(t.per * (ch[0] + ch[1]), 1, batch);
  // longest-first block order: the plan's for full-view launches, the
  // caller's (built for this view list with bp_launch_chunks) for subsets
  static const bool no_order = getenv("MS2G_BP_NO_ORDER") != nullptr;    // experiment switch
  const int* order = no_order ? nullptr : (d_sel ? order_sel : (n_sel == p->V_r ? f.d_bp_order : nullptr));
  const int slot = timing_begin(p, 1, f.factor, s);
  switch (H) {
    case 64: MS2G_TRY(bwd_launch<64>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    case 96: MS2G_TRY(bwd_launch<96>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    case 128: MS2G_TRY(bwd_launch<128>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    case 192: MS2G_TRY(bwd_launch<192>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    case 256: MS2G_TRY(bwd_launch<256>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    case 320: MS2G_TRY(bwd_launch<320>(grid, s, p, f, sino, d_sel, n_sel, ch, vpc, t, order)); break;
    default: return set_error(MS2G_ERR_CONFIG, "adjoint tile height must be 64, 96, 128, 192, 256 or 320");
  }
  MS2G_TRY(check_launch("k_backward"));
  timing_end(p, slot, s);
  if (nplanes_out) *nplanes_out = ch[0] + ch[1];
  if (publish == 2) return MS2G_OK;   // partial planes only: the caller's fused epilogue sums them
  if (publish == 3) return launch_mc_publish(p, p->w_part, ch[0] + ch[1], np, total, scale, s);   // NVLS
  if (publish)   // NEXT-3: the chunk sum goes straight to the peer exchange slot (peer_reduce.cu)
    return launch_chunk_reduce_publish(p, p->w_part, ch[0] + ch[1], np, total, scale, s);
  const int G = plane_groups(np, ch[0] + ch[1]);
  MS2G_CUDA(launch_k(k_chunk_reduce, dim3(plane_blocks(np, G, 4096), batch), dim3(32, kPlaneGroups), 0, s,
                     (const float*)p->w_part, ch[0] + ch[1], np, img, scale, accumulate, G));
  return check_launch("k_chunk_reduce");
}

}  // namespace ms2g
