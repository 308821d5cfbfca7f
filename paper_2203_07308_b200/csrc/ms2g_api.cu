// ms2g_api.cu -- C ABI of libms2g (include/ms2g.h): plan, geometry tables,
// operator entry points, schedule, power iteration and the graph-captured
// PnP-MS2G solve.  Host code only; kernels live in projector.cu/image_ops.cu.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

// NVTX range around every compute entry point (SURVEY §5 tracing): visible
// to Nsight tools (ncu --nvtx-include, nsys) when they are attached; a no-op
// otherwise (NVTX v3 is header-only and binds an injection library lazily).
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace ms2g {

int launch_check_finite(const float* a, size_t na, const float* c, size_t nc_, int* flag, cudaStream_t st);

std::atomic<uint64_t> g_launches{0};
thread_local bool t_capturing = false;
thread_local uint64_t t_captured = 0;
static thread_local std::string t_err;

int set_error(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

const FactorTables* find_factor(const ms2g_plan* p, int factor) {
  for (const auto& f : p->ft)
    if (f.factor == factor) return &f;
  return nullptr;
}

int timing_begin(ms2g_plan* p, int kind, int factor, cudaStream_t st) {
  if (p->root) p = p->root;
  if (!p->timing || !t_capturing) return -1;
  ms2g_plan::TimedLaunch tl{nullptr, nullptr, kind, factor};
  if (cudaEventCreate(&tl.a) != cudaSuccess || cudaEventCreate(&tl.b) != cudaSuccess) return -1;
  if (cudaEventRecordWithFlags(tl.a, st, cudaEventRecordExternal) != cudaSuccess) return -1;
  p->tev.push_back(tl);
  return (int)p->tev.size() - 1;
}

void timing_end(ms2g_plan* p, int slot, cudaStream_t st) {
  if (p->root) p = p->root;
  if (slot < 0) return;
  cudaEventRecordWithFlags(p->tev[slot].b, st, cudaEventRecordExternal);
}

static void clear_timing_events(ms2g_plan* p) {
  for (auto& tl : p->tev) {
    if (tl.a) cudaEventDestroy(tl.a);
    if (tl.b) cudaEventDestroy(tl.b);
  }
  p->tev.clear();
}

// floor / ceil division of a signed 64-bit value by a positive divisor
static long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}
static long long ceil_div(long long a, long long b) { return -floor_div(-a, b); }

// Longest-first (LPT) block orders from the host cost tables, for a launch over
// `views` (rank-local, in launch order).  Adjoint: block = (family, view chunk,
// tile) with the chunking of bp_launch_chunks; forward: block = (view block of
// vpb views, 32-bin block).  The result (a permutation of the block indices,
// longest first) goes to a new device array.
static int upload_order(const std::vector<long long>& cost, int** out) {
  std::vector<int> order(cost.size());
  for (size_t it = 0; it < order.size(); ++it) order[it] = (int)it;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  MS2G_CUDA(cudaMalloc(out, sizeof(int) * std::max<size_t>(order.size(), 1)));
  MS2G_CUDA(cudaMemcpy(*out, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
  return MS2G_OK;
}

static int upload_bp_order(const ms2g_plan* p, const FactorTables& f, const std::vector<int>& views, int** out) {
  const int n_sel = (int)views.size(), V_r = p->V_r;
  const int per_t = bp_tile_count(f.nc, f.bp_h) / 2;
  int ch[2];
  bp_launch_chunks(p, f, n_sel, ch);
  const int n_items = per_t * (ch[0] + ch[1]);
  std::vector<long long> cost(n_items, 0);
  for (int it = 0; it < n_items; ++it) {
    const int fam = it >= per_t * ch[0];
    const int bi = it - fam * per_t * ch[0];
    const int ti = bi % per_t, c = bi / per_t;
    const int vpc = (n_sel + ch[fam] - 1) / ch[fam];
    const uint16_t* row = f.h_bp_cost.data() + (size_t)(fam * per_t + ti) * V_r;
    long long sum = 0;
    for (int k = c * vpc; k < std::min(n_sel, (c + 1) * vpc); ++k) sum += row[views[k]];
    cost[it] = sum;
  }
  return upload_order(cost, out);
}

static int upload_fwd_order(const ms2g_plan* p, const FactorTables& f, const std::vector<int>& views, int vpb,
                            int** out) {
  const int n_sel = (int)views.size();
  const int nbx = (p->B + 31) / 32, nby = (n_sel + vpb - 1) / vpb;
  std::vector<long long> cost((size_t)nbx * nby, 0);
  for (int by = 0; by < nby; ++by)
    for (int k = by * vpb; k < std::min(n_sel, (by + 1) * vpb); ++k)
      for (int bx = 0; bx < nbx; ++bx) cost[(size_t)by * nbx + bx] += f.h_fwd_cost[(size_t)views[k] * nbx + bx];
  return upload_order(cost, out);
}

// Reading Z14 at the boundary: a ray lying ON a grid line of a planned grid
// (exactly axis-parallel, its constant coordinate a grid line) belongs to two
// closed pixel rows at once; the paper and the configs leave that undefined
// (it needs an odd bin count with an even grid side, or a shifted detector).
// The oracle's fp64 crossings then split the ray by rounding noise while the
// fixed-point traversal picks one row, so such geometries are rejected before
// any device work (MS2G_ERR_CONFIG).  Tolerances: |slope| < 1e-9 and within
// 1e-6 pixel of a grid line (the fixed point resolves 2^-32 pixel, and its
// slope floor 2^-32 moves a ray by < 1e-6 pixel across 32767 columns).
static int check_grid_ties(const ms2g_geom_desc& d, double pitch, const int32_t* factors, int n_factors) {
  const double org = -0.5 * d.fov;
  for (int v = d.view_begin; v < d.view_end; ++v) {
    const double th = d.arc_rad * (double)v / (double)d.n_views;
    const double c = std::cos(th), s = std::sin(th);
    const double sx = d.sod * c, sy = d.sod * s;
    for (int t = 0; t < d.n_bins; ++t) {
      const double u = ((double)t - 0.5 * (double)(d.n_bins - 1)) * pitch;
      const double px = -(d.sdd - d.sod) * c - u * s, py = -(d.sdd - d.sod) * s + u * c;
      const double dx = px - sx, dy = py - sy;
      double coord;   // the constant coordinate of an axis-parallel ray
      if (std::fabs(dy) < 1e-9 * std::fabs(dx)) coord = sy + (org - sx) * dy / dx;
      else if (std::fabs(dx) < 1e-9 * std::fabs(dy)) coord = sx + (org - sy) * dx / dy;
      else continue;
      for (int k = 0; k < n_factors; ++k) {
        const int fac = factors[k];
        if (fac < 1 || d.n % fac) continue;       // reported by the caller
        const double hc = d.fov * fac / d.n;
        const double q = (coord - org) / hc;      // grid-line units of this grid
        const double r = std::nearbyint(q);
        if (r >= 0 && r <= d.n / fac && std::fabs(q - r) < 1e-6) {
          std::ostringstream os;
          os << "ray (view " << v << ", bin " << t << ") lies on grid line " << (long long)r << " of the factor-"
             << fac << " grid (reading Z14: ambiguous pixel row); use an even bin count or move the detector";
          return set_error(MS2G_ERR_CONFIG, os.str());
        }
      }
    }
  }
  return MS2G_OK;
}

// Scale bounds of the fixed-point adjoint (projector.cu, k_backward): per
// (tile family, view), an upper bound of the weight one pixel receives from
// the view's rays.  Within a run of one ray class the rays do not cross
// inside the grid and, in a column, ray t covers the minor interval
// [F_t(c), F_t(c) + S_t] (length S_t <= 1, in pixels) with weight Lc_t times
// the covered fraction: a pixel row [rho, rho + 1) meets at most
// (1 + S_max) / delta_min + 1 of them (delta_min = the smallest gap between
// neighbouring rays, at c = 0 or c = n_c since F is linear in c), each
// giving at most Lc_max -- or, per unit of the row, at most
// S_max / delta_min + 1 column steps overlap, each weighing Lc / S per unit
// of minor travel: the smaller bound counts.  Runs of a family add up.
static int plan_bp_bounds(FactorTables& f, const std::vector<RayEntry>& rays, const std::vector<ViewEntry>& views,
                          int V_r, int B, int nc) {
  std::vector<float> w(2 * (size_t)V_r, 0.f);
  double lcm = 0.0;
  for (int v = 0; v < V_r; ++v) {
    const ViewEntry& ve = views[v];
    for (int sg = 0; sg < ve.nseg; ++sg) {
      const int fam = (ve.seg_cls[sg] & kMajorY) ? 1 : 0;
      double lmax = 0.0, smax = 0.0, dmin = 1e300, lymax = 0.0;
      int cnt = 0, prev = -1;
      for (int t = ve.seg_t[sg]; t < ve.seg_t[sg + 1]; ++t) {
        const RayEntry& R = rays[(size_t)v * B + t];
        if (R.c_lo >= R.c_hi) continue;          // misses the grid
        ++cnt;
        lmax = std::max(lmax, (double)R.Lc);
        smax = std::max(smax, (double)R.S / kFix);
        lymax = std::max(lymax, (double)R.Lc / ((double)R.S / kFix));   // length per unit of minor travel
        if (prev >= 0) {
          const RayEntry& Q = rays[(size_t)v * B + prev];
          const double d0 = std::fabs((double)(R.F0 - Q.F0)) / kFix;
          const double d1 = std::fabs((double)(R.F0 - Q.F0) + (double)nc * ((double)R.S - (double)Q.S)) / kFix;
          dmin = std::min(dmin, std::min(d0, d1));
        }
        prev = t;
      }
      if (!cnt) continue;
      const double count = cnt == 1 ? 1.0 : std::min((double)cnt, (1.0 + smax) / std::max(dmin, 1e-6) + 1.0);
      // or: a point of the row lies under at most S_max / delta_min + 1 of
      // the rays' column steps, each weighing Ly = Lc / S per unit of minor
      // travel, so the row receives at most Ly_max (S_max / delta_min + 1)
      const double cover = cnt == 1 ? 1.0 : smax / std::max(dmin, 1e-6) + 1.0;
      const double wb = std::min(lmax * count, lymax * cover);
      w[(size_t)fam * V_r + v] += (float)(wb * 1.001 + 1e-30);
      lcm = std::max(lcm, lmax);
    }
  }
  f.lc_max = (float)(lcm * 1.001);
  MS2G_CUDA(cudaMalloc(&f.d_bpw, sizeof(float) * w.size()));
  MS2G_CUDA(cudaMemcpy(f.d_bpw, w.data(), sizeof(float) * w.size(), cudaMemcpyHostToDevice));
  return MS2G_OK;
}

// Geometry plan: per-view and
// per-ray constants computed in fp64 on the host, rounded once.
static int build_tables(ms2g_plan* p, FactorTables& f, int sm_count) {
  const ms2g_geom_desc& d = p->d;
  const int nc = d.n / f.factor;
  f.nc = nc;
  const double hc = d.fov / nc, org = -0.5 * d.fov;
  const int B = p->B, V_r = p->V_r;
  std::vector<RayEntry> rays((size_t)V_r * B);
  std::vector<ViewEntry> views(V_r);
  const long long M = (long long)nc << 32;
  if (B > 32767) return set_error(MS2G_ERR_CONFIG, "n_bins must be <= 32767");
  for (int vl = 0; vl < V_r; ++vl) {
    const int v = d.view_begin + vl;
    const double th = d.arc_rad * (double)v / (double)d.n_views;
    const double c = std::cos(th), s = std::sin(th);
    const double Sx = (d.sod * c - org) / hc, Sy = (d.sod * s - org) / hc;
    const double dcx = -(d.sdd - d.sod) * c, dcy = -(d.sdd - d.sod) * s;
    ViewEntry ve;
    ve.Sx = (float)Sx; ve.Sy = (float)Sy;
    ve.ex = (float)(-s); ve.ey = (float)c;
    ve.nx = (float)(-c); ve.ny = (float)(-s);
    ve.scale = (float)(d.sdd / p->pitch);
    ve.off = (float)(0.5 * (B - 1));
    ve.nseg = 0;
    int prev_cls = -1;
    for (int t = 0; t < B; ++t) {
      const double u = ((double)t - 0.5 * (double)(B - 1)) * p->pitch;
      const double Px = (dcx - u * s - org) / hc, Py = (dcy + u * c - org) / hc;
      const double Dx = Px - Sx, Dy = Py - Sy;
      RayEntry R;
      int flags = 0;
      double slope, m0c;
      if (std::fabs(Dx) >= std::fabs(Dy)) {
        slope = Dy / Dx;
        m0c = Sy - Sx * slope;
      } else {
        flags |= kMajorY;
        slope = Dx / Dy;
        m0c = Sx - Sy * slope;
      }
      const double Lc = hc * std::sqrt(1.0 + slope * slope);
      if (slope < 0) {
        flags |= kMirror;
        slope = -slope;
        m0c = (double)nc - m0c;
      }
      R.F0 = llround(m0c * kFix);
      // slope in [0, 1]; 1 only at exactly 45 deg.  S >= 1 (a slope below
      // 2^-32 is rounded up to 2^-32): the end-coordinate weights need S > 0.
      const long long Sq = llround(slope * kFix);
      R.S = (unsigned)(Sq > 0xFFFFFFFFLL ? 0xFFFFFFFFLL : (Sq < 1 ? 1 : Sq));
      R.Lc = (float)Lc;
      R.Ly32 = (float)(Lc / (double)R.S);                  // length per 2^-32 of minor travel
      R.flags = flags;
      R.pad = 0;
      if (flags != prev_cls) {                              // a new run of one ray class
        if (ve.nseg == 4) return set_error(MS2G_ERR_CONFIG, "fan wider than 180 degrees: more than 4 ray classes");
        ve.seg_t[ve.nseg] = (short)t;
        ve.seg_cls[ve.nseg] = (char)flags;
        ve.nseg++;
        prev_cls = flags;
      }
      long long lo, hi;
      {
        const long long Sl = (long long)(unsigned long long)R.S;   // >= 1
        lo = floor_div(-R.F0, Sl);
        if (lo < 0) lo = 0;
        hi = ceil_div(M - R.F0, Sl);
        if (hi > nc) hi = nc;
      }
      if (lo >= hi) lo = hi = 0;
      R.c_lo = (short)lo;
      R.c_hi = (short)hi;
      rays[(size_t)vl * B + t] = R;
    }
    ve.seg_t[ve.nseg] = (short)B;
    views[vl] = ve;
    if (f.factor == p->ft[0].factor)   // classes depend on the ray directions only (all factors alike)
      for (int k = 0; k < ve.nseg; ++k) p->class_mask |= 1 << (ve.seg_cls[k] & 3);
  }
  MS2G_CUDA(cudaMalloc(&f.d_rays, sizeof(RayEntry) * rays.size()));
  MS2G_CUDA(cudaMalloc(&f.d_views, sizeof(ViewEntry) * views.size()));
  MS2G_CUDA(cudaMemcpy(f.d_rays, rays.data(), sizeof(RayEntry) * rays.size(), cudaMemcpyHostToDevice));
  {
    std::vector<RayBp> bp(rays.size());
    for (size_t i = 0; i < rays.size(); ++i) bp[i] = RayBp{rays[i].F0, rays[i].S, rays[i].Ly32};
    MS2G_CUDA(cudaMalloc(&f.d_rays_bp, sizeof(RayBp) * bp.size()));
    MS2G_CUDA(cudaMemcpy(f.d_rays_bp, bp.data(), sizeof(RayBp) * bp.size(), cudaMemcpyHostToDevice));
  }
  MS2G_TRY(plan_bp_bounds(f, rays, views, V_r, B, nc));
  MS2G_CUDA(cudaMemcpy(f.d_views, views.data(), sizeof(ViewEntry) * views.size(), cudaMemcpyHostToDevice));
  MS2G_TRY(build_bicubic_tables(f, d.n));
  MS2G_CUDA(cudaMalloc(&f.d_Lcache, 3 * sizeof(double)));
  MS2G_CUDA(cudaMemset(f.d_Lcache, 0, 3 * sizeof(double)));
  {  // adjoint tile/view bin ranges (geometry only, once per plan)
    int* d_err = nullptr;
    f.bp_h = bp_height(nc, V_r);
    MS2G_CUDA(cudaMalloc(&f.d_bpr, sizeof(int4) * (size_t)bp_tile_count(nc, f.bp_h) * V_r));
    MS2G_CUDA(cudaMalloc(&d_err, sizeof(int)));
    MS2G_CUDA(cudaMemset(d_err, 0, sizeof(int)));
    int rc = launch_bp_ranges(f, V_r, B, f.d_bpr, d_err, 0);
    int herr = 0;
    if (rc == MS2G_OK) {
      cudaError_t e = cudaMemcpy(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = set_error(MS2G_ERR_CUDA, std::string("bp ranges: ") + cudaGetErrorString(e));
    }
    cudaFree(d_err);
    if (rc != MS2G_OK) return rc;
    if (herr) return set_error(MS2G_ERR_CONFIG, "a tile's shadow spans more than 2 ray classes (fan too wide)");
  }
  // backprojector view chunks: about 12-24 "waves" of SM-count blocks
  // (measured on B200 with the longest-first order below; with the fp32
  // adjoint 24 was best or within 2 % everywhere, 8 and 64 lost 3-10 %).  The
  // chunk partials are summed by k_chunk_reduce in fixed order.
  // The X- and Y-tile families only see the views with major-x / major-y
  // rays; a contiguous view shard (e.g. 45 degrees at P = 8) is almost all
  // one class, so each family gets view chunks in proportion to its views.
  const long long tiles = (long long)bp_tile_count(nc, f.bp_h) * d.batch;
  const long long per = tiles / 2;
  // 12 "waves" at n_c >= 256 since the fixed-point adjoint with tall tiles
  // (C4 solve 493 -> 500 iterations/s, C3 13.9 -> 13.1 ms, C5 64.9 -> 63.9 ms,
  // the 180-view shard 18.7 -> 17.7 ms, C3 s = 2 subset gradients 20.0 k ->
  // 23.1 k evals/s); 24 below, whose small subset launches need the blocks
  // (C3 s = 4 subset gradient 27.0 k against 22.1 k evals/s)
  const long long waves = getenv("MS2G_BP_WAVES") ? atoi(getenv("MS2G_BP_WAVES")) : (nc >= 256 ? 12 : 24);
  const long long target = waves * sm_count;
  long long nv[2] = {0, 0};
  for (const ViewEntry& ve : views) {
    int mask = 0;
    for (int k = 0; k < ve.nseg; ++k) mask |= (ve.seg_cls[k] & kMajorY) ? 2 : 1;
    nv[0] += mask & 1;
    nv[1] += (mask >> 1) & 1;
  }
  const long long maxch = (V_r + 3) / 4;
  for (int fam = 0; fam < 2; ++fam) {
    const long long share = (target * nv[fam] + (nv[0] + nv[1]) - 1) / std::max(1LL, nv[0] + nv[1]);
    long long ch = (share + per - 1) / per;
    if (ch > maxch) ch = maxch;
    if (ch < 1) ch = 1;
    f.bp_chunks[fam] = (int)ch;
  }
  // Cost tables for the longest-first block orders (LPT): blocks start
  // roughly in index order, so a launch of 2-3 waves of uneven blocks (tiles
  // outside the disk of the fan, families of a view shard) no longer ends on
  // its longest blocks.  Adjoint: rays meeting (tile, view), from the range
  // table; forward: the longest ray column range of (view, 32-bin block).
  {
    const int ntile = bp_tile_count(nc, f.bp_h);
    std::vector<int4> rt((size_t)ntile * V_r);
    MS2G_CUDA(cudaMemcpy(rt.data(), f.d_bpr, sizeof(int4) * rt.size(), cudaMemcpyDeviceToHost));
    f.h_bp_cost.assign(rt.size(), 0);
    for (size_t i = 0; i < rt.size(); ++i) {
      const int4 r = rt[i];
      const int nr = (r.z >> 16) & 0xff;
      int sum = 0;
      if (nr > 0) sum += (short)(r.x >> 16) - (r.x & 0xffff) + 1;
      if (nr > 1) sum += (short)(r.y >> 16) - (r.y & 0xffff) + 1;
      f.h_bp_cost[i] = (uint16_t)std::min(sum, 65535);
    }
    const int nbx = (B + 31) / 32;
    f.h_fwd_cost.assign((size_t)V_r * nbx, 0);
    for (int v = 0; v < V_r; ++v)
      for (int bx = 0; bx < nbx; ++bx) {
        int lo = INT_MAX, hi = INT_MIN;
        for (int t = bx * 32; t < std::min(B, bx * 32 + 32); ++t) {
          const RayEntry& R = rays[(size_t)v * B + t];
          if (R.c_lo < R.c_hi) {
            lo = std::min(lo, (int)R.c_lo);
            hi = std::max(hi, (int)R.c_hi);
          }
        }
        f.h_fwd_cost[(size_t)v * nbx + bx] = (uint16_t)(lo < hi ? hi - lo : 0);
      }
  }
  std::vector<int> all_views(V_r);
  for (int v = 0; v < V_r; ++v) all_views[v] = v;
  MS2G_TRY(upload_bp_order(p, f, all_views, &f.d_bp_order));
  if (d.batch % 2 != 0) {
    f.fwd_order_vpb = fwd_views_per_block(p, V_r, d.batch);
    MS2G_TRY(upload_fwd_order(p, f, all_views, f.fwd_order_vpb, &f.d_fwd_order));
  }
  return MS2G_OK;
}

static void free_plan(ms2g_plan* p) {
  if (!p) return;
  for (auto& f : p->ft) {
    cudaFree(f.d_rays);
    cudaFree(f.d_rays_bp);
    cudaFree(f.d_bpw);
    cudaFree(f.d_views);
    cudaFree(f.d_bpr);
    cudaFree(f.d_bp_order);
    cudaFree(f.d_fwd_order);
    for (int* q : f.d_bp_order_sub) cudaFree(q);
    for (int* q : f.d_fwd_order_sub) cudaFree(q);
    cudaFree(f.d_idx_down);
    cudaFree(f.d_w_down);
    cudaFree(f.d_idx_up);
    cudaFree(f.d_w_up);
  }
  for (auto& f : p->ft) cudaFree(f.d_Lcache);
  cudaFree(p->w_pair);
  float* fl[] = {p->w_v, p->w_rs, p->w_snap, p->w_mu, p->w_G, p->w_res, p->w_part, p->w_x[0], p->w_x[1],
                 p->w_y, p->w_z, p->w_p[0], p->w_p[1], p->w_etaf};
  for (float* q : fl) cudaFree(q);
  cudaFree(p->w_red);
  cudaFree(p->w_scal);
  cudaFree(p->w_pw);
  cudaFree(p->w_ticket);
  cudaFree(p->w_rmaxv);
  cudaFree(p->tvws.flags);
  cudaFree(p->tvws.gen_ticket);
  cudaFree(p->tvws.err);
  cudaFree(p->w_flag);
  cudaFree(p->w_sel);
  cudaFree(p->w_subsets);
  cudaFree(p->w_mb);
  cudaFree(p->w_saga);
  if (p->h_sel) cudaFreeHost(p->h_sel);
  for (cudaEvent_t ev : p->sel_ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& r : p->reg) {
    cudaFree(r.d_sel);
    for (int* q : r.bp_order) cudaFree(q);
    for (int* q : r.fwd_order) cudaFree(q);
  }
  if (p->sg.exec) cudaGraphExecDestroy(p->sg.exec);
  if (p->sg.graph) cudaGraphDestroy(p->sg.graph);
  for (auto& gg : p->grad_graphs) {   // per-call gradient graphs captured without it
    if (gg.exec) cudaGraphExecDestroy(gg.exec);
    if (gg.graph) cudaGraphDestroy(gg.graph);
  }
  p->grad_graphs.clear();
  p->topo_version++;
  for (auto& br : p->pbr) {
    cudaFree(br.w_v);
    cudaFree(br.w_pair);
    cudaFree(br.w_res);
    cudaFree(br.w_G);
    cudaFree(br.w_part);
    cudaFree(br.w_red);
    cudaFree(br.w_pw);
    cudaFree(br.w_ticket);
    cudaFree(br.w_rmaxv);
    if (br.stream) cudaStreamDestroy(br.stream);
    if (br.done) cudaEventDestroy(br.done);
  }
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  for (void* q : p->peer_opened) cudaIpcCloseMemHandle(q);
  mc_release(p);
  cudaFree(p->xch_buf);
  cudaFree(p->xch_pad);
  cudaFree(p->d_peer_bufs);
  cudaFree(p->d_peer_pads);
  cudaFree(p->w_peer_err);
  clear_timing_events(p);
  if (p->comm) ncclCommDestroy(p->comm);
  delete p;
}

// Resolve a host subset of GLOBAL view indices into this rank's compacted
// list on the device (stream ordered).  subset == NULL -> all views.
// Host subsets use a slot of the plan's list ring (*slot, -1 if none); the
// caller releases it with release_subset after enqueueing every consumer.
static int check_subset(const ms2g_plan* p, const int32_t* subset, int n_subset, int* m_local) {
  if (n_subset < 1) return set_error(MS2G_ERR_INPUT, "empty view subset (S:285)");
  int prev = -1, m = 0;
  for (int k = 0; k < n_subset; ++k) {
    const int v = subset[k];
    if (v < 0 || v >= p->d.n_views || v <= prev)
      return set_error(MS2G_ERR_INPUT, "subset must hold ascending view indices in [0, n_views)");
    prev = v;
    m += (v >= p->d.view_begin && v < p->d.view_end);
  }
  *m_local = m;
  return MS2G_OK;
}

static int resolve_subset(ms2g_plan* p, const int32_t* subset, int n_subset, cudaStream_t st, const int** d_sel,
                          int* n_sel, int* n_global, int* slot) {
  *slot = -1;
  if (!subset) {
    *d_sel = nullptr;
    *n_sel = p->V_r;
    *n_global = p->d.n_views;
    return MS2G_OK;
  }
  int m = 0;
  MS2G_TRY(check_subset(p, subset, n_subset, &m));
  const int k = p->sel_next;
  int* h = p->h_sel + (size_t)k * p->V_r;
  int* dv = p->w_sel + (size_t)k * p->V_r;
  if (m > 0) {
    // the slot's previous consumers (any stream) are done: ring depth 8, so
    // this waits only when 8 calls are in flight
    MS2G_CUDA(cudaEventSynchronize(p->sel_ev[k]));
    int q = 0;
    for (int i = 0; i < n_subset; ++i) {
      const int v = subset[i];
      if (v >= p->d.view_begin && v < p->d.view_end) h[q++] = v - p->d.view_begin;
    }
    MS2G_CUDA(cudaMemcpyAsync(dv, h, sizeof(int) * m, cudaMemcpyHostToDevice, st));
    p->sel_next = (k + 1) % ms2g_plan::kSelRing;
    *slot = k;
  }
  *d_sel = dv;
  *n_sel = m;
  *n_global = n_subset;
  return MS2G_OK;
}

static int release_subset(ms2g_plan* p, int slot, cudaStream_t st) {
  if (slot >= 0) MS2G_CUDA(cudaEventRecord(p->sel_ev[slot], st));
  return MS2G_OK;
}

static int peer_ok(const ms2g_plan* p) {
  if (p->peer_failed)
    return set_error(MS2G_ERR_NCCL, "peer exchange failed earlier (barrier time-out): call ms2g_attach_peers again");
  return MS2G_OK;
}

static int allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st) {
  if (p->mc_n > 0) {                        // NEXT-3 NVLS multicast path wins
    MS2G_TRY(peer_ok(p));
    return launch_mc_allreduce(p, buf, count, st);
  }
  if (p->peer_n > 0) {                      // then the NEXT-3 peer path
    MS2G_TRY(peer_ok(p));
    return launch_peer_allreduce(p, buf, count, st);
  }
  if (!p->comm) return MS2G_OK;   // attached communicators are always used (1 rank: NCCL identity)
  MS2G_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, p->comm, st));
  return MS2G_OK;
}

// G = c A_s^T r summed over ranks.  With peers attached the backprojector's
// chunk reduction publishes straight into the exchange slot (fused, no
// separate collective); otherwise backprojection then NCCL (or nothing).
static int backward_sum(ms2g_plan* p, const FactorTables& f, const float* sino, float* G, float c, const int* d_sel,
                        int n_sel, int batch, cudaStream_t st, const int* order_sel = nullptr) {
  const size_t count = (size_t)f.nc * f.nc * batch;
  if (p->mc_n > 0) {
    MS2G_TRY(peer_ok(p));
    MS2G_TRY(launch_backward(p, f, sino, G, c, 0, d_sel, n_sel, batch, st, 3, order_sel));
    return launch_mc_finish(p, count, G, 0, 0, nullptr, nullptr, st);
  }
  if (p->peer_n > 0) {
    MS2G_TRY(peer_ok(p));
    MS2G_TRY(launch_backward(p, f, sino, G, c, 0, d_sel, n_sel, batch, st, 1, order_sel));
    return launch_peer_finish(p, G, count, st);
  }
  MS2G_TRY(launch_backward(p, f, sino, G, c, 0, d_sel, n_sel, batch, st, 0, order_sel));
  return allreduce(p, G, count, st);
}

// Single-rank plans reduce the backprojection's partial planes in a fused
// epilogue (the step, the power iteration); with a communicator or peers the
// partial image is summed over ranks first (G = allreduce), then consumed.
static bool fused_epilogue(const ms2g_plan* p) { return p->peer_n == 0 && p->mc_n == 0 && !p->comm; }

// Pair images of v = S_s(src) for the forward: kind 0 fuses the s x s mean
// into the pair prep (one launch); bicubic resamples into w_v first.
static int prep_pairs(ms2g_plan* p, const FactorTables& f, int kind, int batch, const float* src, cudaStream_t st) {
  if (f.factor > 1 && kind != 0) {
    MS2G_TRY(launch_resample_down(p, f, kind, batch, src, p->w_v, st));   // v = S(y)
    return launch_pair_prep(p, f.nc, batch, p->w_v, st);
  }
  return launch_pair_prep(p, f.nc, batch, src, st, f.factor);          // v = S(y) fused
}

// z = y - eta U_s (c A_s^T r)  (y == NULL: z = U_s (c A_s^T r)), summed over
// ranks when attached: the G-step of Eq. 6/7.
static int backward_step(ms2g_plan* p, const FactorTables& f, int kind, const float* sino, float c, const int* d_sel,
                         int n_sel, int batch, const float* y, const float* eta_dev, float* z, cudaStream_t st,
                         const int* bord) {
  if (kind == 0 && fused_epilogue(p)) {
    int npl = 0;
    MS2G_TRY(launch_backward(p, f, sino, nullptr, c, 0, d_sel, n_sel, batch, st, 2, bord, &npl));
    return launch_reduce_up_step(p->w_part, npl, f.nc, batch, c, y, eta_dev, z, f.factor, st);
  }
  if (kind == 0 && p->mc_n > 0) {     // NEXT-3 NVLS: publish, in-switch reduce + broadcast, step
    MS2G_TRY(peer_ok(p));
    MS2G_TRY(launch_backward(p, f, sino, nullptr, c, 0, d_sel, n_sel, batch, st, 3, bord));
    return launch_mc_finish(p, (size_t)f.nc * f.nc * batch, z, f.nc, f.factor, y, eta_dev, st);
  }
  if (kind == 0 && p->peer_n > 0) {   // NEXT-3: publish (fused chunk sum), reduce-scatter, all-gather + step
    MS2G_TRY(peer_ok(p));
    MS2G_TRY(launch_backward(p, f, sino, nullptr, c, 0, d_sel, n_sel, batch, st, 1, bord));
    return launch_peer_finish_step(p, (size_t)f.nc * f.nc * batch, f.nc, f.factor, y, eta_dev, z, st);
  }
  float* G = (f.factor > 1 || y) ? p->w_G : z;
  MS2G_TRY(backward_sum(p, f, sino, G, c, d_sel, n_sel, batch, st, bord));   // G = c A_s^T r (+ ranks)
  if (f.factor > 1 || y) MS2G_TRY(launch_resample_up_step(p, f, kind, batch, G, y, eta_dev, 0.f, z, st));
  return MS2G_OK;
}

// g = c U_s A_s^T (A_s S_s x - b), into a full-resolution image.
static int enqueue_grad(ms2g_plan* p, const FactorTables& f, int kind, const float* x, const float* b, float* g,
                        const int* d_sel, int n_sel, float c, int batch, cudaStream_t st,
                        const int* ford = nullptr, const int* bord = nullptr) {
  MS2G_TRY(prep_pairs(p, f, kind, batch, x, st));
  MS2G_TRY(launch_forward(p, f, b, p->w_res, d_sel, n_sel, batch, st, ford));  // r = A_s v - b
  return backward_step(p, f, kind, p->w_res, c, d_sel, n_sel, batch, nullptr, nullptr, g, st, bord);
}

// O8 power iteration on the full view set (allreduced over ranks); the last
// Rayleigh quotient goes to L_out / eta_out / etaf_out (device pointers).
// Per iteration: forward, backprojection, the fused chunk-sum + dot/norm
// step (k_reduce_power, last-block finalisation) and the pair prep of the
// next v = w / ||w|| (scaled on the fly): 4 launches.
static int enqueue_power(ms2g_plan* p, const FactorTables& f, int iters, double* L_out, double* eta_out,
                         float* etaf_out, cudaStream_t st) {
  const size_t np = (size_t)f.nc * f.nc;
  const float v0 = (float)(1.0 / (double)f.nc);  // 1 / ||1||
  MS2G_TRY(launch_fill(p->w_v, np, v0, st));
  MS2G_TRY(launch_pair_prep(p, f.nc, 1, p->w_v, st));
  for (int k = 0; k < iters; ++k) {
    MS2G_TRY(launch_forward(p, f, nullptr, p->w_res, nullptr, p->V_r, 1, st));
    const float* part = p->w_G;
    int npl = 1, ch[2];
    bp_launch_chunks(p, f, p->V_r, ch);
    const int npl_bp = ch[0] + ch[1];   // the backprojection's plane count (tiling of the reduction)
    if (fused_epilogue(p)) {
      MS2G_TRY(launch_backward(p, f, p->w_res, nullptr, 1.f, 0, nullptr, p->V_r, 1, st, 2, nullptr, &npl));
      part = p->w_part;
    } else {
      MS2G_TRY(backward_sum(p, f, p->w_res, p->w_G, 1.f, nullptr, p->V_r, 1, st));   // G summed over ranks
    }
    const bool last = (k == iters - 1);
    double* cache = f.d_Lcache;
    MS2G_TRY(launch_reduce_power(p, part, npl, np, p->w_G, p->w_v, p->w_red, p->red_blocks, p->w_ticket, p->w_pw,
                                 last ? cache : nullptr, last ? cache + 1 : nullptr,
                                 last ? reinterpret_cast<float*>(cache + 2) : nullptr, st, npl_bp));
    if (!last) MS2G_TRY(launch_pair_prep(p, f.nc, 1, p->w_G, st, 1, p->w_pw + 1, p->w_v));   // v = w / ||w||
  }
  // the last Rayleigh quotient went to the factor's cache (reused by solves
  // with power_iters = 0); hand it to the caller's slots
  f.L_iters = iters;
  return launch_cached_step(f.d_Lcache, L_out, eta_out, etaf_out, st);
}

static int denoise_mix(ms2g_plan* p, const ms2g_denoiser& den, const float* z, const float* xprev, float* xout,
                       float* yout, float alpha, float a, int mode, int iter, int batch, cudaStream_t st) {
  const int n = p->d.n;
  switch (den.kind) {
    case 0:
      return launch_copy_mix_mom(n, batch, z, xprev, xout, yout, a, mode, p->w_flag, iter, st);
    case 1:
      return launch_gauss_mix_mom(n, batch, den.sigma, z, xprev, xout, yout, alpha, a, mode, p->w_flag, iter, st);
    case 2:
      return launch_tv(n, batch, den.lambda, den.tau, den.inner_iters, z, p->w_p[0], p->w_p[1], xprev, xout, yout,
                       alpha, a, mode, p->w_flag, iter, st, &p->tvws);
    default:
      return set_error(MS2G_ERR_CONFIG, "unknown denoiser kind");
  }
}

static int check_denoiser(const ms2g_denoiser& den) {
  if (den.kind < 0 || den.kind > 2) return set_error(MS2G_ERR_CONFIG, "denoiser kind must be 0, 1 or 2");
  if (den.kind == 1 && !(den.sigma > 0)) return set_error(MS2G_ERR_CONFIG, "gaussian sigma must be > 0");
  if (den.kind == 2) {
    if (!(den.lambda >= 0)) return set_error(MS2G_ERR_CONFIG, "tv lambda must be >= 0");
    if (!(den.tau > 0 && den.tau <= 0.125f)) return set_error(MS2G_ERR_CONFIG, "tv tau must be in (0, 1/8]");
    if (den.inner_iters < 1) return set_error(MS2G_ERR_CONFIG, "tv inner_iters must be >= 1");
  }
  return MS2G_OK;
}

// O13 schedule: SplitMix64 + Fisher-Yates (independent of the oracle's copy).
static uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static int make_schedule(const ms2g_plan* p, const ms2g_solve_desc* sd, std::vector<ms2g_sched_entry>& out) {
  out.clear();
  if (!sd || !sd->stages || sd->n_stages < 1 || sd->n_stages > 63)
    return set_error(MS2G_ERR_CONFIG, "solve needs 1..63 stages");
  if (sd->option < 1 || sd->option > 5) return set_error(MS2G_ERR_CONFIG, "option must be 1..5");
  if (sd->option >= 2 && (sd->n_subsets < 1 || (p && sd->n_subsets > p->d.n_views)))
    return set_error(MS2G_ERR_CONFIG, "n_subsets (option 4: views per minibatch) must be in [1, n_views]");
  uint64_t state = sd->seed;
  int i = 0;
  std::vector<int> perm(sd->option >= 2 ? sd->n_subsets : 1);
  for (int k = 0; k < sd->n_stages; ++k) {
    const ms2g_stage& st = sd->stages[k];
    if (st.factor < 1 || (p && p->d.n % st.factor != 0))
      return set_error(MS2G_ERR_CONFIG, "stage factor must divide n (S:127)");
    if (sd->option == 1 || sd->option == 4) {
      if (st.n_iters < 0) return set_error(MS2G_ERR_CONFIG, "n_iters must be >= 0");
      for (int j = 0; j < st.n_iters; ++j) {
        ++i;
        out.push_back({i, k, st.factor, sd->option == 4 ? i - 1 : -1, 0.0, (double)(i - 1) / (double)(i + 3)});
      }
    } else {
      if (st.n_epochs < 0) return set_error(MS2G_ERR_CONFIG, "n_epochs must be >= 0");
      for (int ep = 0; ep < st.n_epochs; ++ep) {
        for (int q = 0; q < sd->n_subsets; ++q) perm[q] = q;
        for (int q = sd->n_subsets - 1; q >= 1; --q) {
          const int j = (int)(splitmix64(state) % (uint64_t)(q + 1));
          std::swap(perm[q], perm[j]);
        }
        for (int q = 0; q < sd->n_subsets; ++q) {
          ++i;
          out.push_back({i, k, st.factor, perm[q], 0.0, (double)(i - 1) / (double)(i + 3)});
        }
      }
    }
  }
  return MS2G_OK;
}

// Option 4: per step m distinct views drawn uniformly without
// replacement by a partial Fisher-Yates shuffle of [0..V-1] on one SplitMix64
// stream, ascending (independent of the oracle's copy; compared bit-exactly).
static void minibatch_views(int V, int m, uint64_t seed, int n_steps, std::vector<int>& out) {
  uint64_t state = seed;
  std::vector<int> arr(V);
  out.assign((size_t)n_steps * m, 0);
  for (int st = 0; st < n_steps; ++st) {
    for (int q = 0; q < V; ++q) arr[q] = q;
    for (int q = 0; q < m; ++q) {
      const int j = q + (int)(splitmix64(state) % (uint64_t)(V - q));
      std::swap(arr[q], arr[j]);
    }
    std::sort(arr.begin(), arr.begin() + m);
    std::copy(arr.begin(), arr.begin() + m, out.begin() + (size_t)st * m);
  }
}

// Upload the per-step minibatch lists (rank-local) of an Option-4 solve.
static int prepare_minibatches(ms2g_plan* p, const ms2g_solve_desc* sd, int n_steps) {
  std::vector<int> g;
  minibatch_views(p->d.n_views, sd->n_subsets, sd->seed, n_steps, g);
  std::vector<int> all;
  p->mb_off.assign(n_steps, 0);
  p->mb_len.assign(n_steps, 0);
  for (int st = 0; st < n_steps; ++st) {
    p->mb_off[st] = (int)all.size();
    for (int q = 0; q < sd->n_subsets; ++q) {
      const int v = g[(size_t)st * sd->n_subsets + q];
      if (v >= p->d.view_begin && v < p->d.view_end) all.push_back(v - p->d.view_begin);
    }
    p->mb_len[st] = (int)all.size() - p->mb_off[st];
  }
  cudaFree(p->w_mb);
  p->w_mb = nullptr;
  MS2G_CUDA(cudaMalloc(&p->w_mb, sizeof(int) * (all.size() + 1)));
  if (!all.empty()) MS2G_CUDA(cudaMemcpy(p->w_mb, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice));
  p->subsets_n = 0;   // the interleaved-subset cache is independent
  return MS2G_OK;
}

// Upload the n_subsets interleaved subset lists (rank-local) once per solve
// description; synchronous, outside graph capture.
static int prepare_subsets(ms2g_plan* p, int n_subsets) {
  if (p->subsets_n == n_subsets) return MS2G_OK;
  std::vector<int> all;
  p->subset_off.assign(n_subsets, 0);
  p->subset_len.assign(n_subsets, 0);
  p->subset_global_len.assign(n_subsets, 0);
  for (int k = 0; k < n_subsets; ++k) {
    p->subset_off[k] = (int)all.size();
    for (int v = k; v < p->d.n_views; v += n_subsets) {
      p->subset_global_len[k]++;
      if (v >= p->d.view_begin && v < p->d.view_end) all.push_back(v - p->d.view_begin);
    }
    p->subset_len[k] = (int)all.size() - p->subset_off[k];
  }
  cudaFree(p->w_subsets);
  p->w_subsets = nullptr;
  MS2G_CUDA(cudaMalloc(&p->w_subsets, sizeof(int) * (all.size() + 1)));
  if (!all.empty())
    MS2G_CUDA(cudaMemcpy(p->w_subsets, all.data(), sizeof(int) * all.size(), cudaMemcpyHostToDevice));
  // longest-first block orders of every subset launch, per factor
  for (auto& f : p->ft) {
    for (int* q : f.d_bp_order_sub) cudaFree(q);
    for (int* q : f.d_fwd_order_sub) cudaFree(q);
    f.d_bp_order_sub.assign(n_subsets, nullptr);
    f.d_fwd_order_sub.assign(n_subsets, nullptr);
    for (int k = 0; k < n_subsets; ++k) {
      if (p->subset_len[k] == 0) continue;
      const std::vector<int> views(all.begin() + p->subset_off[k], all.begin() + p->subset_off[k] + p->subset_len[k]);
      MS2G_TRY(upload_bp_order(p, f, views, &f.d_bp_order_sub[k]));
      if (p->d.batch % 2 != 0)
        MS2G_TRY(upload_fwd_order(p, f, views, fwd_views_per_block(p, (int)views.size(), p->d.batch),
                                  &f.d_fwd_order_sub[k]));
    }
  }
  p->subsets_n = n_subsets;
  return MS2G_OK;
}

// Branch workspaces for the power chains of the stage factors (allocated
// once, outside any capture).  Returns false when branching is not used.
static bool power_branching(const ms2g_plan* p) {
  static const bool off = getenv("MS2G_SERIAL_POWER") != nullptr;   // experiment switch
  // kernel timing wants each launch's own duration: concurrent branches would
  // share the GPU inside the timed intervals, so an instrumented solve is serial
  return !off && !p->timing && p->nranks == 1 && !p->comm && p->peer_n == 0 && p->mc_n == 0;
}

static int ensure_power_branches(ms2g_plan* p, const ms2g_solve_desc* sd) {
  for (int k = 0; k < sd->n_stages; ++k) {
    const int fac = sd->stages[k].factor;
    bool have = false;
    for (const auto& br : p->pbr) have |= br.factor == fac;
    if (have) continue;
    const FactorTables* f = find_factor(p, fac);
    ms2g_plan::PowerBranch br;
    br.factor = fac;
    const size_t nc = (size_t)f->nc, np = nc * nc;
    br.pair_stride = nc * pair_line(nc);
    const size_t planes = (size_t)(f->bp_chunks[0] + f->bp_chunks[1]);
    MS2G_CUDA(cudaMalloc(&br.w_v, sizeof(float) * np));
    MS2G_CUDA(cudaMalloc(&br.w_pair, sizeof(float2) * 4 * br.pair_stride));
    MS2G_CUDA(cudaMemset(br.w_pair, 0, sizeof(float2) * 4 * br.pair_stride));
    MS2G_CUDA(cudaMalloc(&br.w_res, sizeof(float) * (size_t)p->V_r * p->B));
    MS2G_CUDA(cudaMalloc(&br.w_G, sizeof(float) * np));
    MS2G_CUDA(cudaMalloc(&br.w_part, sizeof(float) * planes * np));
    MS2G_CUDA(cudaMalloc(&br.w_red, sizeof(double) * 2 * p->red_blocks));
    MS2G_CUDA(cudaMalloc(&br.w_pw, sizeof(double) * 8));
    MS2G_CUDA(cudaMalloc(&br.w_ticket, sizeof(unsigned)));
    MS2G_CUDA(cudaMemset(br.w_ticket, 0, sizeof(unsigned)));
    MS2G_CUDA(cudaMalloc(&br.w_rmaxv, sizeof(unsigned) * (size_t)p->V_r));
    MS2G_CUDA(cudaMemset(br.w_rmaxv, 0, sizeof(unsigned) * (size_t)p->V_r));
    MS2G_CUDA(cudaStreamCreateWithFlags(&br.stream, cudaStreamNonBlocking));
    MS2G_CUDA(cudaEventCreateWithFlags(&br.done, cudaEventDisableTiming));
    p->pbr.push_back(br);
  }
  if (!p->ev_fork) MS2G_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  return MS2G_OK;
}

// Fork every stage factor's power chain onto its branch (inside the capture):
// the chain writes the factor's step cache and every stage slot of that
// factor, then records the branch's `done` event for the stage to wait on.
static int enqueue_power_branches(ms2g_plan* p, const ms2g_solve_desc* sd, cudaStream_t st) {
  MS2G_CUDA(cudaEventRecord(p->ev_fork, st));
  for (auto& br : p->pbr) {
    int first = -1;
    for (int k = 0; k < sd->n_stages; ++k)
      if (sd->stages[k].factor == br.factor && first < 0) first = k;
    if (first < 0) continue;
    MS2G_CUDA(cudaStreamWaitEvent(br.stream, p->ev_fork, 0));
    ms2g_plan shadow = *p;                 // same tables, the branch's workspaces
    shadow.root = p;
    shadow.w_v = br.w_v;
    shadow.w_pair = br.w_pair;
    shadow.pair_stride = br.pair_stride;
    shadow.w_res = br.w_res;
    shadow.w_G = br.w_G;
    shadow.w_part = br.w_part;
    shadow.w_red = br.w_red;
    shadow.w_pw = br.w_pw;
    shadow.w_ticket = br.w_ticket;
    shadow.w_rmaxv = br.w_rmaxv;
    const FactorTables* f = find_factor(p, br.factor);
    MS2G_TRY(enqueue_power(&shadow, *f, sd->power_iters, p->w_scal + first, p->w_scal + 64 + first,
                           p->w_etaf + first, br.stream));
    for (int k = first + 1; k < sd->n_stages; ++k)
      if (sd->stages[k].factor == br.factor)
        MS2G_TRY(launch_cached_step(f->d_Lcache, p->w_scal + k, p->w_scal + 64 + k, p->w_etaf + k, br.stream));
    MS2G_CUDA(cudaEventRecord(br.done, br.stream));
  }
  return MS2G_OK;
}

// The whole solve as one stream-ordered sequence (captured into a graph).
static int enqueue_solve(ms2g_plan* p, const ms2g_solve_desc* sd, const std::vector<ms2g_sched_entry>& sch,
                         const float* b, const float* x0, float* x_out, cudaStream_t st) {
  const int n = p->d.n, batch = p->d.batch;
  const size_t img = (size_t)n * n * batch;
  MS2G_TRY(launch_init_flag(p->w_flag, st));
  MS2G_TRY(launch_check_finite(b, (size_t)p->V_r * p->B * batch, x0, img, p->w_flag, st));
  // x_0 = y_0 = x0, x_prev = x_0
  MS2G_CUDA(cudaMemcpyAsync(p->w_x[0], x0, sizeof(float) * img, cudaMemcpyDeviceToDevice, st));
  MS2G_CUDA(cudaMemcpyAsync(p->w_y, x0, sizeof(float) * img, cudaMemcpyDeviceToDevice, st));
  int cur = 0;
  size_t step = 0;
  const bool branched = sd->power_iters > 0 && power_branching(p);
  if (branched) MS2G_TRY(enqueue_power_branches(p, sd, st));
  for (int k = 0; k < sd->n_stages; ++k) {
    const ms2g_stage& stg = sd->stages[k];
    const FactorTables* f = find_factor(p, stg.factor);
    if (branched) {           // this stage's step size comes from its factor's branch
      for (const auto& br : p->pbr)
        if (br.factor == stg.factor) MS2G_CUDA(cudaStreamWaitEvent(st, br.done, 0));
    } else if (sd->power_iters > 0) {
      MS2G_TRY(enqueue_power(p, *f, sd->power_iters, p->w_scal + k, p->w_scal + 64 + k, p->w_etaf + k, st));
    } else {   // reuse the plan's cached step for this factor (geometry-only, S8(e))
      MS2G_TRY(launch_cached_step(f->d_Lcache, p->w_scal + k, p->w_scal + 64 + k, p->w_etaf + k, st));
    }
    int step_in_stage = 0;
    if (sd->option == 5 && step < sch.size() && sch[step].stage == k) {
      // SAGA table at the stage start: phi_q = c_q A_{M_q}^T (A_{M_q} S y - b), avg = mean_q phi_q
      const size_t ncimg = (size_t)f->nc * f->nc * batch;
      float* avg = p->w_saga + (size_t)sd->n_subsets * ncimg;
      MS2G_TRY(launch_fill(avg, ncimg, 0.f, st));
      MS2G_TRY(prep_pairs(p, *f, sd->resampler, batch, p->w_y, st));
      for (int q = 0; q < sd->n_subsets; ++q) {
        float* ph = p->w_saga + (size_t)q * ncimg;
        const float cq = (float)((double)p->d.n_views / (double)p->subset_global_len[q]);
        MS2G_TRY(launch_forward(p, *f, b, p->w_res, p->w_subsets + p->subset_off[q], p->subset_len[q], batch, st,
                                f->d_fwd_order_sub[q]));
        MS2G_TRY(backward_sum(p, *f, p->w_res, ph, cq, p->w_subsets + p->subset_off[q], p->subset_len[q], batch, st,
                              f->d_bp_order_sub[q]));
        MS2G_TRY(launch_axpby(avg, avg, ph, 1.f, 1.f / (float)sd->n_subsets, ncimg, st));
      }
    }
    while (step < sch.size() && sch[step].stage == k) {
      const ms2g_sched_entry& e = sch[step];
      const int* d_sel = nullptr;
      const int *ford = nullptr, *bord = nullptr;   // longest-first block orders of a subset launch
      int n_sel = p->V_r;
      float c = 1.f;
      if (sd->option == 4) {
        d_sel = p->w_mb + p->mb_off[step];
        n_sel = p->mb_len[step];
        c = (float)((double)p->d.n_views / (double)sd->n_subsets);
      } else if (e.subset >= 0) {
        d_sel = p->w_subsets + p->subset_off[e.subset];
        n_sel = p->subset_len[e.subset];
        c = (float)((double)p->d.n_views / (double)p->subset_global_len[e.subset]);
        static const bool sub_off = getenv("MS2G_SUB_NO_ORDER") != nullptr;   // experiment switch
        if ((int)f->d_bp_order_sub.size() == p->subsets_n && !sub_off) {
          bord = f->d_bp_order_sub[e.subset];
          ford = f->d_fwd_order_sub[e.subset];
        }
      }
      // G-step: z = y - eta_k U (c A_s^T (A_s S y - b_M))       (Options 1, 2)
      //         z = y - eta_k U (c A_M^T A_M S (y - xs) + mu)  (Option 3, SVRG)
      const size_t ncimg = (size_t)f->nc * f->nc * batch;
      const int kind = sd->resampler;
      if (sd->option == 3) {
        if (step_in_stage % sd->n_subsets == 0) {   // epoch start: snapshot xs = y, mu = g_s(xs) (all views)
          MS2G_CUDA(cudaMemcpyAsync(p->w_snap, p->w_y, sizeof(float) * img, cudaMemcpyDeviceToDevice, st));
          MS2G_TRY(prep_pairs(p, *f, kind, batch, p->w_y, st));
          MS2G_TRY(launch_forward(p, *f, b, p->w_res, nullptr, p->V_r, batch, st));
          MS2G_TRY(backward_sum(p, *f, p->w_res, p->w_mu, 1.f, nullptr, p->V_r, batch, st));
        }
        MS2G_TRY(launch_axpby(p->w_z, p->w_y, p->w_snap, 1.f, -1.f, img, st));   // d = y - xs
        MS2G_TRY(prep_pairs(p, *f, kind, batch, p->w_z, st));
        MS2G_TRY(launch_forward(p, *f, nullptr, p->w_res, d_sel, n_sel, batch, st, ford));
        MS2G_TRY(backward_sum(p, *f, p->w_res, p->w_G, c, d_sel, n_sel, batch, st, bord));
        MS2G_TRY(launch_axpby(p->w_G, p->w_G, p->w_mu, 1.f, 1.f, ncimg, st));  // + mu
      } else if (sd->option == 5) {
        MS2G_TRY(prep_pairs(p, *f, kind, batch, p->w_y, st));
        MS2G_TRY(launch_forward(p, *f, b, p->w_res, d_sel, n_sel, batch, st, ford));
        MS2G_TRY(backward_sum(p, *f, p->w_res, p->w_G, c, d_sel, n_sel, batch, st, bord));
        // G = new - phi_j + avg; phi_j = new; avg += (new - phi_j)/K
        MS2G_TRY(launch_saga(p->w_G, p->w_saga + (size_t)e.subset * ncimg,
                             p->w_saga + (size_t)sd->n_subsets * ncimg, sd->n_subsets, ncimg, st));
      } else {   // Options 1, 2, 4: v = S y, r = A_s v - b_M, z = y - eta U (c A_s^T r) in 4 launches
        MS2G_TRY(prep_pairs(p, *f, kind, batch, p->w_y, st));
        MS2G_TRY(launch_forward(p, *f, b, p->w_res, d_sel, n_sel, batch, st, ford));
        MS2G_TRY(backward_step(p, *f, kind, p->w_res, c, d_sel, n_sel, batch, p->w_y, p->w_etaf + k, p->w_z, st,
                               bord));
      }
      if (sd->option == 3 || sd->option == 5)
        MS2G_TRY(launch_resample_up_step(p, *f, kind, batch, p->w_G, p->w_y, p->w_etaf + k, 0.f, p->w_z, st));
      // x = (1-alpha) z + alpha D(z);  y = x + a_i (x - x_prev)
      MS2G_TRY(denoise_mix(p, sd->den, p->w_z, p->w_x[cur], p->w_x[cur ^ 1], p->w_y, sd->alpha, (float)e.a, 1,
                           e.i, batch, st));
      cur ^= 1;
      ++step;
      ++step_in_stage;
    }
  }
  MS2G_CUDA(cudaMemcpyAsync(x_out, p->w_x[cur], sizeof(float) * img, cudaMemcpyDeviceToDevice, st));
  return MS2G_OK;
}

// Key of a captured solve graph.  Every parameter baked into the graph's
// kernel arguments enters with its exact bits (floats as their 32-bit
// patterns): two descriptors that differ anywhere never share a graph.
static std::string solve_key(const ms2g_solve_desc* sd, const float* b, const float* x0, const float* x_out) {
  auto bits = [](float f) {
    uint32_t u;
    memcpy(&u, &f, sizeof(u));
    return u;
  };
  std::ostringstream os;
  os << std::hex << sd->n_stages << ':' << sd->option << ':' << sd->n_subsets << ':' << sd->seed << ':'
     << sd->den.kind << ':' << bits(sd->den.sigma) << ':' << bits(sd->den.lambda) << ':' << bits(sd->den.tau) << ':'
     << sd->den.inner_iters << ':' << bits(sd->alpha) << ':' << sd->power_iters << ':' << sd->resampler << ':'
     << (const void*)b << ':' << (const void*)x0 << ':' << (const void*)x_out;
  for (int k = 0; k < sd->n_stages; ++k)
    os << '|' << sd->stages[k].factor << ',' << sd->stages[k].n_iters << ',' << sd->stages[k].n_epochs;
  return os.str();
}

static int solve_launch(ms2g_plan* p, const ms2g_solve_desc* sd, const float* b, const float* x0, float* x_out,
                        cudaStream_t st) {
  if (!b || !x0 || !x_out) return set_error(MS2G_ERR_INPUT, "NULL b/x0/x_out");
  if (p->peer_n > 0 || p->mc_n > 0) MS2G_TRY(peer_ok(p));   // a cached graph would replay the failed exchange
  if (!(sd->alpha > 0.f && sd->alpha <= 1.f)) return set_error(MS2G_ERR_CONFIG, "alpha must be in (0, 1] (S:197)");
  if (sd->power_iters < 0) return set_error(MS2G_ERR_CONFIG, "power_iters must be >= 0");
  if (sd->resampler != 0 && sd->resampler != 1) return set_error(MS2G_ERR_CONFIG, "resampler must be 0 or 1");
  MS2G_TRY(check_denoiser(sd->den));
  std::vector<ms2g_sched_entry> sch;
  MS2G_TRY(make_schedule(p, sd, sch));
  for (int k = 0; k < sd->n_stages; ++k) {
    const FactorTables* f = find_factor(p, sd->stages[k].factor);
    if (!f) return set_error(MS2G_ERR_CONFIG, "stage factor was not planned (ms2g_plan_geometry factors)");
    if (sd->power_iters == 0 && f->L_iters == 0)
      return set_error(MS2G_ERR_CONFIG, "power_iters = 0 reuses a cached step, but no power iteration has run "
                                        "on this plan for a stage factor");
  }
  if (!find_factor(p, 1) && p->nmax_c < p->d.n)
    return set_error(MS2G_ERR_CONFIG, "the solve needs full-resolution workspaces: plan factor 1 as well");
  if (sd->option == 2 || sd->option == 3 || sd->option == 5) MS2G_TRY(prepare_subsets(p, sd->n_subsets));
  if (sd->option == 5) {   // SAGA table (allocated outside capture)
    const size_t need = (size_t)(sd->n_subsets + 1) * p->nmax_c * p->nmax_c * p->d.batch;
    if (need > p->saga_elems) {
      cudaFree(p->w_saga);
      p->w_saga = nullptr;
      p->saga_elems = 0;
      MS2G_CUDA(cudaMalloc(&p->w_saga, sizeof(float) * need));
      p->saga_elems = need;
    }
  }
  const std::string key = solve_key(sd, b, x0, x_out);
  if (sd->option == 4 && (key != p->sg.key || !p->sg.exec)) MS2G_TRY(prepare_minibatches(p, sd, (int)sch.size()));
  if (sd->power_iters > 0 && power_branching(p)) MS2G_TRY(ensure_power_branches(p, sd));
  if (key != p->sg.key || !p->sg.exec) {
    if (p->sg.exec) cudaGraphExecDestroy(p->sg.exec);
    if (p->sg.graph) cudaGraphDestroy(p->sg.graph);
    p->sg = SolveGraph{};
    clear_timing_events(p);
    cudaStream_t cs;
    MS2G_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      cudaStreamDestroy(cs);
      return set_error(MS2G_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
    }
    t_capturing = true;
    t_captured = 0;
    int rc = enqueue_solve(p, sd, sch, b, x0, x_out, cs);
    t_capturing = false;
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc != MS2G_OK) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return set_error(MS2G_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(graph);
      return set_error(MS2G_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    p->sg.key = key;
    p->sg.graph = graph;
    p->sg.exec = exec;
    p->sg.kernel_nodes = t_captured;
  }
  MS2G_CUDA(cudaGraphLaunch(p->sg.exec, st));
  count_launch(p->sg.kernel_nodes);
  p->last_sched = sch;
  return MS2G_OK;
}

static int solve_status(ms2g_plan* p, cudaStream_t st) {
  int flags[2] = {INT_MAX, 0}, perr = 0, tverr = 0;
  MS2G_CUDA(cudaMemcpyAsync(flags, p->w_flag, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  const int flag = flags[0];
  if (p->tvws.err) MS2G_CUDA(cudaMemcpyAsync(&tverr, p->tvws.err, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (p->w_peer_err) MS2G_CUDA(cudaMemcpyAsync(&perr, p->w_peer_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  MS2G_CUDA(cudaStreamSynchronize(st));
  if (tverr) return set_error(MS2G_ERR_CUDA, "persistent TV-prox kernel: a neighbour wait timed out");
  if (flags[1]) return set_error(MS2G_ERR_INPUT, "non-finite value (NaN or Inf) in b or x0 (S:258)");
  if (perr) {
    p->peer_failed = true;     // epochs are out of step: refuse exchanges until every rank re-attaches
    return set_error(MS2G_ERR_NCCL, "peer allreduce: barrier timed out (a rank never arrived); "
                                    "call ms2g_attach_peers again on every rank");
  }
  if (flag != INT_MAX) {
    int stage = -1;
    for (const auto& e : p->last_sched)
      if (e.i == flag) stage = e.stage;
    std::ostringstream os;
    os << "diverged: non-finite iterate at stage " << stage << ", iteration " << flag;
    return set_error(MS2G_ERR_DIVERGED, os.str());
  }
  return MS2G_OK;
}

}  // namespace ms2g

using namespace ms2g;

extern "C" {

const char* ms2g_last_error(void) { return t_err.c_str(); }

uint64_t ms2g_launch_count(void) { return g_launches.load(); }

int ms2g_plan_geometry(const ms2g_geom_desc* desc, const int32_t* factors, int32_t n_factors, ms2g_plan** out) {
  NvtxRange nvtx_range__("ms2g_plan_geometry");
  t_err.clear();
  if (!desc || !out) return set_error(MS2G_ERR_INPUT, "NULL desc/out");
  *out = nullptr;
  ms2g_geom_desc d = *desc;
  if (d.n < 1 || !(d.fov > 0) || d.n_views < 1 || d.n_bins < 1 || !(d.arc_rad > 0))
    return set_error(MS2G_ERR_CONFIG, "need n, fov, n_views, n_bins, arc_rad > 0");
  const double R = d.fov / std::sqrt(2.0);
  if (!(d.sod > R) || !(d.sdd - d.sod > R))
    return set_error(MS2G_ERR_CONFIG, "source and detector must lie outside the FOV circle (sod, sdd-sod > fov/sqrt2)");
  if (d.view_begin == 0 && d.view_end == 0) d.view_end = d.n_views;
  if (d.view_begin < 0 || d.view_end > d.n_views || d.view_begin >= d.view_end)
    return set_error(MS2G_ERR_CONFIG, "view shard [view_begin, view_end) out of range");
  if (d.batch < 1) d.batch = 1;
  if (!factors || n_factors < 1) return set_error(MS2G_ERR_CONFIG, "need at least one factor");
  for (int k = 0; k < n_factors; ++k)
    if (factors[k] < 1 || d.n % factors[k] != 0)
      return set_error(MS2G_ERR_CONFIG, "every factor must be >= 1 and divide n (S:127, S:145)");
  // host-only geometry checks first: they need no device (testable on CPU)
  MS2G_TRY(check_grid_ties(d, d.bin_pitch > 0 ? d.bin_pitch : (d.sdd / d.sod) * d.fov / d.n, factors, n_factors));
  ms2g_plan* p = new ms2g_plan();
  p->d = d;
  p->V_r = d.view_end - d.view_begin;
  p->B = d.n_bins;
  p->pitch = d.bin_pitch > 0 ? d.bin_pitch : (d.sdd / d.sod) * d.fov / d.n;
  int dev = 0, sms = 148;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    delete p;
    return set_error(MS2G_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  for (int k = 0; k < n_factors; ++k) {
    const int s = factors[k];
    if (s < 1 || d.n % s != 0) {
      delete p;
      return set_error(MS2G_ERR_CONFIG, "every factor must be >= 1 and divide n (S:127, S:145)");
    }
    if (d.n / s > 32767) {
      delete p;
      return set_error(MS2G_ERR_CONFIG, "n/factor must be <= 32767");
    }
    if (find_factor(p, s)) continue;
    FactorTables f;
    f.factor = s;
    p->ft.push_back(f);
  }
  int rc = MS2G_OK;
  size_t part = 1;
  p->sm_count = sms;
  p->class_mask = 0;   // filled by build_tables
  for (auto& f : p->ft) {
    rc = build_tables(p, f, sms);
    if (rc != MS2G_OK) {
      free_plan(p);
      return rc;
    }
    if (f.nc > p->nmax_c) p->nmax_c = f.nc;
    const size_t need = (size_t)(f.bp_chunks[0] + f.bp_chunks[1]) * f.nc * f.nc * d.batch;   // family chunks
    if (need > part) part = need;
  }
  const size_t bt = d.batch;
  const size_t cimg = (size_t)p->nmax_c * p->nmax_c * bt, fimg = (size_t)d.n * d.n * bt;
  auto alloc = [&](float** q, size_t count) -> int {
    MS2G_CUDA(cudaMalloc(q, sizeof(float) * (count ? count : 1)));
    return MS2G_OK;
  };
  p->red_blocks = 8 * sms;   // k_reduce_power grid cap (fp64 partials per block)
  p->pair_stride = (size_t)p->nmax_c * pair_line(p->nmax_c) * bt;
  e = cudaMalloc(&p->w_pair, sizeof(float2) * 4 * p->pair_stride);
  if (e != cudaSuccess) {
    free_plan(p);
    return set_error(MS2G_ERR_CUDA, std::string("pair image allocation: ") + cudaGetErrorString(e));
  }
  if ((rc = alloc(&p->w_v, cimg)) || (rc = alloc(&p->w_rs, fimg)) || (rc = alloc(&p->w_snap, fimg)) ||
      (rc = alloc(&p->w_mu, cimg)) ||
      (rc = alloc(&p->w_G, cimg)) || (rc = alloc(&p->w_res, (size_t)p->V_r * p->B * bt)) ||
      (rc = alloc(&p->w_part, part)) || (rc = alloc(&p->w_x[0], fimg)) || (rc = alloc(&p->w_x[1], fimg)) ||
      (rc = alloc(&p->w_y, fimg)) || (rc = alloc(&p->w_z, fimg)) || (rc = alloc(&p->w_p[0], 2 * fimg)) ||
      (rc = alloc(&p->w_p[1], 2 * fimg)) || (rc = alloc(&p->w_etaf, 64))) {
    free_plan(p);
    return rc;
  }
  p->part_elems = part;
  e = cudaMalloc(&p->w_red, sizeof(double) * 2 * p->red_blocks);
  if (e == cudaSuccess) e = cudaMalloc(&p->w_scal, sizeof(double) * 128);
  if (e == cudaSuccess) e = cudaMalloc(&p->w_pw, sizeof(double) * 2);
  if (e == cudaSuccess) e = cudaMalloc(&p->w_ticket, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(p->w_ticket, 0, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMalloc(&p->w_rmaxv, sizeof(unsigned) * (size_t)p->V_r * bt);
  if (e == cudaSuccess) e = cudaMemset(p->w_rmaxv, 0, sizeof(unsigned) * (size_t)p->V_r * bt);
  {  // persistent TV-prox workspace: one CTA per SM at most, rows of the full-resolution grid
    int optin = 0;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    ms2g::TvWs& w = p->tvws;
    w.max_ctas = sms;
    w.smem_optin = optin;
    if (e == cudaSuccess) e = cudaMalloc(&w.flags, sizeof(unsigned long long) * sms);
    if (e == cudaSuccess) e = cudaMemset(w.flags, 0, sizeof(unsigned long long) * sms);
    if (e == cudaSuccess) e = cudaMalloc(&w.gen_ticket, 2 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(w.gen_ticket, 0, 2 * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&w.err, sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(w.err, 0, sizeof(int));
  }
  if (e == cudaSuccess) e = cudaMalloc(&p->w_flag, 2 * sizeof(int));   // {diverged iteration, input flag}
  if (e == cudaSuccess) e = cudaMalloc(&p->w_sel, sizeof(int) * p->V_r * ms2g_plan::kSelRing);
  if (e == cudaSuccess) e = cudaMallocHost(&p->h_sel, sizeof(int) * p->V_r * ms2g_plan::kSelRing);
  for (int k = 0; k < ms2g_plan::kSelRing && e == cudaSuccess; ++k)
    e = cudaEventCreateWithFlags(&p->sel_ev[k], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemset(p->w_flag, 0x7f, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(p->w_flag + 1, 0, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(p->w_scal, 0, sizeof(double) * 128);
  if (e != cudaSuccess) {
    free_plan(p);
    return set_error(MS2G_ERR_CUDA, std::string("workspace allocation: ") + cudaGetErrorString(e));
  }
  *out = p;
  return MS2G_OK;
}

void ms2g_plan_destroy(ms2g_plan* plan) {
  if (plan) cudaDeviceSynchronize();
  free_plan(plan);
}

int ms2g_plan_info(const ms2g_plan* p, int32_t factor, int32_t* n_c, int32_t* vb, int32_t* ve, int32_t* batch) {
  if (!p) return set_error(MS2G_ERR_INPUT, "NULL plan");
  const FactorTables* f = find_factor(p, factor);
  if (n_c) *n_c = f ? f->nc : 0;
  if (vb) *vb = p->d.view_begin;
  if (ve) *ve = p->d.view_end;
  if (batch) *batch = p->d.batch;
  return MS2G_OK;
}

int ms2g_set_kernel_timing(ms2g_plan* p, int32_t enable) {
  if (!p) return set_error(MS2G_ERR_INPUT, "NULL plan");
  if ((enable != 0) != p->timing) {
    p->timing = enable != 0;
    if (p->sg.exec) {   // the cached solve graph is re-captured with / without the event nodes
      cudaGraphExecDestroy(p->sg.exec);
      cudaGraphDestroy(p->sg.graph);
      p->sg = SolveGraph{};
    }
    clear_timing_events(p);
  }
  return MS2G_OK;
}

int ms2g_kernel_time(ms2g_plan* p, int32_t kind, int32_t factor, double* total_ms, int32_t* launches) {
  if (!p || !total_ms || !launches) return set_error(MS2G_ERR_INPUT, "NULL plan/total_ms/launches");
  double t = 0.0;
  int n = 0;
  for (const auto& tl : p->tev) {
    if (tl.kind != kind || tl.factor != factor) continue;
    MS2G_CUDA(cudaEventSynchronize(tl.b));
    float ms = 0.f;
    MS2G_CUDA(cudaEventElapsedTime(&ms, tl.a, tl.b));
    t += ms;
    ++n;
  }
  *total_ms = t;
  *launches = n;
  return MS2G_OK;
}

int ms2g_nccl_unique_id(void* out) {
  if (!out) return set_error(MS2G_ERR_INPUT, "NULL id buffer");
  ncclUniqueId id;
  MS2G_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, sizeof(id));
  return MS2G_OK;
}

int ms2g_attach_nccl(ms2g_plan* p, const void* uid, int32_t rank, int32_t nranks) {
  NvtxRange nvtx_range__("ms2g_attach_nccl");
  if (!p || !uid) return set_error(MS2G_ERR_INPUT, "NULL plan/id");
  if (nranks < 1 || rank < 0 || rank >= nranks) return set_error(MS2G_ERR_CONFIG, "bad rank/nranks");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  if (p->comm) {
    ncclCommDestroy(p->comm);
    p->comm = nullptr;
  }
  MS2G_NCCL(ncclCommInitRank(&p->comm, nranks, id, rank));
  for (auto& gg : p->grad_graphs) {   // per-call gradient graphs captured without it
    if (gg.exec) cudaGraphExecDestroy(gg.exec);
    if (gg.graph) cudaGraphDestroy(gg.graph);
  }
  p->grad_graphs.clear();
  p->topo_version++;
  p->rank = rank;
  p->nranks = nranks;
  if (p->sg.exec) {  // a cached solve graph captured without the communicator
    cudaGraphExecDestroy(p->sg.exec);
    cudaGraphDestroy(p->sg.graph);
    p->sg = SolveGraph{};
  }
  return MS2G_OK;
}

// ---- NEXT-3: peer-memory allreduce (peer_reduce.cu) ----
namespace {
struct PeerBlob {
  uint64_t magic;
  uint64_t slot;                 // floats per exchange slot
  cudaIpcMemHandle_t buf, pad;
};
constexpr uint64_t kPeerMagic = 0x4d53324750454552ULL;   // "MS2GPEER"
constexpr int kPadWords = 256;   // peer_reduce.cu: PUB[64], RED[64], epoch, time-out, ticket
}  // namespace

static int ensure_exchange(ms2g_plan* p) {
  if (p->xch_buf) return MS2G_OK;
  p->xch_slot = (size_t)p->nmax_c * p->nmax_c * p->d.batch;
  MS2G_CUDA(cudaMalloc(&p->xch_buf, sizeof(float) * 2 * p->xch_slot));
  MS2G_CUDA(cudaMalloc(&p->xch_pad, sizeof(unsigned) * kPadWords));
  MS2G_CUDA(cudaMemset(p->xch_pad, 0, sizeof(unsigned) * kPadWords));
  MS2G_CUDA(cudaMalloc(&p->w_peer_err, sizeof(int)));
  MS2G_CUDA(cudaMemset(p->w_peer_err, 0, sizeof(int)));
  return MS2G_OK;
}

int ms2g_peer_blob_size(void) { return (int)sizeof(PeerBlob); }

int ms2g_peer_export(ms2g_plan* p, void* blob) {
  if (!p || !blob) return set_error(MS2G_ERR_INPUT, "NULL plan/blob");
  MS2G_TRY(ensure_exchange(p));
  PeerBlob b{};
  b.magic = kPeerMagic;
  b.slot = p->xch_slot;
  MS2G_CUDA(cudaIpcGetMemHandle(&b.buf, p->xch_buf));
  MS2G_CUDA(cudaIpcGetMemHandle(&b.pad, p->xch_pad));
  memcpy(blob, &b, sizeof(b));
  return MS2G_OK;
}

int ms2g_attach_peers(ms2g_plan* p, const void* blobs, int32_t rank, int32_t nranks) {
  NvtxRange nvtx_range__("ms2g_attach_peers");
  if (!p || !blobs) return set_error(MS2G_ERR_INPUT, "NULL plan/blobs");
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) return set_error(MS2G_ERR_CONFIG, "bad rank/nranks");
  if (p->peer_n > 0 && !p->peer_failed) return set_error(MS2G_ERR_CONFIG, "peers already attached");
  if (p->peer_n > 0) {        // re-attach after a time-out: fresh mappings, epochs and error flag
    MS2G_CUDA(cudaDeviceSynchronize());
    for (void* q : p->peer_opened) cudaIpcCloseMemHandle(q);
    p->peer_opened.clear();
    cudaFree(p->d_peer_bufs);
    cudaFree(p->d_peer_pads);
    p->d_peer_bufs = nullptr;
    p->d_peer_pads = nullptr;
    p->peer_n = 0;
    MS2G_CUDA(cudaMemset(p->xch_pad, 0, sizeof(unsigned) * kPadWords));
    MS2G_CUDA(cudaMemset(p->w_peer_err, 0, sizeof(int)));
    p->peer_failed = false;
  }
  MS2G_TRY(ensure_exchange(p));
  std::vector<float*> bufs(nranks);
  std::vector<unsigned*> pads(nranks);
  for (int q = 0; q < nranks; ++q) {
    PeerBlob b;
    memcpy(&b, (const char*)blobs + (size_t)q * sizeof(PeerBlob), sizeof(b));
    if (b.magic != kPeerMagic || b.slot != p->xch_slot)
      return set_error(MS2G_ERR_CONFIG, "peer blob mismatch (different plan shapes or corrupt exchange)");
    if (q == rank) {
      bufs[q] = p->xch_buf;
      pads[q] = p->xch_pad;
      continue;
    }
    void *pb = nullptr, *pp = nullptr;
    MS2G_CUDA(cudaIpcOpenMemHandle(&pb, b.buf, cudaIpcMemLazyEnablePeerAccess));
    p->peer_opened.push_back(pb);
    MS2G_CUDA(cudaIpcOpenMemHandle(&pp, b.pad, cudaIpcMemLazyEnablePeerAccess));
    p->peer_opened.push_back(pp);
    bufs[q] = (float*)pb;
    pads[q] = (unsigned*)pp;
  }
  MS2G_CUDA(cudaMalloc(&p->d_peer_bufs, sizeof(float*) * nranks));
  MS2G_CUDA(cudaMalloc(&p->d_peer_pads, sizeof(unsigned*) * nranks));
  MS2G_CUDA(cudaMemcpy(p->d_peer_bufs, bufs.data(), sizeof(float*) * nranks, cudaMemcpyHostToDevice));
  MS2G_CUDA(cudaMemcpy(p->d_peer_pads, pads.data(), sizeof(unsigned*) * nranks, cudaMemcpyHostToDevice));
  for (auto& gg : p->grad_graphs) {   // per-call gradient graphs captured without it
    if (gg.exec) cudaGraphExecDestroy(gg.exec);
    if (gg.graph) cudaGraphDestroy(gg.graph);
  }
  p->grad_graphs.clear();
  p->topo_version++;
  p->peer_rank = rank;
  p->peer_n = nranks;
  p->rank = rank;
  p->nranks = nranks;
  if (p->sg.exec) {  // a cached solve graph captured without the peers
    cudaGraphExecDestroy(p->sg.exec);
    cudaGraphDestroy(p->sg.graph);
    p->sg = SolveGraph{};
  }
  return MS2G_OK;
}

// A resolved view selection: an ad-hoc host subset in a ring slot, a
// registered subset (with its longest-first block orders), or all views.
struct Sel {
  const int* d_sel = nullptr;
  int n_sel = 0, n_glob = 0, slot = -1;
  const int* ford = nullptr;
  const int* bord = nullptr;
};

static int sel_host(ms2g_plan* p, const int32_t* subset, int32_t n_subset, cudaStream_t st, Sel* s) {
  return resolve_subset(p, subset, n_subset, st, &s->d_sel, &s->n_sel, &s->n_glob, &s->slot);
}

static int sel_registered(ms2g_plan* p, int32_t id, const FactorTables* f, Sel* s) {
  if (id < 0 || id >= (int)p->reg.size() || !p->reg[id].d_sel)
    return set_error(MS2G_ERR_INPUT, "unknown or released subset id");
  const auto& r = p->reg[id];
  const int fi = (int)(f - p->ft.data());
  s->d_sel = r.d_sel;
  s->n_sel = r.n_sel;
  s->n_glob = r.n_global;
  s->ford = r.fwd_order.empty() ? nullptr : r.fwd_order[fi];
  s->bord = r.bp_order.empty() ? nullptr : r.bp_order[fi];
  return MS2G_OK;
}

static int do_forward(ms2g_plan* p, const FactorTables* f, const float* x, const float* b, float* out,
                      const Sel& s, cudaStream_t st) {
  MS2G_TRY(launch_pair_prep(p, f->nc, p->d.batch, x, st));
  return launch_forward(p, *f, b, out, s.d_sel, s.n_sel, p->d.batch, st, s.ford);
}

// Every launch_backward needs p->w_rmaxv to bound |sino| per view (the
// fixed-point adjoint's scale, projector.cu): written by the launch_forward
// that produced sino (all solve / gradient / power paths), or here by
// launch_view_absmax for a caller's sinogram.  A stale larger bound only
// coarsens the scale; a missing one (0) would give sigma = 1.
static int do_backward(ms2g_plan* p, const FactorTables* f, const float* sino, float* img, float scale,
                       int accumulate, int do_allreduce, const Sel& s, cudaStream_t st) {
  MS2G_TRY(launch_view_absmax(p, sino, s.n_sel, p->d.batch, st));   // a caller's sinogram: its per-view bounds
  MS2G_TRY(launch_backward(p, *f, sino, img, scale, accumulate, s.d_sel, s.n_sel, p->d.batch, st, 0, s.bord));
  if (do_allreduce) MS2G_TRY(allreduce(p, img, (size_t)f->nc * f->nc * p->d.batch, st));
  return MS2G_OK;
}

static int do_grad(ms2g_plan* p, const FactorTables* f, int kind, const float* x, const float* b, float* g,
                   const Sel& s, cudaStream_t st) {
  const float c = (float)((double)p->d.n_views / (double)s.n_glob);
  return enqueue_grad(p, *f, kind, x, b, g, s.d_sel, s.n_sel, c, p->d.batch, st, s.ford, s.bord);
}

static void destroy_graph(SolveGraph& gg) {
  if (gg.exec) cudaGraphExecDestroy(gg.exec);
  if (gg.graph) cudaGraphDestroy(gg.graph);
  gg = SolveGraph{};
}

// The standalone gradient is 4 launches (fused sketch + pair prep, forward,
// backprojection, fused chunk sum + upsample); a loop of such calls (the
// method's inner loop driven from outside) is launch-bound at small sizes,
// so calls without host-side staging (all views or a registered subset) are
// captured once per (factor, kind, selection, pointers) into a CUDA graph and
// replayed: one launch per call (SURVEY §7 "small configs are launch-bound").
static int grad_graph(ms2g_plan* p, const FactorTables* f, int kind, const float* x, const float* b, float* g,
                      const Sel& s, int sel_id, cudaStream_t st) {
  static const bool off = getenv("MS2G_GRAD_GRAPHS") && atoi(getenv("MS2G_GRAD_GRAPHS")) == 0;   // experiment switch
  if (off || p->timing || t_capturing) return do_grad(p, f, kind, x, b, g, s, st);
  if (p->peer_n > 0 || p->mc_n > 0) MS2G_TRY(peer_ok(p));   // a cached graph would replay a failed exchange
  std::ostringstream os;
  os << f->factor << ':' << kind << ':' << sel_id << ':' << (const void*)x << ':' << (const void*)b << ':'
     << (const void*)g << ':' << p->topo_version;
  const std::string key = os.str();
  for (size_t k = 0; k < p->grad_graphs.size(); ++k) {
    if (p->grad_graphs[k].key != key) continue;
    std::rotate(p->grad_graphs.begin(), p->grad_graphs.begin() + k, p->grad_graphs.begin() + k + 1);
    MS2G_CUDA(cudaGraphLaunch(p->grad_graphs[0].exec, st));
    count_launch(p->grad_graphs[0].kernel_nodes);
    return MS2G_OK;
  }
  cudaStream_t cs;
  MS2G_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    cudaStreamDestroy(cs);
    return set_error(MS2G_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
  }
  t_capturing = true;
  t_captured = 0;
  const int rc = do_grad(p, f, kind, x, b, g, s, cs);
  t_capturing = false;
  SolveGraph gg;
  e = cudaStreamEndCapture(cs, &gg.graph);
  cudaStreamDestroy(cs);
  if (rc != MS2G_OK) {
    destroy_graph(gg);
    return rc;
  }
  if (e != cudaSuccess) return set_error(MS2G_ERR_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&gg.exec, gg.graph, 0);
  if (e != cudaSuccess) {
    destroy_graph(gg);
    return set_error(MS2G_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
  }
  gg.key = key;
  gg.kernel_nodes = t_captured;
  if ((int)p->grad_graphs.size() == ms2g_plan::kGradGraphs) {
    destroy_graph(p->grad_graphs.back());
    p->grad_graphs.pop_back();
  }
  p->grad_graphs.insert(p->grad_graphs.begin(), gg);
  MS2G_CUDA(cudaGraphLaunch(p->grad_graphs[0].exec, st));
  count_launch(gg.kernel_nodes);
  return MS2G_OK;
}

static int check_fwd(ms2g_plan* p, int32_t factor, const float* x, const float* out, const FactorTables** f) {
  if (!p || !x || !out) return set_error(MS2G_ERR_INPUT, "NULL plan/x/out");
  *f = find_factor(p, factor);
  if (!*f) return set_error(MS2G_ERR_CONFIG, "factor not in plan");
  return MS2G_OK;
}

static int check_bwd(ms2g_plan* p, int32_t factor, const float* sino, const float* img, int do_allreduce,
                     const FactorTables** f) {
  if (!p || !sino || !img) return set_error(MS2G_ERR_INPUT, "NULL plan/sino/img");
  *f = find_factor(p, factor);
  if (!*f) return set_error(MS2G_ERR_CONFIG, "factor not in plan");
  if (do_allreduce && !p->comm && !p->peer_n && !p->mc_n && p->nranks > 1)
    return set_error(MS2G_ERR_CONFIG, "allreduce needs attach_nccl or attach_peers");
  return MS2G_OK;
}

static int check_grad(ms2g_plan* p, int32_t factor, int32_t kind, const float* x, const float* b, const float* g,
                      const FactorTables** f) {
  if (kind != 0 && kind != 1) return set_error(MS2G_ERR_CONFIG, "kind must be 0 or 1");
  if (!p || !x || !b || !g) return set_error(MS2G_ERR_INPUT, "NULL plan/x/b/g");
  *f = find_factor(p, factor);
  if (!*f) return set_error(MS2G_ERR_CONFIG, "factor not in plan");
  if (factor != 1 && p->nmax_c < (*f)->nc) return set_error(MS2G_ERR_CONFIG, "workspace too small");
  return MS2G_OK;
}

int ms2g_mc_blob_size(void) { return mc_blob_size(); }

int ms2g_mc_create(ms2g_plan* p, int32_t nranks, void* blob_out) {
  if (!p || !blob_out) return set_error(MS2G_ERR_INPUT, "NULL plan/blob");
  if (p->mc_n > 0 || p->mc_handle) return set_error(MS2G_ERR_CONFIG, "multicast already created / attached");
  if (!p->xch_slot) p->xch_slot = (size_t)p->nmax_c * p->nmax_c * p->d.batch;
  return mc_create(p, nranks, blob_out);
}

int ms2g_attach_multicast(ms2g_plan* p, const void* blob_rank0, int32_t rank, int32_t nranks, int32_t phase) {
  if (!p || !blob_rank0) return set_error(MS2G_ERR_INPUT, "NULL plan/blob");
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks || (phase != 0 && phase != 1))
    return set_error(MS2G_ERR_CONFIG, "bad rank/nranks/phase");
  if (p->mc_n > 0) return set_error(MS2G_ERR_CONFIG, "multicast already attached");
  if (!p->xch_slot) p->xch_slot = (size_t)p->nmax_c * p->nmax_c * p->d.batch;
  MS2G_TRY(mc_attach(p, blob_rank0, rank, nranks, phase));
  if (phase == 1) {
    for (auto& gg : p->grad_graphs) {
      if (gg.exec) cudaGraphExecDestroy(gg.exec);
      if (gg.graph) cudaGraphDestroy(gg.graph);
    }
    p->grad_graphs.clear();
    p->topo_version++;
    if (p->sg.exec) {
      cudaGraphExecDestroy(p->sg.exec);
      cudaGraphDestroy(p->sg.graph);
      p->sg = SolveGraph{};
    }
  }
  return MS2G_OK;
}

int ms2g_forward_project(ms2g_plan* p, int32_t factor, const float* x, const float* b, float* out,
                         const int32_t* subset, int32_t n_subset, void* stream) {
  NvtxRange nvtx_range__("ms2g_forward_project");
  const FactorTables* f;
  MS2G_TRY(check_fwd(p, factor, x, out, &f));
  cudaStream_t st = (cudaStream_t)stream;
  Sel s;
  MS2G_TRY(sel_host(p, subset, n_subset, st, &s));
  const int rc = do_forward(p, f, x, b, out, s, st);
  MS2G_TRY(release_subset(p, s.slot, st));
  return rc;
}

int ms2g_back_project(ms2g_plan* p, int32_t factor, const float* sino, float* img, float scale, int32_t accumulate,
                      const int32_t* subset, int32_t n_subset, int32_t do_allreduce, void* stream) {
  NvtxRange nvtx_range__("ms2g_back_project");
  const FactorTables* f;
  MS2G_TRY(check_bwd(p, factor, sino, img, do_allreduce, &f));
  cudaStream_t st = (cudaStream_t)stream;
  Sel s;
  MS2G_TRY(sel_host(p, subset, n_subset, st, &s));
  const int rc = do_backward(p, f, sino, img, scale, accumulate, do_allreduce, s, st);
  MS2G_TRY(release_subset(p, s.slot, st));
  return rc;
}

int ms2g_sketched_grad(ms2g_plan* p, int32_t factor, int32_t kind, const float* x, const float* b, float* g,
                       const int32_t* subset, int32_t n_subset, void* stream) {
  NvtxRange nvtx_range__("ms2g_sketched_grad");
  const FactorTables* f;
  MS2G_TRY(check_grad(p, factor, kind, x, b, g, &f));
  cudaStream_t st = (cudaStream_t)stream;
  Sel s;
  MS2G_TRY(sel_host(p, subset, n_subset, st, &s));
  const int rc = subset ? do_grad(p, f, kind, x, b, g, s, st) : grad_graph(p, f, kind, x, b, g, s, -1, st);
  MS2G_TRY(release_subset(p, s.slot, st));
  return rc;
}

int ms2g_register_subset(ms2g_plan* p, const int32_t* subset, int32_t n_subset, int32_t* id) {
  NvtxRange nvtx_range__("ms2g_register_subset");
  if (!p || !subset || !id) return set_error(MS2G_ERR_INPUT, "NULL plan/subset/id");
  int m = 0;
  MS2G_TRY(check_subset(p, subset, n_subset, &m));
  ms2g_plan::RegSubset r;
  std::vector<int> local;
  for (int i = 0; i < n_subset; ++i)
    if (subset[i] >= p->d.view_begin && subset[i] < p->d.view_end) local.push_back(subset[i] - p->d.view_begin);
  r.n_sel = m;
  r.n_global = n_subset;
  MS2G_CUDA(cudaMalloc(&r.d_sel, sizeof(int) * std::max(m, 1)));
  if (m > 0) MS2G_CUDA(cudaMemcpy(r.d_sel, local.data(), sizeof(int) * m, cudaMemcpyHostToDevice));
  if (m > 0) {
    for (const auto& f : p->ft) {
      int* o = nullptr;
      MS2G_TRY(upload_bp_order(p, f, local, &o));
      r.bp_order.push_back(o);
      o = nullptr;
      if (p->d.batch % 2 != 0) MS2G_TRY(upload_fwd_order(p, f, local, fwd_views_per_block(p, m, p->d.batch), &o));
      r.fwd_order.push_back(o);
    }
  }
  p->reg.push_back(r);
  *id = (int32_t)p->reg.size() - 1;
  return MS2G_OK;
}

int ms2g_release_subset(ms2g_plan* p, int32_t id) {
  if (!p || id < 0 || id >= (int)p->reg.size() || !p->reg[id].d_sel)
    return set_error(MS2G_ERR_INPUT, "unknown or released subset id");
  MS2G_CUDA(cudaDeviceSynchronize());   // no kernel of any stream may still read it
  for (auto& gg : p->grad_graphs) destroy_graph(gg);   // graphs may hold the list
  p->grad_graphs.clear();
  auto& r = p->reg[id];
  cudaFree(r.d_sel);
  for (int* q : r.bp_order) cudaFree(q);
  for (int* q : r.fwd_order) cudaFree(q);
  r = ms2g_plan::RegSubset{};
  return MS2G_OK;
}

int ms2g_forward_project_registered(ms2g_plan* p, int32_t factor, const float* x, const float* b, float* out,
                                    int32_t subset_id, void* stream) {
  NvtxRange nvtx_range__("ms2g_forward_project_registered");
  const FactorTables* f;
  MS2G_TRY(check_fwd(p, factor, x, out, &f));
  Sel s;
  MS2G_TRY(sel_registered(p, subset_id, f, &s));
  return do_forward(p, f, x, b, out, s, (cudaStream_t)stream);
}

int ms2g_back_project_registered(ms2g_plan* p, int32_t factor, const float* sino, float* img, float scale,
                                 int32_t accumulate, int32_t subset_id, int32_t do_allreduce, void* stream) {
  NvtxRange nvtx_range__("ms2g_back_project_registered");
  const FactorTables* f;
  MS2G_TRY(check_bwd(p, factor, sino, img, do_allreduce, &f));
  Sel s;
  MS2G_TRY(sel_registered(p, subset_id, f, &s));
  return do_backward(p, f, sino, img, scale, accumulate, do_allreduce, s, (cudaStream_t)stream);
}

int ms2g_sketched_grad_registered(ms2g_plan* p, int32_t factor, int32_t kind, const float* x, const float* b,
                                  float* g, int32_t subset_id, void* stream) {
  NvtxRange nvtx_range__("ms2g_sketched_grad_registered");
  const FactorTables* f;
  MS2G_TRY(check_grad(p, factor, kind, x, b, g, &f));
  Sel s;
  MS2G_TRY(sel_registered(p, subset_id, f, &s));
  return grad_graph(p, f, kind, x, b, g, s, subset_id, (cudaStream_t)stream);
}

int ms2g_sketch_down(ms2g_plan* p, int32_t factor, int32_t kind, const float* x, float* v, void* stream) {
  NvtxRange nvtx_range__("ms2g_sketch_down");
  if (!p || !x || !v) return set_error(MS2G_ERR_INPUT, "NULL plan/x/v");
  if (factor < 1 || p->d.n % factor) return set_error(MS2G_ERR_CONFIG, "factor must divide n (S:127)");
  if (kind != 0 && kind != 1) return set_error(MS2G_ERR_CONFIG, "kind must be 0 (mean) or 1 (bicubic)");
  if (kind == 0) return launch_sketch_down(p->d.n, factor, p->d.batch, x, v, (cudaStream_t)stream);
  const FactorTables* f = find_factor(p, factor);
  if (!f) return set_error(MS2G_ERR_CONFIG, "bicubic resampling needs the factor in the plan");
  return launch_resample_down(p, *f, kind, p->d.batch, x, v, (cudaStream_t)stream);
}

int ms2g_sketch_up(ms2g_plan* p, int32_t factor, int32_t kind, const float* g, const float* y, float eta, float* z,
                   void* stream) {
  NvtxRange nvtx_range__("ms2g_sketch_up");
  if (!p || !g || !z) return set_error(MS2G_ERR_INPUT, "NULL plan/g/z");
  if (factor < 1 || p->d.n % factor) return set_error(MS2G_ERR_CONFIG, "factor must divide n");
  if (kind != 0 && kind != 1) return set_error(MS2G_ERR_CONFIG, "kind must be 0 (replicate) or 1 (bicubic)");
  if (kind == 0) return launch_up_step(p->d.n, factor, p->d.batch, g, y, nullptr, y ? eta : 0.f, z, (cudaStream_t)stream);
  const FactorTables* f = find_factor(p, factor);
  if (!f) return set_error(MS2G_ERR_CONFIG, "bicubic resampling needs the factor in the plan");
  return launch_resample_up_step(p, *f, kind, p->d.batch, g, y, nullptr, y ? eta : 0.f, z, (cudaStream_t)stream);
}

int ms2g_power_iteration(ms2g_plan* p, int32_t factor, int32_t iters, double* L, void* stream) {
  NvtxRange nvtx_range__("ms2g_power_iteration");
  if (!p || !L) return set_error(MS2G_ERR_INPUT, "NULL plan/L");
  if (iters < 1) return set_error(MS2G_ERR_CONFIG, "iters must be >= 1");
  const FactorTables* f = find_factor(p, factor);
  if (!f) return set_error(MS2G_ERR_CONFIG, "factor not in plan");
  cudaStream_t st = (cudaStream_t)stream;
  MS2G_TRY(enqueue_power(p, *f, iters, p->w_scal + 127, nullptr, nullptr, st));
  MS2G_CUDA(cudaMemcpyAsync(L, p->w_scal + 127, sizeof(double), cudaMemcpyDeviceToHost, st));
  MS2G_CUDA(cudaStreamSynchronize(st));
  return MS2G_OK;
}

int ms2g_denoise(ms2g_plan* p, const ms2g_denoiser* den, const float* z, float* out, void* stream) {
  NvtxRange nvtx_range__("ms2g_denoise");
  if (!p || !den || !z || !out) return set_error(MS2G_ERR_INPUT, "NULL plan/den/z/out");
  if (z == out) return set_error(MS2G_ERR_INPUT, "z and out must not alias");
  MS2G_TRY(check_denoiser(*den));
  return denoise_mix(p, *den, z, nullptr, out, nullptr, 1.f, 0.f, 0, 0, p->d.batch, (cudaStream_t)stream);
}

int ms2g_schedule(const ms2g_plan* p, const ms2g_solve_desc* sd, ms2g_sched_entry* out, int32_t cap, int32_t* n_out) {
  std::vector<ms2g_sched_entry> sch;
  MS2G_TRY(make_schedule(p, sd, sch));
  if (n_out) *n_out = (int32_t)sch.size();
  for (size_t k = 0; k < sch.size() && (int)k < cap && out; ++k) out[k] = sch[k];
  return MS2G_OK;
}

int ms2g_schedule_views(const ms2g_plan* p, const ms2g_solve_desc* sd, int32_t step, int32_t* out, int32_t cap,
                        int32_t* n_out) {
  if (!p || !sd) return set_error(MS2G_ERR_INPUT, "NULL plan/desc");
  std::vector<ms2g_sched_entry> sch;
  MS2G_TRY(make_schedule(p, sd, sch));
  if (step < 0 || step >= (int)sch.size()) return set_error(MS2G_ERR_INPUT, "step out of range");
  std::vector<int> v;
  int m = 0;
  if (sd->option == 1) {
    m = p->d.n_views;
    v.resize(m);
    for (int q = 0; q < m; ++q) v[q] = q;
  } else if (sd->option == 4) {
    std::vector<int> g;
    minibatch_views(p->d.n_views, sd->n_subsets, sd->seed, step + 1, g);
    m = sd->n_subsets;
    v.assign(g.begin() + (size_t)step * m, g.begin() + (size_t)(step + 1) * m);
  } else {
    for (int q = sch[step].subset; q < p->d.n_views; q += sd->n_subsets) v.push_back(q);
    m = (int)v.size();
  }
  if (n_out) *n_out = m;
  for (int q = 0; q < m && q < cap && out; ++q) out[q] = v[q];
  return MS2G_OK;
}

int ms2g_pnp_ms2g_solve_async(ms2g_plan* p, const ms2g_solve_desc* sd, const float* b, const float* x0,
                              float* x_out, void* stream) {
  NvtxRange nvtx_range__("ms2g_pnp_ms2g_solve_async");
  if (!p || !sd) return set_error(MS2G_ERR_INPUT, "NULL plan/desc");
  return solve_launch(p, sd, b, x0, x_out, (cudaStream_t)stream);
}

int ms2g_solve_status(ms2g_plan* p, void* stream) {
  if (!p) return set_error(MS2G_ERR_INPUT, "NULL plan");
  return solve_status(p, (cudaStream_t)stream);
}

int ms2g_pnp_ms2g_solve(ms2g_plan* p, const ms2g_solve_desc* sd, const float* b, const float* x0, float* x_out,
                        ms2g_sched_entry* trace, void* stream) {
  NvtxRange nvtx_range__("ms2g_pnp_ms2g_solve");
  if (!p || !sd) return set_error(MS2G_ERR_INPUT, "NULL plan/desc");
  cudaStream_t st = (cudaStream_t)stream;
  MS2G_TRY(solve_launch(p, sd, b, x0, x_out, st));
  const int rc = solve_status(p, st);
  if (trace) {
    double etas[64];
    MS2G_CUDA(cudaMemcpy(etas, p->w_scal + 64, sizeof(double) * 64, cudaMemcpyDeviceToHost));
    for (size_t k = 0; k < p->last_sched.size(); ++k) {
      trace[k] = p->last_sched[k];
      trace[k].eta = etas[trace[k].stage];
    }
  }
  return rc;
}

}  // extern "C"
