// internal.cuh -- shared declarations of libms2g (CUDA product path).
// Independent of oracle/: no code, header or table is shared with it.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <atomic>
#include <map>
#include <string>
#include <vector>

#include "../../include/ms2g.h"

namespace ms2g {

// Device bounds checks for the debug build (-DMS2G_DEBUG=1, `build.py --debug`):
// a violated index traps the kernel (the launch then fails with an error)
// instead of reading or writing out of bounds.  compute-sanitizer is closed on
// this GPU pool, so the GPU test suite is also run against this build.
#if defined(MS2G_DEBUG) && MS2G_DEBUG
#define MS2G_DASSERT(cond) \
  do {                     \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define MS2G_DASSERT(cond) \
  do {                     \
  } while (0)
#endif

// Zero entries on each side of every pair-image line beyond the two the
// layout needs: a forward warp whose rays leave the grid by at most this many
// rows inside its column range reads them without a clamp (projector.cu).
constexpr int kPairPad = 64;
__host__ __device__ inline size_t pair_line(int nc) { return (size_t)nc + 3 + 2 * kPairPad; }

// Fixed-point minor coordinate: 32 fractional bits (1 unit = 2^-32 pixel).
constexpr double kFix = 4294967296.0;

enum RayFlags : int { kMajorY = 1, kMirror = 2 };

// One ray of one view on the grid of one factor (32 bytes).  The ray is a
// line "minor = F0 + S * major" in pixel units of the n_c grid, in a frame
// where the minor axis may be mirrored (minor' = n_c - minor) so that the
// slope S is in [0, 1).  major = x (column) for |dx| >= |dy|, else y (row).
// The ray "class" is flags & 3 (major axis, mirror).
struct __align__(16) RayEntry {
  long long F0;             // minor' at major coordinate 0, 2^-32 units
  unsigned S;               // minor' step per unit major step, 2^-32 units (< 2^32)
  float Lc;                 // physical length per unit major step: h_c sqrt(1 + slope^2)
  float Ly32;               // Lc / slope' * 2^-32 (0 when S == 0)
  int flags;                // kMajorY | kMirror
  short c_lo, c_hi;         // major indices [c_lo, c_hi) where the ray meets the grid
  int pad;
};
static_assert(sizeof(RayEntry) == 32, "RayEntry must be 32 bytes");

// The adjoint's half of a ray (16 bytes, same values as RayEntry): its
// record loads are part of the L1 data pipe the adjoint is bound by.
struct __align__(16) RayBp {
  long long F0;
  unsigned S;
  float Ly32;
};
static_assert(sizeof(RayBp) == 16, "RayBp must be 16 bytes");

// Per-view constants.  Detector coordinate of a point P (pixel units of the
// n_c grid): tau(P) = off + scale * ((P-S).e) / ((P-S).n).  The bins of a view
// split into <= 4 contiguous runs of one ray class (the ray angle is monotone
// in t): run k covers t in [seg_t[k], seg_t[k+1]) with class seg_cls[k].
struct __align__(16) ViewEntry {
  float Sx, Sy, ex, ey, nx, ny, scale, off;
  short seg_t[5];
  char seg_cls[4];
  short nseg;
};
static_assert(sizeof(ViewEntry) == 48, "ViewEntry must be 48 bytes");

struct FactorTables {
  int factor = 0, nc = 0;
  RayEntry* d_rays = nullptr;     // [V_r][B]
  RayBp* d_rays_bp = nullptr;     // [V_r][B], the adjoint's fields
  // adjoint fixed-point scale bounds: per (tile family, view) an upper bound
  // of the weight one pixel receives from the view's rays; the largest Lc
  float* d_bpw = nullptr;         // [2][V_r]
  float lc_max = 0.f;
  ViewEntry* d_views = nullptr;   // [V_r]
  int bp_chunks[2] = {1, 1};      // view chunks of the backprojector per tile family (X, Y)
  int bp_h = 64;                  // minor extent of the adjoint's tiles (bp_height)
  // step size cached per factor by the last power iteration on this plan:
  // d_Lcache = {L, eta} (double), then eta as float; L_iters = its iteration
  // count as enqueued (0 = none yet).  L depends on the geometry only.
  double* d_Lcache = nullptr;
  mutable int L_iters = 0;
  int4* d_bpr = nullptr;          // per (adjoint tile, view): bin runs meeting the tile
  int* d_bp_order = nullptr;      // full-view launches: block -> work item, longest first
  int* d_fwd_order = nullptr;     // same for the single-image forward (for fwd_order_vpb views per block)
  int fwd_order_vpb = 0;
  // host cost tables behind the orders (also used for subset orders):
  // rays meeting (tile, view) [2 tiles-per-family][V_r]; longest ray column
  // range of (view, 32-bin block) [V_r][ceil(B/32)]
  std::vector<uint16_t> h_bp_cost, h_fwd_cost;
  // per interleaved subset of the current Option-2/3/5 partition: block orders
  std::vector<int*> d_bp_order_sub, d_fwd_order_sub;
  // bicubic resampling tables (NEXT-1), [n_out][taps] clamped input index / weight
  int taps_down = 0, taps_up = 0;
  int* d_idx_down = nullptr;
  float* d_w_down = nullptr;
  int* d_idx_up = nullptr;
  float* d_w_up = nullptr;
};

// workspace of the persistent TV-prox kernel (plan-owned, zero-initialised)
struct TvWs {
  unsigned long long* flags = nullptr;   // [max_ctas]
  unsigned* gen_ticket = nullptr;        // {generation, ticket}
  int* err = nullptr;
  int max_ctas = 0, smem_optin = 0;      // (the round halos go through the plan's dual buffers w_p)
};

struct SolveGraph {
  std::string key;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t kernel_nodes = 0;
};

}  // namespace ms2g

struct ms2g_plan {
  ms2g_geom_desc d{};
  int V_r = 0;                         // views in this rank's shard
  int B = 0;
  double pitch = 0;
  std::vector<ms2g::FactorTables> ft;
  int nmax_c = 0;                      // largest coarse side among the factors
  int sm_count = 148;                  // SMs of the plan's device
  int class_mask = 15;                 // ray classes (flags & 3) present in the rank's views, bit per class
  // workspaces (all sized for batch)
  float2* w_pair = nullptr;            // forward gather images: 4 x [batch][n_c][n_c + 3 + 2 kPairPad] float2
  size_t pair_stride = 0;              // float2 elements per pair image
  float* w_v = nullptr;                // coarse sketch
  float* w_rs = nullptr;               // separable-resampling intermediate [batch][n][n]
  float* w_G = nullptr;                // coarse gradient / backprojection
  float* w_res = nullptr;              // residual / projection [batch][V_r][B]
  float* w_part = nullptr;             // backprojection partial planes [batch][X chunks, Y chunks][n_c^2]
  size_t part_elems = 0;
  float* w_x[2] = {nullptr, nullptr};  // iterate double buffer (full res)
  float* w_y = nullptr;                // extrapolated point
  float* w_z = nullptr;                // pre-denoiser point
  float* w_snap = nullptr;             // SVRG snapshot (full res)
  float* w_mu = nullptr;               // SVRG snapshot gradient (coarse)
  float* w_p[2] = {nullptr, nullptr};  // TV dual double buffer [batch][2][n][n]
  ms2g::TvWs tvws;                     // persistent TV-prox kernel workspace
  double* w_red = nullptr;             // reduction partials
  int red_blocks = 0;
  double* w_scal = nullptr;            // device scalars: [0..63] L per stage, [64..127] eta
  float* w_etaf = nullptr;             // fp32 eta per stage [64]
  double* w_pw = nullptr;              // power-iteration scalars (dot, inv_norm)
  unsigned* w_ticket = nullptr;        // last-block ticket of k_reduce_power (0 between launches)
  unsigned* w_rmaxv = nullptr;         // [batch][V_r] max |r| per view (float bits) of the last forward(s)
  int* w_flag = nullptr;               // first non-finite global iteration (INT_MAX = none)
  // ad-hoc host subsets: a ring of kSelRing (pinned host, device) list slots;
  // slot k is reused only after the event recorded behind its last consumer
  // (on that consumer's stream) has completed, so calls on different streams
  // never overwrite a list a kernel still reads
  static constexpr int kSelRing = 8;
  int* w_sel = nullptr;                // device lists [kSelRing][V_r]
  int* h_sel = nullptr;                // pinned host staging [kSelRing][V_r]
  cudaEvent_t sel_ev[kSelRing] = {};
  int sel_next = 0;
  // registered subsets (ms2g_register_subset): device list + longest-first
  // block orders per factor, built once; id = index (nullptr d_sel: released)
  struct RegSubset {
    int* d_sel = nullptr;
    int n_sel = 0, n_global = 0;
    std::vector<int*> bp_order, fwd_order;   // per plan factor (index into ft)
  };
  std::vector<RegSubset> reg;
  int* w_subsets = nullptr;            // precomputed Option-2 subset lists
  int* w_mb = nullptr;                 // precomputed Option-4 minibatch lists
  float* w_saga = nullptr;             // Option-5 table: K coarse gradients + their mean
  size_t saga_elems = 0;
  std::vector<int> mb_off, mb_len;
  std::vector<int> subset_off, subset_len, subset_global_len;
  int subsets_n = 0;
  // NCCL
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // peer-memory allreduce (NEXT-3, peer_reduce.cu): exchange buffer of two
  // regions (PUB: this rank's partial, RED: its chunk of the sum), signal pad
  // (PUB / RED epochs by rank, local epoch, time-out, ticket), device tables
  // of every rank's buffer / pad
  float* xch_buf = nullptr;
  size_t xch_slot = 0;                 // floats per slot
  unsigned* xch_pad = nullptr;
  float** d_peer_bufs = nullptr;
  unsigned** d_peer_pads = nullptr;
  int* w_peer_err = nullptr;
  int peer_rank = 0, peer_n = 0;       // peer_n > 0: attached
  bool peer_failed = false;            // a barrier timed out: exchanges refused until re-attached
  // NVLS multicast exchange (multicast.cu): object + physical memory handles,
  // unicast and multicast views of the PUB | RED | flags buffer
  unsigned long long mc_handle = 0, mc_mem = 0;
  size_t mc_size = 0;
  void* mc_uc = nullptr;
  void* mc_mc = nullptr;
  int mc_rank = 0, mc_n = 0;           // mc_n > 0: attached
  std::vector<void*> peer_opened;      // IPC mappings to close
  // Power-iteration branches of the solve graph: one per stage factor, each
  // with its own workspaces (batch 1), so the geometry-only power chains of
  // all stages run concurrently with each other and with the earlier stages'
  // steps.  Single rank only (a communicator is not used from two branches).
  struct PowerBranch {
    int factor = 0;
    float* w_v = nullptr;
    float2* w_pair = nullptr;
    size_t pair_stride = 0;
    float* w_res = nullptr;
    float* w_G = nullptr;
    float* w_part = nullptr;
    double* w_red = nullptr;
    double* w_pw = nullptr;
    unsigned* w_ticket = nullptr;
    unsigned* w_rmaxv = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::vector<PowerBranch> pbr;
  cudaEvent_t ev_fork = nullptr;
  ms2g_plan* root = nullptr;           // set on shadow copies that borrow a branch's workspaces
  // per-kernel timing inside the captured solve graph (ms2g_set_kernel_timing):
  // external event-record nodes around every k_forward / k_backward launch
  struct TimedLaunch { cudaEvent_t a, b; int kind, factor; };
  bool timing = false;
  std::vector<TimedLaunch> tev;
  // graph cache
  ms2g::SolveGraph sg;
  // per-call graphs of the standalone gradient (all views or a registered
  // subset: no host-side staging), most recent first, at most kGradGraphs
  static constexpr int kGradGraphs = 16;
  std::vector<ms2g::SolveGraph> grad_graphs;
  uint64_t topo_version = 0;           // bumped when a communicator / peers attach (graphs re-captured)
  int last_total_steps = 0;
  std::vector<ms2g_sched_entry> last_sched;
  std::vector<int> last_stage_of_step;
};

namespace ms2g {

// ---- programmatic dependent launch (PDL) ----
// launch_k_pdl launches with programmatic stream serialisation: the kernel is
// scheduled while its predecessor drains, reads only what does not depend on
// the predecessor before griddepcontrol.wait (pdl_wait: the predecessor has
// completed and its writes are visible), then lets its own successor launch
// (pdl_release, after the wait, so visibility stays transitive).  Used for
// the TV chain (K + 1 short dependent launches per denoise).  The other hot
// kernels also wait / release (no-ops for an ordinary launch) but are
// launched ordinarily with launch_k: launched with PDL, their resident
// waiting CTAs took occupancy from the predecessor's last wave (C3 cached-
// step solve 5.48 -> 6.85 ms, C4 355 -> 350 iterations/s).  MS2G_PDL=0
// disables PDL everywhere.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release() { asm volatile("griddepcontrol.launch_dependents;" :::); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_cfg(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
  return launch_cfg(false, kern, grid, block, smem, st, args...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args... args) {
  return launch_cfg(true, kern, grid, block, smem, st, args...);
}

// ---- the fixed-order sum of the backprojection's partial planes ----
// Every consumer of the partial planes (k_chunk_reduce, the fused step and
// power epilogues, the NEXT-3 publishes) sums them with THIS rule, so all
// paths give bitwise equal images.  Two orders, chosen from (np, nplanes)
// alone by plane_groups() -- identically for every consumer of a launch:
//  * G = 1 (large images: the common case) -- thread t of a 256-thread block
//    adds all planes of pixel p0 + t in increasing plane order (a 256-pixel
//    tile per block iteration, loads of independent planes in flight);
//  * G = 8 (small coarse grids with many view-chunk planes, e.g. 128^2 with
//    360 planes): too few pixels to fill the GPU one thread per pixel, so
//    thread (x, g) of the (32 x 8) block adds planes g, g + 8, ... of pixel
//    p0 + x (a 32-pixel tile), then the 8 group sums are added in order
//    g = 0..7.
// sm.tot[t] receives the total of pixel p0 + t (t < plane_tile(G)); all
// threads of the block must call it; pixels >= np read nothing.
constexpr int kPlaneGroups = 8;
struct PlaneSmem {
  float g[kPlaneGroups][33];
  float tot[256];
};
__host__ __device__ inline int plane_tile(int G) { return G == 1 ? 256 : 32; }
inline int plane_groups(size_t np, int nplanes) { return (np <= 65536 && nplanes >= 16) ? kPlaneGroups : 1; }
__device__ __forceinline__ void sum_planes(const float* __restrict__ part, int nplanes, size_t np, size_t p0, int G,
                                           PlaneSmem& sm) {
  const int tid = threadIdx.y * 32 + threadIdx.x;
  if (G == 1) {
    const size_t p = p0 + tid;
    float s = 0.f;
    if (p < np)
      for (int c = 0; c < nplanes; ++c) s += part[(size_t)c * np + p];
    sm.tot[tid] = s;
    __syncthreads();
    return;
  }
  const size_t p = p0 + threadIdx.x;
  float s = 0.f;
  if (p < np)
    for (int c = threadIdx.y; c < nplanes; c += kPlaneGroups) s += part[(size_t)c * np + p];
  sm.g[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (tid < 32) {
    float t = 0.f;
#pragma unroll
    for (int g = 0; g < kPlaneGroups; ++g) t += sm.g[g][tid];
    sm.tot[tid] = t;
  }
  __syncthreads();
}
// blocks for the plane sums of np pixels: one tile each, at most `cap`
inline int plane_blocks(size_t np, int G, int cap) {
  const size_t t = (np + plane_tile(G) - 1) / plane_tile(G);
  return (int)(t < (size_t)cap ? (t ? t : 1) : cap);
}

// error handling (thread-local message)
int set_error(int code, const std::string& msg);
#define MS2G_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e__ = (call);                                                             \
    if (e__ != cudaSuccess)                                                               \
      return ::ms2g::set_error(MS2G_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
  } while (0)
#define MS2G_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r__ = (call);                                                            \
    if (r__ != ncclSuccess)                                                               \
      return ::ms2g::set_error(MS2G_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r__)); \
  } while (0)
#define MS2G_TRY(call)         \
  do {                         \
    int rc__ = (call);         \
    if (rc__ != MS2G_OK) return rc__; \
  } while (0)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// launches issued while a solve graph is being captured (not yet executed)
extern thread_local bool t_capturing;
extern thread_local uint64_t t_captured;
inline void note_launch() {
  if (t_capturing) ++t_captured;
  else count_launch();
}
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(MS2G_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  note_launch();
  return MS2G_OK;
}

const FactorTables* find_factor(const ms2g_plan* p, int factor);
// timing of one projector launch inside a solve capture (no-op otherwise);
// kind 0 forward, 1 backward; returns the slot for timing_end (-1: none)
int timing_begin(ms2g_plan* p, int kind, int factor, cudaStream_t st);
void timing_end(ms2g_plan* p, int slot, cudaStream_t st);

// ---- kernel launchers (projector.cu) ----
// pair images of v for the forward; v = x (factor 1), the factor x factor mean
// of the full-resolution x (fused S_s), times *scale_dev if given; v_out
// (optional) receives v
int launch_pair_prep(ms2g_plan* p, int nc, int batch, const float* x, cudaStream_t s, int factor = 1,
                     const double* scale_dev = nullptr, float* v_out = nullptr);
// order_sel: longest-first block order for a subset launch (d_sel != NULL),
// built for this view list (subset_orders in ms2g_api.cu); NULL = grid order
int launch_forward(ms2g_plan* p, const FactorTables& f, const float* b, float* out, const int* d_sel, int n_sel,
                   int batch, cudaStream_t s, const int* order_sel = nullptr);
int bp_tile_count(int nc, int H);   // adjoint tiles (both families) of an n_c grid, minor extent H
int bp_height(int nc, int V_r);      // that minor extent for a plan's factor
int fwd_views_per_block(const ms2g_plan* p, int n_sel, int batch);
int launch_bp_ranges(const FactorTables& f, int V_r, int B, int4* out, int* err, cudaStream_t s);
// publish: 0 = img = scale A_s^T sino (+ img), 1 = write scale * A_s^T sino
// into the peer exchange slot (not img), 2 = leave the partial planes in
// p->w_part for a fused epilogue; *nplanes_out = their count
int launch_backward(ms2g_plan* p, const FactorTables& f, const float* sino, float* img, float scale,
                    int accumulate, const int* d_sel, int n_sel, int batch, cudaStream_t s, int publish = 0,
                    const int* order_sel = nullptr, int* nplanes_out = nullptr);
// fused epilogues of the backprojection (projector.cu)
int launch_reduce_up_step(const float* part, int nplanes, int nc, int batch, float c, const float* y,
                          const float* eta_dev, float* z, int s, cudaStream_t st);
// per-view max |sino| (float bits) into p->w_rmaxv, for a backprojection of a
// sinogram that did not come from launch_forward (the fixed-point scale)
int launch_view_absmax(ms2g_plan* p, const float* sino, int n_sel, int batch, cudaStream_t s);
int launch_reduce_power(ms2g_plan* p, const float* part, int nplanes, size_t np, float* w_out, const float* v,
                        double* red, int red_blocks, unsigned* ticket, double* pw, double* L_out, double* eta_out,
                        float* etaf_out, cudaStream_t st, int tile_planes = 0);
void bp_launch_chunks(const ms2g_plan* p, const FactorTables& f, int n_sel, int* ch);

// ---- peer-memory allreduce (peer_reduce.cu, NEXT-3) ----
int launch_peer_allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st);
int launch_peer_finish(ms2g_plan* p, float* out, size_t count, cudaStream_t st);
// reduce-scatter + all-gather fused with z = y - eta U_s G (y == NULL: z = U_s G)
int launch_peer_finish_step(ms2g_plan* p, size_t count, int nc, int s, const float* y, const float* eta_dev,
                            float* z, cudaStream_t st);
int launch_chunk_reduce_publish(ms2g_plan* p, const float* part, int nplanes, size_t np, size_t total, float scale,
                                cudaStream_t st);

// ---- NVLS multicast allreduce (multicast.cu, NEXT-3) ----
int mc_blob_size();
int mc_create(ms2g_plan* p, int nranks, void* blob_out);
int mc_attach(ms2g_plan* p, const void* blob0, int rank, int nranks, int phase);
void mc_release(ms2g_plan* p);
int launch_mc_publish(ms2g_plan* p, const float* part, int nplanes, size_t np, size_t total, float scale,
                      cudaStream_t st);
// reduce in the switch + all-gather into out (s == 0) or the step z = y - eta U_s G (out = z, s >= 1)
int launch_mc_finish(ms2g_plan* p, size_t count, float* out, int nc, int s, const float* y, const float* eta_dev,
                     cudaStream_t st);
int launch_mc_allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st);

// ---- image kernels (image_ops.cu) ----
int launch_sketch_down(int n, int s, int batch, const float* x, float* v, cudaStream_t st);
int launch_up_step(int n, int s, int batch, const float* g, const float* y, const float* eta_dev,
                   float eta, float* z, cudaStream_t st);
// kind 0: average pool / replication; kind 1: bicubic (tables in f)
int launch_resample_down(ms2g_plan* p, const FactorTables& f, int kind, int batch, const float* x, float* v,
                         cudaStream_t st);
int launch_resample_up_step(ms2g_plan* p, const FactorTables& f, int kind, int batch, const float* g,
                            const float* y, const float* eta_dev, float eta, float* z, cudaStream_t st);
int build_bicubic_tables(FactorTables& f, int n);
int launch_gauss_mix_mom(int n, int batch, float sigma, const float* z, const float* xprev, float* xout,
                         float* yout, float alpha, float a, int mode, int* flag, int iter, cudaStream_t st);
// ws != NULL: the persistent single-launch form when it fits, else K + 1 launches
int launch_tv(int n, int batch, float lambda, float tau, int iters, const float* f, float* p0, float* p1,
              const float* xprev, float* xout, float* yout, float alpha, float a, int mode, int* flag,
              int iter, cudaStream_t st, const TvWs* ws = nullptr);
int launch_copy_mix_mom(int n, int batch, const float* z, const float* xprev, float* xout, float* yout,
                        float a, int mode, int* flag, int iter, cudaStream_t st);
int launch_fill(float* x, size_t count, float value, cudaStream_t st);
int launch_axpby(float* out, const float* x, const float* y, float a, float b, size_t count, cudaStream_t st);
int launch_saga(float* nw, float* phi, float* avg, int K, size_t count, cudaStream_t st);
int launch_init_flag(int* flag, cudaStream_t st);
int launch_cached_step(const double* cache, double* L_out, double* eta_out, float* etaf_out, cudaStream_t st);

}  // namespace ms2g
