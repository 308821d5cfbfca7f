/*
 * ms2g.h -- C ABI of libms2g.so, the B200 (sm_100a) hot path of PnP-MS2G
 * (Tang, "Multi-Stage Sketched Gradient ... Plug-and-Play", arXiv 2203.07308).
 *
 * Citation keys: P:NN = PAPER.md line NN (the paper), S:NN = SPEC.md line NN,
 * Z1..Z23 / O1..O13 = the readings listed in DESIGN.md.
 *
 * Conventions for every call
 *  - Return value: MS2G_OK (0) or an error code; ms2g_last_error() returns a
 *    thread-local message for the last failing call on this thread.
 *  - Image / sinogram pointers are caller-owned DEVICE pointers to contiguous
 *    fp32 arrays.  The library never frees or retains them past the call.
 *      image     [batch][n_c][n_c], row i along +y, column j along +x, n_c = n/factor
 *      sinogram  [batch][V_r][B]   (this rank's views [view_begin, view_end))
 *      compacted [batch][n_sel][B] (views selected by a subset, ascending order)
 *  - `stream` is a cudaStream_t passed as void*.  Every call is asynchronous
 *    and ordered on that stream, except where "synchronous" is stated.
 *  - A plan is used by one host thread at a time.  Device memory is
 *    allocated by ms2g_plan_geometry / ms2g_attach_nccl / ms2g_attach_peers
 *    and, on a solve description's first use, before its graph is captured
 *    (Option-5 table, power-iteration branch workspaces, subset block
 *    orders); the per-operator calls never allocate, so sequences of them
 *    are CUDA-graph capturable.
 *  - Configuration errors are detected on the host before any launch.
 */
#ifndef MS2G_H
#define MS2G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MS2G_OK = 0,
  MS2G_ERR_CONFIG = 2,    /* invalid description / shapes (SPEC exit code 2) */
  MS2G_ERR_DIVERGED = 3,  /* non-finite iterate (SPEC exit code 3)      */
  MS2G_ERR_CUDA = 5,      /* CUDA runtime failure                                      */
  MS2G_ERR_NCCL = 6,      /* NCCL failure                                              */
  MS2G_ERR_INPUT = 7      /* invalid pointer / subset / argument value                 */
};

typedef struct ms2g_plan ms2g_plan;  /* opaque: owns device geometry tables + workspaces */

/* Fan-beam geometry (views equally spaced over an arc;
 * flat detector S:92; reading Z12).  Pixel (i,j) of the n x n grid covers
 * [-fov/2 + j h, -fov/2 + (j+1) h] x [-fov/2 + i h, ...], h = fov/n.
 * View v: theta = arc_rad * v / n_views, source sod*(cos, sin), detector
 * centre -(sdd-sod)*(cos, sin), axis (-sin, cos); bin t at offset
 * (t - (n_bins-1)/2) * bin_pitch.  One ray per bin. */
typedef struct {
  int32_t n;                       /* image side N; every factor must divide it          */
  double fov;                      /* physical side W (> 0)                               */
  int32_t n_views;                 /* V, global view count                                */
  double arc_rad;                  /* angular range (2 pi full scan, pi limited angle)    */
  int32_t n_bins;                  /* B                                                   */
  double sod, sdd;                 /* source-centre / source-detector distances;          */
                                   /* need sod > fov/sqrt2 and sdd - sod > fov/sqrt2      */
  double bin_pitch;                /* <= 0 selects (sdd/sod) * fov / n                     */
  int32_t view_begin, view_end;    /* this rank's contiguous shard; (0,0) = all views     */
  int32_t batch;                   /* images per call (>= 1)                              */
} ms2g_geom_desc;

/* Build the per-factor ray tables (host fp64, cast once) and every workspace.
 * factors: the sketch factors s (each divides n) the plan will be used with.
 * Synchronous.  Errors: MS2G_ERR_CONFIG (bad desc / factor, or a ray lying
 * exactly on a grid line of a planned grid -- reading Z14: such a ray meets
 * two closed pixel rows and its row is undefined; it needs an odd bin count
 * with views at multiples of 90 deg -- checked on the host before any device
 * work), MS2G_ERR_CUDA. */
int ms2g_plan_geometry(const ms2g_geom_desc* desc, const int32_t* factors, int32_t n_factors,
                       ms2g_plan** out);
void ms2g_plan_destroy(ms2g_plan* plan);

/* Multi-GPU view sharding: rank 0 creates a 128-byte
 * ncclUniqueId, the caller broadcasts it, then every rank attaches.  After
 * attaching, back_project(..., allreduce=1) sums partial images over ranks
 * in place (ncclAllReduce, fp32, sum).  Synchronous.  MS2G_ERR_NCCL. */
int ms2g_nccl_unique_id(void* out_128_bytes);
int ms2g_attach_nccl(ms2g_plan* plan, const void* unique_id_128_bytes, int32_t rank, int32_t nranks);

/* NEXT-3: the same cross-rank sum over NVLink peer memory,
 * fused into the backprojection (no separate collective).  The plan owns an
 * IPC-shareable exchange buffer (2 x n_cmax^2 x batch fp32: this rank's
 * partial, and its chunk of the sum) and a signal pad; ms2g_peer_export
 * writes this rank's ms2g_peer_blob_size() bytes (CUDA IPC handles + region
 * size), the caller all-gathers the blobs in rank order (nranks x size
 * bytes, host memory) and every rank calls ms2g_attach_peers (one process per
 * GPU of one node, nranks <= 64).  From then on every allreduce of the plan
 * (back_project(..., allreduce=1), sketched_grad, power_iteration, the solve)
 * is a reduce-scatter + all-gather over peer loads in three launches with
 * the barrier folded in: publish (fused into the backprojector's chunk
 * reduction; its last block signals the peers), reduce-scatter (each rank
 * sums its 1/P chunk over the ranks in FIXED rank order, then signals),
 * all-gather (fused with the step z = y - eta U_s G in the solve) -- all
 * ranks get bitwise identical images.  Peers take precedence over an
 * attached NCCL communicator.  Synchronous; MS2G_ERR_CUDA (IPC),
 * MS2G_ERR_CONFIG (blob mismatch: plans of different shapes).  A wait that
 * lasts 20 s of wall time (a rank never arrived) gives up: the next
 * ms2g_solve_status / synchronous solve returns MS2G_ERR_NCCL and the plan
 * refuses exchanges until every rank calls ms2g_attach_peers again. */
/* NEXT-3, NVLS form: the same sum reduced IN the NVSwitch (multimem.ld_reduce
 * on a multicast object, broadcast with multimem.st), precedence over peers
 * and NCCL once attached.  Rank 0 calls ms2g_mc_create (creates the object
 * for nranks devices, writes ms2g_mc_blob_size() bytes: its pid and a POSIX
 * file descriptor of the object); the caller broadcasts rank 0's blob; every
 * rank calls ms2g_attach_multicast(phase 0) (import via pidfd_getfd, add its
 * device), then -- after a process-group barrier -- phase 1 (allocate, bind,
 * map).  MS2G_ERR_CUDA names the failing driver call: where NVLS multicast
 * is unavailable (one GPU; no NVSwitch multicast) ms2g_mc_create fails
 * cleanly and the plan keeps its other paths.  Unexercised beyond that
 * failure on the single-GPU development pool. */
int ms2g_mc_blob_size(void);
int ms2g_mc_create(ms2g_plan* plan, int32_t nranks, void* blob_out);
int ms2g_attach_multicast(ms2g_plan* plan, const void* blob_rank0, int32_t rank, int32_t nranks, int32_t phase);

int ms2g_peer_blob_size(void);
int ms2g_peer_export(ms2g_plan* plan, void* blob_out);
int ms2g_attach_peers(ms2g_plan* plan, const void* blobs_all_ranks, int32_t rank, int32_t nranks);

/* Forward projection with fused residual (Eq. 6-7 "A_s S(x) - b"):
 *   out[b][k][t] = (A_s x_b)[v_k][t] - bsino[b][v_k][t]
 * A_s = Siddon exact intersection lengths on the n_c = n/factor grid.
 * x     image [batch][n_c][n_c] (the library first packs it into its gather
 *       layout, a plan workspace).
 * bsino [batch][V_r][B] indexed by rank-local view, or NULL (plain A_s x).
 * subset: ascending GLOBAL view indices (NULL = all views); views outside
 *       this rank's shard are skipped; out is compacted over the rest.
 * Errors: CONFIG (factor not in plan), INPUT (NULL x/out, bad subset). */
int ms2g_forward_project(ms2g_plan* plan, int32_t factor, const float* x, const float* bsino, float* out,
                         const int32_t* subset, int32_t n_subset, void* stream);

/* Exact adjoint ("A_s^T"):  img[b] = scale * A_s^T sino[b]
 * (accumulate != 0: img += ...).  sino is compacted [batch][n_sel][B] in the
 * same view order forward_project used.  allreduce != 0 sums the partial
 * images over the ranks in place (requires attach_nccl or attach_peers; with
 * one rank and neither attached it is a no-op).  Accumulation is fixed point
 * (DESIGN.md 7a): each contribution is rounded to 2^-22 of the largest one
 * the tile's views can give, so the result is deterministic and
 * order-independent, ~1e-6 relative; a non-finite sinogram value makes the
 * affected tiles NaN. */
int ms2g_back_project(ms2g_plan* plan, int32_t factor, const float* sino, float* img, float scale,
                      int32_t accumulate, const int32_t* subset, int32_t n_subset, int32_t allreduce,
                      void* stream);

/* Resampler kinds for S and U:
 *   0  s x s average pool / nearest replication (BASELINE configs; reading Z2)
 *   1  bicubic, the paper's own choice "MATLAB imresize ... bicubic" (P:156,
 *      P:92): Keys a = -0.5, centre-aligned, antialiased downscale, clamped
 *      boundary (NEXT-1; needs the factor in the plan). */
enum { MS2G_RESAMPLE_MEAN = 0, MS2G_RESAMPLE_BICUBIC = 1 };

/* Image-space sketch S (north-star D): x [batch][n][n] -> v [batch][n/s][n/s]. */
int ms2g_sketch_down(ms2g_plan* plan, int32_t factor, int32_t kind, const float* x, float* v, void* stream);

/* Upsample + step ("z = y - eta U G"):  z = y - eta * U g.  y == NULL
 * gives z = U g.  kind 0: U = nearest replication = s^2 S^T (reading Z2). */
int ms2g_sketch_up(ms2g_plan* plan, int32_t factor, int32_t kind, const float* g, const float* y, float eta,
                   float* z, void* stream);

/* Sketched data-fidelity gradient (Eq. 6, Eq. 7):
 *   g = (V/|M|) U A_s^T (A_s S x - b_M)      (full resolution n x n)
 * factor 1 gives A^T(Ax - b).  subset NULL = all views (|M| = V).
 * kind selects S/U (see MS2G_RESAMPLE_*).  With NCCL or peers attached the
 * partial A_s^T is summed over the ranks before U. */
int ms2g_sketched_grad(ms2g_plan* plan, int32_t factor, int32_t kind, const float* x, const float* bsino, float* g,
                       const int32_t* subset, int32_t n_subset, void* stream);

/* Registered view subsets (P:72, P:95-97 minibatches M_i reused every
 * epoch).  ms2g_register_subset validates the ascending GLOBAL view list
 * (MS2G_ERR_INPUT as above), uploads this rank's part once, builds the
 * longest-first block orders of its projector launches for every planned
 * factor and returns an id (synchronous; allocates).  The *_registered calls
 * are the calls above with the list given by id: no host->device copy, no
 * host synchronisation, so a loop of them is launch-bound only (and graph
 * capturable).  ms2g_release_subset frees it (synchronises the device).
 * MS2G_ERR_INPUT on an unknown or released id.  Ad-hoc `subset` arguments of
 * the calls above use a ring of 8 staged lists per plan, each reused only
 * after the kernels of its previous call (on whatever stream) completed. */
int ms2g_register_subset(ms2g_plan* plan, const int32_t* subset, int32_t n_subset, int32_t* id);
int ms2g_release_subset(ms2g_plan* plan, int32_t id);
int ms2g_forward_project_registered(ms2g_plan* plan, int32_t factor, const float* x, const float* bsino,
                                    float* out, int32_t subset_id, void* stream);
int ms2g_back_project_registered(ms2g_plan* plan, int32_t factor, const float* sino, float* img, float scale,
                                 int32_t accumulate, int32_t subset_id, int32_t allreduce, void* stream);
int ms2g_sketched_grad_registered(ms2g_plan* plan, int32_t factor, int32_t kind, const float* x,
                                  const float* bsino, float* g, int32_t subset_id, void* stream);

/* Lipschitz constant of the factor-s fidelity ("eta = O(1/L)"; reading
 * Z5/Z6): v0 = 1/||1||, w = A_s^T A_s v, L = <v,w>, v = w/||w||, `iters`
 * times over all views (allreduced when NCCL is attached).  fp64 dots.
 * Synchronous: *L is written on return. */
int ms2g_power_iteration(ms2g_plan* plan, int32_t factor, int32_t iters, double* L, void* stream);

/* Denoiser D: kind 0 identity, 1 Gaussian 3x3 (sigma, replicate
 * boundary), 2 TV-prox by Chambolle's dual iteration (lambda, tau <= 1/8,
 * inner_iters).  z, out: [batch][n][n], must not alias. */
typedef struct {
  int32_t kind;
  float sigma;
  float lambda;
  float tau;
  int32_t inner_iters;
} ms2g_denoiser;
int ms2g_denoise(ms2g_plan* plan, const ms2g_denoiser* den, const float* z, float* out, void* stream);

/* Algorithm 1.  Option 1: n_iters steps per stage on all views.
 * Option 2: n_epochs per stage, each epoch visits the n_subsets interleaved
 * view subsets {v : v mod n_subsets == k} in a Fisher-Yates order drawn from
 * one SplitMix64 stream seeded with `seed` (reading Z8/Z9; O13).
 * Option 3 (NEXT-4, "variance-reduced estimator ... SVRG"): the Option 2
 * schedule with the SVRG estimator: at each epoch start xs = y and
 * mu = A_s^T (A_s S xs - b) on all views; a step uses
 * G = (V/|M|) A_M^T A_M S (y - xs) + mu.
 * Option 4 (NEXT-4, "randomly sampled minibatch", "uniformly
 * sampled"): n_iters steps per stage, each on m = n_subsets views drawn
 * uniformly without replacement (partial Fisher-Yates on the SplitMix64
 * stream), scaled by V/m; ms2g_schedule_views returns a step's views.
 * Option 5 (NEXT-4, "SAGA"): the Option 2 schedule with a table of
 * the K scaled subset gradients (filled at every stage start); a step on
 * subset j uses G = new - phi_j + mean(phi) and stores phi_j = new. */
typedef struct {
  int32_t factor, n_iters, n_epochs;
} ms2g_stage;
typedef struct {
  const ms2g_stage* stages;
  int32_t n_stages;
  int32_t option;        /* 1 | 2 | 3 SVRG | 4 uniform minibatches | 5 SAGA */
  int32_t n_subsets;     /* Options 2/3: subsets; Option 4: views per step */
  uint64_t seed;
  ms2g_denoiser den;
  float alpha;           /* RED-PRO mix weight, 0 < alpha <= 1      */
  int32_t power_iters;   /* per-stage power iterations (20 in the configs); 0 = reuse, for
                            each stage factor, the step L, eta = 1/L of the last power
                            iteration run on this plan for that factor (by an earlier solve
                            or ms2g_power_iteration): L depends on the geometry only
                            (SURVEY 8(e)).  MS2G_ERR_CONFIG if none has run. */
  int32_t check_every;   /* unused by the graph path: every step is checked on device */
  int32_t resampler;     /* MS2G_RESAMPLE_MEAN (configs) | MS2G_RESAMPLE_BICUBIC (paper) */
} ms2g_solve_desc;
/* One global iteration: i (1-based, continuous over stages), stage,
 * factor, subset (-1 = all views), eta = 1/L_stage, a_i = (i-1)/(i+3). */
typedef struct {
  int32_t i, stage, factor, subset;
  double eta, a;
} ms2g_sched_entry;

/* Host-only, bit-exact schedule (eta left 0).  *n_out = total steps; at most
 * `cap` entries are written.  MS2G_ERR_CONFIG on a bad description.  plan
 * may be NULL (then factor divisibility and n_subsets <= n_views are not
 * checked); no device is touched. */
int ms2g_schedule(const ms2g_plan* plan, const ms2g_solve_desc* desc, ms2g_sched_entry* out, int32_t cap,
                  int32_t* n_out);

/* Host-only: the ascending GLOBAL view indices used by schedule step `step`
 * (0-based): all views (Option 1), interleaved subset (Options 2/3) or the
 * drawn minibatch (Option 4).  *n_out = their count; <= cap are written. */
int ms2g_schedule_views(const ms2g_plan* plan, const ms2g_solve_desc* desc, int32_t step, int32_t* out,
                        int32_t cap, int32_t* n_out);

/* Whole PnP-MS2G solve, captured once as a CUDA graph per (plan, desc,
 * pointers) and replayed: per stage the power iteration, then per step
 *   v = S_s y; r = A_s v - b_M; G = c A_s^T r (+allreduce); z = y - eta U_s G;
 *   x = (1-alpha) z + alpha D(z); y = x + a_i (x - x_prev).
 * x0 = y0, b [batch][V_r][B], x_out [batch][n][n] (may alias x0).
 * trace (optional, host) receives the schedule with eta filled in.
 * Synchronous on return (the flags are read back): a NaN / Inf in b or x0
 * (checked on the device at the solve's start) returns MS2G_ERR_INPUT; a
 * non-finite iterate returns MS2G_ERR_DIVERGED naming the stage and
 * iteration. */
int ms2g_pnp_ms2g_solve(ms2g_plan* plan, const ms2g_solve_desc* desc, const float* b, const float* x0,
                        float* x_out, ms2g_sched_entry* trace, void* stream);

/* Same solve, asynchronous: the graph is launched and the call returns; the
 * divergence flag is left on the device (read it with ms2g_solve_status). */
int ms2g_pnp_ms2g_solve_async(ms2g_plan* plan, const ms2g_solve_desc* desc, const float* b,
                              const float* x0, float* x_out, void* stream);
/* Synchronous: MS2G_OK, MS2G_ERR_INPUT (non-finite b / x0) or
 * MS2G_ERR_DIVERGED for the last solve. */
int ms2g_solve_status(ms2g_plan* plan, void* stream);

/* Per-kernel timing inside the solve graph (measurement support).
 * ms2g_set_kernel_timing(plan, 1): the next captured solve graph records an
 * external CUDA event before and after every projector launch (k_forward,
 * k_backward); 0 removes them (the cached graph is re-captured either way).
 * An instrumented solve runs its power iterations serially (no concurrent
 * branches), so each timed interval holds one kernel alone on the GPU.
 * ms2g_kernel_time: for the LAST replayed solve, the summed device time (ms)
 * and count of the launches of one kind (0 forward, 1 backward) at one
 * factor.  Synchronizes on those events.  MS2G_ERR_INPUT on NULL. */
int ms2g_set_kernel_timing(ms2g_plan* plan, int32_t enable);
int ms2g_kernel_time(ms2g_plan* plan, int32_t kind, int32_t factor, double* total_ms, int32_t* launches);

/* Thread-local message of the last failing call ("" if none). */
const char* ms2g_last_error(void);

/* Number of device kernels libms2g has launched in this process (graph
 * replays count their kernel nodes).  For the bench's gpu_launches claim. */
uint64_t ms2g_launch_count(void);

/* Plan facts for the binding: coarse side for a factor (0 if not planned),
 * rank-local view range and batch. */
int ms2g_plan_info(const ms2g_plan* plan, int32_t factor, int32_t* n_c, int32_t* view_begin,
                   int32_t* view_end, int32_t* batch);

#ifdef __cplusplus
}
#endif
#endif /* MS2G_H */
