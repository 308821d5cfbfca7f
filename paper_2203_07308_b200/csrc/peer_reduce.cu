// peer_reduce.cu -- NEXT-3: the backprojection's cross-rank sum
// over NVLink peer memory instead of a separate NCCL collective.
//
// Every rank's plan owns an IPC-shareable exchange buffer of two regions --
// PUB (this rank's partial image) and RED (the chunk of the sum this rank
// owns) -- and a signal pad.  After ms2g_attach_peers each rank holds device
// pointers to every peer's buffer and pad.  One allreduce of the view-sharded
// partial images G_r is a reduce-scatter + all-gather in three
// launches, with the barrier folded into them:
//   1. publish: the backprojector's chunk reduction writes scale * G_r into
//      PUB (fused epilogue; a generic allreduce copies the buffer instead);
//      the LAST block of the launch (atomic ticket) bumps the epoch e and
//      stores it into word PUB+rank of every peer's pad (release, system
//      scope, after __threadfence_system);
//   2. reduce-scatter: every block first waits until all P words PUB+q of
//      the local pad reach e (acquire), then rank r sums its contiguous 1/P
//      chunk of the image over the P PUB regions in FIXED rank order 0..P-1
//      (peer loads over NVLink) into its RED region; the last block signals
//      RED+rank = e to every peer;
//   3. all-gather: every block waits for all RED words, then copies each
//      element from the RED region of the rank that owns it -- or, fused,
//      takes the step z = y - eta U_s G there with no G round trip.
// Every rank ends with the bitwise same G (each chunk is summed once, by its
// owner, in rank order).  NVLink traffic per rank: 2 (P-1)/P of the image
// instead of (P-1) images for the one-shot sum.  One region of each kind
// suffices: a rank rewrites PUB (next allreduce) only after its all-gather,
// which waited for every peer's RED signal, which each peer raised after its
// reduce-scatter had read every PUB region; and it rewrites RED only after
// the next reduce-scatter's wait, i.e. after every peer published again,
// which each did after its all-gather had read every RED region.
// Waits are bounded by 20 s of wall time (%globaltimer): on a time-out the
// kernel raises the plan's error flag (every later wait of the plan then
// returns at once and the sum kernels leave their outputs untouched), the
// host sees MS2G_ERR_NCCL and the plan refuses further exchanges until every
// rank calls ms2g_attach_peers again (epochs restart from 0).
#include "internal.cuh"

namespace ms2g {

// pad layout (unsigned words): [0, 64) PUB epochs by rank, [64, 128) RED
// epochs by rank, then the local epoch, the time-out mark and the last-block
// ticket of the running exchange kernel
constexpr int kPub = 0, kRed = 64, kEpoch = 128, kTimeout = 129, kTicket = 130;

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct PeerArgs {
  float* const* bufs;          // every rank's exchange buffer (PUB region first, RED at + slot)
  unsigned* const* pads;       // every rank's signal pad
  int rank, nranks;
  size_t slot;                 // floats per region
  int* err;                    // plan error flag (time-out)
};

// Wait until the words [base, base + P) of the local pad reach epoch e.
// Bounded by WALL time, not a spin count; returns false on a time-out (after
// raising the error flag) or at once when the flag is already up.
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;   // 20 s
__device__ bool wait_words(const PeerArgs& a, int base, unsigned e) {
  if (*(volatile int*)a.err) return false;
  unsigned* mine = a.pads[a.rank];
  const unsigned long long t0 = globaltimer_ns();
  for (int q = 0; q < a.nranks; ++q) {
    while ((int)(ld_acquire_sys(mine + base + q) - e) < 0) {
      if (globaltimer_ns() - t0 > kPeerTimeoutNs || *(volatile int*)a.err) {
        atomicExch(a.err, 1);
        mine[kTimeout] = 1u;
        return false;
      }
      __nanosleep(64);
    }
  }
  return true;
}

// Block-wide wait: thread 0 polls, the block proceeds together; false when
// the exchange has failed (outputs are then left untouched).
__device__ bool block_wait(const PeerArgs& a, int base, unsigned e) {
  __shared__ int ok;
  if (threadIdx.x == 0) ok = wait_words(a, base, e) ? 1 : 0;
  __syncthreads();
  return ok != 0;
}

// The last block of the launch to finish signals word base + rank = e at
// every peer (after all blocks' stores are visible system-wide); with
// bump != 0 it first records e as the local epoch.
__device__ void last_block_signal(const PeerArgs& a, int base, unsigned e, int bump) {
  __syncthreads();
  if (threadIdx.x != 0 || threadIdx.y != 0) return;
  unsigned* mine = a.pads[a.rank];
  __threadfence_system();
  if (atomicAdd(mine + kTicket, 1u) != gridDim.x * gridDim.y - 1) return;
  mine[kTicket] = 0u;
  if (bump) mine[kEpoch] = e;
  __threadfence_system();
  for (int q = 0; q < a.nranks; ++q) st_release_sys(a.pads[q] + base + a.rank, e);
}

// 1a. publish, fused with the backprojection's chunk sum: PUB = scale * sum
// of the nplanes partial planes (fixed order).  grid.y = batch image.
__global__ void k_chunk_reduce_publish(const float* __restrict__ part, int nplanes, size_t np, PeerArgs a,
                                       float scale, int G) {
  __shared__ PlaneSmem sm;
  const unsigned e = *(volatile unsigned*)(a.pads[a.rank] + kEpoch) + 1u;
  const size_t b = blockIdx.y;
  float* dst = a.bufs[a.rank] + b * np;
  const float* src = part + b * nplanes * np;
  const int tid = threadIdx.y * 32 + threadIdx.x, tile = plane_tile(G);
  for (size_t p0 = (size_t)blockIdx.x * tile; p0 < np; p0 += (size_t)gridDim.x * tile) {
    sum_planes(src, nplanes, np, p0, G, sm);
    const size_t p = p0 + tid;
    if (tid < tile && p < np) dst[p] = scale * sm.tot[tid];
    if (G != 1) __syncthreads();   // tot is rewritten by the next tile
  }
  last_block_signal(a, kPub, e, 1);
}

// 1b. publish a buffer (generic allreduce: back_project(allreduce=1), ...)
__global__ void k_publish_copy(const float* __restrict__ buf, size_t count, PeerArgs a) {
  const unsigned e = *(volatile unsigned*)(a.pads[a.rank] + kEpoch) + 1u;
  float* dst = a.bufs[a.rank];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = buf[i];
  last_block_signal(a, kPub, e, 1);
}

__device__ __forceinline__ size_t chunk_lo(int q, int P, size_t count) { return ((size_t)q * count) / P; }

// 2. reduce-scatter: this rank's chunk of the sum, in rank order, into RED
__global__ void k_peer_rs(size_t count, PeerArgs a) {
  const unsigned e = *(volatile unsigned*)(a.pads[a.rank] + kEpoch);
  if (block_wait(a, kPub, e)) {
    const size_t lo = chunk_lo(a.rank, a.nranks, count), hi = chunk_lo(a.rank + 1, a.nranks, count);
    float* red = a.bufs[a.rank] + a.slot;
    for (size_t i = lo + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi; i += (size_t)gridDim.x * blockDim.x) {
      float s = 0.f;
      for (int q = 0; q < a.nranks; ++q) s += a.bufs[q][i];
      red[i] = s;
    }
  }
  last_block_signal(a, kRed, e, 0);
}

__device__ __forceinline__ float gathered(const PeerArgs& a, size_t i, size_t count) {
  const int q = (int)((((unsigned long long)i + 1) * (unsigned long long)a.nranks - 1) / count);   // chunk owner
  return a.bufs[q][a.slot + i];
}

// 3a. all-gather into out
__global__ void k_peer_ag(size_t count, PeerArgs a, float* __restrict__ out) {
  const unsigned e = *(volatile unsigned*)(a.pads[a.rank] + kEpoch);
  if (!block_wait(a, kRed, e)) return;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    out[i] = gathered(a, i, count);
}

// 3b. all-gather fused with the step z = y - eta U_s G (y == NULL: z = U_s G);
// element i = coarse pixel (b, I, J) of the [batch][nc][nc] sum
__global__ void k_peer_ag_step(size_t count, PeerArgs a, int nc, int s, const float* __restrict__ y,
                               const float* __restrict__ eta_dev, float* __restrict__ z) {
  const unsigned e = *(volatile unsigned*)(a.pads[a.rank] + kEpoch);
  if (!block_wait(a, kRed, e)) return;
  const float et = eta_dev ? *eta_dev : 0.f;
  const int n = nc * s;
  const size_t np = (size_t)nc * nc;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const float G = gathered(a, i, count);
    const size_t b = i / np, r = i - b * np;
    const int I = (int)(r / nc), J = (int)(r - (size_t)I * nc);
    for (int u = 0; u < s; ++u) {
      const size_t row = (b * n + (size_t)(s * I + u)) * n + (size_t)s * J;
      for (int q = 0; q < s; ++q) z[row + q] = y ? fmaf(-et, G, y[row + q]) : G;
    }
  }
}

static int grid_for(size_t n, int cap) {
  const size_t b = (n + 255) / 256;
  return (int)(b < (size_t)cap ? (b ? b : 1) : cap);
}

static PeerArgs peer_args(ms2g_plan* p) {
  return PeerArgs{p->d_peer_bufs, p->d_peer_pads, p->peer_rank, p->peer_n, p->xch_slot, p->w_peer_err};
}

int launch_peer_finish(ms2g_plan* p, float* out, size_t count, cudaStream_t st) {
  const PeerArgs a = peer_args(p);
  k_peer_rs<<<grid_for((count + p->peer_n - 1) / p->peer_n, 2 * p->sm_count), 256, 0, st>>>(count, a);
  MS2G_TRY(check_launch("k_peer_rs"));
  k_peer_ag<<<grid_for(count, 4 * p->sm_count), 256, 0, st>>>(count, a, out);
  return check_launch("k_peer_ag");
}

int launch_peer_finish_step(ms2g_plan* p, size_t count, int nc, int s, const float* y, const float* eta_dev,
                            float* z, cudaStream_t st) {
  const PeerArgs a = peer_args(p);
  k_peer_rs<<<grid_for((count + p->peer_n - 1) / p->peer_n, 2 * p->sm_count), 256, 0, st>>>(count, a);
  MS2G_TRY(check_launch("k_peer_rs"));
  k_peer_ag_step<<<grid_for(count, 4 * p->sm_count), 256, 0, st>>>(count, a, nc, s, y, eta_dev, z);
  return check_launch("k_peer_ag_step");
}

int launch_peer_allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st) {
  if (count > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "peer allreduce larger than the exchange slot");
  k_publish_copy<<<grid_for(count, 4 * p->sm_count), 256, 0, st>>>(buf, count, peer_args(p));
  MS2G_TRY(check_launch("k_publish_copy"));
  return launch_peer_finish(p, buf, count, st);
}

int launch_chunk_reduce_publish(ms2g_plan* p, const float* part, int nplanes, size_t np, size_t total, float scale,
                                cudaStream_t st) {
  if (total > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "peer allreduce larger than the exchange slot");
  const int G = plane_groups(np, nplanes);
  k_chunk_reduce_publish<<<dim3(plane_blocks(np, G, 4096), (unsigned)(total / np)), dim3(32, kPlaneGroups), 0, st>>>(
      part, nplanes, np, peer_args(p), scale, G);
  return check_launch("k_chunk_reduce_publish");
}

}  // namespace ms2g
