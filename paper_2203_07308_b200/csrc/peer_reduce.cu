// peer_reduce.cu -- NEXT-3: the backprojection's cross-rank sum
// over NVLink peer memory instead of a separate NCCL collective.
//
// Every rank's plan owns an IPC-shareable exchange buffer (two slots of
// n_cmax^2 x batch floats) and a signal pad.  After ms2g_attach_peers each
// rank holds device pointers to every peer's buffer and pad.  One allreduce
// of the view-sharded partial image G_r:
//   1. publish: the backprojector's chunk reduction writes scale * G_r
//      straight into slot (epoch + 1) & 1 of the local exchange buffer (fused
//      epilogue; a generic allreduce copies the buffer there instead),
//   2. barrier: epoch += 1; store it into slot `rank` of every peer's pad
//      (release, system scope); wait until every slot of the local pad holds
//      it (acquire),
//   3. sum: G = sum_{q = 0..P-1} slot_q of rank q's buffer, peer loads over
//      NVLink in FIXED rank order: every rank gets a bitwise identical G and
//      the result does not depend on a collective's algorithm.
// Two slots alternate: a rank reuses a slot two allreduces later only after
// the barrier in between, which every peer passes only after finishing its
// sum of that slot (stream order), so no extra barrier is needed.
// The wait in the barrier is bounded by 20 s of wall time (%globaltimer); on a
// time-out it raises the plan's error flag instead of hanging the device, and
// every later barrier / sum of the plan returns at once.  The host then sees
// MS2G_ERR_NCCL and the plan refuses further exchanges until every rank calls
// ms2g_attach_peers again (epochs restart from 0).
#include "internal.cuh"

namespace ms2g {

constexpr int kEpoch = 64;                // pad word holding the local epoch
constexpr int kTimeout = 65;              // pad word set on a barrier time-out

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// scale * (sum of nplanes partial planes) -> the local exchange slot of the
// NEXT epoch (fused publish of the backprojection).
// grid.y = batch image (no index division)
__global__ void k_chunk_reduce_publish(const float* __restrict__ part, int nplanes, size_t np,
                                       float* __restrict__ xbuf, size_t slot_elems, const unsigned* __restrict__ pad,
                                       float scale) {
  const size_t b = blockIdx.y;
  float* dst = xbuf + (size_t)((pad[kEpoch] + 1u) & 1u) * slot_elems + b * np;
  const float* src0 = part + b * nplanes * np;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < np; p += (size_t)gridDim.x * blockDim.x) {
    const float* src = src0 + p;
    float s = 0.f;
    for (int c = 0; c < nplanes; ++c) s += src[(size_t)c * np];
    dst[p] = scale * s;
  }
}

__global__ void k_publish_copy(const float* __restrict__ buf, size_t count, float* __restrict__ xbuf,
                               size_t slot_elems, const unsigned* __restrict__ pad) {
  float* dst = xbuf + (size_t)((pad[kEpoch] + 1u) & 1u) * slot_elems;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = buf[i];
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Wait until *slot has reached epoch e.  Bounded by WALL time (%globaltimer,
// kPeerTimeoutNs), not by a spin count; returns false on a time-out (after
// raising the plan's error flag) or at once when the flag is already up, so
// a failed exchange costs one time-out, not one per later barrier.
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;   // 20 s
__device__ bool wait_epoch(const unsigned* slot, unsigned e, int* err_flag, unsigned* timeout_word) {
  if (*(volatile int*)err_flag) return false;
  const unsigned long long t0 = globaltimer_ns();
  while ((int)(ld_acquire_sys(slot) - e) < 0) {
    if (globaltimer_ns() - t0 > kPeerTimeoutNs || *(volatile int*)err_flag) {
      atomicExch(err_flag, 1);
      *timeout_word = 1u;
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// one warp: lane q signals peer q and waits for peer q's signal
__global__ void k_peer_barrier(unsigned* const* __restrict__ pads, int rank, int nranks, int* err_flag) {
  unsigned* mine = pads[rank];
  __shared__ unsigned e;
  if (threadIdx.x == 0) {
    e = mine[kEpoch] + 1u;
    mine[kEpoch] = e;
  }
  __syncthreads();
  __threadfence_system();            // this rank's published slot before the signal
  for (int q = threadIdx.x; q < nranks; q += blockDim.x) st_release_sys(pads[q] + rank, e);
  for (int q = threadIdx.x; q < nranks; q += blockDim.x) wait_epoch(mine + q, e, err_flag, mine + kTimeout);
}

// out = sum over ranks (fixed order) of the current epoch's slots
__global__ void k_peer_sum(const float* const* __restrict__ bufs, int nranks, size_t slot_elems,
                           const unsigned* __restrict__ pad, float* __restrict__ out, size_t count,
                           const int* __restrict__ err_flag) {
  if (*(volatile const int*)err_flag) return;   // a peer never arrived: its slot holds stale data
  const size_t off = (size_t)(pad[kEpoch] & 1u) * slot_elems;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < nranks; ++q) s += bufs[q][off + i];
    out[i] = s;
  }
}

static int grid_for(size_t n) {
  const size_t b = (n + 255) / 256;
  return (int)(b < 4096 ? (b ? b : 1) : 4096);
}

int launch_peer_finish(ms2g_plan* p, float* out, size_t count, cudaStream_t st) {
  k_peer_barrier<<<1, 32, 0, st>>>(p->d_peer_pads, p->peer_rank, p->peer_n, p->w_peer_err);
  MS2G_TRY(check_launch("k_peer_barrier"));
  k_peer_sum<<<grid_for(count), 256, 0, st>>>(p->d_peer_bufs, p->peer_n, p->xch_slot, p->xch_pad, out, count,
                                               p->w_peer_err);
  return check_launch("k_peer_sum");
}

int launch_peer_allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st) {
  if (count > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "peer allreduce larger than the exchange slot");
  k_publish_copy<<<grid_for(count), 256, 0, st>>>(buf, count, p->xch_buf, p->xch_slot, p->xch_pad);
  MS2G_TRY(check_launch("k_publish_copy"));
  return launch_peer_finish(p, buf, count, st);
}

int launch_chunk_reduce_publish(ms2g_plan* p, const float* part, int nplanes, size_t np, size_t total, float scale,
                                cudaStream_t st) {
  if (total > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "peer allreduce larger than the exchange slot");
  k_chunk_reduce_publish<<<dim3(grid_for(np), (unsigned)(total / np)), 256, 0, st>>>(part, nplanes, np, p->xch_buf,
                                                                                     p->xch_slot, p->xch_pad, scale);
  return check_launch("k_chunk_reduce_publish");
}

}  // namespace ms2g
