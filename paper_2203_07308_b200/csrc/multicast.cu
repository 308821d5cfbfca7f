// multicast.cu -- NEXT-3, NVLS form ("symmetric memory plus
// in-switch multimem reduction"): the cross-rank sum of the view-sharded
// partial backprojections through an NVSwitch multicast object, reduced IN
// THE SWITCH by multimem.ld_reduce and broadcast by multimem.st.
//
// Attach (host): rank 0 creates a multicast object for P devices
// (cuMulticastCreate) and exports it as a POSIX file descriptor; the caller
// all-gathers the blob; every other rank imports it (pidfd_getfd) and every
// rank adds its device (phase 0); after a process-group barrier every rank
// allocates its physical buffer, binds it to the object and maps both the
// unicast and the multicast address (phase 1).  The driver API is reached
// through cudaGetDriverEntryPointByVersion (no libcuda link dependency).
// Where multicast is unavailable -- e.g. this pool's single-GPU boxes, where
// cuMulticastCreate returns CUDA_ERROR_INVALID_VALUE (gpurun_out/probe_mc.log)
// -- ms2g_mc_create fails cleanly with MS2G_ERR_CUDA and the plan keeps its
// other exchange paths.  UNEXERCISED beyond that failure: no multi-GPU box.
//
// One allreduce (buffer regions PUB | RED | flags, identical on every rank):
//   1. publish: the chunk sum writes scale * G_r into the local PUB region
//      (unicast); the last block adds 1 to flag word 0 of EVERY rank's copy
//      with one multimem.red.release (the switch fans it out);
//   2. reduce: every block waits until its local flag 0 reaches P e, then
//      rank r reads its 1/P chunk as the switch-reduced sum over all ranks'
//      PUB regions (multimem.ld_reduce.add.f32) and writes it to every rank's
//      RED region (multimem.st); the last block bumps flag 1 everywhere;
//   3. finish: wait for flag 1 = P e, read RED locally (or take the step
//      z = y - eta U_s G from it).  Every rank reads the same reduced words.
// Ordering between allreduces follows the same argument as peer_reduce.cu.
#include <cuda.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace ms2g {

namespace {
typedef CUresult (*PFN_mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
typedef CUresult (*PFN_mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
typedef CUresult (*PFN_mcAddDev)(CUmemGenericAllocationHandle, CUdevice);
typedef CUresult (*PFN_mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                                  unsigned long long);
typedef CUresult (*PFN_export)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType, unsigned long long);
typedef CUresult (*PFN_import)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
typedef CUresult (*PFN_create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
typedef CUresult (*PFN_reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
typedef CUresult (*PFN_map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
typedef CUresult (*PFN_access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
typedef CUresult (*PFN_unmap)(CUdeviceptr, size_t);
typedef CUresult (*PFN_free)(CUdeviceptr, size_t);
typedef CUresult (*PFN_release)(CUmemGenericAllocationHandle);

struct Drv {
  PFN_mcCreate mcCreate = nullptr;
  PFN_mcGran mcGran = nullptr;
  PFN_mcAddDev mcAddDev = nullptr;
  PFN_mcBindMem mcBindMem = nullptr;
  PFN_export exportH = nullptr;
  PFN_import importH = nullptr;
  PFN_create create = nullptr;
  PFN_reserve reserve = nullptr;
  PFN_map map = nullptr;
  PFN_access access = nullptr;
  PFN_unmap unmap = nullptr;
  PFN_free freeVA = nullptr;
  PFN_release release = nullptr;
  bool ok = false;
};

template <class F>
bool entry(const char* name, F* fn) {
  cudaDriverEntryPointQueryResult q;
  void* p = nullptr;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    x.ok = entry("cuMulticastCreate", &x.mcCreate) && entry("cuMulticastGetGranularity", &x.mcGran) &&
           entry("cuMulticastAddDevice", &x.mcAddDev) && entry("cuMulticastBindMem", &x.mcBindMem) &&
           entry("cuMemExportToShareableHandle", &x.exportH) &&
           entry("cuMemImportFromShareableHandle", &x.importH) && entry("cuMemCreate", &x.create) &&
           entry("cuMemAddressReserve", &x.reserve) && entry("cuMemMap", &x.map) &&
           entry("cuMemSetAccess", &x.access) && entry("cuMemUnmap", &x.unmap) &&
           entry("cuMemAddressFree", &x.freeVA) && entry("cuMemRelease", &x.release);
    return x;
  }();
  return d;
}

struct McBlob {
  uint64_t magic;
  int32_t pid, fd;
  uint64_t size;
  int32_t nranks, pad;
};
constexpr uint64_t kMcMagic = 0x4d5332474d434153ULL;   // "MS2GMCAS"

int drv_error(const char* what, CUresult r) {
  return set_error(MS2G_ERR_CUDA, std::string("NVLS multicast: ") + what + " returned CUresult " + std::to_string((int)r));
}
}  // namespace

// ------------------------------------------------------------- device side
constexpr unsigned long long kMcTimeoutNs = 20ull * 1000 * 1000 * 1000;   // 20 s

__device__ __forceinline__ unsigned long long mc_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned mc_ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void mc_red_add(unsigned* mc_word, unsigned v) {
  asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_word), "r"(v) : "memory");
}
__device__ __forceinline__ float mc_ld_reduce(const float* mc) {
  float v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc) : "memory");
  return v;
}
__device__ __forceinline__ void mc_st(float* mc, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "f"(v) : "memory");
}

struct McArgs {
  float* uc;            // local unicast view: PUB [slot] | RED [slot] | flags
  float* mc;            // multicast view of the same layout
  size_t slot;
  int rank, nranks;
  int* err;
};
__device__ __forceinline__ unsigned* mc_flags(float* base, size_t slot) {
  return reinterpret_cast<unsigned*>(base + 2 * slot);
}

// block-wide wait until local flag word w reaches target (false: failed)
__device__ bool mc_wait(const McArgs& a, int w, unsigned target) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    const unsigned* f = mc_flags(a.uc, a.slot) + w;
    const unsigned long long t0 = mc_clock();
    while ((int)(mc_ld_acquire(f) - target) < 0) {
      if (*(volatile int*)a.err || mc_clock() - t0 > kMcTimeoutNs) {
        atomicExch(a.err, 1);
        ok = 0;
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
  return ok != 0;
}

// the last block of the launch adds 1 to flag word w on every rank
__device__ void mc_last_block_signal(const McArgs& a, int w) {
  __syncthreads();
  if (threadIdx.x != 0 || threadIdx.y != 0) return;
  unsigned* local = mc_flags(a.uc, a.slot);
  __threadfence_system();
  if (atomicAdd(local + 3, 1u) != gridDim.x * gridDim.y - 1) return;   // word 3: ticket
  local[3] = 0u;
  __threadfence_system();
  mc_red_add(mc_flags(a.mc, a.slot) + w, 1u);
}

__global__ void k_mc_publish(const float* __restrict__ part, int nplanes, size_t np, McArgs a, float scale, int G) {
  __shared__ PlaneSmem sm;
  const size_t b = blockIdx.y;
  float* dst = a.uc + b * np;
  const float* src = part + b * nplanes * np;
  const int tid = threadIdx.y * 32 + threadIdx.x, tile = plane_tile(G);
  for (size_t p0 = (size_t)blockIdx.x * tile; p0 < np; p0 += (size_t)gridDim.x * tile) {
    sum_planes(src, nplanes, np, p0, G, sm);
    const size_t p = p0 + tid;
    if (tid < tile && p < np) dst[p] = scale * sm.tot[tid];
    if (G != 1) __syncthreads();   // tot is rewritten by the next tile
  }
  mc_last_block_signal(a, 0);
}

__global__ void k_mc_publish_copy(const float* __restrict__ buf, size_t count, McArgs a) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    a.uc[i] = buf[i];
  mc_last_block_signal(a, 0);
}

// epoch e = this allreduce's number (local word 2, bumped by the reducer's
// last block after its wait): targets P e on words 0 and 1
__global__ void k_mc_reduce(size_t count, McArgs a) {
  const unsigned e = *(volatile unsigned*)(mc_flags(a.uc, a.slot) + 2) + 1u;
  if (mc_wait(a, 0, e * (unsigned)a.nranks)) {
    const size_t lo = ((size_t)a.rank * count) / a.nranks, hi = ((size_t)(a.rank + 1) * count) / a.nranks;
    for (size_t i = lo + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi; i += (size_t)gridDim.x * blockDim.x)
      mc_st(a.mc + a.slot + i, mc_ld_reduce(a.mc + i));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* local = mc_flags(a.uc, a.slot);
    __threadfence_system();
    if (atomicAdd(local + 4, 1u) == gridDim.x - 1) {   // word 4: ticket of this kernel
      local[4] = 0u;
      local[2] = e;
      __threadfence_system();
      mc_red_add(mc_flags(a.mc, a.slot) + 1, 1u);
    }
  }
}

__global__ void k_mc_finish(size_t count, McArgs a, float* __restrict__ out, int nc, int s,
                            const float* __restrict__ y, const float* __restrict__ eta_dev) {
  const unsigned e = *(volatile unsigned*)(mc_flags(a.uc, a.slot) + 2);
  if (!mc_wait(a, 1, e * (unsigned)a.nranks)) return;
  const float* red = a.uc + a.slot;
  if (s == 0) {   // plain all-gather into out
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
      out[i] = red[i];
    return;
  }
  const float et = eta_dev ? *eta_dev : 0.f;
  const int n = nc * s;
  const size_t np = (size_t)nc * nc;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const float G = red[i];
    const size_t b = i / np, r = i - b * np;
    const int I = (int)(r / nc), J = (int)(r - (size_t)I * nc);
    for (int u = 0; u < s; ++u) {
      const size_t row = (b * n + (size_t)(s * I + u)) * n + (size_t)s * J;
      for (int q = 0; q < s; ++q) out[row + q] = y ? fmaf(-et, G, y[row + q]) : G;
    }
  }
}

static McArgs mc_args(ms2g_plan* p) {
  return McArgs{(float*)p->mc_uc, (float*)p->mc_mc, p->xch_slot, p->mc_rank, p->mc_n, p->w_peer_err};
}
static int mc_grid(size_t n, int cap) {
  const size_t b = (n + 255) / 256;
  return (int)(b < (size_t)cap ? (b ? b : 1) : cap);
}

int launch_mc_publish(ms2g_plan* p, const float* part, int nplanes, size_t np, size_t total, float scale,
                      cudaStream_t st) {
  if (total > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "multicast allreduce larger than the exchange slot");
  const int G = plane_groups(np, nplanes);
  k_mc_publish<<<dim3(plane_blocks(np, G, 4096), (unsigned)(total / np)), dim3(32, kPlaneGroups), 0, st>>>(
      part, nplanes, np, mc_args(p), scale, G);
  return check_launch("k_mc_publish");
}

int launch_mc_finish(ms2g_plan* p, size_t count, float* out, int nc, int s, const float* y, const float* eta_dev,
                     cudaStream_t st) {
  const McArgs a = mc_args(p);
  k_mc_reduce<<<mc_grid((count + p->mc_n - 1) / p->mc_n, 2 * p->sm_count), 256, 0, st>>>(count, a);
  MS2G_TRY(check_launch("k_mc_reduce"));
  k_mc_finish<<<mc_grid(count, 4 * p->sm_count), 256, 0, st>>>(count, a, out, nc, s, y, eta_dev);
  return check_launch("k_mc_finish");
}

int launch_mc_allreduce(ms2g_plan* p, float* buf, size_t count, cudaStream_t st) {
  if (count > p->xch_slot) return set_error(MS2G_ERR_CONFIG, "multicast allreduce larger than the exchange slot");
  k_mc_publish_copy<<<mc_grid(count, 4 * p->sm_count), 256, 0, st>>>(buf, count, mc_args(p));
  MS2G_TRY(check_launch("k_mc_publish_copy"));
  return launch_mc_finish(p, count, buf, 0, 0, nullptr, nullptr, st);
}

// --------------------------------------------------------------- host side
static size_t mc_bytes(const ms2g_plan* p) { return sizeof(float) * 2 * p->xch_slot + 256; }

int mc_create(ms2g_plan* p, int nranks, void* blob_out) {
  const Drv& d = drv();
  if (!d.ok) return set_error(MS2G_ERR_CUDA, "NVLS multicast: driver entry points unavailable");
  if (nranks < 1 || nranks > 64) return set_error(MS2G_ERR_CONFIG, "bad nranks");
  CUmulticastObjectProp prop = {};
  prop.numDevices = (unsigned)nranks;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = mc_bytes(p);
  size_t gran = 0;
  CUresult r = d.mcGran(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return drv_error("cuMulticastGetGranularity", r);
  prop.size = (prop.size + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle mc = 0;
  r = d.mcCreate(&mc, &prop);
  if (r != CUDA_SUCCESS)
    return drv_error("cuMulticastCreate (unavailable here: one GPU, or no NVSwitch multicast on this system)", r);
  int fd = -1;
  r = d.exportH(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) {
    d.release(mc);
    return drv_error("cuMemExportToShareableHandle", r);
  }
  p->mc_handle = (unsigned long long)mc;
  p->mc_size = prop.size;
  McBlob b{kMcMagic, (int32_t)getpid(), fd, prop.size, nranks, 0};
  memcpy(blob_out, &b, sizeof(b));
  return MS2G_OK;
}

int mc_attach(ms2g_plan* p, const void* blob0, int rank, int nranks, int phase) {
  const Drv& d = drv();
  if (!d.ok) return set_error(MS2G_ERR_CUDA, "NVLS multicast: driver entry points unavailable");
  McBlob b;
  memcpy(&b, blob0, sizeof(b));
  if (b.magic != kMcMagic || b.nranks != nranks) return set_error(MS2G_ERR_CONFIG, "multicast blob mismatch");
  int dev = 0;
  MS2G_CUDA(cudaGetDevice(&dev));
  CUresult r;
  if (phase == 0) {
    if (rank != 0) {   // import rank 0's object through its file descriptor
      const long pidfd = syscall(SYS_pidfd_open, (pid_t)b.pid, 0);
      if (pidfd < 0) return set_error(MS2G_ERR_CUDA, "NVLS multicast: pidfd_open failed");
      const long fd = syscall(SYS_pidfd_getfd, (int)pidfd, b.fd, 0);
      close((int)pidfd);
      if (fd < 0) return set_error(MS2G_ERR_CUDA, "NVLS multicast: pidfd_getfd failed (ptrace permission?)");
      CUmemGenericAllocationHandle mc = 0;
      r = d.importH(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close((int)fd);
      if (r != CUDA_SUCCESS) return drv_error("cuMemImportFromShareableHandle", r);
      p->mc_handle = (unsigned long long)mc;
      p->mc_size = b.size;
    }
    r = d.mcAddDev((CUmemGenericAllocationHandle)p->mc_handle, (CUdevice)dev);
    if (r != CUDA_SUCCESS) return drv_error("cuMulticastAddDevice", r);
    return MS2G_OK;
  }
  // phase 1 (after every rank's phase 0): physical memory, bind, map both views
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  CUmemGenericAllocationHandle mem = 0;
  if ((r = d.create(&mem, p->mc_size, &ap, 0)) != CUDA_SUCCESS) return drv_error("cuMemCreate", r);
  if ((r = d.mcBindMem((CUmemGenericAllocationHandle)p->mc_handle, 0, mem, 0, p->mc_size, 0)) != CUDA_SUCCESS)
    return drv_error("cuMulticastBindMem", r);
  CUdeviceptr uc = 0, mcva = 0;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((r = d.reserve(&uc, p->mc_size, 0, 0, 0)) != CUDA_SUCCESS) return drv_error("cuMemAddressReserve", r);
  if ((r = d.map(uc, p->mc_size, 0, mem, 0)) != CUDA_SUCCESS) return drv_error("cuMemMap (unicast)", r);
  if ((r = d.access(uc, p->mc_size, &acc, 1)) != CUDA_SUCCESS) return drv_error("cuMemSetAccess (unicast)", r);
  if ((r = d.reserve(&mcva, p->mc_size, 0, 0, 0)) != CUDA_SUCCESS) return drv_error("cuMemAddressReserve", r);
  if ((r = d.map(mcva, p->mc_size, 0, (CUmemGenericAllocationHandle)p->mc_handle, 0)) != CUDA_SUCCESS)
    return drv_error("cuMemMap (multicast)", r);
  if ((r = d.access(mcva, p->mc_size, &acc, 1)) != CUDA_SUCCESS) return drv_error("cuMemSetAccess (multicast)", r);
  p->mc_mem = (unsigned long long)mem;
  p->mc_uc = (void*)uc;
  p->mc_mc = (void*)mcva;
  MS2G_CUDA(cudaMemset(p->mc_uc, 0, p->mc_size));
  if (!p->w_peer_err) {
    MS2G_CUDA(cudaMalloc(&p->w_peer_err, sizeof(int)));
    MS2G_CUDA(cudaMemset(p->w_peer_err, 0, sizeof(int)));
  }
  p->mc_rank = rank;
  p->mc_n = nranks;
  p->rank = rank;
  p->nranks = nranks;
  return MS2G_OK;
}

void mc_release(ms2g_plan* p) {
  const Drv& d = drv();
  if (!d.ok) return;
  if (p->mc_mc) {
    d.unmap((CUdeviceptr)p->mc_mc, p->mc_size);
    d.freeVA((CUdeviceptr)p->mc_mc, p->mc_size);
  }
  if (p->mc_uc) {
    d.unmap((CUdeviceptr)p->mc_uc, p->mc_size);
    d.freeVA((CUdeviceptr)p->mc_uc, p->mc_size);
  }
  if (p->mc_mem) d.release((CUmemGenericAllocationHandle)p->mc_mem);
  if (p->mc_handle) d.release((CUmemGenericAllocationHandle)p->mc_handle);
  p->mc_mc = p->mc_uc = nullptr;
  p->mc_mem = p->mc_handle = 0;
  p->mc_n = 0;
}

int mc_blob_size() { return (int)sizeof(McBlob); }

}  // namespace ms2g
