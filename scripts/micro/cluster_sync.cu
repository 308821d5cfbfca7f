// Microbenchmark (dev aid): cost of one thread-block-cluster barrier
// (barrier.cluster.arrive.release + wait.acquire) per iteration, alone and
// with a distributed-shared-memory read of the neighbour CTAs' boundary rows
// (2 x 512 floats), for cluster sizes 2..16, one cluster per image strip.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cluster_sync cluster_sync.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
constexpr int NIT = 2000;
template <bool DS>
__global__ void k(float* out) {
  __shared__ float row[2][2][512];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), n = cl.num_blocks();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) (&row[0][0][0])[i] = (float)(r + i);
  cl.sync();
  float acc = 0.f;
  for (int it = 0; it < NIT; ++it) {
    const int b = it & 1;
    if (DS) {
      const float* up = cl.map_shared_rank(&row[b][1][0], (r + n - 1) % n);
      const float* dn = cl.map_shared_rank(&row[b][0][0], (r + 1) % n);
      for (int i = threadIdx.x; i < 512; i += blockDim.x) acc += up[i] + dn[i];
      for (int i = threadIdx.x; i < 512; i += blockDim.x) { row[b ^ 1][0][i] = acc; row[b ^ 1][1][i] = acc + 1.f; }
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) out[blockIdx.x] = acc;
}
template <bool DS>
float run(int cs, int nclusters, float* out) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * nclusters);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k<DS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchKernelEx(&cfg, k<DS>, out);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, k<DS>, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("cs %d: %s\n", cs, cudaGetErrorString(e)); return -1; }
  return ms * 1e3f / NIT;   // us per iteration
}
int main() {
  float* out; cudaMalloc(&out, 4096 * 4);
  for (int cs : {2, 4, 8, 16}) {
    int ncl = (cs == 16) ? 8 : 144 / cs;
    printf("cluster %2d x %3d clusters: barrier %.3f us/iter, barrier + DSMEM rows %.3f us/iter\n", cs, ncl,
           run<false>(cs, ncl, out), run<true>(cs, ncl, out));
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
