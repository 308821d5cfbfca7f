// Microbenchmark (dev aid): cost of the adjoint's per-step shared-memory
// update on sm_100a.  Each warp walks NSTEP "steps"; per step one broadcast
// 16-B record load plus two updates at (row_lane, lane) and (row_lane+1, lane)
// (distinct banks, rows varying per lane), as in k_backward.
//   V0: fp32 read-modify-write (LDS, FADD, STS) x 2
//   V1: red.shared.add.u32 x 2 (integer, order-independent)
//   V2: red.shared.add.f32 x 2
//   V3: red.shared.add.u64 x 1 on a packed pair
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/smem_rmw smem_rmw.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NSTEP = 8192, ROWS = 36, WARPS = 4;
template <int V>
__global__ void __launch_bounds__(128) k(const int4* rec, int* out, int seed) {
  __shared__ int4 R[64];
  __shared__ unsigned T[WARPS][ROWS + 4][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < WARPS * (ROWS + 4) * 32; i += blockDim.x) (&T[0][0][0])[i] = 0;
  if (threadIdx.x < 64) R[threadIdx.x] = rec[threadIdx.x];
  __syncthreads();
  const unsigned e0 = seed * 2654435761u + lane * 40503u;
#pragma unroll 4
  for (int s = 0; s < NSTEP; ++s) {
    const int4 r = R[s & 63];                       // broadcast record
    const unsigned e = e0 + (unsigned)r.x * (unsigned)(lane + 1);   // independent steps
    const int row = (e >> 27) + 1;                   // 1..32, varies per lane
    const float wv = __int_as_float(r.y) * (float)(e & 0xffff);
    if (V == 0) {
      float* a = reinterpret_cast<float*>(&T[w][row][lane]);
      float* b = reinterpret_cast<float*>(&T[w][row + 1][lane]);
      *a += wv; *b += __int_as_float(r.z) - wv;
    } else if (V == 1) {
      const int iv = (int)(e & 0xffff) * r.w;
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row][lane])), "r"(iv));
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row + 1][lane])), "r"(r.z - iv));
    } else if (V == 2) {
      asm volatile("red.shared.add.f32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row][lane])), "f"(wv));
      asm volatile("red.shared.add.f32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row + 1][lane])), "f"(__int_as_float(r.z) - wv));
    } else if (V == 4) {
      const int iv = __float2int_rn(wv);
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row][lane])), "r"(iv));
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row + 1][lane])), "r"(r.z - iv));
  } else if (V == 5) {
      const int iv = __umulhi(e & 0xffffff, (unsigned)r.w);
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row][lane])), "r"(iv));
      asm volatile("red.shared.add.u32 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(&T[w][row + 1][lane])), "r"(r.z - iv));
  } else {
      const unsigned long long iv = (unsigned long long)((e & 0xffff) * (unsigned)r.w);
      unsigned long long* p = reinterpret_cast<unsigned long long*>(&T[w][row][lane & ~1]);
      asm volatile("red.shared.add.u64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(p)), "l"(iv));
    }
  }
  __syncthreads();
  unsigned acc = 0;
  for (int i = threadIdx.x; i < WARPS * (ROWS + 4) * 32; i += blockDim.x) acc += (&T[0][0][0])[i];
  atomicAdd(out, (int)acc);
}
template <int V>
float run(const int4* rec, int* out, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<V><<<blocks, 128>>>(rec, out, 1);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k<V><<<blocks, 128>>>(rec, out, i);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  if (cudaGetLastError() != cudaSuccess) { printf("error V%d\n", V); return -1; }
  return ms / 5;
}
int main() {
  int4* rec; int* out;
  cudaMalloc(&rec, 64 * sizeof(int4)); cudaMalloc(&out, 4);
  int4 h[64];
  for (int i = 0; i < 64; ++i) h[i] = make_int4(0x01234567 * (i + 1), 0x3727c5ac, 3, 7);
  cudaMemcpy(rec, h, sizeof h, cudaMemcpyHostToDevice);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {3, 4, 6, 8}) {
    const int blocks = sms * per;
    const double steps = (double)blocks * WARPS * NSTEP;   // warp-steps
    float t0 = run<0>(rec, out, blocks), t1 = run<1>(rec, out, blocks), t2 = run<2>(rec, out, blocks), t3 = run<3>(rec, out, blocks);
    float t4 = run<4>(rec, out, blocks), t5 = run<5>(rec, out, blocks);
    auto clk = [&](float ms) { return ms * 1e-3 * 1.965e9 * sms / steps; };   // SM clocks per warp-step per SM
    printf("blocks/SM %d: fp32 RMW %.3f ms (%.2f clk/warp-step)  red.u32 %.3f (%.2f)  red.f32 %.3f (%.2f)  red.u64x1 %.3f (%.2f)  F2I+red.u32 %.3f (%.2f)  mulhi+red.u32 %.3f (%.2f)\n",
           per, t0, clk(t0), t1, clk(t1), t2, clk(t2), t3, clk(t3), t4, clk(t4), t5, clk(t5));
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
}
