// ubench2.cu -- cycle cost of the loop's building blocks in isolation (dev tool).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2202_12380_b200/csrc -o ubench2 ubench2.cu
#include <cstdio>
#include "argmax.cuh"

__device__ __forceinline__ long long tclock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <typename R>
__global__ void blocks(long long* out, int nrec, int reps) {
  extern __shared__ __align__(32) unsigned char smem[];
  Rec<R>* rec = reinterpret_cast<Rec<R>*>(smem);
  for (int i = threadIdx.x; i < nrec; i += blockDim.x) {
    rec[i].s = (R)((i * 7919) % 1000);
    rec[i].re = (R)i;
    rec[i].im = 0;
    rec[i].p = i;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  long long acc = 0;
  // (a) warp_node: one 32-record node -> argmax (redux) -> winner stores
  long long t0 = tclock();
  int node = 0;
  for (int r = 0; r < reps; ++r) {
    const Rec<R> x = rec[(node * 32 + lane) % nrec];
    R s;
    uint32_t p;
    const int wl = warp_argmax(x.s, x.p, s, p);
    if (lane == wl) rec[nrec - 1 - (node & 63)] = x;
    node = (node + 1 + (int)p) & 127;
    __syncwarp();
  }
  long long t1 = tclock();
  // (b) warp_best (full record argmax)
  Rec<R> b = rec[lane];
  for (int r = 0; r < reps; ++r) {
    b = warp_best(b);
    b.s += (R)lane;
  }
  long long t2 = tclock();
  // (c) top scan of 81 records + warp_best
  for (int r = 0; r < reps; ++r) {
    Rec<R> bb = empty_rec(R(0));
    for (int i = lane; i < 81; i += 32) {
      const Rec<R> x = rec[(i + r) % nrec];
      if (better(x.s, x.p, bb.s, bb.p)) bb = x;
    }
    bb = warp_best(bb);
    acc += bb.p;
  }
  long long t3 = tclock();
  // (d) __syncwarp + smem atomicExch/atomicAdd dirty marking
  for (int r = 0; r < reps; ++r) {
    int* st = reinterpret_cast<int*>(smem + 65536);
    if (lane == 0) {
      if (atomicExch(&st[r & 31], r) != r) st[64 + atomicAdd(&st[100], 1) % 32] = r;
    }
    __syncwarp();
  }
  long long t4 = tclock();
  if (lane == 0) {
    out[0] = (t1 - t0) / reps;
    out[1] = (t2 - t1) / reps;
    out[2] = (t3 - t2) / reps;
    out[3] = (t4 - t3) / reps;
    out[4] = acc + b.p;
  }
}

// __syncthreads cost with 8 warps doing nothing else
__global__ void bars(long long* out, int reps) {
  long long t0 = tclock();
  for (int r = 0; r < reps; ++r) __syncthreads();
  long long t1 = tclock();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  long long h[8];
  cudaFuncSetAttribute(blocks<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(blocks<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  blocks<double><<<1, 256, 200 * 1024>>>(d, 2048, 1000);
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("f64: warp_node %lld | warp_best %lld | top scan 81 %lld | dirty mark %lld cycles\n", h[0], h[1], h[2], h[3]);
  blocks<float><<<1, 256, 200 * 1024>>>(d, 2048, 1000);
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("f32: warp_node %lld | warp_best %lld | top scan 81 %lld | dirty mark %lld cycles\n", h[0], h[1], h[2], h[3]);
  bars<<<1, 256>>>(d, 1000);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (8 warps) %lld cycles\n", h[0]);
  bars<<<1, 512>>>(d, 1000);
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (16 warps) %lld cycles\n", h[0]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
