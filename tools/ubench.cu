// ubench.cu -- latency microbenchmarks on the B200 (dev tool, not part of the library):
// dependent global loads (L2 / DRAM), shared-memory atomics, fences, redux.sync,
// DSMEM st.async + mbarrier ping-pong between two CTAs of a cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ubench ubench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

__global__ void chase(const unsigned* __restrict__ next, int steps, unsigned start, long long* out, unsigned* sink) {
  unsigned p = start;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) {
    unsigned q;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(q) : "l"(next + p));
    p = q;
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
  *sink = p;
}

__global__ void misc(long long* out, int* sink) {
  __shared__ int a[64];
  __shared__ double d[64];
  if (threadIdx.x < 64) { a[threadIdx.x] = 0; d[threadIdx.x] = 1.0; }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int N = 1000;
  // dependent smem atomics
  long long t0 = clock64();
  int v = 0;
  for (int i = 0; i < N; ++i) v = atomicAdd(&a[v & 7], 1) & 1;
  long long t1 = clock64();
  // fences
  for (int i = 0; i < N; ++i) { a[threadIdx.x] = i; __threadfence_block(); }
  long long t2 = clock64();
  // dependent redux
  unsigned r = threadIdx.x;
  for (int i = 0; i < N; ++i) r = __reduce_max_sync(0xffffffffu, r + i) - i;
  long long t3 = clock64();
  // dependent shfl
  for (int i = 0; i < N; ++i) r = __shfl_sync(0xffffffffu, r, (r + 1) & 31);
  long long t4 = clock64();
  // dependent fp64 division
  double x = 1.0 + threadIdx.x;
  for (int i = 0; i < N; ++i) x = 3.0 / (x + 1.0);
  long long t5 = clock64();
  // dependent LDS
  int q = threadIdx.x & 7;
  for (int i = 0; i < N; ++i) q = a[q & 63] & 7;
  long long t6 = clock64();
  // __syncwarp + gtime reading
  long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  for (int i = 0; i < N; ++i) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1)); }
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[0] = (t1 - t0) / N; out[1] = (t2 - t1) / N; out[2] = (t3 - t2) / N; out[3] = (t4 - t3) / N;
    out[4] = (t5 - t4) / N; out[5] = (t6 - t5) / N; out[6] = (t7 - t6) / N; out[7] = g1 - g0;
  }
  sink[threadIdx.x] = v + (int)r + (int)x + q;
}

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// two CTAs of a cluster play ping-pong through st.async + mbarrier complete_tx
__global__ void __cluster_dims__(2, 1, 1) pingpong(long long* out, int rounds) {
  __shared__ __align__(16) unsigned long long mbar;
  __shared__ __align__(16) uint4 box;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  if (threadIdx.x != 0) return;
  const uint32_t rb = saddr(&mbar), rd = saddr(&box);
  uint32_t peer_bar, peer_box;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_bar) : "r"(rb), "r"(rank ^ 1));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(peer_box) : "r"(rd), "r"(rank ^ 1));
  long long t0 = clock64();
  for (int i = 0; i < rounds; ++i) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(rb) : "memory");
    if (rank == (i & 1)) {
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%1,%1,%1}, [%2];" ::"r"(peer_box),
                   "r"(i), "r"(peer_bar) : "memory");
      // the peer answers in the next round; arrive locally so this phase completes too
    }
    // every round both sides expect 16 B: the one that did not send waits for the data,
    // the sender receives its answer next round -> each round = one one-way trip
    if (rank != (i & 1)) {
      uint32_t ok = 0;
      do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok) : "r"(rb), "r"((unsigned)((i >> 1) & 1)) : "memory");
      } while (!ok);
    }
  }
  long long t1 = clock64();
  if (rank == 0) out[0] = (t1 - t0) / rounds;
}

int main() {
  long long* d_out;
  unsigned* sink;
  cudaMalloc(&d_out, 64 * sizeof(long long));
  cudaMalloc(&sink, 4096);
  for (size_t mb : {1ull, 8ull, 35ull, 100ull, 512ull, 2048ull}) {
    size_t n = mb * 1024 * 1024 / 4;
    std::vector<unsigned> h(n);
    // random cyclic permutation with 128-B stride granularity
    size_t lines = n / 32;
    std::vector<unsigned> perm(lines);
    for (size_t i = 0; i < lines; ++i) perm[i] = (unsigned)i;
    unsigned long long s = 88172645463325252ull;
    for (size_t i = lines - 1; i > 0; --i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      size_t j = s % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    for (size_t i = 0; i < lines; ++i) h[perm[i] * 32] = perm[(i + 1) % lines] * 32;
    unsigned* d;
    cudaMalloc(&d, n * 4);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(d, 20000, 0, d_out, sink);   // warm L2
    chase<<<1, 1>>>(d, 20000, 0, d_out, sink);
    long long c;
    cudaMemcpy(&c, d_out, 8, cudaMemcpyDeviceToHost);
    printf("chase %5zu MB: %lld cycles/load\n", mb, c / 20000);
    cudaFree(d);
  }
  int* isink;
  cudaMalloc(&isink, 4096);
  misc<<<1, 64>>>(d_out, isink);
  long long m[8];
  cudaMemcpy(m, d_out, sizeof m, cudaMemcpyDeviceToHost);
  printf("smem atomicAdd dep %lld | fence.cta %lld | redux dep %lld | shfl dep %lld | fp64 div dep %lld | lds dep %lld | "
         "globaltimer read %lld cyc, 1000 reads span %lld ns\n",
         m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7]);
  pingpong<<<2, 32>>>(d_out, 10000);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(m, d_out, 8, cudaMemcpyDeviceToHost);
  printf("st.async+mbarrier one-way (cluster 2): %lld cycles  (%s)\n", m[0], cudaGetErrorString(e));
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
