// synth.cu -- N6: synthesis of the approximation from an atom list (Eq. (18)):
//   y = sum_atoms c~ d (self-conjugate m = 0, M/2) or 2 Re(c~ d) (pairs).
// The atoms are first scattered into a solution grid (complex, unpadded), then
// every frame is inverted with one half-length complex IFFT in shared memory
// (c2r with Hermitian extension, X[M-m] = conj X[m]) and the windowed frames are
// overlap-added by a gather over output samples (fixed order -> deterministic).
#include <algorithm>
#include "launch.h"
#include "fft.cuh"

// Deterministic scatter of the atom list into the solution grid: sol(p) = 0 + c~_i1 +
// c~_i2 + ... over the atoms selecting p, in atom-list order -- the order of Alg. 1 step 2a
// (reading Z19) and of the oracle.  Rounds of one cooperative launch: every
// pending atom offers its list index to first[p] (atomicMin, an order-free result); the
// atom holding first[p] adds itself (one writer per p per round) and retires.  A p
// selected m times takes m rounds; the sum order never depends on scheduling.
__device__ __forceinline__ void synth_grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned int v;
    const long long t0 = clock64();
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
      if (clock64() - t0 > (1LL << 35)) __trap();  // a CTA that never arrives: fail, do not hang
    } while (v < target);
  }
  __syncthreads();
}

__global__ void synth_scatter_kernel(const AtomOut* __restrict__ atoms, int64_t n, const DictGeo* __restrict__ dg,
                                     double2* __restrict__ sol, unsigned int* __restrict__ first,
                                     unsigned char* __restrict__ done, unsigned int* __restrict__ ctl) {
  // ctl[0] barrier counter, ctl[1 + r % 3] "atoms left" flag of round r (all zero at launch):
  // round r clears the slot of round r + 1, last read (by every CTA) before round r - 1 ended
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned int gen = 0;
  for (int round = 0;; ++round) {
    if (i0 == 0) ctl[1 + (round + 1) % 3] = 0;
    for (int64_t i = i0; i < n; i += stride) {
      if (done[i]) continue;
      const AtomOut a = atoms[i];
      const DictGeo d = dg[a.w];
      atomicMin(first + d.off + (int64_t)a.n * d.MR + a.m, (unsigned int)i);
    }
    synth_grid_barrier(ctl, ++gen * gridDim.x);
    bool left = false;
    for (int64_t i = i0; i < n; i += stride) {
      if (done[i]) continue;
      const AtomOut a = atoms[i];
      const DictGeo d = dg[a.w];
      const int64_t p = d.off + (int64_t)a.n * d.MR + a.m;
      if (first[p] == (unsigned int)i) {
        double2 c = sol[p];
        c.x += a.re;
        c.y += a.im;
        sol[p] = c;
        first[p] = 0xffffffffu;
        done[i] = 1;
      } else {
        left = true;
      }
    }
    if (__syncthreads_or(left) && threadIdx.x == 0) ctl[1 + round % 3] = 1;
    synth_grid_barrier(ctl, ++gen * gridDim.x);
    if (*(volatile unsigned int*)&ctl[1 + round % 3] == 0) break;
  }
}

// frame n: t[s] = sum_{m=0}^{M-1} X[m] e^{+2 pi i m s/M}, X[0], X[M/2] real parts,
// X[M-m] = conj X[m]; via Z[m] = A[m] + i B[m], A = X[m] + conj X[n-m],
// B = (X[m] - conj X[n-m]) e^{+2 pi i m/M}, z = IFFT_n(Z), t[2r] = Re z[r], t[2r+1] = Im z[r].
__global__ void synth_frames_kernel(const double2* __restrict__ sol, int64_t off, int M, int MR, int N,
                                    const double2* __restrict__ tw, int twres, double* __restrict__ frames, int F) {
  extern __shared__ double2 z[];
  const int n = M / 2;
  const int lgn = 31 - __clz(n);
  const int frame0 = blockIdx.x * F;
  for (int idx = threadIdx.x; idx < F * n; idx += blockDim.x) {
    const int f = idx / n, m = idx - f * n;
    const int frame = frame0 + f;
    double2 Zm = make_double2(0.0, 0.0);
    if (frame < N) {
      const double2* X = sol + off + (int64_t)frame * MR;
      double2 a = X[m];
      double2 b = X[n - m];
      if (m == 0) {
        a.y = 0.0;
        b.y = 0.0;
      }
      const double2 bc = cconj(b);
      const double2 A = cadd(a, bc);
      double2 wp = __ldg(&tw[(int64_t)m * (twres / M)]);
      wp.y = -wp.y;  // e^{+2 pi i m/M}
      const double2 B = cmul(csub(a, bc), wp);
      Zm = make_double2(A.x - B.y, A.y + B.x);  // A + iB
    }
    z[f * n + bitrev(m, lgn)] = Zm;
  }
  __syncthreads();
  smem_fft(z, lgn, F, tw, twres, +1);
  for (int idx = threadIdx.x; idx < F * n; idx += blockDim.x) {
    const int f = idx / n, r = idx - f * n;
    const int frame = frame0 + f;
    if (frame >= N) continue;
    const double2 v = z[f * n + r];
    frames[(int64_t)frame * M + 2 * r] = v.x;
    frames[(int64_t)frame * M + 2 * r + 1] = v.y;
  }
}

// y[l] (+)= sum over frames nn covering l, ascending: g(j) t_nn(j mod M), j = l - nn a
__global__ void synth_ola_kernel(const double* __restrict__ frames, int a, int M, int N, int gl,
                                 const double* __restrict__ g, int64_t L, int64_t Ls, double* __restrict__ y,
                                 int accumulate) {
  const int j0 = -(gl / 2), j1 = j0 + gl - 1;
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < Ls; l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nlo = -fdiv64(-(l - j1), a);  // ceil((l - j1)/a)
    const int64_t nhi = fdiv64(l - j0, a);
    double acc = 0.0;
    for (int64_t nn = nlo; nn <= nhi; ++nn) {
      const int64_t j = l - nn * a;
      const int64_t fr = fmod64(nn, N);
      acc += g[j - j0] * frames[fr * M + fmod64(j, M)];
    }
    y[l] = accumulate ? y[l] + acc : acc;
  }
  (void)L;
}

cudaError_t launch_synth_scatter(const AtomOut* atoms, int64_t n_atoms, const DictGeo* dg_dev, int W, double2* sol,
                                 unsigned int* first, unsigned char* done, unsigned int* ctl, cudaStream_t st) {
  (void)W;
  if (n_atoms <= 0) return cudaSuccess;
  // co-resident CTAs (cooperative launch): at most the occupancy limit, at least one
  static int maxb = 0;
  if (maxb == 0) {
    int per_sm = 0, dev = 0, sms = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, synth_scatter_kernel, 256, 0));
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    maxb = std::max(1, std::min(per_sm, 4) * sms);
  }
  const int blocks = (int)std::min<int64_t>(maxb, (n_atoms + 255) / 256);
  void* args[] = {(void*)&atoms, (void*)&n_atoms, (void*)&dg_dev, (void*)&sol, (void*)&first, (void*)&done, (void*)&ctl};
  return cudaLaunchCooperativeKernel((const void*)synth_scatter_kernel, dim3(blocks), dim3(256), args, 0, st);
}

cudaError_t launch_synth_frames(const double2* sol, const DictGeo& d, const double2* tw, int twres, double* frames,
                                cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    CUDA_OK(cudaFuncSetAttribute(synth_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const int n = d.M / 2;
  const int F = max(1, 2048 / n);
  synth_frames_kernel<<<(d.N + F - 1) / F, 256, (size_t)F * n * sizeof(double2), st>>>(sol, d.off, d.M, d.MR, d.N,
                                                                                       tw, twres, frames, F);
  return cudaGetLastError();
}

cudaError_t launch_synth_ola(const double* frames, const DictGeo& d, const double* g, int64_t L, double* y,
                             int accumulate, cudaStream_t st) {
  // y has Ls = L entries here (caller passes the truncated length as L)
  const int blocks = (int)std::min<int64_t>(148 * 16, (L + 255) / 256);
  synth_ola_kernel<<<blocks, 256, 0, st>>>(frames, d.a, d.M, d.N, d.gl, g, L, L, y, accumulate);
  return cudaGetLastError();
}

// r -= y (Alg. 2 step 2c, r_out <- r_out - D c), grid-stride over n samples
__global__ void sub_kernel(double* __restrict__ r, const double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] -= y[i];
}

cudaError_t launch_sub(double* r, const double* y, int64_t n, cudaStream_t st) {
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((n + threads - 1) / threads, 148 * 8);
  sub_kernel<<<(unsigned)std::max<int64_t>(blocks, 1), threads, 0, st>>>(r, y, n);
  return cudaGetLastError();
}
