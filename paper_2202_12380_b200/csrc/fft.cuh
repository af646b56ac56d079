// fft.cuh -- shared-memory real FFT building block (fp64) for the DGT analysis
// (N1), the Gram-kernel precompute (N2) and the synthesis (N6).
//
// A real sequence b of even length M is transformed through a half-length
// complex FFT: z[r] = b[2r] + i b[2r+1], Z = FFT_{M/2}(z),
//   X[m] = E[m] + W^m O[m],  E[m] = (Z[m] + conj Z[n-m])/2,  O[m] = (Z[m] - conj Z[n-m])/(2i),
// W = e^{-2 pi i/M}, n = M/2, m = 0..n.  Radix-2 decimation in time, one CTA
// transforms F frames at once; twiddles come from a table tw[k] = e^{-2 pi i k/res}
// (k < res/2) computed once per handle with sincospi.
#pragma once
#include "common.cuh"

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__device__ __forceinline__ int bitrev(int i, int lg) { return lg == 0 ? 0 : (int)(__brev((unsigned)i) >> (32 - lg)); }

// In-place radix-2 DIT FFT of F consecutive length-n sequences in shared memory,
// input already in bit-reversed order.  sign = -1 forward (e^{-}), +1 inverse (e^{+}),
// unnormalised.  All threads of the block must call it.
__device__ inline void smem_fft(double2* z, int lgn, int F, const double2* __restrict__ tw, int twres,
                                int sign) {
  const int n = 1 << lgn;
  const int nb = F << (lgn - (lgn > 0 ? 1 : 0));  // butterflies per stage = F*n/2
  if (lgn == 0) return;
  for (int lh = 0; lh < lgn; ++lh) {               // half = 2^lh, len = 2^(lh+1)
    const int half = 1 << lh;
    const int tstep = twres >> (lh + 1);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int f = b >> (lgn - 1);
      const int i = b & ((n >> 1) - 1);
      const int jj = i & (half - 1);
      const int i0 = (f << lgn) + ((i >> lh) << (lh + 1)) + jj;
      const int i1 = i0 + half;
      double2 w = __ldg(&tw[jj * tstep]);
      if (sign > 0) w.y = -w.y;
      const double2 a = z[i0];
      const double2 t = cmul(w, z[i1]);
      z[i0] = cadd(a, t);
      z[i1] = csub(a, t);
    }
    __syncthreads();
  }
}

// X[m] of the real sequence packed in frame f (n = 2^lgn complex values), m in [0, n].
// W^m = e^{-2 pi i m / (2n)} = tw[m * twres / (2n)] for m < n; W^n = -1.
__device__ __forceinline__ double2 rfft_bin(const double2* zf, int lgn, int m, const double2* __restrict__ tw,
                                            int twres) {
  const int n = 1 << lgn;
  const double2 Zm = zf[m & (n - 1)];
  const double2 Zc = cconj(zf[(n - m) & (n - 1)]);
  const double2 E = make_double2(0.5 * (Zm.x + Zc.x), 0.5 * (Zm.y + Zc.y));
  const double2 D = csub(Zm, Zc);
  const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);  // D / (2i)
  double2 W;
  if (m == n) W = make_double2(-1.0, 0.0);
  else W = __ldg(&tw[(int64_t)m * (twres / (2 * n))]);
  return cadd(E, cmul(W, O));
}
