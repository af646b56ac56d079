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

// ---------------------------------------------------------------------------
// Register-blocked Stockham FFT (fp64) for the DGT analysis of M >= 32 (N1).
//
// F frames of n = 2^lgn complex values live in shared memory in natural order at the
// padded index PZ(f n + i) = (f n + i) + ((f n + i) >> 4) (one 16-byte pad per 16 values:
// the stride-16 stores of a radix-16 pass then spread over all banks).  A frame has
// n/16 threads; every pass each thread loads 16 values (16/R butterflies of radix R =
// 2^LGR, butterfly j touching j + r n/R), the CTA synchronises, the butterflies run in
// registers (twiddle e^{-2 pi i r k/(Ns R)}, k = j mod Ns, then an in-register DFT_R)
// and are stored at (j - k) R + k + r Ns (Stockham auto-sort: natural order out, no
// bit reversal).  lgn = 4 p + q: one radix-2^q pass (if q > 0), then p radix-16 passes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int pz(int i) { return i + (i >> 4); }

// e^{-2 pi i t / twres} for 0 <= t < twres from the half-circle table tw (t < twres/2)
__device__ __forceinline__ double2 tw_full(const double2* __restrict__ tw, int t, int twres) {
  const int h = twres >> 1;
  const bool up = t >= h;
  double2 w = __ldg(&tw[up ? t - h : t]);
  w.x = up ? -w.x : w.x;
  w.y = up ? -w.y : w.y;
  return w;
}

__host__ __device__ constexpr int brev_c(int i, int lg) {
  int r = 0;
  for (int b = 0; b < lg; ++b) r |= ((i >> b) & 1) << (lg - 1 - b);
  return r;
}
// cos / sin of 2 pi k / 16
__device__ constexpr double C16[16] = {1.0, 0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,
                                       -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,
                                       -0.92387953251128674, -0.70710678118654757, -0.38268343236508978, 0.0,
                                       0.38268343236508978, 0.70710678118654757, 0.92387953251128674};
__device__ constexpr double S16[16] = {0.0, 0.38268343236508978, 0.70710678118654757, 0.92387953251128674, 1.0,
                                       0.92387953251128674, 0.70710678118654757, 0.38268343236508978, 0.0,
                                       -0.38268343236508978, -0.70710678118654757, -0.92387953251128674, -1.0,
                                       -0.92387953251128674, -0.70710678118654757, -0.38268343236508978};

// in-register DFT of size 2^LGR, natural order in and out, X[r] = sum_q v[q] e^{SIGN 2 pi i q r / R}
template <int LGR, int SIGN>
__device__ __forceinline__ void reg_dft(double2* v) {
  constexpr int R = 1 << LGR;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int j = brev_c(i, LGR);
    if (j > i) {
      const double2 t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
#pragma unroll
  for (int lh = 0; lh < LGR; ++lh) {
    const int half = 1 << lh;
#pragma unroll
    for (int i = 0; i < R / 2; ++i) {
      const int jj = i & (half - 1);
      const int i0 = ((i >> lh) << (lh + 1)) + jj, i1 = i0 + half;
      const int e = jj * (16 >> (lh + 1));   // e^{SIGN 2 pi i jj / (2 half)} = root16^e
      const double2 b = v[i1];
      double2 t;
      if (e == 0) {
        t = b;
      } else if (e == 4) {                   // SIGN i
        t = SIGN < 0 ? make_double2(b.y, -b.x) : make_double2(-b.y, b.x);
      } else {
        const double wr = C16[e], wi = SIGN < 0 ? -S16[e] : S16[e];
        t = make_double2(b.x * wr - b.y * wi, b.x * wi + b.y * wr);
      }
      v[i1] = csub(v[i0], t);
      v[i0] = cadd(v[i0], t);
    }
  }
}

// one Stockham pass of radix 2^LGR over the CTA's frames (all threads; ends with a barrier)
template <int LGR, int SIGN>
__device__ __forceinline__ void stockham_pass(double2* z, int lgn, int lgNs, int lgtpf, const double2* __restrict__ tw,
                                              int twres) {
  constexpr int R = 1 << LGR, B = 16 >> LGR;
  const int f = threadIdx.x >> lgtpf, t = threadIdx.x & ((1 << lgtpf) - 1);
  const int fb = f << lgn;
  const int qstride = 1 << (lgn - LGR);   // n / R
  double2 v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + (b << lgtpf);
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = z[pz(fb + j + r * qstride)];
  }
  __syncthreads();
  const int Ns = 1 << lgNs;
  const int tws = twres >> (lgNs + LGR);    // twres / (Ns R)
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + (b << lgtpf);
    const int k = j & (Ns - 1);
    if (lgNs > 0) {
      // w_r = w_1^r: one table load (w_1; consecutive k are tws entries apart, so every
      // load of the table is its own sector), the powers by squaring and products --
      // at most 4 roundings deep, ~1e-15 relative
      double2 w1 = tw_full(tw, k * tws, twres);
      if (SIGN > 0) w1.y = -w1.y;
      double2 wp[R];
      wp[1] = w1;
#pragma unroll
      for (int r = 2; r < R; ++r) {
        const int hb = 1 << (31 - __clz(r));   // highest power of two in r (compile time)
        wp[r] = r == hb ? cmul(wp[r >> 1], wp[r >> 1]) : cmul(wp[hb], wp[r - hb]);
      }
#pragma unroll
      for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], wp[r]);
    }
    reg_dft<LGR, SIGN>(v[b]);
    const int base = ((j - k) << LGR) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) z[pz(fb + base + r * Ns)] = v[b][r];
  }
  __syncthreads();
}

// the whole transform of every frame of the CTA (n >= 16; n/16 threads per frame)
template <int SIGN>
__device__ __forceinline__ void stockham_fft(double2* z, int lgn, int lgtpf, const double2* __restrict__ tw,
                                             int twres) {
  const int q = lgn & 3;
  int lgNs = 0;
  if (q == 1) stockham_pass<1, SIGN>(z, lgn, 0, lgtpf, tw, twres);
  else if (q == 2) stockham_pass<2, SIGN>(z, lgn, 0, lgtpf, tw, twres);
  else if (q == 3) stockham_pass<3, SIGN>(z, lgn, 0, lgtpf, tw, twres);
  lgNs = q;
  for (; lgNs < lgn; lgNs += 4) stockham_pass<4, SIGN>(z, lgn, lgNs, lgtpf, tw, twres);
}
