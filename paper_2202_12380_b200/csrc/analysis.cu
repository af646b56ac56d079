// analysis.cu -- setup and analysis kernels of libmpgabor (sm_100a):
//   windows (O2 reading Z1/Z2), twiddle/root tables, signal padding + energy,
//   N1 DGT analysis, N2 Gram cross-kernel precompute + threshold +
//   compaction (Eqs. (14)-(17); Eq. (7)), N4 tile-max init.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "launch.h"
#include "fft.cuh"
#include "argmax.cuh"
#include "loopcore.cuh"

// ---------------------------------------------------------------------------
// windows: g(j), j = -floor(gl/2) .. ceil(gl/2)-1, unit norm
// ---------------------------------------------------------------------------
__global__ void window_kernel(int win, int gl, int a, int M, double* __restrict__ g) {
  __shared__ double part[1024];
  const int j0 = -(gl / 2);
  double acc = 0.0;
  for (int i = threadIdx.x; i < gl; i += blockDim.x) {
    const double j = (double)(j0 + i);
    double v;
    if (win == 1) v = 0.5 + 0.5 * cospi(2.0 * j / gl);
    else if (win == 2) v = 0.42 + 0.5 * cospi(2.0 * j / gl) + 0.08 * cospi(4.0 * j / gl);
    else v = exp(-M_PI * j * j / ((double)a * (double)M));
    g[i] = v;
    acc += v * v;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  const double inv = 1.0 / sqrt(part[0]);
  for (int i = threadIdx.x; i < gl; i += blockDim.x) g[i] *= inv;
}

// tw[k] = e^{-2 pi i k / res}, k < res/2 ;  roots[r] = e^{+2 pi i r / R}, r < R
__global__ void tables_kernel(double2* __restrict__ tw, int twres, double2* __restrict__ roots, int R) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < twres / 2) {
    double s, c;
    sincospi(-2.0 * (double)i / (double)twres, &s, &c);
    tw[i] = make_double2(c, s);
  }
  if (i < R) {
    double s, c;
    sincospi(2.0 * (double)i / (double)R, &s, &c);
    roots[i] = make_double2(c, s);
  }
}

// ---------------------------------------------------------------------------
// padding, finiteness and E0 = ||x||^2 (Alg. 1 init); deterministic
// two-stage reduction (fixed block partition, fixed tree order)
// ---------------------------------------------------------------------------
__global__ void pad_energy_kernel(const double* __restrict__ x, int64_t Ls, double* __restrict__ xp, int64_t L,
                                  double* __restrict__ partial, int* __restrict__ nonfinite) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L; i += (int64_t)gridDim.x * blockDim.x) {
    double v = i < Ls ? x[i] : 0.0;
    if (!isfinite(v)) { *nonfinite = 1; v = 0.0; }
    xp[i] = v;
    acc += v * v;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int n, double* __restrict__ out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ---------------------------------------------------------------------------
// N1 DGT: c(m,n) = sum_j x(na+j) g(j) e^{-2 pi i m j/M}, m = 0..M/2 (Eq. (3)),
// frames folded mod M then one real FFT of length M per frame in shared memory.
// F frames per CTA.  Output row stride `stride` (>= M/2+1, zero padded).
// ---------------------------------------------------------------------------
template <typename R>
__global__ void __launch_bounds__(1024) dgt_kernel(const double* __restrict__ x, int64_t L, int a, int M, int gl, int N,
                                                   const double* __restrict__ g, const double2* __restrict__ tw,
                                                   int twres, typename cplx<R>::t* __restrict__ out, int stride, int F,
                                                   uint32_t stride_magic) {
  using C2 = typename cplx<R>::t;
  extern __shared__ double2 z[];
  const int n = M / 2;
  const int lgn = 31 - __clz(n), lgM = lgn + 1;
  const int j0 = -(gl / 2);
  const int frame0 = blockIdx.x * F;
  // fold the windowed frame modulo M (M a power of two: masks, no integer division;
  // sample positions wrap circularly by one conditional add / subtract of L)
  for (int idx = threadIdx.x; idx < F << lgM; idx += blockDim.x) {
    const int f = idx >> lgM, s = idx & (M - 1);
    const int frame = frame0 + f;
    double v = 0.0;
    if (frame < N) {
      const int64_t base = (int64_t)frame * a;
      for (int j = j0 + ((s - j0) & (M - 1)); j < j0 + gl; j += M) {
        int64_t pos = base + j;
        pos += pos < 0 ? L : 0;
        pos -= pos >= L ? L : 0;
        v += x[pos] * g[j - j0];
      }
    }
    double* zz = reinterpret_cast<double*>(&z[f * n + bitrev(s >> 1, lgn)]);
    zz[s & 1] = v;
  }
  __syncthreads();
  smem_fft(z, lgn, F, tw, twres, -1);
  // row f of the output: bins 0..n, then zero padding up to the row stride;
  // f = idx / stride by a multiply-high with the host's magic (exact for idx < 2^16)
  for (int idx = threadIdx.x; idx < F * stride; idx += blockDim.x) {
    const int f = (int)__umulhi((uint32_t)idx, stride_magic), m = idx - f * stride;
    const int frame = frame0 + f;
    if (frame >= N) continue;
    C2 o;
    if (m <= n) {
      const double2 X = rfft_bin(z + f * n, lgn, m, tw, twres);
      o.x = (R)X.x;
      o.y = (R)X.y;
    } else {
      o.x = 0;
      o.y = 0;
    }
    out[(int64_t)frame * stride + m] = o;
  }
}

// The same analysis for M >= 32 with the register-blocked Stockham FFT (fft.cuh):
// n/16 threads per frame, F frames per CTA, the frames in natural order at padded
// shared-memory indices (no bit reversal, conflict-free radix-16 stores); the output
// rows of the CTA's frames are contiguous in `out`, written by consecutive threads.
template <typename R>
__global__ void __launch_bounds__(512) dgt_stockham_kernel(const double* __restrict__ x, int64_t L, int a, int M, int gl,
                                                           int N, const double* __restrict__ g,
                                                           const double2* __restrict__ tw, int twres,
                                                           typename cplx<R>::t* __restrict__ out, int stride, int F,
                                                           uint32_t stride_magic, int write_pad) {
  using C2 = typename cplx<R>::t;
  extern __shared__ double2 z[];
  const int n = M / 2;
  const int lgn = 31 - __clz(n), lgM = lgn + 1;
  const int lgtpf = lgn - 4;
  const int j0 = -(gl / 2);
  const int frame0 = blockIdx.x * F;
  double* zd = reinterpret_cast<double*>(z);
  // the post-processing twiddles W^m = e^{-2 pi i m/M}, m < n: consecutive m lie twstep
  // table entries apart; for twstep >= 4 (scattered loads) they are staged in shared
  // memory behind the frames, one table load per CTA instead of one per output
  const int twstep = twres / (2 * n);
  double2* wt = z + (F * n + ((F * n) >> 4));
  const bool use_wt = twstep >= 4;
  if (use_wt)
    for (int m = threadIdx.x; m < n; m += blockDim.x) wt[m] = __ldg(&tw[(int64_t)m * twstep]);
  // windowed frame folded modulo M, natural order: sample s -> value s >> 1, part s & 1
  if (gl <= M) {  // one window sample per s: UF independent loads in flight per thread
    constexpr int UF = 8;
    const int total = F << lgM;
    for (int i0 = threadIdx.x; i0 < total; i0 += UF * blockDim.x) {
      double xv[UF], gv[UF];
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        const int idx = i0 + u * blockDim.x;
        const int f = idx >> lgM, s = idx & (M - 1);
        const int frame = frame0 + f;
        const int j = j0 + ((s - j0) & (M - 1));
        const bool ok = idx < total && frame < N && j < j0 + gl;
        int64_t pos = (int64_t)frame * a + j;
        pos += pos < 0 ? L : 0;
        pos -= pos >= L ? L : 0;
        xv[u] = ok ? __ldg(&x[pos]) : 0.0;
        gv[u] = ok ? __ldg(&g[j - j0]) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UF; ++u) {
        const int idx = i0 + u * blockDim.x;
        if (idx < total) zd[2 * pz(idx >> 1) + (idx & 1)] = xv[u] * gv[u];
      }
    }
  } else {
    for (int idx = threadIdx.x; idx < F << lgM; idx += blockDim.x) {
      const int f = idx >> lgM, s = idx & (M - 1);
      const int frame = frame0 + f;
      double v = 0.0;
      if (frame < N) {
        const int64_t base = (int64_t)frame * a;
        for (int j = j0 + ((s - j0) & (M - 1)); j < j0 + gl; j += M) {
          int64_t pos = base + j;
          pos += pos < 0 ? L : 0;
          pos -= pos >= L ? L : 0;
          v += x[pos] * g[j - j0];
        }
      }
      zd[2 * pz(idx >> 1) + (s & 1)] = v;
    }
  }
  __syncthreads();
  stockham_fft<-1>(z, lgn, lgtpf, tw, twres);
  // X[m] = E[m] + W^m O[m] (fft.cuh rfft_bin), rows of the CTA's frames back to back
  const int64_t o0 = (int64_t)frame0 * stride;
  const int nval = min(F, N - frame0) * stride;
  constexpr int UO = 4;   // outputs per thread per batch: their twiddle loads in flight together
  for (int i0 = threadIdx.x; i0 < nval; i0 += UO * blockDim.x) {
    double2 Wv[UO];
    int mv[UO], fv[UO];
#pragma unroll
    for (int u = 0; u < UO; ++u) {
      const int idx = i0 + u * blockDim.x;
      const int f = (int)__umulhi((uint32_t)idx, stride_magic), m = idx - f * stride;
      fv[u] = f;
      mv[u] = idx < nval ? m : INT_MAX;
      Wv[u] = (idx < nval && m < n) ? (use_wt ? wt[m] : __ldg(&tw[(int64_t)m * twstep])) : make_double2(-1.0, 0.0);  // W^n = -1
    }
#pragma unroll
    for (int u = 0; u < UO; ++u) {
      const int idx = i0 + u * blockDim.x, m = mv[u];
      if (m == INT_MAX) continue;
      C2 o;
      if (m <= n) {
        const int fb = fv[u] << lgn;
        const double2 Zm = z[pz(fb + (m & (n - 1)))];
        const double2 Zn = z[pz(fb + ((n - m) & (n - 1)))];
        const double2 Zc = cconj(Zn);
        const double2 E = make_double2(0.5 * (Zm.x + Zc.x), 0.5 * (Zm.y + Zc.y));
        const double2 D = csub(Zm, Zc);
        const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
        const double2 X = cadd(E, cmul(Wv[u], O));
        o.x = (R)X.x;
        o.y = (R)X.y;
      } else {
        if (!write_pad) continue;
        o.x = 0;
        o.y = 0;
      }
      out[o0 + idx] = o;
    }
  }
}

// ---------------------------------------------------------------------------
// The same analysis with the frame size a compile-time constant (n = 2^LGN complex
// points, M = 2n, LGN = 4..13) for the common window shape gl <= M, gl % 4 == 0, a even
// (every configuration of the paper and C0-C4).  The profile of the runtime-size kernel
// above (profiles/r02an_dgt_sass_mix.md) spent 39 % of its instructions folding the
// frame into shared memory and 43 % on the post-processing, almost all of it integer
// index arithmetic; here
//  * the fold is fused into the first Stockham pass: the pass's 16 inputs per thread,
//    z[i] = (x_w[2i], x_w[2i+1]), are read straight from the signal as 16-byte pairs
//    (gl % 4 == 0 and a even keep each pair adjacent, aligned and inside one window
//    period), multiplied by the window pair and transformed in registers -- no
//    shared-memory round trip and no barrier;
//  * every index of the passes is a compile-time offset from one per-thread base;
//  * the post-processing produces X[m] and X[n-m] from one pair of shared loads:
//    with T = W^m O[m], X[m] = E[m] + T and X[n-m] = conj(E[m] - T)
//    (E[n-m] = conj E[m], O[n-m] = conj O[m], W^{n-m} = -conj W^m).
// ---------------------------------------------------------------------------
template <int LGN>
struct DgtC {
  static constexpr int n = 1 << LGN, M = 2 * n;
  static constexpr int LGTPF = LGN - 4, TPF = 1 << LGTPF;   // threads per frame (16 values each)
  static constexpr int Q = LGN & 3;                         // first pass radix 2^Q (16 if Q == 0)
  static constexpr int LGR0 = Q ? Q : 4;
};

// one compile-time Stockham pass (LGNS > 0: after the first), radix 2^LGR, as stockham_pass
template <int LGN, int LGR, int LGNS, int SIGN>
__device__ __forceinline__ void spass_ct(double2* z, int fb, int t, const double2* __restrict__ tw, int twres) {
  constexpr int R = 1 << LGR, B = 16 >> LGR, TPF = DgtC<LGN>::TPF;
  constexpr int QS = 1 << (LGN - LGR), NS = 1 << LGNS;
  double2 v[B][R];
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + b * TPF;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b][r] = z[pz(fb + j + r * QS)];
  }
  __syncthreads();
  const int tws = twres >> (LGNS + LGR);
#pragma unroll
  for (int b = 0; b < B; ++b) {
    const int j = t + b * TPF;
    const int k = j & (NS - 1);
    double2 w1 = tw_full(tw, k * tws, twres);
    if (SIGN > 0) w1.y = -w1.y;
    double2 wp[R];
    wp[1] = w1;
#pragma unroll
    for (int r = 2; r < R; ++r) {
      const int hb = 1 << (31 - __clz(r));
      wp[r] = r == hb ? cmul(wp[r >> 1], wp[r >> 1]) : cmul(wp[hb], wp[r - hb]);
    }
#pragma unroll
    for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], wp[r]);
    reg_dft<LGR, SIGN>(v[b]);
    const int base = ((j - k) << LGR) + k;
#pragma unroll
    for (int r = 0; r < R; ++r) z[pz(fb + base + r * NS)] = v[b][r];
  }
  __syncthreads();
}

template <int LGN, int LGNS>
__device__ __forceinline__ void spass_rest(double2* z, int fb, int t, const double2* __restrict__ tw, int twres) {
  if constexpr (LGNS < LGN) {
    spass_ct<LGN, 4, LGNS, -1>(z, fb, t, tw, twres);
    spass_rest<LGN, LGNS + 4>(z, fb, t, tw, twres);
  }
}

#ifndef MPG_DGT_STAGE
#define MPG_DGT_STAGE 0   // 1: the CTA's signal range staged by a TMA bulk copy (measured slower)
#endif
#ifndef MPG_DGT_THREADS
#define MPG_DGT_THREADS 128   // threads per CTA (at least one frame: n/16 threads)
#endif
#ifndef MPG_DGT_MINB
#define MPG_DGT_MINB 5   // resident CTAs per SM the register allocation targets (<= 102 registers)
#endif
template <int LGN>
constexpr int dgt_ct_threads() { return DgtC<LGN>::TPF > MPG_DGT_THREADS ? DgtC<LGN>::TPF : MPG_DGT_THREADS; }
template <int LGN>
constexpr int dgt_ct_minb() { return dgt_ct_threads<LGN>() > MPG_DGT_THREADS ? 1 : MPG_DGT_MINB; }
template <typename R, int LGN>
__global__ void __launch_bounds__(dgt_ct_threads<LGN>(), dgt_ct_minb<LGN>()) dgt_ct_kernel(
    const double* __restrict__ x, int64_t L, int a, int gl, int N, const double* __restrict__ g,
    const double2* __restrict__ tw, int twres, typename cplx<R>::t* __restrict__ out, int stride, int write_pad) {
  using C2 = typename cplx<R>::t;
  using S = DgtC<LGN>;
  constexpr int n = S::n, M = S::M, TPF = S::TPF, LGR0 = S::LGR0;
  constexpr int R0 = 1 << LGR0, B0 = 16 >> LGR0, QS0 = n >> LGR0;
  extern __shared__ double2 z[];
  const int F = blockDim.x >> S::LGTPF;
  const int f = threadIdx.x >> S::LGTPF, t = threadIdx.x & (TPF - 1);
  const int frame = blockIdx.x * F + f;
  const int fb = f << LGN;
  // post-processing twiddles W^m, m < n/2 + 1, staged in shared memory when the table
  // entries are scattered (twstep >= 4)
  const int twstep = twres / M;
  double2* wt = z + (F * n + ((F * n) >> 4));
  const bool use_wt = twstep >= 4;
  if (use_wt)
    for (int m = threadIdx.x; m <= n / 2; m += blockDim.x) wt[m] = __ldg(&tw[(int64_t)m * twstep]);
  // ---- first pass (Ns = 1, no twiddles), inputs from the signal ----
  // The CTA's signal range [frame0 a + j0, (frame0 + F - 1) a + j0 + M) (its frames
  // overlap M/a-fold) is staged into the frame buffer by one TMA bulk copy
  // (cp.async.bulk, completion on an mbarrier) when it does not wrap around the signal
  // ends; each sample then leaves HBM/L2 once per CTA instead of M/a times through L1.
  // The pass's inputs are taken into registers before the barrier after which its
  // outputs overwrite the staged signal.  Wrapping CTAs (the first and the last) load
  // from global memory with the circular index.
  {
    const int j0 = -(gl >> 1);
    const int frame0 = blockIdx.x * F;
    const int nfr = min(F, N - frame0);
    const int64_t lo = (int64_t)frame0 * a + j0;
    const int64_t cnt = (int64_t)(nfr - 1) * a + M;   // doubles (even: 16-byte multiple)
    const bool staged = MPG_DGT_STAGE && lo >= 0 && lo + cnt <= L;    // (uniform over the CTA)
    __shared__ alignas(8) unsigned long long xbar;
    if (staged) {
      if (threadIdx.x == 0) {
        mpcore::mbar_init(mpcore::smem_addr(&xbar), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mpcore::mbar_arm(mpcore::smem_addr(&xbar), (uint32_t)(cnt * 8));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         mpcore::smem_addr(z)),
                     "l"(x + lo), "r"((uint32_t)(cnt * 8)), "r"(mpcore::smem_addr(&xbar))
                     : "memory");
      }
      __syncthreads();
      mpcore::mbar_wait(mpcore::smem_addr(&xbar), 0);
    }
    const int64_t base = (int64_t)min(frame, N - 1) * a;
    const bool fok = frame < N;
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* xs = reinterpret_cast<const double2*>(z) + ((f * a) >> 1);   // staged frame f
    const double2* g2 = reinterpret_cast<const double2*>(g);
    double2 v[B0][R0];
#pragma unroll
    for (int b = 0; b < B0; ++b) {
      const int j = t + b * TPF;
#pragma unroll
      for (int r = 0; r < R0; ++r) {
        const int i = j + r * QS0;
        const int jw = (2 * i - j0) & (M - 1);     // window index of sample 2i (even)
        const bool ok = fok && jw < gl;
        double2 xv;
        if (staged) {
          xv = ok ? xs[jw >> 1] : make_double2(0.0, 0.0);
        } else {
          int64_t pos = base + j0 + jw;
          pos += pos < 0 ? L : 0;
          pos -= pos >= L ? L : 0;
          xv = ok ? __ldg(&x2[pos >> 1]) : make_double2(0.0, 0.0);
        }
        const double2 gv = ok ? __ldg(&g2[jw >> 1]) : make_double2(0.0, 0.0);
        v[b][r] = make_double2(xv.x * gv.x, xv.y * gv.y);
      }
    }
    __syncthreads();   // every input is in registers: the staged signal may be overwritten
#pragma unroll
    for (int b = 0; b < B0; ++b) {
      const int j = t + b * TPF;
      reg_dft<LGR0, -1>(v[b]);
#pragma unroll
      for (int r = 0; r < R0; ++r) z[pz(fb + (j << LGR0) + r)] = v[b][r];
    }
    __syncthreads();
  }
  spass_rest<LGN, LGR0>(z, fb, t, tw, twres);
  // ---- X[m], X[n-m] for m = t + k TPF < n/2; X[n/2] by thread 0; zero padding ----
  if (frame >= N) return;
  C2* orow = out + (int64_t)frame * stride;
  const double2* zf = z + pz(fb);   // (fb is a multiple of 16: pz(fb + i) = pz(fb) + pz(i))
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int m = t + k * TPF;
    const double2 Zm = zf[pz(m)];
    const double2 Zc = cconj(zf[pz((n - m) & (n - 1))]);
    const double2 E = make_double2(0.5 * (Zm.x + Zc.x), 0.5 * (Zm.y + Zc.y));
    const double2 D = csub(Zm, Zc);
    const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
    const double2 W = use_wt ? wt[m] : __ldg(&tw[(int64_t)m * twstep]);
    const double2 T = cmul(W, O);
    C2 o1, o2;
    o1.x = (R)(E.x + T.x);
    o1.y = (R)(E.y + T.y);
    o2.x = (R)(E.x - T.x);
    o2.y = (R)(T.y - E.y);
    orow[m] = o1;
    orow[n - m] = o2;
  }
  if (t == 0) {
    const int m = n / 2;
    const double2 Zm = zf[pz(m)];
    const double2 Zc = cconj(Zm);
    const double2 E = make_double2(0.5 * (Zm.x + Zc.x), 0.5 * (Zm.y + Zc.y));
    const double2 D = csub(Zm, Zc);
    const double2 O = make_double2(0.5 * D.y, -0.5 * D.x);
    const double2 W = use_wt ? wt[m] : __ldg(&tw[(int64_t)m * twstep]);
    const double2 X = cadd(E, cmul(W, O));
    C2 o;
    o.x = (R)X.x;
    o.y = (R)X.y;
    orow[m] = o;
  }
  if (write_pad)
    for (int m = n + 1 + t; m < stride; m += TPF) {
      C2 o;
      o.x = 0;
      o.y = 0;
      orow[m] = o;
    }
}

template <typename R, int LGN>
static cudaError_t launch_dgt_ct(const double* xp, int64_t L, const DictGeo& d, const double* g, const double2* tw,
                                 int twres, typename cplx<R>::t* out, cudaStream_t st, int write_pad) {
  using S = DgtC<LGN>;
  const int threads = dgt_ct_threads<LGN>();
  const int F = threads / S::TPF;
  const int n = S::n;
  const bool use_wt = twres / S::M >= 4;
  const size_t smem = (size_t)(F * n + (F * n) / 16 + (use_wt ? n / 2 + 1 : 0)) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    // (<= 140 KB for every LGN; the kernel has 16 bytes of static shared memory besides)
    CUDA_OK(cudaFuncSetAttribute(dgt_ct_kernel<R, LGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    attr = true;
  }
  dgt_ct_kernel<R, LGN><<<(d.N + F - 1) / F, threads, smem, st>>>(xp, L, d.a, d.gl, d.N, g, tw, twres, out, d.stride,
                                                                  write_pad);
  return cudaGetLastError();
}

// the compile-time kernel applies: gl <= M, gl % 4 == 0, a even, 16-byte aligned x and g
static bool dgt_ct_applies(const double* xp, const DictGeo& d, const double* g) {
  return d.M >= 32 && d.M <= 16384 && d.gl <= d.M && d.gl % 4 == 0 && d.a % 2 == 0 &&
         ((uintptr_t)xp & 15) == 0 && ((uintptr_t)g & 15) == 0;
}

template <typename R>
static cudaError_t launch_dgt_ct_any(const double* xp, int64_t L, const DictGeo& d, const double* g,
                                     const double2* tw, int twres, typename cplx<R>::t* out, cudaStream_t st,
                                     int write_pad) {
  switch (31 - __builtin_clz((unsigned)d.M / 2)) {
    case 4: return launch_dgt_ct<R, 4>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 5: return launch_dgt_ct<R, 5>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 6: return launch_dgt_ct<R, 6>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 7: return launch_dgt_ct<R, 7>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 8: return launch_dgt_ct<R, 8>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 9: return launch_dgt_ct<R, 9>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 10: return launch_dgt_ct<R, 10>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 11: return launch_dgt_ct<R, 11>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 12: return launch_dgt_ct<R, 12>(xp, L, d, g, tw, twres, out, st, write_pad);
    case 13: return launch_dgt_ct<R, 13>(xp, L, d, g, tw, twres, out, st, write_pad);
    default: return cudaErrorInvalidValue;
  }
}

// ---------------------------------------------------------------------------
// N2 kernel rows: for lag nu = nu_first + blockIdx.x
//   b[s mod M_c] += g_u(s + nu a_c) g_v(s),  H[i][m] = sum_s b e^{-2 pi i m s/M_c}, m = 0..M_c/2
// i.e. h_{u,v}(m, nu) for m >= 0 (h(-m,nu) = conj h(m,nu), real windows).
// ---------------------------------------------------------------------------
__global__ void kern_rows_kernel(int a_c, int M_c, int nu_first, const double* __restrict__ gu, int glu,
                                 const double* __restrict__ gv, int glv, const double2* __restrict__ tw,
                                 int twres, double2* __restrict__ H) {
  extern __shared__ double2 z[];
  const int n = M_c / 2;
  const int lgn = 31 - __clz(n);
  const int nu = nu_first + blockIdx.x;
  const int ju0 = -(glu / 2), ju1 = ju0 + glu - 1;
  const int jv0 = -(glv / 2), jv1 = jv0 + glv - 1;
  const int slo = max(jv0, ju0 - nu * a_c), shi = min(jv1, ju1 - nu * a_c);
  for (int r = threadIdx.x; r < M_c; r += blockDim.x) {
    double v = 0.0;
    if (slo <= shi)
      for (int s = slo + fmod32(r - slo, M_c); s <= shi; s += M_c) v += gu[s + nu * a_c - ju0] * gv[s - jv0];
    double* zz = reinterpret_cast<double*>(&z[bitrev(r >> 1, lgn)]);
    zz[r & 1] = v;
  }
  __syncthreads();
  smem_fft(z, lgn, 1, tw, twres, -1);
  double2* row = H + (int64_t)blockIdx.x * (n + 1);
  for (int m = threadIdx.x; m <= n; m += blockDim.x) row[m] = rfft_bin(z, lgn, m, tw, twres);
}

__device__ __forceinline__ double cabs2(double2 v) { return sqrt(v.x * v.x + v.y * v.y); }

// max |h| over the pair (order independent: max of non-negative doubles via their bit patterns)
__global__ void kern_max_kernel(const double2* __restrict__ H, int64_t count, unsigned long long* __restrict__ mx) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, cabs2(H[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, (unsigned long long)__double_as_longlong(m));
}

// bounding box of entries with |h| > thr * max (strict, relative; Z5-Z7), signed mu in (-M_c/2, M_c/2]
// box[0..3] = mu_lo, mu_hi, nu_lo, nu_hi (init to +inf,-inf,+inf,-inf); box[4] += kept count
__global__ void kern_box_kernel(const double2* __restrict__ H, int nlag, int M_c, int nu_first, double thr,
                                const unsigned long long* __restrict__ mxp, int* __restrict__ box) {
  const int n = M_c / 2;
  const double lim = thr * __longlong_as_double((long long)*mxp);
  const int64_t count = (int64_t)nlag * (n + 1);
  int mlo = INT_MAX, mhi = INT_MIN, nlo = INT_MAX, nhi = INT_MIN, kept = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    if (cabs2(H[i]) > lim) {
      const int row = (int)(i / (n + 1)), m = (int)(i - (int64_t)row * (n + 1));
      const int nu = nu_first + row;
      const bool mirror = (m > 0 && m < n);
      mhi = max(mhi, m);
      mlo = min(mlo, mirror ? -m : m);
      nlo = min(nlo, nu);
      nhi = max(nhi, nu);
      kept += mirror ? 2 : 1;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mlo = min(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
    mhi = max(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
    nlo = min(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
    nhi = max(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
    kept += __shfl_xor_sync(0xffffffffu, kept, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&box[0], mlo);
    atomicMax(&box[1], mhi);
    atomicMin(&box[2], nlo);
    atomicMax(&box[3], nhi);
    atomicAdd(&box[4], kept);
  }
}

// Compact the box into the per-alignment-class layout of PairGeo:
// class (on, om) = (i_nu mod s_n, i_mu mod s_m) holds rows i_nu = on + r s_n and
// columns i_mu = om + c s_m as a contiguous [nr(on)][nc(om)] block at
// koff + cnt_lt(on) * nmu + nr(on) * cnt_lt(om).  Sub-threshold entries are 0.
// Also writes the fp64 box copy (row-major [nu][mu]) used by parity tests and
// the fp64 conjugate-pair row (nu = 0) when u == v.
template <typename R>
__global__ void kern_compact_kernel(const double2* __restrict__ H, int M_c, int nu_first, double thr,
                                    const unsigned long long* __restrict__ mxp, PairGeo pg,
                                    typename cplx<R>::t* __restrict__ kern, double2* __restrict__ boxcopy,
                                    RhoEnt* __restrict__ rho_row) {
  using C2 = typename cplx<R>::t;
  const int n = M_c / 2;
  const double lim = thr * __longlong_as_double((long long)*mxp);
  const int64_t count = (int64_t)pg.nmu * pg.nnu;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int inu = (int)(i / pg.nmu), imu = (int)(i - (int64_t)inu * pg.nmu);
    const int mu = pg.mu_lo + imu, nu = pg.nu_lo + inu;
    const int m = mu < 0 ? -mu : mu;
    double2 v = H[(int64_t)(nu - nu_first) * (n + 1) + m];
    if (mu < 0) v.y = -v.y;
    if (!(cabs2(v) > lim)) v = make_double2(0.0, 0.0);
    const int on = inu % pg.s_n, r = inu / pg.s_n;
    const int om = imu % pg.s_m, c = imu / pg.s_m;
    const int nr = cnt_eq(on, pg.nnu, pg.s_n), nc = cnt_eq(om, pg.nmu, pg.s_m);
    const int64_t dst = pg.koff + (int64_t)cnt_lt(on, pg.nnu, pg.s_n) * pg.nmu +
                        (int64_t)nr * cnt_lt(om, pg.nmu, pg.s_m) + (int64_t)r * nc + c;
    C2 o;
    o.x = (R)v.x;
    o.y = (R)v.y;
    kern[dst] = o;
    if (boxcopy) boxcopy[i] = v;
    if (rho_row && nu == 0) {
      RhoEnt e;
      e.re = v.x;
      e.im = v.y;
      e.inv = 1.0 / (1.0 - (v.x * v.x + v.y * v.y));
      e.pad_ = 0.0;
      rho_row[imu] = e;
    }
  }
}

// ---------------------------------------------------------------------------
// N4 init: one warp per tile computes the tile record (best |c|^2, lowest index)
// and stores it at rec[(g % C) * Lc + g / C] (CTA-major slices of the loop kernel).
// ---------------------------------------------------------------------------
template <typename R, int TW>
__global__ void tile_init_kernel(const typename cplx<R>::t* __restrict__ grid, const DictGeo* __restrict__ dg,
                                 const OwnGeo* __restrict__ own, int W, int64_t total, int C, int64_t Lc,
                                 Rec<R>* __restrict__ rec, SelScore sel) {
  // tile g of dictionary v, frame n goes to its owner CTA c = (frame_off_v + n) mod C,
  // local index loc_base(c,v) + ((n - n_first(c,v)) / C) * T_v + t (frame-major)
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g < total; g += nwarps) {
    Rec<R> best = empty_rec(R(0));
    int64_t dst;
    {
      int v = 0;
      while (v + 1 < W && dg[v + 1].tile_off <= g) ++v;
      const DictGeo d = dg[v];
      const int64_t loc = g - d.tile_off;
      const int64_t n = loc / d.T;
      const int t = (int)(loc - n * d.T);
      const int c = (int)((d.frame_off + n) % C);
      const OwnGeo o = own[c * W + v];
      dst = (int64_t)c * Lc + o.loc_base + ((n - o.n_first) / C) * d.T + t;
      const typename cplx<R>::t* row = grid + d.grid_off + n * d.stride;
#pragma unroll
      for (int ch = 0; ch < TW / 32; ++ch) {
        const int b = t * TW + ch * 32 + lane;
        if (b < d.MR) {
          const typename cplx<R>::t c = row[b];
          // selection score (mpcore::sel_score: |c|^2, or the pedantic Eq. (20) energy)
          const R s = sel.pedantic ? mpcore::sel_score<R>(c.x, c.y, b, d.M, true, sel.rho + sel.rho_meta[2 * W + v],
                                                          sel.rho_meta[v], sel.rho_meta[W + v])
                                   : mpcore::sel_score<R>(c.x, c.y, b, d.M, false, nullptr, 0, 0);
          const uint32_t p = (uint32_t)(d.off + n * d.MR + b);
          if (better(s, p, best.s, best.p)) {
            best.s = s;
            best.p = p;
            best.re = c.x;
            best.im = c.y;
          }
        }
      }
    }
    best = warp_best(best);
    if (lane == 0) rec[dst] = best;
  }
}

// empty records in every slot (run before tile_init_kernel: slices are padded to Lc)
template <typename R>
__global__ void rec_clear_kernel(Rec<R>* __restrict__ rec, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    rec[i] = empty_rec(R(0));
}

// residual export: padded grid (cplx<R>) -> complex double in global index order p
template <typename R>
__global__ void grid_export_kernel(const typename cplx<R>::t* __restrict__ grid, const DictGeo* __restrict__ dg,
                                   int W, int64_t P, double2* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    int v = 0;
    while (v + 1 < W && dg[v + 1].off <= p) ++v;
    const DictGeo d = dg[v];
    const int64_t q = p - d.off;
    const int64_t n = q / d.MR;
    const int64_t m = q - n * d.MR;
    const typename cplx<R>::t c = grid[d.grid_off + n * d.stride + m];
    out[p] = make_double2((double)c.x, (double)c.y);
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_window(int win, int gl, int a, int M, double* g, cudaStream_t st) {
  window_kernel<<<1, 1024, 0, st>>>(win, gl, a, M, g);
  return cudaGetLastError();
}

cudaError_t launch_tables(double2* tw, int twres, double2* roots, int R, cudaStream_t st) {
  const int n = max(twres / 2, R);
  tables_kernel<<<(n + 255) / 256, 256, 0, st>>>(tw, twres, roots, R);
  return cudaGetLastError();
}

cudaError_t launch_pad_energy(const double* x, int64_t Ls, double* xp, int64_t L, double* partial,
                              int* nonfinite, double* E0, cudaStream_t st) {
  pad_energy_kernel<<<256, 256, 0, st>>>(x, Ls, xp, L, partial, nonfinite);
  sum_partials_kernel<<<1, 256, 0, st>>>(partial, 256, E0);
  return cudaGetLastError();
}

// frames per CTA: 4096 complex values of shared memory (64 KB) per CTA, threads up to
// 1024 so that a large-M transform (one frame) still has every SM busy
static int dgt_frames_per_cta(int M) { return max(1, 4096 / (M / 2)); }

template <typename R>
cudaError_t launch_dgt(const double* xp, int64_t L, const DictGeo& d, const double* g, const double2* tw,
                       int twres, typename cplx<R>::t* out, cudaStream_t st, int write_pad) {
  // the compile-time-size kernel where it applies (MPGABOR_DGT_RT=1: the runtime-size
  // kernels below, kept for every other window shape and as the tests' second path)
  const char* rt = std::getenv("MPGABOR_DGT_RT");
  if (!(rt != nullptr && rt[0] == '1') && dgt_ct_applies(xp, d, g))
    return launch_dgt_ct_any<R>(xp, L, d, g, tw, twres, out, st, write_pad);
  if (d.M >= 32) {  // Stockham: n/16 threads per frame, >= 256 threads per CTA
    const int tpf = d.M / 32;
    int F = std::max(1, 256 / tpf);
    while (F > 1 && (int64_t)F * d.stride >= (1 << 16)) F >>= 1;
    if ((int64_t)F * d.stride >= (1 << 16)) return cudaErrorInvalidValue;
    const int n = d.M / 2;
    const bool use_wt = twres / d.M >= 4;   // (twstep = twres / (2n))
    const size_t smem = (size_t)(F * n + (F * n) / 16 + (use_wt ? n : 0)) * sizeof(double2);
    static bool attr_s = false;
    if (!attr_s) {
      CUDA_OK(cudaFuncSetAttribute(dgt_stockham_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr_s = true;
    }
    const uint32_t magic = (uint32_t)((0x100000000ull + (uint64_t)d.stride - 1) / (uint64_t)d.stride);
    dgt_stockham_kernel<R><<<(d.N + F - 1) / F, F * tpf, smem, st>>>(xp, L, d.a, d.M, d.gl, d.N, g, tw, twres, out,
                                                                      d.stride, F, magic, write_pad);
    return cudaGetLastError();
  }
  // (F * stride < 2^16 keeps the output row index by multiply-high exact)
  const int F = std::max(1, std::min(dgt_frames_per_cta(d.M), 65535 / d.stride));
  const size_t smem = (size_t)F * (d.M / 2) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    CUDA_OK(cudaFuncSetAttribute(dgt_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  if ((int64_t)F * d.stride >= (1 << 16)) return cudaErrorInvalidValue;
  const uint32_t magic = (uint32_t)((0x100000000ull + (uint64_t)d.stride - 1) / (uint64_t)d.stride);
  const int threads = (int64_t)F * (d.M / 2) >= 8192 ? 1024 : 512;
  dgt_kernel<R><<<(d.N + F - 1) / F, threads, smem, st>>>(xp, L, d.a, d.M, d.gl, d.N, g, tw, twres, out, d.stride, F,
                                                          magic);
  return cudaGetLastError();
}
template cudaError_t launch_dgt<double>(const double*, int64_t, const DictGeo&, const double*, const double2*, int,
                                        double2*, cudaStream_t, int);
template cudaError_t launch_dgt<float>(const double*, int64_t, const DictGeo&, const double*, const double2*, int,
                                       float2*, cudaStream_t, int);

cudaError_t launch_kern_rows(int a_c, int M_c, int nu_first, int nlag, const double* gu, int glu, const double* gv,
                             int glv, const double2* tw, int twres, double2* H, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    CUDA_OK(cudaFuncSetAttribute(kern_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const size_t smem = (size_t)(M_c / 2) * sizeof(double2);
  kern_rows_kernel<<<nlag, 512, smem, st>>>(a_c, M_c, nu_first, gu, glu, gv, glv, tw, twres, H);
  return cudaGetLastError();
}

cudaError_t launch_kern_max_box(const double2* H, int nlag, int M_c, int nu_first, double thr,
                                unsigned long long* mx, int* box, cudaStream_t st) {
  const int64_t count = (int64_t)nlag * (M_c / 2 + 1);
  const int blocks = (int)std::min<int64_t>(1184, (count + 255) / 256);
  kern_max_kernel<<<blocks, 256, 0, st>>>(H, count, mx);
  kern_box_kernel<<<blocks, 256, 0, st>>>(H, nlag, M_c, nu_first, thr, mx, box);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_kern_compact(const double2* H, int M_c, int nu_first, double thr, const unsigned long long* mx,
                                const PairGeo& pg, typename cplx<R>::t* kern, double2* boxcopy, RhoEnt* rho_row,
                                cudaStream_t st) {
  const int64_t count = (int64_t)pg.nmu * pg.nnu;
  const int blocks = (int)std::min<int64_t>(1184, (count + 255) / 256);
  kern_compact_kernel<R><<<blocks, 256, 0, st>>>(H, M_c, nu_first, thr, mx, pg, kern, boxcopy, rho_row);
  return cudaGetLastError();
}
template cudaError_t launch_kern_compact<double>(const double2*, int, int, double, const unsigned long long*,
                                                 const PairGeo&, double2*, double2*, RhoEnt*, cudaStream_t);
template cudaError_t launch_kern_compact<float>(const double2*, int, int, double, const unsigned long long*,
                                                const PairGeo&, float2*, double2*, RhoEnt*, cudaStream_t);

template <typename R>
cudaError_t launch_tile_init(const typename cplx<R>::t* grid, const DictGeo* dg, const OwnGeo* own, int W,
                             int64_t total, int C, int64_t Lc, int TW, Rec<R>* rec, SelScore sel, cudaStream_t st) {
  const int64_t slots = (int64_t)C * Lc;
  rec_clear_kernel<R><<<(int)std::min<int64_t>(1184, (slots + 255) / 256), 256, 0, st>>>(rec, slots);
  const int blocks = (int)std::min<int64_t>(148 * 8, (total + 7) / 8);
  switch (TW) {
    case 32: tile_init_kernel<R, 32><<<blocks, 256, 0, st>>>(grid, dg, own, W, total, C, Lc, rec, sel); break;
    case 64: tile_init_kernel<R, 64><<<blocks, 256, 0, st>>>(grid, dg, own, W, total, C, Lc, rec, sel); break;
    case 128: tile_init_kernel<R, 128><<<blocks, 256, 0, st>>>(grid, dg, own, W, total, C, Lc, rec, sel); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
template <typename R>
cudaError_t launch_grid_export(const typename cplx<R>::t* grid, const DictGeo* dg, int W, int64_t P, double2* out,
                               cudaStream_t st) {
  grid_export_kernel<R><<<(int)std::min<int64_t>(1184, (P + 255) / 256), 256, 0, st>>>(grid, dg, W, P, out);
  return cudaGetLastError();
}
template cudaError_t launch_grid_export<double>(const double2*, const DictGeo*, int, int64_t, double2*, cudaStream_t);
template cudaError_t launch_grid_export<float>(const float2*, const DictGeo*, int, int64_t, double2*, cudaStream_t);

template cudaError_t launch_tile_init<double>(const double2*, const DictGeo*, const OwnGeo*, int, int64_t, int,
                                              int64_t, int, Rec<double>*, SelScore, cudaStream_t);
template cudaError_t launch_tile_init<float>(const float2*, const DictGeo*, const OwnGeo*, int, int64_t, int,
                                             int64_t, int, Rec<float>*, SelScore, cudaStream_t);
