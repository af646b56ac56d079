// common.cuh -- shared device/host helpers of libmpgabor (CUDA path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MPG_HD __host__ __device__ __forceinline__

MPG_HD int64_t fdiv64(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b) != 0 && ((a < 0) != (b < 0))) --q;
  return q;
}
MPG_HD int64_t fmod64(int64_t a, int64_t b) {
  int64_t r = a % b;
  return r < 0 ? r + b : r;
}
MPG_HD int fmod32(int a, int b) {
  int r = a % b;
  return r < 0 ? r + b : r;
}
// number of i in [0, n) with i mod s < o   (class prefix counts of the kernel layout)
MPG_HD int cnt_lt(int o, int n, int s) { return o * (n / s) + (o < n % s ? o : n % s); }
// number of i in [0, n) with i mod s == o
MPG_HD int cnt_eq(int o, int n, int s) { return n / s + (o < n % s ? 1 : 0); }

template <typename R> struct cplx;
template <> struct cplx<double> { using t = double2; };
template <> struct cplx<float> { using t = float2; };

// ---------------------------------------------------------------------------
// Per-dictionary and per-pair geometry shared by host runtime and kernels.
// ---------------------------------------------------------------------------
struct DictGeo {
  int32_t win, gl, a, M;
  int32_t N, MR;          // frames L/a, reduced bins M/2+1
  int32_t T, stride;      // tiles per frame, padded row stride (= T*TW)
  int32_t frame_off;      // global frame id of frame 0 (frames of all dictionaries in order)
  uint32_t mr_magic;      // ceil(2^32 / MR): q / MR = umulhi(q, mr_magic) or one less (decode)
  int64_t off;            // global coefficient index of (n=0, m=0)
  int64_t grid_off;       // element offset of this dictionary in the padded grid
  int64_t tile_off;       // global tile id of (n=0, t=0)
};

// Frame ownership of the loop cluster: frame f (global id) belongs to CTA f mod C.
// For CTA c and dictionary v: its first owned frame, its number of owned frames and
// the local index of its first tile record (tiles of owned frames in frame order).
struct OwnGeo {
  int32_t n_first, n_own;
  int32_t loc_base, pad_;
};

struct PairGeo {          // u = selected dictionary, v = updated dictionary
  int32_t a_c, M_c, R;    // common grid and modulation period R = M_c/a_c
  int32_t s_m, s_n;       // frequency subsampling M_c/M_v, time subsampling a_v/a_c (>=1)
  int32_t mu_lo, mu_hi, nu_lo, nu_hi;
  int32_t nmu, nnu;       // box size
  int32_t rstep;          // Rmax / R: index step into the common root table
  int32_t sh;             // packed shifts (5 bits each, PG_SH_*): log2 a_c, s_m, s_n, M_c/M_u, a_u/a_c, a_v, a_u
  int64_t koff;           // element offset of this pair's kernel storage
};

enum { PG_SH_AC = 0, PG_SH_SM = 5, PG_SH_SN = 10, PG_SH_MCU = 15, PG_SH_AUC = 20, PG_SH_AV = 25 };
MPG_HD int pg_sh(int32_t sh, int f) { return (sh >> f) & 31; }

// Tile record: best |c|^2 of a tile with its global index and value.  Scores are
// >= +0 so their IEEE bit patterns order like the values; an empty record is
// (s = 0, p = 0xffffffff) and loses every tie (Z10).
template <typename R> struct Rec;
template <> struct __align__(32) Rec<double> {
  double s, re, im;
  uint32_t p, pad;
};
template <> struct __align__(16) Rec<float> {
  float s, re, im;
  uint32_t p;
};
constexpr uint32_t NO_INDEX = 0xffffffffu;

// conjugate-pair entry rho = <d, conj d> = h_uu(mu, 0) and 1/(1 - |rho|^2) (Eq. (19))
struct RhoEnt {
  double re, im, inv, pad_;
};

MPG_HD int ilog2(int x) {  // x a power of two
#ifdef __CUDA_ARCH__
  return __ffs(x) - 1;
#else
  return __builtin_ctz((unsigned)x);
#endif
}

// lexicographic order: higher score wins, equal scores -> lower index (Z10)
template <typename S, typename P>
MPG_HD bool better(S s1, P p1, S s2, P p2) { return s1 > s2 || (s1 == s2 && p1 < p2); }

// Debug builds (-DMPG_CHECKS, tools/build_variant.sh): device-side protocol and bounds
// checks that trap with a message (the launch then fails with a CUDA error).  They stand
// in for compute-sanitizer, which this GPU pool does not offer.
#ifdef MPG_CHECKS
#include <cstdio>
#define MPG_CHECK(cond, what)                                                                              \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("MPG_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                            \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define MPG_CHECK(cond, what) \
  do {                        \
  } while (0)
#endif

#define CUDA_OK(x)                                   \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) return e_;                \
  } while (0)
