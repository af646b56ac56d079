// argmax.cuh -- warp-wide argmax of tile records with redux.sync (sm_80+):
// maximise the score, ties to the lowest global index (Z10).  Scores are
// non-negative, so comparing their IEEE bit patterns as unsigned integers is exact.
#pragma once
#include "common.cuh"

__device__ __forceinline__ Rec<double> empty_rec(double) {
  Rec<double> r;
  r.s = 0.0; r.re = 0.0; r.im = 0.0; r.p = NO_INDEX; r.pad = 0;
  return r;
}
__device__ __forceinline__ Rec<float> empty_rec(float) {
  Rec<float> r;
  r.s = 0.0f; r.re = 0.0f; r.im = 0.0f; r.p = NO_INDEX;
  return r;
}

// Returns the winning lane; every lane gets the winning score and index.
__device__ __forceinline__ int warp_argmax(double s, uint32_t p, double& sbest, uint32_t& pbest) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const bool top = (hi == mhi) && (lo == mlo);
  pbest = __reduce_min_sync(0xffffffffu, top ? p : NO_INDEX);
  sbest = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  return __ffs(__ballot_sync(0xffffffffu, top && p == pbest)) - 1;
}
__device__ __forceinline__ int warp_argmax(float s, uint32_t p, float& sbest, uint32_t& pbest) {
  const unsigned b = (unsigned)__float_as_int(s);
  const unsigned mb = __reduce_max_sync(0xffffffffu, b);
  const bool top = (b == mb);
  pbest = __reduce_min_sync(0xffffffffu, top ? p : NO_INDEX);
  sbest = __int_as_float((int)mb);
  return __ffs(__ballot_sync(0xffffffffu, top && p == pbest)) - 1;
}

// Only the winning lane (score desc, index asc): one redux on the upper score word and a
// ballot in the common case; the full comparison only when the upper words tie.
__device__ __forceinline__ int warp_argmax_lane(double s, uint32_t p) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(s);
  const unsigned hi = (unsigned)(b >> 32);
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned m = __ballot_sync(0xffffffffu, hi == mhi);
  if ((m & (m - 1)) == 0) return __ffs(m) - 1;
  double sb;
  uint32_t pb;
  return warp_argmax(s, p, sb, pb);
}
__device__ __forceinline__ int warp_argmax_lane(float s, uint32_t p) {
  const unsigned b = (unsigned)__float_as_int(s);
  const unsigned mb = __reduce_max_sync(0xffffffffu, b);
  const unsigned m = __ballot_sync(0xffffffffu, b == mb);
  if ((m & (m - 1)) == 0) return __ffs(m) - 1;
  const uint32_t pb = __reduce_min_sync(0xffffffffu, b == mb ? p : NO_INDEX);
  return __ffs(__ballot_sync(0xffffffffu, b == mb && p == pb)) - 1;
}

// Full-record argmax: every lane ends with the winning record.
template <typename R>
__device__ __forceinline__ Rec<R> warp_best(const Rec<R>& r) {
  Rec<R> o;
  const int wl = warp_argmax(r.s, r.p, o.s, o.p);
  o.re = __shfl_sync(0xffffffffu, r.re, wl);
  o.im = __shfl_sync(0xffffffffu, r.im, wl);
  if constexpr (sizeof(R) == 8) o.pad = 0;
  return o;
}
