// loopcore.cuh -- device building blocks shared by the persistent MP loop kernels
// (mploop.cu: one selection per iteration; mpmulti.cu: exact multi-selection rounds).
//
//   * ScoreOps      |c|^2 without FMA contraction (both sides of the argmax parity,
//                   DESIGN.md §2 note under Z21)
//   * VGeo/vgeo()   the Alg. 3 index sets of one target dictionary v
//                   for a selected atom (u, k, j): alignment class of the kernel box,
//                   first frame / bin, folded bin hull in tiles, this CTA's rows
//   * mailbox       st.async into remote shared memory + mbarrier complete_tx
//   * warp_node     32-ary max-tree node re-reduction
#pragma once
#include "argmax.cuh"
#include "launch.h"

namespace mpcore {

template <typename R>
struct ScoreOps;
template <>
struct ScoreOps<double> {
  static __device__ __forceinline__ double score(double re, double im) {
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
  }
};
template <>
struct ScoreOps<float> {
  static __device__ __forceinline__ float score(float re, float im) {
    return __fadd_rn(__fmul_rn(re, re), __fmul_rn(im, im));
  }
};

// Correctly rounded arithmetic without FMA contraction, so that every loop kernel
// (and the oracle, compiled with -ffp-contract=off) rounds the update identically.
template <typename R>
struct Ar;
template <>
struct Ar<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
};
template <>
struct Ar<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
};

// z0 = c~ omega (fp64, then rounded to R) for one kernel row (Eq. (15))
template <typename C2, typename R>
__device__ __forceinline__ C2 row_z0(double tre, double tim, double2 w) {
  C2 z;
  z.x = (R)__dsub_rn(__dmul_rn(tre, w.x), __dmul_rn(tim, w.y));
  z.y = (R)__dadd_rn(__dmul_rn(tre, w.y), __dmul_rn(tim, w.x));
  return z;
}

// One target bin of Alg. 3 with the fold rule (Z14): z = z0 h; the direct term
// c -= z_d and the conjugate term c -= conj(z_c), in ascending source-column order.
template <typename R, typename C2>
__device__ __forceinline__ C2 fold_update(C2 c, C2 z0, C2 hd, C2 hc, bool fd, bool fc, bool cfirst) {
  using A = Ar<R>;
  const R zdx = A::sub(A::mul(z0.x, hd.x), A::mul(z0.y, hd.y));
  const R zdy = A::add(A::mul(z0.x, hd.y), A::mul(z0.y, hd.x));
  const R zcx = A::sub(A::mul(z0.x, hc.x), A::mul(z0.y, hc.y));
  const R zcy = A::add(A::mul(z0.x, hc.y), A::mul(z0.y, hc.x));
  if (fc && cfirst) {
    c.x = A::sub(c.x, zcx);
    c.y = A::add(c.y, zcy);
  }
  if (fd) {
    c.x = A::sub(c.x, zdx);
    c.y = A::sub(c.y, zdy);
  }
  if (fc && !cfirst) {
    c.x = A::sub(c.x, zcx);
    c.y = A::add(c.y, zcy);
  }
  return c;
}

// Selection score of coefficient c of atom (v, bin k) (Alg. 1 step 1).  Non-pedantic
// (default, reading Z9): |c|^2.  Pedantic: the energy E~ that selecting the
// atom removes, Eq. (20) with c~ of Eq. (19) -- c~ = Re c, E~ = c~^2 for a self-conjugate
// atom (Z13); else rho = h_vv(-2k, 0) from the kept nu = 0 row (0 outside it, Z12),
// c~ = (c - conj(rho) conj(c)) / (1 - |rho|^2) and E~ = 2 [X^2 + Y^2 + Re rho (X^2 - Y^2)
// - 2 Im rho X Y]; with rho = 0 this is exactly 2 |c|^2.
template <typename R>
__device__ __forceinline__ R sel_score(R cre, R cim, int k, int M, bool pedantic, const RhoEnt* rho_row, int rho_lo,
                                       int rho_n) {
  using A = Ar<R>;
  const R s2 = A::add(A::mul(cre, cre), A::mul(cim, cim));
  if (!pedantic) return s2;
  if (k == 0 || 2 * k == M) return A::mul(cre, cre);
  int mu = (-2 * k) & (M - 1);
  if (2 * mu > M) mu -= M;
  const int ri = mu - rho_lo;
  if (ri < 0 || ri >= rho_n) return A::add(s2, s2);
  const RhoEnt rv = rho_row[ri];
  const double cr = (double)cre, ci = (double)cim;
  const double nre = __dsub_rn(cr, __dsub_rn(__dmul_rn(rv.re, cr), __dmul_rn(rv.im, ci)));
  const double nim = __dadd_rn(ci, __dadd_rn(__dmul_rn(rv.re, ci), __dmul_rn(rv.im, cr)));
  const double X = __dmul_rn(nre, rv.inv), Y = __dmul_rn(nim, rv.inv);
  const double X2 = __dmul_rn(X, X), Y2 = __dmul_rn(Y, Y), XY = __dmul_rn(X, Y);
  const double t = __dsub_rn(__dadd_rn(__dadd_rn(X2, Y2), __dmul_rn(rv.re, __dsub_rn(X2, Y2))),
                             __dmul_rn(__dmul_rn(2.0, rv.im), XY));
  return (R)__dmul_rn(2.0, t);
}

// This lane's best (score desc, index asc) over its NCH bins bin0 + 32 ch of a tile row
// (only bins < MR count); the pedantic test is taken once, outside the bin loop.
template <typename R, typename C2, int NCH>
__device__ __forceinline__ void lane_best(const C2 (&c)[NCH], int bin0, int MR, int M, uint32_t pbase, bool pedantic,
                                          const RhoEnt* rho_row, int rho_lo, int rho_n, R& bs, uint32_t& bp, R& bre,
                                          R& bim) {
  bs = 0;
  bp = NO_INDEX;
  bre = 0;
  bim = 0;
  if (pedantic) {
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int bin = bin0 + ch * 32;
      if (bin < MR) {
        const R s = sel_score<R>(c[ch].x, c[ch].y, bin, M, true, rho_row, rho_lo, rho_n);
        if (better(s, pbase + (uint32_t)bin, bs, bp)) {
          bs = s;
          bp = pbase + (uint32_t)bin;
          bre = c[ch].x;
          bim = c[ch].y;
        }
      }
    }
  } else {
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      const int bin = bin0 + ch * 32;
      if (bin < MR) {
        const R s = sel_score<R>(c[ch].x, c[ch].y, bin, M, false, nullptr, 0, 0);
        if (better(s, pbase + (uint32_t)bin, bs, bp)) {
          bs = s;
          bp = pbase + (uint32_t)bin;
          bre = c[ch].x;
          bim = c[ch].y;
        }
      }
    }
  }
}

struct VGeo {           // update geometry for one target dictionary v, seen from this CTA
  long long kbase;      // first kernel entry of the alignment class
  int nr, nc;           // rows (frames) and columns (bins) of the class sub-box
  int n0, q0;           // first target frame, first target bin (before folding)
  int t0, Tr;           // first tile and tile count of the folded bin hull
  int rA, rhoA, cntA;   // rows [0, rA) do not wrap; owned rows rhoA + i*C, i < cntA
  int rhoB, cntB;       // rows [rA, nr) wrap to frame 0..; owned rows rA + rhoB + i*C, i < cntB
  int base, nitems;     // this CTA's items of v: (cntA + cntB) * Tr tiles
  int rr0, rrstep;      // modulation exponent of row 0 and its per-row step (mod R)
  int pad;
};

// fold(Q) = min(Q mod M, M - Q mod M) over the run Q = q0 .. q0+nc-1 (q0 in [0,M)):
// hull [bmin, bmax] of the reduced bins that receive a direct or conjugate term
__device__ __forceinline__ void target_hull(int q0, int nc, int M, int& bmin, int& bmax) {
  const int qa = q0, qb = q0 + nc - 1;
  const int half = M >> 1;
  const int ra = qa & (M - 1), rb = qb & (M - 1);
  const int fa = ra <= half ? ra : M - ra, fb = rb <= half ? rb : M - rb;
  const bool trough = (qa == 0) || (qb >= M);
  const bool peak = (qa <= half && qb >= half) || (qb >= M + half);
  bmin = trough ? 0 : min(fa, fb);
  bmax = peak ? half : max(fa, fb);
}

// Update geometry of target dictionary v for the atom (u, k, j) of dictionary u
// (SURVEY O7e / Alg. 3): the alignment class (o_n, o_m) of the (u, v) kernel box,
// its nr x nc sub-box, the first target frame n0 and bin q0, the folded bin hull
// in tiles [t0, t0 + Tr), the rows owned by CTA `rank` of a C-CTA cluster and the
// modulation exponents.  Every stride is a power of two (shift/mask arithmetic).
// Returns this CTA's item count (rows x hull tiles).
template <int LGTW>
__device__ __forceinline__ int vgeo(const PairGeo& pg, const DictGeo& du, const DictGeo& dv, int k, int j, int rank,
                                    int C, int lgC, VGeo& g) {
  // every stride is a power of two; the shifts come precomputed with the pair (PairGeo::sh)
  const int lgac = pg_sh(pg.sh, PG_SH_AC), lgsm = pg_sh(pg.sh, PG_SH_SM), lgsn = pg_sh(pg.sh, PG_SH_SN);
  const int lgauc = pg_sh(pg.sh, PG_SH_AUC);
  const int kp = k << pg_sh(pg.sh, PG_SH_MCU);                              // k' = k M_c/M_u
  const int on = (-(j << lgauc) - pg.nu_lo) & (pg.s_n - 1);
  const int om = (-kp - pg.mu_lo) & (pg.s_m - 1);
  g.nr = on < pg.nnu ? (pg.nnu - on + pg.s_n - 1) >> lgsn : 0;
  g.nc = om < pg.nmu ? (pg.nmu - om + pg.s_m - 1) >> lgsm : 0;
  const int tnum = ((j << lgauc) + pg.nu_lo + on) << lgac;                  // divisible by a_v
  int n0 = tnum >> pg_sh(pg.sh, PG_SH_AV);
  if (n0 < 0) n0 += dv.N;
  if (n0 >= dv.N) n0 -= dv.N;
  g.n0 = n0;
  g.q0 = ((kp + pg.mu_lo + om) >> lgsm) & (dv.M - 1);
  g.kbase = pg.koff + (long long)(on * (pg.nnu >> lgsn) + min(on, pg.nnu & (pg.s_n - 1))) * pg.nmu +
            (long long)g.nr * (om * (pg.nmu >> lgsm) + min(om, pg.nmu & (pg.s_m - 1)));
  int bmin = 0, bmax = 0;
  if (g.nc > 0) target_hull(g.q0, g.nc, dv.M, bmin, bmax);
  g.t0 = bmin >> LGTW;
  g.Tr = (bmax >> LGTW) - g.t0 + 1;
  // rows owned by this CTA: frame f = frame_off_v + n belongs to CTA f mod C
  g.rA = min(g.nr, dv.N - n0);
  g.rhoA = (rank - (dv.frame_off + n0)) & (C - 1);
  g.cntA = g.rhoA < g.rA ? ((g.rA - 1 - g.rhoA) >> lgC) + 1 : 0;
  const int nB = g.nr - g.rA;
  g.rhoB = (rank - dv.frame_off) & (C - 1);
  g.cntB = (nB > 0 && g.rhoB < nB) ? ((nB - 1 - g.rhoB) >> lgC) + 1 : 0;
  const int nitems = g.nc > 0 ? (g.cntA + g.cntB) * g.Tr : 0;
  g.rr0 = (kp * (pg.nu_lo + on)) & (pg.R - 1);
  g.rrstep = (kp << lgsn) & (pg.R - 1);
  g.nitems = nitems;
  g.base = 0;
  g.pad = 0;
  return nitems;
}

// ---- named CTA barriers (id 0 is __syncthreads) ----
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- cluster mailbox: st.async into remote shared memory + mbarrier complete_tx ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Inter-CTA waits are bounded: a peer that never arrives (a logic error, or a CTA that
// left the loop early) traps after ~2^35 SM cycles (~17 s) instead of hanging the GPU;
// the launch then fails with a CUDA error (MPG_ECUDA) instead of spinning forever.
constexpr long long SPIN_LIMIT_CYCLES = 1LL << 35;
__device__ __forceinline__ void spin_check(long long t0) {
  if (clock64() - t0 > SPIN_LIMIT_CYCLES) __trap();
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  const long long t0 = clock64();
  do {
    spin_check(t0);
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void st_async16(uint32_t raddr, uint32_t rbar, uint4 v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
               : "memory");
}
template <typename R>
__device__ __forceinline__ void push_record(const Rec<R>& r, uint32_t raddr, uint32_t rbar) {
  const uint4* w = reinterpret_cast<const uint4*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(Rec<R>) / 16); ++i) st_async16(raddr + 16 * i, rbar, w[i]);
}

// Bulk prefetch of [p, p + bytes) into L2 by the TMA unit (cp.async.bulk.prefetch.L2,
// fire and forget: no completion, no register or shared-memory destination); the range
// is widened to 16-byte granules as the instruction requires.
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  const unsigned long long a = (unsigned long long)p & ~15ull;
  const uint32_t n = (uint32_t)(((unsigned long long)p + bytes - a + 15ull) & ~15ull);
  if (bytes != 0) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(n) : "memory");
}

// one warp re-reduces node `node` of a level from its (up to) 32 children
template <typename R>
__device__ __forceinline__ void warp_node(const Rec<R>* child, long long nchild, int node, Rec<R>* out, int lane) {
  const long long c = (long long)node * 32 + lane;
  const Rec<R> r = c < nchild ? child[c] : empty_rec(R(0));
  if (lane == warp_argmax_lane(r.s, r.p)) out[node] = r;
}

// 32-bit conservative key of a score for the multi-selection verification:
// fp32 -- the exact bit pattern; fp64 -- the upper word (the score rounded down
// to 20 mantissa bits).  key(s1) < key(s2) implies s1 < s2.
__device__ __forceinline__ uint32_t score_key(double s) {
  return (uint32_t)((unsigned long long)__double_as_longlong(s) >> 32);
}
__device__ __forceinline__ uint32_t score_key(float s) { return (uint32_t)__float_as_int(s); }
// exact 64-bit order key of a (non-negative) score
__device__ __forceinline__ uint64_t skey64(double s) { return (uint64_t)__double_as_longlong(s); }
__device__ __forceinline__ uint64_t skey64(float s) { return (uint64_t)(uint32_t)__float_as_int(s) << 32; }

}  // namespace mpcore
