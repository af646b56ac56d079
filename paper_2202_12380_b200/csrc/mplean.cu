// mplean.cu -- N3 + N4 + N5: the persistent coefficient-domain matching pursuit loop.
//
// One thread-block cluster of C CTAs (one CTA per SM, C <= 16, a power of two)
// runs every iteration of Alg. 1 (approximate recursion Eq. (9)
// P:424-434) on the device.  Frame f (global id over all dictionaries) and all
// its coefficients belong to CTA f mod C; tile records (best |c|^2 per TW bins of
// a frame) and a 32-ary max tree over them live in that CTA's shared memory
// (or global memory for the largest grids).  Per iteration:
//
//  A  warp 0: read the C roots from the local mailbox, argmax with redux.sync
//             (score desc, index asc -- DESIGN.md Z10), stop tests (Z15), scalar
//             step: rho from the auto-kernel row, c~ (Eq. (19), Z11),
//             E~ (Eq. (20)), E_{k+1}; rank 0 appends the atom.
//     warp 1: the same argmax, then lane v computes the update geometry of
//             target dictionary v (Alg. 3 index sets: alignment class, first
//             frame and bin, folded bin hull, this CTA's rows) and writes one
//             descriptor per owned row into shared memory.
//  B  all warps: work item = segment of SEG tiles of one owned row; loads of
//             the residual and of the subsampled, modulated kernel row
//             (Eqs. (15)-(17)) for the whole segment are issued first, then the
//             fold-rule update (Z14), stores, and one redux argmax per tile.
//  C  dirty level-1 nodes are re-reduced; D warp 0 refreshes upper levels,
//     scans the top level and pushes the new root into every CTA's mailbox
//     (st.async + mbarrier complete_tx); the mailbox barrier is the only
//     inter-CTA synchronisation.
// Every coefficient is touched by one CTA only: no atomics on data, deterministic.
#include <cooperative_groups.h>
#include "argmax.cuh"
#include "launch.h"

namespace cg = cooperative_groups;

namespace {

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

constexpr int SEG = 2;          // tiles per work item
constexpr int MAX_ROWS = 512;   // owned-row descriptors per iteration (per CTA)

struct Sel {
  double tre, tim;
  double E[2];                  // E_k in E[k & 1]
  int u, k, j, selfc, stop, nseg, nrows, nnode;
};

struct RowDesc {                // one owned row of one target dictionary
  long long grow;               // element offset of the row in the residual grid
  long long krow;               // element offset of the kernel class row
  unsigned pbase;               // global index of bin 0 of the row
  int v, MR, Mmask;
  int q0, nc, t0, Tr;           // first target bin, class columns, tile hull
  int lbase;                    // local tile record index of tile t0
  int rr;                       // modulation exponent (mod R), index rr * rstep into the root table
  int rstep, seg0;              // root-table step; first segment id of this row
  int nd0, ndbase;              // first level-1 node of the row's tiles; first node item id
  int nnd, pad_;                // level-1 nodes spanned by the row's tiles
};

struct Smem {
  size_t mbar, mail, trec, lev, sel, rows, vseg, pairs, dicts, own, roots, rho, rho_meta, stamp, list, cnt, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem smem_layout(const LoopParams& P, size_t recsz) {
  Smem s;
  int levtot = 0;
  for (int l = 0; l < P.nlev; ++l) levtot += P.lev_n[l];
  size_t o = 0;
  s.mbar = o;
  o += 32;
  s.mail = o;
  o += 2 * MAX_CLUSTER * recsz;
  s.trec = o;
  o += P.srec ? (size_t)P.Lc * recsz : 0;
  s.lev = o;
  o += (size_t)levtot * recsz;
  s.sel = o;
  o += align_up(sizeof(Sel), 16);
  s.rows = o;
  o += sizeof(RowDesc) * MAX_ROWS;
  s.vseg = o;
  o += sizeof(int) * 2 * 32;
  s.pairs = o;
  o += sizeof(PairGeo) * P.W * P.W;
  o = align_up(o, 16);
  s.dicts = o;
  o += sizeof(DictGeo) * P.W;
  o = align_up(o, 16);
  s.own = o;
  o += sizeof(OwnGeo) * P.W;
  o = align_up(o, 16);
  s.roots = o;
  o += P.Rmax <= 4096 ? sizeof(double2) * P.Rmax : 0;
  s.rho = o;
  o += sizeof(RhoEnt) * P.rho_total;
  s.rho_meta = o;
  o += sizeof(int) * 3 * P.W;
  o = align_up(o, 16);
  s.stamp = o;
  o += sizeof(int) * levtot;
  s.list = o;
  o += sizeof(int) * levtot;
  s.cnt = o;
  o += sizeof(int) * MAX_LEVELS;
  s.total = align_up(o, 16);
  return s;
}

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
// CTA-scope acquire: only shared memory written by st.async crosses CTAs (a cluster-scope
// acquire would invalidate L1 on every poll)
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
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

template <typename R>
__device__ __forceinline__ void warp_node(const Rec<R>* child, long long nchild, int node, Rec<R>* out, int lane) {
  const long long c = (long long)node * 32 + lane;
  const Rec<R> r = c < nchild ? child[c] : empty_rec(R(0));
  R s;
  uint32_t p;
  const int wl = warp_argmax(r.s, r.p, s, p);
  if (lane == wl) out[node] = r;
}

__device__ __forceinline__ long long tclock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}

template <typename R, int TW, bool SREC>
__global__ void __launch_bounds__(512, 1) mp_lean_kernel(const LoopParams P) {
  using C2 = typename cplx<R>::t;
  using RecT = Rec<R>;
  constexpr int LGTW = TW == 32 ? 5 : (TW == 64 ? 6 : 7);
  constexpr int NCH = TW / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = P.C, lgC = ilog2(P.C);
  const int rank = (int)cluster.block_rank();
  const int W = P.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;

  extern __shared__ __align__(32) unsigned char smem[];
  const Smem L = smem_layout(P, sizeof(RecT));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  RecT* mail = reinterpret_cast<RecT*>(smem + L.mail);
  RecT* lev = reinterpret_cast<RecT*>(smem + L.lev);
  Sel* sel = reinterpret_cast<Sel*>(smem + L.sel);
  RowDesc* rows = reinterpret_cast<RowDesc*>(smem + L.rows);
  int* vseg = reinterpret_cast<int*>(smem + L.vseg);   // [0..31] first segment of v, [32..63] first row of v
  PairGeo* sp = reinterpret_cast<PairGeo*>(smem + L.pairs);
  DictGeo* sd = reinterpret_cast<DictGeo*>(smem + L.dicts);
  OwnGeo* sown = reinterpret_cast<OwnGeo*>(smem + L.own);
  const double2* roots = P.Rmax <= 4096 ? reinterpret_cast<const double2*>(smem + L.roots) : P.roots;
  RhoEnt* srho = reinterpret_cast<RhoEnt*>(smem + L.rho);
  int* rho_lo = reinterpret_cast<int*>(smem + L.rho_meta);
  int* rho_n = rho_lo + W;
  int* rho_off = rho_n + W;
  int* stamp = reinterpret_cast<int*>(smem + L.stamp);
  int* list = reinterpret_cast<int*>(smem + L.list);
  int* cnt = reinterpret_cast<int*>(smem + L.cnt);
  RecT* grec = reinterpret_cast<RecT*>(P.rec) + (long long)rank * P.Lc;
  RecT* trec = SREC ? reinterpret_cast<RecT*>(smem + L.trec) : grec;
  C2* grid = reinterpret_cast<C2*>(P.grid);
  const C2* kern = reinterpret_cast<const C2*>(P.kern);

  // ---- tables -------------------------------------------------------------------
  for (int i = threadIdx.x; i < W * W; i += blockDim.x) sp[i] = P.pairs[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    sd[i] = P.dicts[i];
    sown[i] = P.own[rank * W + i];
    rho_lo[i] = P.rho_lo[i];
    rho_n[i] = P.rho_n[i];
    rho_off[i] = P.rho_off[i];
  }
  if (P.Rmax <= 4096)
    for (int i = threadIdx.x; i < P.Rmax; i += blockDim.x) reinterpret_cast<double2*>(smem + L.roots)[i] = P.roots[i];
  for (int i = threadIdx.x; i < P.rho_total; i += blockDim.x) srho[i] = P.rho[i];
  int levtot = 0;
  for (int l = 0; l < P.nlev; ++l) levtot += P.lev_n[l];
  for (int i = threadIdx.x; i < levtot; i += blockDim.x) stamp[i] = 0;
  if (threadIdx.x < MAX_LEVELS) cnt[threadIdx.x] = 0;
  if (SREC)
    for (long long i = threadIdx.x; i < P.Lc; i += blockDim.x) trec[i] = grec[i];
  __syncthreads();

  // ---- node levels, mailbox barriers, first root --------------------------------
  for (int i = warp; i < P.lev_n[0]; i += NW) warp_node(trec, P.Lc, i, lev, lane);
  __syncthreads();
  for (int l = 1; l < P.nlev; ++l) {
    for (int i = warp; i < P.lev_n[l]; i += NW)
      warp_node(lev + P.lev_off[l - 1], (long long)P.lev_n[l - 1], i, lev + P.lev_off[l], lane);
    __syncthreads();
  }
  const uint32_t recbytes = (uint32_t)sizeof(RecT);
  if (threadIdx.x == 0) {
    mbar_init(smem_addr(&mbar[0]), 1);
    mbar_init(smem_addr(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(smem_addr(&mbar[0]), C * recbytes);
    mbar_arm(smem_addr(&mbar[1]), C * recbytes);
    sel->E[0] = P.E0;
    sel->stop = 0;
  }
  __syncthreads();
  cluster.sync();
  // warp 0: top scan (<= TOP_SCAN nodes: independent loads, then compares of (s, p)
  // only), winner record fetched once and pushed into every CTA's mailbox
  auto publish_root = [&](int slot) {
    const int top = P.nlev - 1;
    const RecT* tl = lev + P.lev_off[top];
    const int nt = P.lev_n[top];
    constexpr int PER = TOP_SCAN / 32;
    R sv[PER];
    uint32_t pv[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = q * 32 + lane;
      sv[q] = i < nt ? tl[i].s : (R)0;
      pv[q] = i < nt ? tl[i].p : NO_INDEX;
    }
    R bs = sv[0];
    uint32_t bp = pv[0];
    int bi = lane;
#pragma unroll
    for (int q = 1; q < PER; ++q)
      if (better(sv[q], pv[q], bs, bp)) {
        bs = sv[q];
        bp = pv[q];
        bi = q * 32 + lane;
      }
    R ws;
    uint32_t wp;
    const int wl = warp_argmax(bs, bp, ws, wp);
    const int wi = __shfl_sync(0xffffffffu, bi, wl);
    const RecT b = wi < nt ? tl[wi] : empty_rec(R(0));
    if (lane < C)
      push_record(b, mapa(smem_addr(&mail[slot * MAX_CLUSTER + rank]), lane), mapa(smem_addr(&mbar[slot]), lane));
  };
  if (warp == 0) publish_root(0);

  long long it = 0;
  int stop = 0;
  const bool prof = P.prof != nullptr && rank == 0 && threadIdx.x == 0;
  long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
  long long tprev = tclock();
#define PROF_MARK(i)                \
  if (prof) {                        \
    const long long tn = tclock();   \
    ph[i] += tn - tprev;             \
    tprev = tn;                      \
  }
#define TRACE(slot, val)                                                                         \
  if (P.trace && it >= P.trace_it0 && it < P.trace_it0 + P.trace_n)                                \
    P.trace[((it - P.trace_it0) * C + rank) * P.trace_slots + (slot)] = (val);

  for (;; ++it) {
    const int par = (int)(it & 1);
    // ---- A. selection (warps 0, 1) ------------------------------------------------
    if (warp < 2) {
      mbar_wait(smem_addr(&mbar[par]), (uint32_t)((it >> 1) & 1));
      if (warp == 0 && lane == 0) {
        mbar_arm(smem_addr(&mbar[par]), C * recbytes);  // slot reused at it + 2
        TRACE(0, tclock());
      }
      const RecT best = warp_best(lane < C ? mail[par * MAX_CLUSTER + lane] : empty_rec(R(0)));
      const double Ecur = sel->E[par];
      int st = 0;
      if (it >= P.maxit) st = 1;
      else if (Ecur <= P.Etol) st = 2;
      else if (Ecur < 0.0) st = 3;
      else if (!(best.s > (R)0)) st = 4;
      if (st) {
        if (warp == 0 && lane == 0) sel->stop = st;
      } else {
        const uint32_t p = best.p;
        const int u = __popc(__ballot_sync(0xffffffffu, lane > 0 && lane < W && (uint32_t)sd[lane].off <= p));
        const uint32_t qq = p - (uint32_t)sd[u].off;
        const int MRu = sd[u].MR;
        const int j = (int)(qq / (uint32_t)MRu);
        const int k = (int)(qq - (uint32_t)j * (uint32_t)MRu);
        const int Mu = sd[u].M;
        const bool selfc = (k == 0) || (2 * k == Mu);
        if (warp == 0) {
          // scalar step (Eq. (19)-(20))
          double tre, tim, Et;
          const double cre = (double)best.re, cim = (double)best.im;
          if (selfc) {
            tre = cre;
            tim = 0.0;
            Et = tre * tre;
          } else {
            int mu = (-2 * k) & (Mu - 1);
            if (2 * mu > Mu) mu -= Mu;
            double rre = 0.0, rim = 0.0, inv = 1.0;
            const int ri = mu - rho_lo[u];
            if (ri >= 0 && ri < rho_n[u]) {
              const RhoEnt rv = srho[rho_off[u] + ri];
              rre = rv.re;
              rim = rv.im;
              inv = rv.inv;
            }
            const double nre = cre - (rre * cre - rim * cim);
            const double nim = cim + (rre * cim + rim * cre);
            tre = nre * inv;
            tim = nim * inv;
            const double X2 = tre * tre, Y2 = tim * tim, XY = tre * tim;
            Et = 2.0 * (X2 + Y2 + rre * (X2 - Y2) - 2.0 * rim * XY);
          }
          const double En = Ecur - Et;
          if (lane == 0) {
            sel->tre = tre;
            sel->tim = tim;
            sel->E[par ^ 1] = En;
            sel->u = u;
            sel->k = k;
            sel->j = j;
            sel->selfc = selfc ? 1 : 0;
            sel->stop = 0;
            TRACE(1, tclock());
            if (rank == 0) {
              AtomOut a;
              a.w = u;
              a.m = k;
              a.n = j;
              a.flags = selfc ? 1 : 0;
              a.re = tre;
              a.im = tim;
              P.atoms[it] = a;
              P.energy[it + 1] = En;
            }
          }
        } else {
          // geometry of target dictionary v = lane (Alg. 3 index sets)
          int nrv = 0, segs = 0;
          int q0 = 0, nc = 0, t0 = 0, Tr = 0, n0 = 0, rA = 0, rhoA = 0, cntA = 0, rhoB = 0, rr0 = 0, rrstep = 0;
          long long kbase = 0;
          if (lane < W) {
            const int v = lane;
            const PairGeo& pg = sp[u * W + v];
            const DictGeo& dv = sd[v];
            const int lgac = ilog2(pg.a_c), lgsm = ilog2(pg.s_m), lgsn = ilog2(pg.s_n);
            const int kp = k << (ilog2(pg.M_c) - ilog2(Mu));
            const int on = (-(j << (ilog2(sd[u].a) - lgac)) - pg.nu_lo) & (pg.s_n - 1);
            const int om = (-kp - pg.mu_lo) & (pg.s_m - 1);
            const int nr = on < pg.nnu ? (pg.nnu - on + pg.s_n - 1) >> lgsn : 0;
            nc = om < pg.nmu ? (pg.nmu - om + pg.s_m - 1) >> lgsm : 0;
            n0 = ((j << ilog2(sd[u].a)) + ((pg.nu_lo + on) << lgac)) >> ilog2(dv.a);
            if (n0 < 0) n0 += dv.N;
            if (n0 >= dv.N) n0 -= dv.N;
            q0 = ((kp + pg.mu_lo + om) >> lgsm) & (dv.M - 1);
            kbase = pg.koff + (long long)(on * (pg.nnu >> lgsn) + min(on, pg.nnu & (pg.s_n - 1))) * pg.nmu +
                    (long long)nr * (om * (pg.nmu >> lgsm) + min(om, pg.nmu & (pg.s_m - 1)));
            int bmin = 0, bmax = 0;
            if (nc > 0) target_hull(q0, nc, dv.M, bmin, bmax);
            t0 = bmin >> LGTW;
            Tr = (bmax >> LGTW) - t0 + 1;
            rA = min(nr, dv.N - n0);
            rhoA = (rank - (dv.frame_off + n0)) & (C - 1);
            cntA = rhoA < rA ? ((rA - 1 - rhoA) >> lgC) + 1 : 0;
            const int nB = nr - rA;
            rhoB = (rank - dv.frame_off) & (C - 1);
            const int cntB = (nB > 0 && rhoB < nB) ? ((nB - 1 - rhoB) >> lgC) + 1 : 0;
            nrv = (nc > 0 && !(P.floor_mode & 1)) ? cntA + cntB : 0;
            segs = (Tr + SEG - 1) / SEG;
            rr0 = (kp * (pg.nu_lo + on)) & (pg.R - 1);
            rrstep = (kp << lgsn) & (pg.R - 1);
          }
          // prefix sums over v of rows and segments
          int rinc = nrv, sinc = nrv * segs;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y1 = __shfl_up_sync(0xffffffffu, rinc, o);
            const int y2 = __shfl_up_sync(0xffffffffu, sinc, o);
            if (lane >= o) {
              rinc += y1;
              sinc += y2;
            }
          }
          const int rbase = rinc - nrv, sbase = sinc - nrv * segs;
          const int nrows = __shfl_sync(0xffffffffu, rinc, 31);
          const int nseg = __shfl_sync(0xffffffffu, sinc, 31);
          // level-1 nodes spanned by each owned row (the nodes to refresh in phase C)
          auto row_of = [&](int i, int& r, int& nrow, int& lb) {
            const DictGeo& dv = sd[lane];
            r = i < cntA ? rhoA + (i << lgC) : rA + rhoB + ((i - cntA) << lgC);
            nrow = n0 + r;
            if (nrow >= dv.N) nrow -= dv.N;
            lb = sown[lane].loc_base + ((nrow - sown[lane].n_first) >> lgC) * dv.T + t0;
          };
          int ndv = 0;
          if (lane < W)
            for (int i = 0; i < nrv; ++i) {
              int r, nrow, lb;
              row_of(i, r, nrow, lb);
              ndv += ((lb + Tr - 1) >> 5) - (lb >> 5) + 1;
            }
          int ninc = ndv;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, ninc, o);
            if (lane >= o) ninc += y;
          }
          int ndb = ninc - ndv;
          const int nnode = __shfl_sync(0xffffffffu, ninc, 31);
          if (lane < W) {
            vseg[lane] = sbase;
            vseg[32 + lane] = rbase;
            const int v = lane;
            const DictGeo& dv = sd[v];
            const PairGeo& pg = sp[u * W + v];
            for (int i = 0; i < nrv && rbase + i < MAX_ROWS; ++i) {
              int r, nrow, lb;
              row_of(i, r, nrow, lb);
              RowDesc d;
              d.nd0 = lb >> 5;
              d.nnd = ((lb + Tr - 1) >> 5) - d.nd0 + 1;
              d.ndbase = ndb;
              ndb += d.nnd;
              d.grow = dv.grid_off + (long long)nrow * dv.stride;
              d.krow = kbase + (long long)r * nc;
              d.pbase = (unsigned)dv.off + (unsigned)nrow * (unsigned)dv.MR;
              d.v = v;
              d.MR = dv.MR;
              d.Mmask = dv.M - 1;
              d.q0 = q0;
              d.nc = nc;
              d.t0 = t0;
              d.Tr = Tr;
              d.lbase = lb;
              d.rr = (rr0 + r * rrstep) & (pg.R - 1);
              d.rstep = pg.rstep;
              d.seg0 = sbase + i * segs;
              rows[rbase + i] = d;
            }
          }
          if (lane == 0) {
            sel->nseg = nseg;
            sel->nrows = min(nrows, MAX_ROWS);
            sel->nnode = nnode;
            TRACE(2, tclock());
          }
        }
      }
    }
    PROF_MARK(0);
    __syncthreads();
    PROF_MARK(1);
    if (warp == 0 && lane == 0) {
      TRACE(3, tclock());
      TRACE(5, sel->nseg);
    }
    if (sel->stop) {
      stop = sel->stop;
      break;
    }
    // ---- B. residual update: segments of SEG tiles of the owned rows ---------------
    const int stampv = (int)(it + 1);
    {
      const double tre = sel->tre, tim = sel->tim;
      const bool selfc = sel->selfc != 0;
      const int nseg = sel->nseg, nrows = sel->nrows;
      if (rank == 0 && warp == NW - 1 && lane == 0 && P.sol) {  // solution c(p) += c~ (Alg. 1 step 2a)
        const DictGeo& du = sd[sel->u];
        double2* s = P.sol + du.off + (long long)sel->j * du.MR + sel->k;
        double2 c = *s;
        c.x += tre;
        c.y += tim;
        *s = c;
      }
      for (int sid = warp; sid < nseg; sid += NW) {
        // owning row: the last row whose first segment is <= sid (rows are ordered)
        int ri = 0;
        for (int base = 0; base < nrows; base += 32) {
          const int c = base + lane;
          const bool le = c < nrows && rows[c].seg0 <= sid;
          ri += __popc(__ballot_sync(0xffffffffu, le));
        }
        ri -= 1;
        const RowDesc d = rows[ri];
        const int sg = sid - d.seg0;
        const int tbeg = sg * SEG, tend = min(tbeg + SEG, d.Tr);
        const double2 w = roots[d.rr * d.rstep];
        C2 z0;
        z0.x = (R)(tre * w.x - tim * w.y);
        z0.y = (R)(tre * w.y + tim * w.x);
        const C2* hrow = kern + d.krow;
        C2* row = grid + d.grow;
        C2 cv[SEG][NCH], hd[SEG][NCH], hc[SEG][NCH];
        bool fd[SEG][NCH], fc[SEG][NCH], cf[SEG][NCH];
#pragma unroll
        for (int s = 0; s < SEG; ++s) {   // every load of the segment first
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int bin = ((d.t0 + tbeg + s) << LGTW) + ch * 32 + lane;
            const bool valid = tbeg + s < tend && bin < d.MR;
            const int cd = (bin - d.q0) & d.Mmask;          // direct source column  (q = bin)
            const int cc = (-bin - d.q0) & d.Mmask;         // conjugate source column (q = M - bin)
            fd[s][ch] = valid && cd < d.nc;
            fc[s][ch] = valid && !selfc && cc < d.nc;
            cf[s][ch] = cc < cd;                            // oracle order: ascending column
            cv[s][ch] = valid ? row[bin] : C2{0, 0};
            hd[s][ch] = fd[s][ch] ? hrow[cd] : C2{0, 0};
            hc[s][ch] = fc[s][ch] ? hrow[cc] : C2{0, 0};
          }
        }
#pragma unroll
        for (int s = 0; s < SEG; ++s) {
          if (tbeg + s >= tend) break;
          R bs = 0, bre = 0, bim = 0;
          uint32_t bp = NO_INDEX;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int bin = ((d.t0 + tbeg + s) << LGTW) + ch * 32 + lane;
            C2 c = cv[s][ch];
            // z = z0 h;  direct: c -= z;  conjugate: c -= conj(z)
            const R zdx = z0.x * hd[s][ch].x - z0.y * hd[s][ch].y, zdy = z0.x * hd[s][ch].y + z0.y * hd[s][ch].x;
            const R zcx = z0.x * hc[s][ch].x - z0.y * hc[s][ch].y, zcy = z0.x * hc[s][ch].y + z0.y * hc[s][ch].x;
            if (fc[s][ch] && cf[s][ch]) {
              c.x -= zcx;
              c.y += zcy;
            }
            if (fd[s][ch]) {
              c.x -= zdx;
              c.y -= zdy;
            }
            if (fc[s][ch] && !cf[s][ch]) {
              c.x -= zcx;
              c.y += zcy;
            }
            if (fd[s][ch] || fc[s][ch]) row[bin] = c;
            if (bin < d.MR) {
              const R sc = ScoreOps<R>::score(c.x, c.y);
              const uint32_t pp = d.pbase + (uint32_t)bin;
              if (better(sc, pp, bs, bp)) {
                bs = sc;
                bp = pp;
                bre = c.x;
                bim = c.y;
              }
            }
          }
          R ws;
          uint32_t wp;
          const int wl = warp_argmax(bs, bp, ws, wp);
          if (lane == wl) {
            RecT rec;
            rec.s = bs;
            rec.re = bre;
            rec.im = bim;
            rec.p = bp;
            if constexpr (sizeof(R) == 8) rec.pad = 0;
            trec[d.lbase + tbeg + s] = rec;
          }
        }
      }
    }
    PROF_MARK(2);
    if (lane == 0) TRACE(8 + warp, tclock());
    __syncthreads();
    PROF_MARK(3);
    // ---- C. level-1 refresh: the nodes spanned by the owned rows ---------------------
    {
      const int nnode = sel->nnode, nrows = sel->nrows;
      for (int q = warp; q < nnode; q += NW) {
        int ri = 0;
        for (int base = 0; base < nrows; base += 32) {
          const int c = base + lane;
          ri += __popc(__ballot_sync(0xffffffffu, c < nrows && rows[c].ndbase <= q));
        }
        ri -= 1;
        const int node = rows[ri].nd0 + (q - rows[ri].ndbase);
        warp_node(trec, P.Lc, node, lev, lane);
      }
    }
    __syncthreads();
    PROF_MARK(4);
    if (warp == 0 && lane == 0) TRACE(7, tclock());
    // ---- D. upper levels, top scan, publish (warp 0) -----------------------------------
    if (warp == 0) {
      const int nrows = sel->nrows;
      for (int l = 1; l < P.nlev; ++l) {   // level l nodes spanned by the rows, in order
        const int sh = 5 * (l + 1);
        int last = -1;   // skip immediate repeats (adjacent rows share nodes); repeats are harmless
        for (int i = 0; i < nrows; ++i) {
          const RowDesc& d = rows[i];
          const int lo = d.lbase >> sh, hi = (d.lbase + d.Tr - 1) >> sh;
          for (int node = lo; node <= hi; ++node) {
            if (node == last) continue;
            warp_node(lev + P.lev_off[l - 1], (long long)P.lev_n[l - 1], node, lev + P.lev_off[l], lane);
            __syncwarp();
            last = node;
          }
        }
      }
      publish_root(par ^ 1);
      if (lane == 0) {
        TRACE(4, tclock());
        for (int l = 0; l < P.nlev; ++l) cnt[l] = 0;
      }
    }
    PROF_MARK(5);
  }
  if (rank == 0 && threadIdx.x == 0) {
    P.result->n_done = it;
    P.result->stop = stop;
    P.result->E_final = sel->E[it & 1];
  }
  if (prof) {
    for (int i = 0; i < 7; ++i) P.prof[i] = ph[i];
    P.prof[7] = it;
  }
#undef PROF_MARK
#undef TRACE
  __syncthreads();
  cluster.sync();  // keep every CTA's shared memory alive until all remote stores are done
}

inline cudaLaunchConfig_t cluster_cfg(int C, int threads, size_t smem, cudaStream_t st, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

template <typename R, int TW, bool SREC>
cudaError_t launch_t(const LoopParams& P, int threads, cudaStream_t st) {
  const void* kfn = (const void*)mp_lean_kernel<R, TW, SREC>;
  CUDA_OK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_bytes));
  if (P.C > 8) CUDA_OK(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = cluster_cfg(P.C, threads, P.smem_bytes, st, attr);
  void* args[] = {const_cast<LoopParams*>(&P)};
  return cudaLaunchKernelExC(&cfg, kfn, args);
}

template <typename R, int TW, bool SREC>
int max_cluster_t(int threads, size_t smem) {
  const void* kfn = (const void*)mp_lean_kernel<R, TW, SREC>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int c = MAX_CLUSTER; c >= 1; c >>= 1) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = cluster_cfg(c, threads, smem, 0, attr);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) == cudaSuccess && n > 0) return c;
    cudaGetLastError();
  }
  return 0;
}

template <typename R, bool SREC>
cudaError_t launch_r(const LoopParams& P, int threads, cudaStream_t st) {
  switch (P.TW) {
    case 32: return launch_t<R, 32, SREC>(P, threads, st);
    case 64: return launch_t<R, 64, SREC>(P, threads, st);
    case 128: return launch_t<R, 128, SREC>(P, threads, st);
  }
  return cudaErrorInvalidValue;
}
template <typename R, bool SREC>
int max_cluster_r(int TW, int threads, size_t smem) {
  switch (TW) {
    case 32: return max_cluster_t<R, 32, SREC>(threads, smem);
    case 64: return max_cluster_t<R, 64, SREC>(threads, smem);
    case 128: return max_cluster_t<R, 128, SREC>(threads, smem);
  }
  return 0;
}

}  // namespace

size_t lean_smem_bytes(const LoopParams& P, bool f64) {
  return smem_layout(P, f64 ? sizeof(Rec<double>) : sizeof(Rec<float>)).total;
}

cudaError_t launch_lean_loop(const LoopParams& P, bool f64, int threads, cudaStream_t st) {
  if (f64) return P.srec ? launch_r<double, true>(P, threads, st) : launch_r<double, false>(P, threads, st);
  return P.srec ? launch_r<float, true>(P, threads, st) : launch_r<float, false>(P, threads, st);
}

int lean_max_cluster(bool f64, bool srec, int TW, int threads, size_t smem) {
  if (f64) return srec ? max_cluster_r<double, true>(TW, threads, smem) : max_cluster_r<double, false>(TW, threads, smem);
  return srec ? max_cluster_r<float, true>(TW, threads, smem) : max_cluster_r<float, false>(TW, threads, smem);
}
