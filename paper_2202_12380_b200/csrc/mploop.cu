// mploop.cu -- N3 + N4 + N5: the persistent coefficient-domain matching pursuit loop.
//
// One thread-block cluster of C CTAs (one CTA per SM, C <= 16, a power of two)
// runs every iteration of Alg. 1 (approximate recursion Eq. (9)
// P:424-434) without returning to the host.  Per iteration:
//
//   A  (warp 0)   read the C per-CTA roots from the local mailbox (pushed by
//                 every CTA through distributed shared memory), argmax with
//                 redux.sync (score desc, index asc -- DESIGN.md Z10), stop tests
//                 (Z15), scalar step: rho from the auto-kernel, c~
//                 (Eq. (19), reading Z11), E~ (Eq. (20)); lane v computes the
//                 update geometry of target dictionary v (all power-of-two
//                 shift/mask arithmetic); rank 0 appends the atom.
//   B  (all)      Alg. 3: every touched tile (TW bins of one frame
//                 row) owned by this CTA (tile id g, owner g mod C) is loaded once
//                 by one warp, the subsampled, modulated cross-kernel entries
//                 (Eqs. (15)-(17)) are applied with the fold rule (Z14), touched
//                 bins are stored and the tile's new best is reduced in registers.
//   C  (all)      dirty level-1 nodes (32 tiles each) are re-reduced.
//   D  (warp 0)   dirty upper nodes, top scan, and the new root is pushed into
//                 every CTA's mailbox; one cluster barrier ends the iteration.
//
// Every coefficient is touched only by its tile's owner CTA, so the update needs
// no atomics and no second cluster barrier.  The run is deterministic.
#include <algorithm>
#include <cooperative_groups.h>
#include "loopcore.cuh"

namespace cg = cooperative_groups;

namespace {

using namespace mpcore;

struct Sel {            // the selection of the current iteration, published by warps 0 and 1
  double tre, tim;
  double E[2];          // E_k in E[k & 1] (double-buffered: read and written in the same phase)
  int u, k, j, selfc, stop, total;
};

struct Smem {
  size_t mbar, mail, trec, lev, sel, vg, own, pairs, dicts, roots, rho, rho_meta, stamp, list, cnt, total;
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
  o += sizeof(Sel);
  s.vg = o;
  o += sizeof(VGeo) * P.W;
  o = align_up(o, 16);
  s.own = o;
  o += sizeof(OwnGeo) * P.W;
  o = align_up(o, 16);
  s.pairs = o;
  o += sizeof(PairGeo) * P.W * P.W;
  o = align_up(o, 16);
  s.dicts = o;
  o += sizeof(DictGeo) * P.W;
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

// global-exchange helpers (GX): a CTA's root record and its iteration stamp in global
// memory; the stamp is written with release and polled with acquire semantics (gpu scope)
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// GX = false: one thread-block cluster of C <= 16 CTAs exchanging roots through
// distributed shared memory.  GX = true: a cooperative grid of C CTAs (C a power of
// two up to 128, one per SM) exchanging roots through global memory (release/acquire
// stamps); everything else is identical.
// PED: pedantic selection scores (compile-time, so the default path has no trace of it)
template <typename R, int TW, bool SREC, bool GX, bool PED>
__global__ void __launch_bounds__(512, 1) mp_loop_kernel(const LoopParams P) {
  using C2 = typename cplx<R>::t;
  using RecT = Rec<R>;
  const int C = P.C, lgC = ilog2(P.C);
  const int rank = GX ? (int)blockIdx.x : (int)cg::this_cluster().block_rank();
  const int W = P.W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  constexpr int LGTW = TW == 32 ? 5 : (TW == 64 ? 6 : 7);
  constexpr int NCH = TW / 32;

  extern __shared__ __align__(32) unsigned char smem[];
  const Smem L = smem_layout(P, sizeof(RecT));
  RecT* mail = reinterpret_cast<RecT*>(smem + L.mail);
  RecT* lev = reinterpret_cast<RecT*>(smem + L.lev);
  Sel* sel = reinterpret_cast<Sel*>(smem + L.sel);
  VGeo* vg = reinterpret_cast<VGeo*>(smem + L.vg);
  OwnGeo* sown = reinterpret_cast<OwnGeo*>(smem + L.own);
  PairGeo* sp = reinterpret_cast<PairGeo*>(smem + L.pairs);
  DictGeo* sd = reinterpret_cast<DictGeo*>(smem + L.dicts);
  const double2* roots = P.Rmax <= 4096 ? reinterpret_cast<const double2*>(smem + L.roots) : P.roots;
  RhoEnt* srho = reinterpret_cast<RhoEnt*>(smem + L.rho);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  int* rho_lo = reinterpret_cast<int*>(smem + L.rho_meta);
  int* rho_n = rho_lo + W;
  int* rho_off = rho_n + W;
  int* stamp = reinterpret_cast<int*>(smem + L.stamp);
  int* list = reinterpret_cast<int*>(smem + L.list);
  int* cnt = reinterpret_cast<int*>(smem + L.cnt);
  // batched independent signals: cluster `slot` works on signal `slot` (its own grids,
  // records, atoms, energies and result; the kernels are shared)
  const int slot = GX ? 0 : (int)(blockIdx.x / (unsigned)C);
  const double E0s = P.E0v ? P.E0v[slot] : P.E0;
  const double Etols = P.etol_mode == 1 ? P.etol_val * E0s : (P.etol_mode == 2 ? P.etol_val : -INFINITY);
  if (P.nonfinite != nullptr && *P.nonfinite) {  // x holds NaN/Inf: report, run nothing (uniform exit)
    if (rank == 0 && threadIdx.x == 0) {
      P.result[slot].n_done = 0;
      P.result[slot].stop = STOP_NONFINITE;
      P.result[slot].E_final = E0s;
      P.result[slot].rounds = 0;
      P.result[slot].E0 = E0s;
    }
    return;
  }
  AtomOut* atoms_out = P.atoms + (long long)slot * P.slot_atoms;
  double* energy_out = P.energy + (long long)slot * (P.slot_atoms + 1);
  RecT* grec = reinterpret_cast<RecT*>(P.rec) + (long long)slot * C * P.Lc + (long long)rank * P.Lc;
  RecT* trec = SREC ? reinterpret_cast<RecT*>(smem + L.trec) : grec;
  C2* grid = reinterpret_cast<C2*>(P.grid) + (long long)slot * P.slot_grid;
  const C2* kern = reinterpret_cast<const C2*>(P.kern);

  // ---- load tables -------------------------------------------------------
  for (int i = threadIdx.x; i < W * W; i += blockDim.x) sp[i] = P.pairs[i];
  for (int i = threadIdx.x; i < W; i += blockDim.x) {
    sd[i] = P.dicts[i];
    sown[i] = P.own[rank * W + i];
    rho_lo[i] = P.rho_lo[i];
    rho_n[i] = P.rho_n[i];
    rho_off[i] = P.rho_off[i];
  }
  if (P.Rmax <= 4096)
    for (int i = threadIdx.x; i < P.Rmax; i += blockDim.x)
      reinterpret_cast<double2*>(smem + L.roots)[i] = P.roots[i];
  for (int i = threadIdx.x; i < P.rho_total; i += blockDim.x) srho[i] = P.rho[i];
  int levtot = 0;
  for (int l = 0; l < P.nlev; ++l) levtot += P.lev_n[l];
  for (int i = threadIdx.x; i < levtot; i += blockDim.x) stamp[i] = 0;
  if (threadIdx.x < MAX_LEVELS) cnt[threadIdx.x] = 0;
  if (SREC)
    for (long long i = threadIdx.x; i < P.Lc; i += blockDim.x) trec[i] = grec[i];
  __syncthreads();

  // ---- build the node levels and the first root --------------------------
  for (int i = warp; i < P.lev_n[0]; i += NW) warp_node(trec, P.Lc, i, lev, lane);
  __syncthreads();
  for (int l = 1; l < P.nlev; ++l) {
    for (int i = warp; i < P.lev_n[l]; i += NW)
      warp_node(lev + P.lev_off[l - 1], (long long)P.lev_n[l - 1], i, lev + P.lev_off[l], lane);
    __syncthreads();
  }
  // mailbox barriers: slot s completes once all C roots (C * sizeof(Rec) bytes) arrived
  const uint32_t recbytes = (uint32_t)sizeof(RecT);
  if (threadIdx.x == 0) {
    mbar_init(smem_addr(&mbar[0]), 1);
    mbar_init(smem_addr(&mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(smem_addr(&mbar[0]), C * recbytes);
    mbar_arm(smem_addr(&mbar[1]), C * recbytes);
    sel->E[0] = E0s;
    sel->stop = 0;
  }
  if constexpr (GX) __syncthreads();
  else cg::this_cluster().sync();
  // warp 0: scan the top level, push the root into slot `slot` of every CTA's mailbox
  unsigned long long stampnext = 1;  // GX: stamp of the root published next (= iteration + 1)
  auto publish_root = [&](int slot) {
    const int top = P.nlev - 1;
    const RecT* tl = lev + P.lev_off[top];
    RecT b = empty_rec(R(0));
    for (int i = lane; i < P.lev_n[top]; i += 32) {
      const RecT r = tl[i];
      if (better(r.s, r.p, b.s, b.p)) b = r;
    }
    b = warp_best(b);
    if constexpr (GX) {
      if (lane == 0) {  // record, then its stamp (release): iteration `stamp - 1` may read it
        reinterpret_cast<RecT*>(P.gx_rec)[slot * C + rank] = b;
        st_release_u64(P.gx_stamp + slot * C + rank, stampnext);
      }
    } else if (lane < C) {
      push_record(b, mapa(smem_addr(&mail[slot * MAX_CLUSTER + rank]), lane), mapa(smem_addr(&mbar[slot]), lane));
    }
  };
  if (warp == 0) publish_root(0);
  long long it = 0;
  int stop = 0;
  const bool prof = P.prof != nullptr && rank == 0 && slot == 0 && threadIdx.x == 0;
  long long ph[7] = {0, 0, 0, 0, 0, 0, 0};
#define PROF_MARK(i)                \
  if (prof) {                        \
    const long long tn = clock64(); \
    ph[i] += tn - tprev;             \
    tprev = tn;                      \
  }
  long long tprev = clock64();
  for (;; ++it) {
    const int par = (int)(it & 1);
    // ---- A. selection (warps 0, 1); scalar step (warp 0); geometry (warp 1) ----
    if (!GX && warp < 2) mbar_wait(smem_addr(&mbar[par]), (uint32_t)((it >> 1) & 1));
    if (GX && warp < 2) {  // every CTA's root of this iteration: stamps == it + 1
      const unsigned long long want = (unsigned long long)it + 1;
      for (int c = lane; c < C; c += 32) {
        const long long t0 = clock64();
        while (ld_acquire_u64(P.gx_stamp + par * C + c) != want) {
          spin_check(t0);
        }
      }
      __syncwarp();
    }
    PROF_MARK(0);
    if (warp < 2) {
      RecT cand = empty_rec(R(0));
      if constexpr (GX) {
        for (int c = lane; c < C; c += 32) {
          const RecT r = reinterpret_cast<const RecT*>(P.gx_rec)[par * C + c];
          if (better(r.s, r.p, cand.s, cand.p)) cand = r;
        }
      } else {
        if (lane < C) cand = mail[par * MAX_CLUSTER + lane];
        if (warp == 0 && lane == 0) mbar_arm(smem_addr(&mbar[par]), C * recbytes);  // slot reused at it + 2
      }
      const RecT best = warp_best(cand);
      const double Ecur = sel->E[par];
      int st = 0;
      if (it >= P.maxit) st = 1;
      else if (Ecur <= Etols) st = 2;
      else if (Ecur < 0.0) st = 3;
      else if (!(best.s > (R)0)) st = 4;
      if (st) {
        if (warp == 0 && lane == 0) sel->stop = st;
      } else {
        // decode p = off_u + j * MR_u + k
        const uint32_t p = best.p;
        const int u = __popc(__ballot_sync(0xffffffffu, lane > 0 && lane < W && (uint32_t)sd[lane].off <= p));
        const uint32_t q = p - (uint32_t)sd[u].off;
        const int MRu = sd[u].MR;
        const int j = (int)(q / (uint32_t)MRu);
        const int k = (int)(q - (uint32_t)j * (uint32_t)MRu);
        const int Mu = sd[u].M;
        if (warp == 0) {
          const bool selfc = (k == 0) || (2 * k == Mu);
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
              inv = rv.inv;                                  // 1 / (1 - |rho|^2)
            }
            const double nre = cre - (rre * cre - rim * cim);
            const double nim = cim + (rre * cim + rim * cre);
            tre = nre * inv;
            tim = nim * inv;
            const double X2 = tre * tre, Y2 = tim * tim, XY = tre * tim;
            Et = 2.0 * (X2 + Y2 + rre * (X2 - Y2) - 2.0 * rim * XY);
          }
          // (latency-floor mode: no update, so the energy is not reduced either -- the floor run
          // does exactly the requested selections, whatever the atom energies)
          const double En = P.floor_mode ? Ecur : Ecur - Et;
          if (lane == 0) {
            sel->tre = tre;
            sel->tim = tim;
            sel->E[par ^ 1] = En;
            sel->u = u;
            sel->k = k;
            sel->j = j;
            sel->selfc = selfc ? 1 : 0;
            sel->stop = 0;
            if (rank == 0) {
              AtomOut a;
              a.w = u;
              a.m = k;
              a.n = j;
              a.flags = selfc ? 1 : 0;
              a.re = tre;
              a.im = tim;
              atoms_out[it] = a;
              energy_out[it + 1] = En;
            }
          }
        } else {
          // lane v: geometry of target dictionary v (Alg. 3 index sets)
          int nitems = 0;
          VGeo g;
          if (lane < W) nitems = vgeo<LGTW>(sp[u * W + lane], sd[u], sd[lane], k, j, rank, C, lgC, g);
          int incl = nitems;  // exclusive scan of the item counts over lanes
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (lane < W) {
            g.base = incl - nitems;
            vg[lane] = g;
          }
          const int total = __shfl_sync(0xffffffffu, incl, 31);
          if (lane == 0) sel->total = P.floor_mode ? 0 : total;
        }
      }
    }
    PROF_MARK(1);
    __syncthreads();
    PROF_MARK(2);
    if (sel->stop) {
      stop = sel->stop;
      break;
    }
    // ---- B. residual update over the owned touched tiles ------------------
    const int stampv = (int)(it + 1);
    {
      const double tre = sel->tre, tim = sel->tim;
      const int u = sel->u;
      const bool selfc = sel->selfc != 0;
      const int total = sel->total;
      if (rank == 0 && warp == NW - 1 && lane == 0 && P.sol) {  // solution c(p) += c~ (Alg. 1 step 2a)
        const DictGeo du = sd[u];
        double2* s = P.sol + du.off + (long long)sel->j * du.MR + sel->k;
        double2 c = *s;
        c.x += tre;
        c.y += tim;
        *s = c;
      }
      // item ends of the target dictionaries in lanes v < W (items are v-major)
      const int vend = lane < W ? vg[lane].base + vg[lane].nitems : 0x7fffffff;
      for (int gi = warp; gi < total; gi += NW) {
        const int v = __popc(__ballot_sync(0xffffffffu, gi >= vend));
        const VGeo& g = vg[v];
        const DictGeo& dv = sd[v];
        const PairGeo& pg = sp[u * W + v];
        const int loc = gi - g.base;
        const int i = (int)((unsigned)loc / (unsigned)g.Tr), tt = loc - i * g.Tr;
        const int r = i < g.cntA ? g.rhoA + (i << lgC) : g.rA + g.rhoB + ((i - g.cntA) << lgC);
        int nrow = g.n0 + r;
        if (nrow >= dv.N) nrow -= dv.N;
        const int t = g.t0 + tt;
        const int l = sown[v].loc_base + ((nrow - sown[v].n_first) >> lgC) * dv.T + t;
        // modulation omega_R^{(k' nu) mod R} of this row (Eq. (15))
        const int rr = (g.rr0 + r * g.rrstep) & (pg.R - 1);
        const double2 w = roots[rr * pg.rstep];
        const C2 z0 = row_z0<C2, R>(tre, tim, w);
        const C2* hrow = kern + g.kbase + (long long)r * g.nc;
        C2* row = grid + dv.grid_off + (long long)nrow * dv.stride;
        const int Mv = dv.M;
        C2 cv[NCH], hd[NCH], hc[NCH];
        bool fd[NCH], fc[NCH], cfirst[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {  // issue every load of the tile before any store
          const int bin = t * TW + ch * 32 + lane;
          const bool valid = bin < dv.MR;
          const int cd = (bin - g.q0) & (Mv - 1);          // direct source column  (q = bin)
          const int cc = (-bin - g.q0) & (Mv - 1);         // conjugate source column (q = M - bin)
          fd[ch] = valid && cd < g.nc;
          fc[ch] = valid && !selfc && cc < g.nc;
          cfirst[ch] = cc < cd;                            // oracle order: ascending source column
          cv[ch] = valid ? row[bin] : C2{0, 0};
          hd[ch] = fd[ch] ? hrow[cd] : C2{0, 0};
          hc[ch] = fc[ch] ? hrow[cc] : C2{0, 0};
        }
        R bs = 0;
        uint32_t bp = NO_INDEX;
        R bre = 0, bim = 0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int bin = t * TW + ch * 32 + lane;
          // z = z0 h;  direct: c -= z;  conjugate: c -= conj(z)   (fold rule Z14)
          const C2 c = fold_update<R>(cv[ch], z0, hd[ch], hc[ch], fd[ch], fc[ch], cfirst[ch]);
          if (bin < dv.MR) {
            if (fd[ch] || fc[ch]) row[bin] = c;
            const R s = sel_score<R>(c.x, c.y, bin, dv.M, PED, srho + rho_off[v], rho_lo[v], rho_n[v]);
            const uint32_t p = (uint32_t)dv.off + (uint32_t)nrow * (uint32_t)dv.MR + (uint32_t)bin;
            if (better(s, p, bs, bp)) {
              bs = s;
              bp = p;
              bre = c.x;
              bim = c.y;
            }
          }
        }
        if (lane == warp_argmax_lane(bs, bp)) {
          RecT rec;
          rec.s = bs;
          rec.re = bre;
          rec.im = bim;
          rec.p = bp;
          if constexpr (sizeof(R) == 8) rec.pad = 0;
          trec[l] = rec;
          const int node = l >> 5;
          if (atomicExch(&stamp[node], stampv) != stampv) list[atomicAdd(&cnt[0], 1)] = node;
        }
      }
    }
    PROF_MARK(3);
    __syncthreads();
    PROF_MARK(4);
    // ---- C. level-1 refresh -------------------------------------------------
    {
      const int n1 = cnt[0];
      for (int idx = warp; idx < n1; idx += NW) {
        const int node = list[idx];
        const long long c = (long long)node * 32 + lane;
        const RecT r = c < P.Lc ? trec[c] : empty_rec(R(0));
        if (lane == warp_argmax_lane(r.s, r.p)) {
          lev[node] = r;
          if (P.nlev > 1) {
            const int par2 = node >> 5;
            int* st2 = stamp + P.lev_off[1];
            if (atomicExch(&st2[par2], stampv) != stampv) list[P.lev_off[1] + atomicAdd(&cnt[1], 1)] = par2;
          }
        }
      }
    }
    __syncthreads();
    PROF_MARK(5);
    // ---- D. upper node levels.  Grid mode (GX, the very large grids with nlev > 1):
    //      one level at a time, the dirty nodes spread over the warps; one cluster:
    //      warp 0 alone (measured faster there)
    if constexpr (GX) {
      for (int l = 1; l < P.nlev; ++l) {
        const int nl = cnt[l];
        for (int idx = warp; idx < nl; idx += NW) {
          const int node = list[P.lev_off[l] + idx];
          const int c = node * 32 + lane;
          const RecT r = c < P.lev_n[l - 1] ? lev[P.lev_off[l - 1] + c] : empty_rec(R(0));
          if (lane == warp_argmax_lane(r.s, r.p)) {
            lev[P.lev_off[l] + node] = r;
            if (l + 1 < P.nlev) {
              const int par2 = node >> 5;
              int* st2 = stamp + P.lev_off[l + 1];
              if (atomicExch(&st2[par2], stampv) != stampv) list[P.lev_off[l + 1] + atomicAdd(&cnt[l + 1], 1)] = par2;
            }
          }
        }
        __syncthreads();
      }
    }
    // ---- D. upper levels, top scan, publish root (warp 0) ------------------
    if (warp == 0) {
      for (int l = 1; l < (GX ? 1 : P.nlev); ++l) {
        const int nl = cnt[l];
        for (int idx = 0; idx < nl; ++idx) {
          const int node = list[P.lev_off[l] + idx];
          const int c = node * 32 + lane;
          const RecT r = c < P.lev_n[l - 1] ? lev[P.lev_off[l - 1] + c] : empty_rec(R(0));
          if (lane == warp_argmax_lane(r.s, r.p)) {
            lev[P.lev_off[l] + node] = r;
            if (l + 1 < P.nlev) {
              const int par2 = node >> 5;
              int* st2 = stamp + P.lev_off[l + 1];
              if (atomicExch(&st2[par2], stampv) != stampv) list[P.lev_off[l + 1] + atomicAdd(&cnt[l + 1], 1)] = par2;
            }
          }
          __syncwarp();
        }
      }
      stampnext = (unsigned long long)it + 2;
      publish_root(par ^ 1);
      if (lane == 0)
        for (int l = 0; l < P.nlev; ++l) cnt[l] = 0;
    }
    PROF_MARK(6);
  }
  if (rank == 0 && threadIdx.x == 0) {
    P.result[slot].n_done = it;
    P.result[slot].stop = stop;
    P.result[slot].E_final = sel->E[it & 1];
    P.result[slot].E0 = E0s;
  }
  if (prof) {
    for (int i = 0; i < 7; ++i) P.prof[i] = ph[i];
    P.prof[7] = it;
  }
#undef PROF_MARK
  if constexpr (!GX) cg::this_cluster().sync();  // keep shared memory alive until all remote stores are done
}

template <typename R, int TW, bool SREC, bool GX>
cudaError_t launch_t(const LoopParams& P, int threads, cudaStream_t st) {
  auto kfn = P.pedantic ? mp_loop_kernel<R, TW, SREC, GX, true> : mp_loop_kernel<R, TW, SREC, GX, false>;
  CUDA_OK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_bytes));
  if (!GX && P.C > 8) CUDA_OK(cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.C * (GX ? 1 : std::max(1, P.nslot)), 1, 1);   // one cluster per signal
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = P.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (GX) {  // all CTAs co-resident: they spin on each other's stamps
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  } else {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P.C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kfn, P);
}

template <typename R, int TW, bool SREC>
int max_cluster_t(int threads, size_t smem) {
  auto kfn = mp_loop_kernel<R, TW, SREC, false, false>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
      cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int c = MAX_CLUSTER; c >= 1; c >>= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kfn, &cfg) == cudaSuccess && n > 0) return c;
    cudaGetLastError();
  }
  return 0;
}

// co-resident CTAs of the global-exchange kernel (one per SM at most)
template <typename R, int TW, bool SREC>
int max_grid_t(int threads, size_t smem) {
  auto kfn = mp_loop_kernel<R, TW, SREC, true, false>;
  if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, threads, smem) != cudaSuccess ||
      cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * sms;
}

template <typename R, bool SREC, bool GX>
cudaError_t launch_r(const LoopParams& P, int threads, cudaStream_t st) {
  switch (P.TW) {
    case 32: return launch_t<R, 32, SREC, GX>(P, threads, st);
    case 64: return launch_t<R, 64, SREC, GX>(P, threads, st);
    case 128: return launch_t<R, 128, SREC, GX>(P, threads, st);
  }
  return cudaErrorInvalidValue;
}
template <typename R, bool SREC>
int max_cluster_r(int TW, int threads, size_t smem, bool gx) {
  switch (TW) {
    case 32: return gx ? max_grid_t<R, 32, SREC>(threads, smem) : max_cluster_t<R, 32, SREC>(threads, smem);
    case 64: return gx ? max_grid_t<R, 64, SREC>(threads, smem) : max_cluster_t<R, 64, SREC>(threads, smem);
    case 128: return gx ? max_grid_t<R, 128, SREC>(threads, smem) : max_cluster_t<R, 128, SREC>(threads, smem);
  }
  return 0;
}

}  // namespace

size_t loop_smem_bytes(const LoopParams& P, bool f64) {
  return smem_layout(P, f64 ? sizeof(Rec<double>) : sizeof(Rec<float>)).total;
}

cudaError_t launch_mp_loop(const LoopParams& P, bool f64, int threads, cudaStream_t st) {
  const bool gx = P.gx_rec != nullptr;
  if (gx) {
    if (f64) return P.srec ? launch_r<double, true, true>(P, threads, st) : launch_r<double, false, true>(P, threads, st);
    return P.srec ? launch_r<float, true, true>(P, threads, st) : launch_r<float, false, true>(P, threads, st);
  }
  if (f64) return P.srec ? launch_r<double, true, false>(P, threads, st) : launch_r<double, false, false>(P, threads, st);
  return P.srec ? launch_r<float, true, false>(P, threads, st) : launch_r<float, false, false>(P, threads, st);
}

int loop_max_cluster(bool f64, bool srec, int TW, int threads, size_t smem, bool gx) {
  if (f64) return srec ? max_cluster_r<double, true>(TW, threads, smem, gx) : max_cluster_r<double, false>(TW, threads, smem, gx);
  return srec ? max_cluster_r<float, true>(TW, threads, smem, gx) : max_cluster_r<float, false>(TW, threads, smem, gx);
}
