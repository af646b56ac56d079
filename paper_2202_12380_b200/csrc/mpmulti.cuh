// mpmulti.cuh -- the exact multi-selection loop kernel (included by the mpmulti_*.cu
// translation units, one per precision and exchange mode, to build in parallel).
#pragma once
// mpmulti.cu -- exact multi-selection rounds of the coefficient-domain MP loop
// (DESIGN.md §8).
//
// The sequential loop of Alg. 1 (recursion Eq. (9)) spends
// almost all of its time in the dependency chain select -> update -> refresh ->
// select (mploop.cu).  Eq. (16)'s locality makes most
// consecutive selections independent: an update only changes the coefficients
// inside the kernel footprint of the selected atom.  A round therefore picks up
// to B atoms at once and proves, one round later, that they are exactly the
// atoms the sequential loop would have selected:
//
//   tiles(p)  the set of tiles (TW bins of one frame row) the update of atom p
//             reads and writes: in every target dictionary v the rows of the
//             kernel's alignment-class sub-box times the folded bin hull.
//   Round: p_1 = global argmax.  p_i (i >= 2) = the best coefficient outside
//   X_i = tiles(p_1) u ... u tiles(p_{i-1}) in the state before the round,
//   taken only if tiles(p_i) is disjoint from X_i.  All updates are applied
//   (they touch disjoint tiles, so each coefficient receives exactly the
//   arithmetic of the sequential loop), every CTA records per candidate the
//   largest post-update score over its tiles, and p_i is *accepted* iff that
//   maximum over X_i is below |c(p_i)|^2.  Then p_i is the sequential argmax
//   after p_1..p_{i-1}: outside X_i nothing changed and p_i is the best there,
//   inside X_i every value is smaller.  c(p_i) is unchanged by the earlier
//   updates (p_i is outside X_i), so c~ and E~ (Eqs. (19)-(20)) are the
//   sequential ones.  The comparison uses a conservative 32-bit score key
//   (equality rejects): it can only cause spurious rejections, never a wrong
//   acceptance.
//   Rejected candidates are rolled back bit-exactly in the next round from a
//   backup of their tiles (a copy, not an inverse update), and that round does
//   no selection.
//
// The candidates come from per-CTA top-K lists: at the end of a round every CTA
// extracts its K best tile records (exact, from its 32-ary max tree) and pushes
// them, with its per-candidate maxima, into every CTA's mailbox (st.async +
// mbarrier complete_tx, as in mploop.cu; in grid mode into global memory with a
// release stamp, see the kernel).  Every CTA then runs the same
// deterministic merge/walk: entries in descending (score, -index) order; an
// entry whose tile lies in X is skipped; passing the K-th entry of a CTA's list
// ends the walk (that CTA's unlisted tiles are unknown); the walk also ends at
// the first candidate whose tiles meet X, at the first candidate after a skipped
// entry (a heuristic: that entry likely still outscores it after the update, which
// would reject it), at a stop rule (Z15) or after B picks.
//
// Frame ownership, tile records, node tree and the per-tile update arithmetic
// are those of mploop.cu; the run is deterministic and its atom sequence is
// identical to the one-selection loop.
#include <cooperative_groups.h>
#include <type_traits>
#include "loopcore.cuh"

namespace cg = cooperative_groups;

namespace {

using namespace mpcore;

#ifndef MPG_NE
#define MPG_NE 8
#endif
#ifndef MPG_BMAX
#define MPG_BMAX 8
#endif
#ifndef MPG_LB_THREADS
#define MPG_LB_THREADS 512  // launch bound (max threads per CTA; 256 leaves 255 registers per thread)
#endif
#ifndef MPG_PUSH_WARPS
#define MPG_PUSH_WARPS 1  // publication: one 16-byte chunk per thread over the first warps (0: warp 0 alone)
#endif
#ifndef MPG_SCAN_W1
#define MPG_SCAN_W1 1     // the round's item bases by warp 1 while warp 0 runs the energy chain
#endif
#ifndef MPG_ECHAIN_BF
#define MPG_ECHAIN_BF 1   // the round's energy chain without branches (0: the branching form)
#endif
constexpr int NE = MPG_NE;      // walk window: best merged list entries considered per round
constexpr int BMAX = MPG_BMAX;  // candidates per round (upper bound; LoopParams::spec lowers it)
static_assert(BMAX == 8 || BMAX == 16, "candidate slots: 8 or 16");
static_assert(NE <= 16, "walk window <= 16 entries");
constexpr int IPL = BMAX * 16 / 32;  // (candidate, dictionary) item bases per lane
// tiles per work item (consecutive tiles of one row): 2, or MPG_TPI32 for 32-bin tiles
#ifndef MPG_TPI32
#define MPG_TPI32 2
#endif
template <int TW>
__host__ __device__ constexpr int tiles_per_item() { return TW == 32 ? MPG_TPI32 : 2; }
// update items in flight per warp for 32-bin tiles (1 or 2)
#ifndef MPG_ITEMS_IN_FLIGHT
#define MPG_ITEMS_IN_FLIGHT 1
#endif

template <typename R, int K>
struct Msg {              // published by every CTA to every CTA at the end of a round
  Rec<R> list[K];         // its K best tile records, (score desc, index asc)
  uint32_t vkey[BMAX];    // per candidate: max score key over the candidate's tiles owned by the CTA
#ifdef MPG_CHECKS
  uint32_t tag, pad_[3];  // debug builds: the round stamp the message was published with
#endif
};

struct Ent {              // one merged list entry of the walk window
  double tre, tim, Et;    // c~ (Eq. (19)) and E~ (Eq. (20)) if selected
  uint32_t key;           // score_key of |c|^2
  int u, k, j;            // dictionary, bin, frame
  int tile;               // k / TW
  int last;               // 1: the K-th entry of its CTA's list
  int pos;                // 1: |c|^2 > 0 and a real record
  int selfc;              // self-conjugate (k = 0 or M_u/2, Z13)
};

struct St {               // round state (shared memory)
  double E;               // E_k after the accepted atoms
  long long it;           // accepted atoms
  double Enext[BMAX];     // E after candidate g
  int G;                  // candidates of the round just run (verified by the next round)
  int Gw;                 // picks of the walk before the energy stop rules (>= G; warp 1's item bases)
  int mode;               // 0 select, 1 roll back candidates rb_from..G-1
  int rb_from;
  int stop;
  int pick[BMAX];         // walk-window position of candidate g (its egeo row)
  uint32_t ckey[BMAX];    // score key of candidate g
  alignas(16) int ibase[BMAX * 16 + 4];  // this CTA's items (tile pairs) before (g, v), index g * 16 + v
  alignas(16) int tbase[BMAX * 16 + 4];  // this CTA's tiles (backup slots) before (g, v)
};

struct TkE {              // a top-K candidate: order key, index, id (tile; -1 = none)
  uint64_t key;
  uint32_t p;
  int id;
};

struct Smem {
  size_t mbar, mail, mymsg, trec, lev, ent, egeo, wmask, rect, ecnt, st, vkey, sorted, hsel, tk, wk, stamp, list, cnt, pairs, dicts, own, roots,
      rho, rho_meta, cls, clid, hist, inl, rcp, hk, nmax, total;
};

// Candidate list of a CTA (top-K mode 2): the tiles whose score key is >= theta, held
// across rounds.  Invariant: every tile NOT in the list has key < theta, so the K best
// list entries are the CTA's exact top K whenever at least K entries remain (or theta
// is the smallest positive key: the CTA has fewer than K positive tiles, and empty
// records stand for its zero tiles).  A round only adds the tiles its items rewrote and
// that reach theta, and drops entries that fell below it; when fewer than K remain (or
// the list overflows) it is rebuilt by a radix select of theta over all tile records.
constexpr int CL_CAP = 128;      // list capacity (4 entries per lane of one warp)
#ifndef MPG_CL_TARGET
#define MPG_CL_TARGET 48
#endif
constexpr int CL_TARGET = MPG_CL_TARGET;  // entries a rebuild aims at
struct ClState {
  uint64_t theta;                // list threshold (order key of the score, >= 1)
  uint64_t prefix;               // radix select: key prefix of the current range
  int n;                         // entries (may exceed CL_CAP: overflow -> rebuild)
  int above;                     // radix select: entries above the current range
  int done;                      // radix select finished
  int valid;                     // 0: the rebuild could not make an exact list (ties) -> scan
  int need;                      // 1: the list could not give the exact top K (scan), rebuild it
  int soon;                      // 1: fewer than CL_LOW entries left -- rebuild after the publications
  int stage;                     // staged rebuild: 0 idle, 1 node maxima taken, 2 threshold chosen
  int pad_;
  uint64_t pend_theta;           // staged rebuild: the chosen threshold (order key)
};
#ifndef MPG_CL_LOW
#define MPG_CL_LOW 12
#endif
constexpr int CL_LOW = MPG_CL_LOW;   // list length below which the list is rebuilt pre-emptively
constexpr int CL_NBK = 256;          // rebuild: buckets of node maxima below the largest
constexpr int CL_BSH = 16;           //   of 2^16 in the upper score word each (1/16 octave of the score)

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
// items per row hp = ceil(hull tiles / tiles per item) <= ceil(257 / 2) (M <= 16384, TW >= 32)
constexpr int RCP_N = 256;


__host__ __device__ inline Smem smem_layout(const LoopParams& P, size_t recsz, size_t msgsz) {
  Smem s;
  int levtot = 0;
  for (int l = 0; l < P.nlev; ++l) levtot += P.lev_n[l];
  size_t o = 0;
  s.mbar = o;
  o += 32;
  s.mail = o;
  o += P.gx ? (size_t)P.C * msgsz : 2 * MAX_CLUSTER * msgsz;  // grid mode: one copy of the C messages
  s.mymsg = o;
  o += msgsz;
  s.trec = o;
  o += P.srec ? (size_t)P.Lc * recsz : 0;
  s.lev = o;
  o += (size_t)levtot * recsz;
  o = align_up(o, 16);
  s.ent = o;
  o += sizeof(Ent) * NE;
  o = align_up(o, 16);
  s.egeo = o;
  o += sizeof(VGeo) * NE * P.W;
  o = align_up(o, 16);
  s.wmask = o;
  o += sizeof(uint32_t) * 2 * NE;
  o = align_up(o, 16);
  s.rect = o;
  o += sizeof(uint2) * NE * P.W;
  o = align_up(o, 16);
  s.ecnt = o;                 // per (window entry, dictionary): this CTA's items and tiles
  o += sizeof(int2) * NE * 16;
  o = align_up(o, 16);
  s.st = o;
  o += sizeof(St);
  o = align_up(o, 16);
  s.vkey = o;
  o += sizeof(uint32_t) * BMAX;
  s.sorted = o;
  o += sizeof(int) * NE;
  s.hsel = o;                 // grid mode: the lists of the NE best heads
  o += sizeof(int) * NE;
  s.tk = o;
  o += sizeof(int) * 64;
  o = align_up(o, 16);
  s.wk = o;                   // scan top-K: warp winners (<= 16 warps x K) + the final K
  o += sizeof(TkE) * (64 + MULTI_K);
  s.stamp = o;
  o += sizeof(int) * levtot;
  s.list = o;
  o += sizeof(int) * levtot;
  s.cnt = o;
  o += sizeof(int) * MAX_LEVELS;
  o = align_up(o, 16);
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
  s.cls = o;
  o += P.topk_scan == 2 ? sizeof(ClState) : 0;
  s.clid = o;
  o += P.topk_scan == 2 ? sizeof(int) * CL_CAP : 0;
  s.hist = o;
  s.inl = o;
  o += P.topk_scan == 2 ? (size_t)P.Lc : 0;
  o = align_up(o, 16);
  s.rcp = o;                  // 0xFFFFFFFF / h + 1 for h < RCP_N (items per row -> row index by umulhi)
  o += sizeof(uint32_t) * RCP_N;
  s.hk = o;                   // candidate lists: upper 32 bits of every tile's score key
  o += P.topk_scan == 2 ? sizeof(uint32_t) * (size_t)P.Lc : 0;
  s.nmax = o;                 // candidate lists: node maxima of hk and their bucket counts (rebuilds)
  o += P.topk_scan == 2 ? sizeof(uint32_t) * (size_t)((P.Lc + 31) / 32 + CL_NBK + 1) : 0;
  s.total = align_up(o, 16);
  return s;
}

// One warp, one candidate per lane (64-bit order key, index p; empty: 0 / NO_INDEX):
// K pops of the warp-wide best (key desc, index asc), resolved on the upper key word
// and only on ties on the lower word / the index.  The winner of pop t writes
// out[t] = its id (-1 when empty).
template <int K>
__device__ __forceinline__ void warp_pop_k(uint64_t key, uint32_t p, int id, int* out, int lane) {
#pragma unroll
  for (int t = 0; t < K; ++t) {
    const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
    const uint32_t mhi = __reduce_max_sync(0xffffffffu, hi);
    unsigned m = __ballot_sync(0xffffffffu, hi == mhi);
    if (m & (m - 1)) {
      const uint32_t mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      m = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
      if (m & (m - 1)) {
        const bool in = (m >> lane) & 1u;
        const uint32_t mp = __reduce_min_sync(0xffffffffu, in ? p : NO_INDEX);
        m = __ballot_sync(0xffffffffu, in && p == mp);
      }
    }
    if (lane == __ffs(m) - 1) {
      out[t] = p == NO_INDEX ? -1 : id;
      key = 0;
      p = NO_INDEX;
    }
  }
}

// One warp, NC candidates per lane (lane holds candidates c * 32 + lane): the K best
// (key desc, index asc) by pops of the lanes' sorted heads -- no barrier, no merge.
// Writes the ids (-1 = none) to out[0..K-1].
template <int K, int NC>
__device__ __forceinline__ void warp_topk_nc(uint64_t (&k)[NC], uint32_t (&p)[NC], int (&id)[NC], int* out,
                                             int lane) {
  auto ce = [&](int a, int b) {  // compare-exchange: position a gets the better one
    const bool sw = (k[b] > k[a]) | ((k[b] == k[a]) & (p[b] < p[a]));
    const uint64_t tk = sw ? k[b] : k[a], uk = sw ? k[a] : k[b];
    const uint32_t tp = sw ? p[b] : p[a], up = sw ? p[a] : p[b];
    const int ti = sw ? id[b] : id[a], ui = sw ? id[a] : id[b];
    k[a] = tk; k[b] = uk; p[a] = tp; p[b] = up; id[a] = ti; id[b] = ui;
  };
  static_assert(NC == 1 || NC == 2 || NC == 4, "sorting network for 1, 2 or 4 candidates per lane");
  if constexpr (NC == 1) {
  } else if constexpr (NC == 2) {
    ce(0, 1);
  } else {
    ce(0, 1); ce(2, 3); ce(0, 2); ce(1, 3); ce(1, 2);
  }
#pragma unroll
  for (int t = 0; t < K; ++t) {
    const uint64_t key = k[0];
    const uint32_t pp = p[0];
    const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
    const uint32_t mhi = __reduce_max_sync(0xffffffffu, hi);
    unsigned m = __ballot_sync(0xffffffffu, hi == mhi);
    if (m & (m - 1)) {
      const uint32_t mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
      m = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
      if (m & (m - 1)) {
        const bool in = (m >> lane) & 1u;
        const uint32_t mp = __reduce_min_sync(0xffffffffu, in ? pp : NO_INDEX);
        m = __ballot_sync(0xffffffffu, in && pp == mp);
      }
    }
    const bool me = lane == __ffs(m) - 1;
    if (me) out[t] = pp == NO_INDEX ? -1 : id[0];
#pragma unroll
    for (int c = 0; c + 1 < NC; ++c) {  // the winner shifts its sorted list
      k[c] = me ? k[c + 1] : k[c];
      p[c] = me ? p[c + 1] : p[c];
      id[c] = me ? id[c + 1] : id[c];
    }
    k[NC - 1] = me ? 0ull : k[NC - 1];
    p[NC - 1] = me ? NO_INDEX : p[NC - 1];
  }
}

// Exact top-K tiles of this CTA down its node tree, by all warps: at every level
// the candidates are the children of the previous level's K winners (all nodes at
// the top level; the top-K nodes of a level contain the top-K of the level below),
// split in chunks of 32; warp q pops the K best of chunk q, warp 0 pops the K best
// of the chunk winners.  Leaves the tile ids (-1 = none) in tk[0..K-1]; tk[16..]
// holds the chunk winners.  Needs a barrier before; ends with one.
template <typename R, int K>
__device__ __forceinline__ void cta_topk(const LoopParams& P, const Rec<R>* lev, const Rec<R>* trec, int* tk,
                                         int lane, int warp, int NW) {
  static_assert(K * 8 <= 32, "the merge holds 8 chunks x K winners in one warp");
  int* part = tk + 16;
  const int top = P.nlev - 1;
  for (int l = top; l >= -1; --l) {
    const bool first = l == top;
    const int count = l >= 0 ? P.lev_n[l] : (int)P.Lc;
    const Rec<R>* arr = l >= 0 ? lev + P.lev_off[l] : trec;
    const int nq = first ? (count + 31) >> 5 : K;
    if (nq <= 4) {  // <= 128 candidates: warp 0 alone, 4 per lane (the other warps wait)
      if (warp == 0) {
        uint64_t kk[4];
        uint32_t pk[4];
        int ik[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          int id = c < nq ? (first ? c * 32 + lane : (tk[c] >= 0 ? tk[c] * 32 + lane : -1)) : -1;
          kk[c] = 0;
          pk[c] = NO_INDEX;
          if (id >= 0 && id < count) {
            kk[c] = skey64(arr[id].s);
            pk[c] = arr[id].p;
          } else {
            id = -1;
          }
          ik[c] = id;
        }
        __syncwarp();
        warp_topk_nc<K, 4>(kk, pk, ik, tk, lane);
        __syncwarp();
      }
      if (l == -1) __syncthreads();
      continue;
    }
    for (int q = warp; q < nq; q += NW) {  // chunk q (fewer warps than chunks: several each)
      int id = first ? q * 32 + lane : (tk[q] >= 0 ? tk[q] * 32 + lane : -1);
      uint64_t key = 0;
      uint32_t p = NO_INDEX;
      if (id >= 0 && id < count) {
        key = skey64(arr[id].s);
        p = arr[id].p;
      } else {
        id = -1;
      }
      warp_pop_k<K>(key, p, id, nq == 1 ? tk : part + q * K, lane);  // one chunk: no merge
    }
    __syncthreads();
    if (nq == 1) continue;
    if (warp == 0) {
      int id = lane < nq * K ? part[lane] : -1;
      uint64_t key = 0;
      uint32_t p = NO_INDEX;
      if (id >= 0) {
        key = skey64(arr[id].s);
        p = arr[id].p;
      }
      warp_pop_k<K>(key, p, id, tk, lane);
    }
    __syncthreads();
  }
}

// Exact top-K tiles of this CTA by a scan of all its tile records (records in shared
// memory, small slices): every lane keeps its K best of a strided share in a sorted
// register list (branch-free insertion), each warp pops its K best lane heads, warp 0
// pops the K best of the NW warps' lists.  No node tree is needed (the caller skips
// its upkeep).  Leaves the tile ids (-1 = none) in tk[0..K-1]; ends with a barrier.
template <typename R, int K>
__device__ __forceinline__ void cta_topk_scan(const Rec<R>* trec, long long Lc, int* tk, TkE* wk, int lane, int warp,
                                              int NW) {
  static_assert(K == 4, "sorted 4-lists");
  uint64_t k[4] = {0ull, 0ull, 0ull, 0ull};
  uint32_t p[4] = {NO_INDEX, NO_INDEX, NO_INDEX, NO_INDEX};
  int id[4] = {-1, -1, -1, -1};
  for (long long i = (long long)warp * 32 + lane; i < Lc; i += (long long)NW * 32) {
    const uint64_t kc = skey64(trec[i].s);
    const uint32_t pc = trec[i].p;
    const int ic = (int)i;
    bool b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = (kc > k[j]) | ((kc == k[j]) & (pc < p[j]));
#pragma unroll
    for (int j = 3; j >= 1; --j) {  // slot j takes slot j-1 if c beats it, c if c beats only slot j
      k[j] = b[j] ? (b[j - 1] ? k[j - 1] : kc) : k[j];
      p[j] = b[j] ? (b[j - 1] ? p[j - 1] : pc) : p[j];
      id[j] = b[j] ? (b[j - 1] ? id[j - 1] : ic) : id[j];
    }
    k[0] = b[0] ? kc : k[0];
    p[0] = b[0] ? pc : p[0];
    id[0] = b[0] ? ic : id[0];
  }
  // K pops of the lanes' heads (the winner shifts its list)
  auto pop4 = [&](TkE* out) {
#pragma unroll
    for (int t = 0; t < K; ++t) {
      const uint64_t key = k[0];
      const uint32_t pp = p[0];
      const uint32_t hi = (uint32_t)(key >> 32), lo = (uint32_t)key;
      const uint32_t mhi = __reduce_max_sync(0xffffffffu, hi);
      unsigned m = __ballot_sync(0xffffffffu, hi == mhi);
      if (m & (m - 1)) {
        const uint32_t mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        m = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
        if (m & (m - 1)) {
          const bool in = (m >> lane) & 1u;
          const uint32_t mp = __reduce_min_sync(0xffffffffu, in ? pp : NO_INDEX);
          m = __ballot_sync(0xffffffffu, in && pp == mp);
        }
      }
      const bool me = lane == __ffs(m) - 1;
      if (me) {
        TkE e;
        e.key = key;
        e.p = pp;
        e.id = pp == NO_INDEX ? -1 : id[0];
        out[t] = e;
      }
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        k[c] = me ? k[c + 1] : k[c];
        p[c] = me ? p[c + 1] : p[c];
        id[c] = me ? id[c + 1] : id[c];
      }
      k[3] = me ? 0ull : k[3];
      p[3] = me ? NO_INDEX : p[3];
      id[3] = me ? -1 : id[3];
    }
  };
  pop4(wk + warp * K);
  __syncthreads();
  if (warp == 0) {  // the NW * K warp winners (<= 64: two per lane), sorted per lane, K pops
    const int n = NW * K;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      k[c] = 0ull;
      p[c] = NO_INDEX;
      id[c] = -1;
    }
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int x = lane + 32 * c;
      if (x < n) {
        const TkE e = wk[x];
        k[c] = e.key;
        p[c] = e.p;
        id[c] = e.id;
      }
    }
    const bool sw = (k[1] > k[0]) | ((k[1] == k[0]) & (p[1] < p[0]));
    if (sw) {
      const uint64_t tk0 = k[0];
      const uint32_t tp0 = p[0];
      const int ti0 = id[0];
      k[0] = k[1]; p[0] = p[1]; id[0] = id[1];
      k[1] = tk0; p[1] = tp0; id[1] = ti0;
    }
    pop4(wk + 64);
    __syncwarp();
    if (lane < K) tk[lane] = wk[64 + lane].id;
  }
  __syncthreads();
}

// upper word of a score's order key for the candidate-list radix select, rounded up when
// the lower word is non-zero: a tile whose word is below w has a key below w << 32, and
// the word is 0 only for a zero score
template <typename R>
__device__ __forceinline__ uint32_t hkey(R s) {
  const uint64_t k = skey64(s);
  return (uint32_t)(k >> 32) | ((uint32_t)k != 0u ? 1u : 0u);
}

// Candidate-list rebuild (all threads; needs a barrier before, ends with one), from the
// words hk[] (the upper 32 bits of every tile's score key, rounded up -- hkey() -- kept
// current by the items):
//   1. node maxima nm[q] = max of the words of tiles 32q .. 32q+31 (one warp reduction
//      per node);
//   2. thw = the lower edge of the first bucket of node maxima (1/16 octave each below the
//      largest, one shared atomic per node) at which the node count reaches T -- at least
//      T nodes, hence tiles, lie at or above it -- or every positive word when fewer than T
//      nodes lie within 16 octaves (a rank count over the nodes took 3.2k-9.3k cycles);
//   3. the list = every tile whose word is >= thw, gathered from the nodes whose maximum
//      reaches thw (one ballot per node).  At least T tiles qualify; if more than
//      CL_CAP do, T is halved and the list gathered again.
// theta = thw << 32: a tile left out has word < thw, hence key < theta.  If even T = 1
// overflows (one word tied more than CL_CAP times), the list is marked invalid and the
// caller extracts by a full scan until a later rebuild succeeds.
template <typename R, int K>
// mode 0: the whole rebuild.  Staged over three publications (1, 2, 3), each short enough
// to hide in the CTA's wait for its peers' messages while the old list keeps serving:
// 1 node maxima (and their histogram), 2 the threshold for CL_TARGET into pend_theta (the
// node maxima may be a round old: only a choice of threshold), 3 the gather of every tile
// word >= it over ALL nodes (current words: the invariant), replacing the old list; an
// overflow there leaves the list invalid and the next extraction falls back to mode 0.
__device__ __noinline__ void cl_rebuild(const uint32_t* hk, long long Lc, ClState* cs, int* clid, uint32_t* nm,
                                        unsigned char* inl, int lane, int warp, unsigned long long* pf,
                                        bool hist_first, int mode) {
  const int tid = threadIdx.x, nthr = blockDim.x, NW = nthr >> 5;
  const int nn = (int)((Lc + 31) >> 5);
  // profile (pf != null on thread 0 of CTA 0): [0] node maxima, [1] thresholds, [2] gathers,
  // [3] rank-halving retries, [4] calls -- cycles summed over the rebuilds
  long long tp = pf ? clock64() : 0;
  auto mark = [&](int i) {
    if (pf) {
      const long long tn = clock64();
      atomicAdd(pf + i, (unsigned long long)(tn - tp));
      tp = tn;
    }
  };
  if (pf && mode <= 1) atomicAdd(pf + 4, 1ull);
  uint32_t* hist = nm + nn;   // [CL_NBK] node counts per bucket, [CL_NBK] = the largest node maximum
  if (mode == 3) {            // staged gather: every current word >= the pending threshold
    const uint64_t tpend = cs->pend_theta;
    const uint32_t thw = tpend == 1ull ? 1u : (uint32_t)(tpend >> 32);
    {
      const int n0 = min(cs->n, CL_CAP);
      for (int i = tid; i < n0; i += nthr) inl[clid[i]] = 0;
    }
    __syncthreads();
    if (tid == 0) cs->n = 0;
    __syncthreads();
    for (int q = warp; q < nn; q += NW) {
      const long long i = (long long)q * 32 + lane;
      const bool in = i < Lc && hk[i] >= thw;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (m == 0u) continue;   // (warp-uniform)
      int base = 0;
      if (lane == 0) base = atomicAdd(&cs->n, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int idx = base + __popc(m & ((1u << lane) - 1u));
      if (in && idx < CL_CAP) {
        clid[idx] = (int)i;
        inl[i] = 1;
      }
    }
    __syncthreads();
    mark(2);
    if (cs->n <= CL_CAP) {
      if (tid == 0) {
        cs->theta = tpend;
        cs->valid = 1;
      }
      __syncthreads();
      return;
    }
    // overflow (the threshold was chosen on older node maxima): unmark the stored entries
    // and rebuild in full now
    for (int i = tid; i < CL_CAP; i += nthr) inl[clid[i]] = 0;
    __syncthreads();
    if (tid == 0) cs->n = 0;
    __syncthreads();
    mode = 0;
  }
  if (mode == 0) {  // the old list's membership flags (inl[l] = 1 exactly for the stored entries)
    const int n0 = min(cs->n, CL_CAP);
    for (int i = tid; i < n0; i += nthr) inl[clid[i]] = 0;
  }
  if (mode <= 1) {
  for (int b = tid; b <= CL_NBK; b += nthr) hist[b] = 0u;
  __syncthreads();
  {
    uint32_t wm = 0u;
    for (int q = warp; q < nn; q += NW) {
      const long long i = (long long)q * 32 + lane;
      const uint32_t m = __reduce_max_sync(0xffffffffu, i < Lc ? hk[i] : 0u);
      if (lane == 0) nm[q] = m;
      wm = max(wm, m);
    }
    if (lane == 0 && wm != 0u) atomicMax(&hist[CL_NBK], wm);
  }
  __syncthreads();
  mark(0);
  // node maxima by bucket below the largest: (mx - m) >> CL_BSH, the last bucket holding
  // everything further down (one shared atomic per node)
  if (hist_first) {
    const uint32_t mx1 = hist[CL_NBK];
    for (int q = tid; q < nn; q += nthr) {
      const uint32_t m = nm[q];
      if (m != 0u) atomicAdd(&hist[min((mx1 - m) >> CL_BSH, (uint32_t)(CL_NBK - 1))], 1u);
    }
    __syncthreads();
  }
  if (mode == 1) return;
  }
  const uint32_t mx = hist[CL_NBK];
  // the threshold goes to the live list (mode 0) or to the pending one (mode 2, the live
  // list keeps serving until the gather)
  uint64_t* thp = mode == 2 ? &cs->pend_theta : &cs->theta;
  // first target: CL_TARGET, at most half the nodes (small slices, C1: a target above the
  // node count makes every positive word the list, which overflows) -- unless the whole
  // slice fits the list (C0: every positive word, no rebuild again)
  const int T0 = Lc <= CL_CAP ? CL_TARGET : min(CL_TARGET, max(1, nn >> 1));
  for (int T = T0;; T >>= 1) {
    if (T < T0 || !hist_first) {
      // the exact node maximum of rank T-1, by a rank count over the nodes (two threads per
      // node, ties by node index): after an overflow (crowded bucket), and for the grid
      // kernels (C4: its late rounds' crowded buckets overflow often, 5.03 -> 5.08 us/atom)
      if (tid == 0) {
        if (mode != 2) {
          cs->n = 0;
          cs->valid = 1;
        }
        *thp = 1ull;   // (no node of rank T-1 with a positive maximum: every positive word)
      }
      __syncthreads();
      for (int t2 = tid; t2 < 2 * ((nn + 15) & ~15); t2 += nthr) {
        const int t = t2 >> 1, h = t2 & 1;
        const uint32_t v = t < nn ? nm[t] : 0u;
        const int half = (nn + 1) >> 1;
        const int j0 = h * half, j1 = min(nn, j0 + half);
        int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
        int j = j0;
        for (; j + 3 < j1; j += 4) {
          const uint32_t u0 = nm[j], u1 = nm[j + 1], u2 = nm[j + 2], u3 = nm[j + 3];
          r0 += (u0 > v) | ((u0 == v) & (j < t));
          r1 += (u1 > v) | ((u1 == v) & (j + 1 < t));
          r2 += (u2 > v) | ((u2 == v) & (j + 2 < t));
          r3 += (u3 > v) | ((u3 == v) & (j + 3 < t));
        }
        for (; j < j1; ++j) {
          const uint32_t u = nm[j];
          r0 += (u > v) | ((u == v) & (j < t));
        }
        int r = r0 + r1 + r2 + r3;
        r += __shfl_xor_sync(0xffffffffu, r, 1);
        if (h == 0 && t < nn && r == T - 1 && v != 0u) *thp = (uint64_t)v << 32;
      }
    } else if (warp == 0) {
      // the first bucket (below the last) at which the node count reaches T: its lower edge
      // thw has at least T nodes -- hence tiles -- at or above it; none: every positive word
      constexpr int PL = CL_NBK / 32;
      uint32_t c[PL], sum = 0u;
#pragma unroll
      for (int k = 0; k < PL; ++k) {
        const int b = lane * PL + k;
        c[k] = b < CL_NBK - 1 ? hist[b] : 0u;
        sum += c[k];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      uint32_t run = incl - sum;
      int bsel = -1;
#pragma unroll
      for (int k = 0; k < PL; ++k) {
        run += c[k];
        if (bsel < 0 && run >= (uint32_t)T) bsel = lane * PL + k;
      }
      const unsigned has = __ballot_sync(0xffffffffu, bsel >= 0);
      const int b = has ? __shfl_sync(0xffffffffu, bsel, __ffs(has) - 1) : -1;
      if (lane == 0) {
        const unsigned long long span = (unsigned long long)(b + 1) << CL_BSH;
        const uint32_t thw = (b < 0 || span >= (unsigned long long)mx) ? 1u : (uint32_t)(mx - span + 1u);
        if (mode != 2) {
          cs->n = 0;
          cs->valid = 1;
        }
        *thp = thw == 1u ? 1ull : (uint64_t)thw << 32;
      }
    }
    __syncthreads();
    mark(1);
    if (mode == 2) return;   // staged: the gather follows after the next publication
    const uint64_t th = cs->theta;
    const uint32_t thw = th == 1ull ? 1u : (uint32_t)(th >> 32);
    for (int q = warp; q < nn; q += NW) {
      if (nm[q] < thw) continue;   // (warp-uniform)
      const long long i = (long long)q * 32 + lane;
      const bool in = i < Lc && hk[i] >= thw;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      int base = 0;
      if (lane == 0) base = atomicAdd(&cs->n, __popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      const int idx = base + __popc(m & ((1u << lane) - 1u));
      if (in && idx < CL_CAP) {
        clid[idx] = (int)i;
        inl[i] = 1;
      }
    }
    __syncthreads();
    mark(2);
    const int n = cs->n;
    if (n <= CL_CAP) break;
    if (pf) atomicAdd(pf + 3, 1ull);
    // overflow: unmark, retry with half the rank target (T = 1 cannot shrink further)
    for (int i = tid; i < CL_CAP; i += nthr) inl[clid[i]] = 0;
    if (T == 1) {
      __syncthreads();
      if (tid == 0) {
        cs->n = 0;
        cs->valid = 0;
      }
      break;
    }
    __syncthreads();
  }
  __syncthreads();
}

// Candidate-list extraction (warp 0): drop the entries that fell below theta (clearing
// their membership flags), compact the list, and pop the K best (score key desc, index
// asc) into tk[0..K-1] (-1 = none).  NC list slots per lane (the list's length picks
// 1, 2 or 4: the sorting network and the pops' shifts are the cost).  Returns (to every
// lane) whether the result is the CTA's exact top K (see ClState); if not, the caller
// rebuilds and extracts again.
template <typename R, int K, int NC>
__device__ __forceinline__ bool cl_extract_nc(const Rec<R>* trec, ClState* cs, int* clid, unsigned char* inl, int* tk,
                                              int lane, int n) {
  const uint64_t th = cs->theta;
  uint64_t kk[NC];
  uint32_t pk[NC];
  int ik[NC];
  int base = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {  // read every slot first (the compaction below overwrites them)
    const int slot = c * 32 + lane;
    const int id = slot < n && slot < CL_CAP ? clid[slot] : -1;
    uint64_t key = 0ull;
    uint32_t p = NO_INDEX;
    if (id >= 0) {
      key = skey64(trec[id].s);
      p = trec[id].p;
    }
    const bool keep = id >= 0 && key >= th;
    if (id >= 0 && !keep) inl[id] = 0;
    kk[c] = keep ? key : 0ull;
    pk[c] = keep ? p : NO_INDEX;
    ik[c] = keep ? id : -1;
  }
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NC; ++c) {  // the compacted list, in slot order
    const bool keep = ik[c] >= 0;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (keep) clid[base + __popc(km & ((1u << lane) - 1u))] = ik[c];
    base += __popc(km);
  }
  __syncwarp();
  if (lane == 0) {
    cs->n = base;
    cs->soon = base < CL_LOW ? 1 : 0;
  }
  warp_topk_nc<K, NC>(kk, pk, ik, tk, lane);
  __syncwarp();
  return n <= CL_CAP && (base >= K || th == 1ull);
}
template <typename R, int K>
__device__ __forceinline__ bool cl_extract(const Rec<R>* trec, ClState* cs, int* clid, unsigned char* inl, int* tk,
                                           int lane) {
  static_assert(CL_CAP == 128, "at most 4 list slots per lane");
  const int n = cs->n;
  if (n <= 32) return cl_extract_nc<R, K, 1>(trec, cs, clid, inl, tk, lane, n);
  if (n <= 64) return cl_extract_nc<R, K, 2>(trec, cs, clid, inl, tk, lane, n);
  return cl_extract_nc<R, K, 4>(trec, cs, clid, inl, tk, lane, n);
}

// global reduced index p -> dictionary u, bin k, frame j (p = off_u + j * M_R,u + k, Z10)
__device__ __forceinline__ void decode_p(uint32_t p, const DictGeo* sd, int W, int& u, int& k, int& j) {
  u = 0;
  for (int w = 1; w < W; ++w) u += (uint32_t)sd[w].off <= p ? 1 : 0;
  const uint32_t q = p - (uint32_t)sd[u].off;
  const int MR = sd[u].MR;
  // q / MR by the rounded-up reciprocal: umulhi gives the quotient or one more
  uint32_t jq = __umulhi(q, sd[u].mr_magic);
  int r = (int)(q - jq * (uint32_t)MR);
  jq = r < 0 ? jq - 1u : jq;
  j = (int)jq;
  k = r < 0 ? r + MR : r;
}

// packed rect of the tiles an update touches in one target dictionary:
// x = first row n0 | rows nr << 20 (rows [n0, n0+nr) mod N), y = first tile t0 | tiles Tr << 16
__device__ __forceinline__ uint2 pack_rect(const VGeo& g) {
  const bool empty = g.nr == 0 || g.nc == 0;
  return make_uint2(empty ? 0u : ((uint32_t)g.n0 | ((uint32_t)g.nr << 20)), (uint32_t)g.t0 | ((uint32_t)g.Tr << 16));
}
__device__ __forceinline__ bool rects_meet(uint2 a, uint2 b, int N) {
  const int an = a.x & 0xFFFFF, ar = a.x >> 20, bn = b.x & 0xFFFFF, br = b.x >> 20;
  const int at = a.y & 0xFFFF, aT = a.y >> 16, bt = b.y & 0xFFFF, bT = b.y >> 16;
  int d1 = bn - an, d2 = an - bn;
  d1 += d1 < 0 ? N : 0;
  d2 += d2 < 0 ? N : 0;
  return (at < bt + bT) & (bt < at + aT) & ((d1 < ar) | (d2 < br)) & (ar > 0) & (br > 0);
}
__device__ __forceinline__ bool rect_has(uint2 a, int n, int t, int N) {
  const int an = a.x & 0xFFFFF, ar = a.x >> 20, at = a.y & 0xFFFF, aT = a.y >> 16;
  int d = n - an;
  d += d < 0 ? N : 0;
  return (d < ar) & (t >= at) & (t < at + aT);
}

// grid-mode exchange (GX): a CTA's message and its round stamp in global memory; the
// stamp is written with release and polled with acquire semantics (gpu scope)
__device__ __forceinline__ void gx_st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gx_ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gx_add_acq_rel(unsigned long long* p, unsigned long long v) {
  unsigned long long o;
  asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
  return o;
}
__device__ __forceinline__ void gx_st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Grid-mode exchange protocol.  MPG_GX_COUNTER = 0 (default): every CTA releases its own
// round stamp after its message; thread c of every CTA polls stamp c.  = 1: after writing
// its message a CTA increments the round's arrival counter (acq_rel); the last arrival
// resets it and releases one round flag, which a single thread per CTA polls (C pollers
// of one line instead of C x C pollers of C stamps).  Measured slower (C4 5.29 vs 5.07
// us/atom, C3 2.58 vs 2.56): the serialised increments cost more than the polling.
// Counter and flag of parity ps at gx_stamp[32 + 16 ps] and gx_stamp[16 ps] (separate
// 128-byte lines).  Correctness: the increments form a release sequence that the last
// arrival's acq_rel read synchronises with, so every message happens-before the flag's
// release; the reset happens-before the counter's next use two rounds later (every CTA
// acquires the flag in between).
#ifndef MPG_GX_COUNTER
#define MPG_GX_COUNTER 0
#endif

// GX = false: one thread-block cluster of C <= 16 CTAs exchanging messages through
// distributed shared memory (st.async + mbarrier).  GX = true: a cooperative grid of C
// CTAs (32..128, one per SM) exchanging them through global memory (release/acquire
// stamps; the messages are copied into shared memory) and ranking the C*K entries in
// two stages (the NE best list heads, then their lists' entries); everything else is
// identical.
// TOPK: how a CTA finds its K best tiles each round -- 0 down the 32-ary node tree, 1 by a
// scan of all its tile records, 2 from its candidate list (ClState).
template <typename R, int TW, bool SREC, int K, bool GX, int TOPK = 0>
__global__ void __launch_bounds__(MPG_LB_THREADS, 1) mp_multi_kernel(const LoopParams P) {
  using C2 = typename cplx<R>::t;
  using RecT = Rec<R>;
  using MsgT = Msg<R, K>;
  const int C = P.C, lgC = ilog2(P.C);
  const int rank = GX ? (int)blockIdx.x : (int)cg::this_cluster().block_rank();
  const int W = P.W;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  constexpr int LGTW = TW == 32 ? 5 : (TW == 64 ? 6 : 7);
  constexpr int NCH = TW / 32;
  constexpr int TPI = tiles_per_item<TW>();
  constexpr bool notree = TOPK != 0;  // top-K without the node tree (no tree upkeep per round)
  static_assert(TOPK != 1 || SREC, "the scan top-K reads shared-memory tile records");
  const int NEc = min(NE, C * K);
  const int B = max(1, min(BMAX, P.spec));
  const bool floorm = P.floor_mode != 0;   // latency-floor measurement (no update)

  extern __shared__ __align__(32) unsigned char smem[];
  const Smem L = smem_layout(P, sizeof(RecT), sizeof(MsgT));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  MsgT* mail = reinterpret_cast<MsgT*>(smem + L.mail);
  MsgT* mymsg = reinterpret_cast<MsgT*>(smem + L.mymsg);
  RecT* lev = reinterpret_cast<RecT*>(smem + L.lev);
  Ent* ent = reinterpret_cast<Ent*>(smem + L.ent);
  VGeo* egeo = reinterpret_cast<VGeo*>(smem + L.egeo);
  uint32_t* wmeet = reinterpret_cast<uint32_t*>(smem + L.wmask);
  uint32_t* wcover = wmeet + NE;
  uint2* rect = reinterpret_cast<uint2*>(smem + L.rect);
  int2* ecnt = reinterpret_cast<int2*>(smem + L.ecnt);
  St* st = reinterpret_cast<St*>(smem + L.st);
  uint32_t* vkey = reinterpret_cast<uint32_t*>(smem + L.vkey);
  int* sorted = reinterpret_cast<int*>(smem + L.sorted);
  int* hsel = reinterpret_cast<int*>(smem + L.hsel);
  int* tk = reinterpret_cast<int*>(smem + L.tk);
  TkE* wk = reinterpret_cast<TkE*>(smem + L.wk);
  int* stamp = reinterpret_cast<int*>(smem + L.stamp);   // dirty-node stamps and lists per level
  int* list = reinterpret_cast<int*>(smem + L.list);
  int* cnt = reinterpret_cast<int*>(smem + L.cnt);
  PairGeo* sp = reinterpret_cast<PairGeo*>(smem + L.pairs);
  DictGeo* sd = reinterpret_cast<DictGeo*>(smem + L.dicts);
  OwnGeo* sown = reinterpret_cast<OwnGeo*>(smem + L.own);
  const double2* roots = P.Rmax <= 4096 ? reinterpret_cast<const double2*>(smem + L.roots) : P.roots;
  RhoEnt* srho = reinterpret_cast<RhoEnt*>(smem + L.rho);
  int* rho_lo = reinterpret_cast<int*>(smem + L.rho_meta);
  int* rho_n = rho_lo + W;
  int* rho_off = rho_n + W;
  ClState* cls = reinterpret_cast<ClState*>(smem + L.cls);
  int* clid = reinterpret_cast<int*>(smem + L.clid);
  unsigned char* inl = smem + L.inl;
  uint32_t* hk = reinterpret_cast<uint32_t*>(smem + L.hk);
  uint32_t* nmx = reinterpret_cast<uint32_t*>(smem + L.nmax);
  uint32_t* rcp = reinterpret_cast<uint32_t*>(smem + L.rcp);
  // batched independent signals: cluster `slot` works on signal `slot` (its own grids,
  // records, backups, atoms, energies, result; the kernels are shared)
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
  C2* backup = reinterpret_cast<C2*>(P.backup) + ((long long)slot * C + rank) * P.bk_cap * TW;

  // ---- load tables -------------------------------------------------------
  for (int i = tid; i < W * W; i += blockDim.x) sp[i] = P.pairs[i];
  for (int i = tid; i < W; i += blockDim.x) {
    sd[i] = P.dicts[i];
    sown[i] = P.own[rank * W + i];
    rho_lo[i] = P.rho_lo[i];
    rho_n[i] = P.rho_n[i];
    rho_off[i] = P.rho_off[i];
  }
  if (P.Rmax <= 4096)
    for (int i = tid; i < P.Rmax; i += blockDim.x) reinterpret_cast<double2*>(smem + L.roots)[i] = P.roots[i];
  for (int i = tid; i < P.rho_total; i += blockDim.x) srho[i] = P.rho[i];
  {
    int levtot = 0;
    for (int l = 0; l < P.nlev; ++l) levtot += P.lev_n[l];
    for (int i = tid; i < levtot; i += blockDim.x) stamp[i] = 0;
  }
  for (int i = tid; i < RCP_N; i += blockDim.x) rcp[i] = i > 1 ? 0xFFFFFFFFu / (uint32_t)i + 1u : 0u;
  if (tid < MAX_LEVELS) cnt[tid] = 0;
  if (tid < BMAX) vkey[tid] = 0;
  if (SREC)
    for (long long i = tid; i < P.Lc; i += blockDim.x) trec[i] = grec[i];
  if (TOPK == 2)
    for (long long i = tid; i < P.Lc; i += blockDim.x) {
      hk[i] = hkey(grec[i].s);
      inl[i] = 0;
    }
  __syncthreads();

  // ---- node levels -------------------------------------------------------
  for (int i = warp; i < P.lev_n[0]; i += NW) warp_node(trec, P.Lc, i, lev, lane);
  __syncthreads();
  for (int l = 1; l < P.nlev; ++l) {
    for (int i = warp; i < P.lev_n[l]; i += NW)
      warp_node(lev + P.lev_off[l - 1], (long long)P.lev_n[l - 1], i, lev + P.lev_off[l], lane);
    __syncthreads();
  }
  const uint32_t msgbytes = (uint32_t)sizeof(MsgT);
  if (tid == 0) {
    if constexpr (!GX) {
      mbar_init(smem_addr(&mbar[0]), 1);
      mbar_init(smem_addr(&mbar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_arm(smem_addr(&mbar[0]), C * msgbytes);
      mbar_arm(smem_addr(&mbar[1]), C * msgbytes);
    }
    st->E = E0s;
    st->it = 0;
    st->G = 0;
    st->mode = 0;
    st->rb_from = 0;
    st->stop = 0;
  }
  if constexpr (GX) __syncthreads();
  else cg::this_cluster().sync();

  const bool prof = P.prof != nullptr && slot == 0 && rank == 0 && tid == 0;
  long long tprev = clock64();
#define PROF_MARK(i)                                                                                     \
  if (prof) {                                                                                             \
    const long long tn = clock64();                                                                      \
    atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + (i), (unsigned long long)(tn - tprev)); \
    tprev = tn;                                                                                           \
  }

  // The message (top-K records + per-candidate maxima): warp 0 forms it in shared memory
  // (form_msg, before the top-K's closing barrier), then the first warps push it into slot
  // `ps` of every CTA, one 16-byte chunk per thread (push_msg; MPG_PUSH_WARPS = 0: warp 0
  // alone, 5 stores per lane -- 578 cycles of every round)
  auto form_msg = [&](unsigned long long stamp) {
    if (lane < K) mymsg->list[lane] = tk[lane] >= 0 ? trec[tk[lane]] : empty_rec(R(0));
#ifdef MPG_CHECKS
    if (lane == 0) mymsg->tag = (uint32_t)stamp;
#else
    (void)stamp;
#endif
    if (lane < BMAX) {
      mymsg->vkey[lane] = vkey[lane];
      vkey[lane] = 0;
    }
    __syncwarp();
  };
  auto push_msg = [&](int ps, unsigned long long stamp) {
    PROF_MARK(13);
    const int NCHUNK = (int)(msgbytes / 16);
    const uint4* src = reinterpret_cast<const uint4*>(mymsg);
    if constexpr (GX) {  // message, then its stamp (release, same thread): round `stamp - 1` may read it
      if (tid == 0) {
        uint4* dstg = reinterpret_cast<uint4*>(reinterpret_cast<MsgT*>(P.gx_rec) + (long long)ps * C + rank);
#pragma unroll
        for (int ch = 0; ch < (int)(sizeof(MsgT) / 16); ++ch) dstg[ch] = src[ch];
        if constexpr (MPG_GX_COUNTER) {
          unsigned long long* cntp = P.gx_stamp + 32 + 16 * ps;
          if (gx_add_acq_rel(cntp, 1ull) == (unsigned long long)(C - 1)) {
            gx_st_relaxed(cntp, 0ull);
            gx_st_release(P.gx_stamp + 16 * ps, stamp);
          }
        } else {
          gx_st_release(P.gx_stamp + (long long)ps * C + rank, stamp);
        }
      }
    } else {
      (void)stamp;
      const uint32_t dst = smem_addr(&mail[ps * MAX_CLUSTER + rank]);
      const uint32_t bar = smem_addr(&mbar[ps]);
#if MPG_PUSH_WARPS
      for (int t = tid; t < C * NCHUNK; t += blockDim.x) {
#else
      for (int t = warp == 0 ? lane : C * NCHUNK; t < C * NCHUNK; t += 32) {
#endif
        const int d = t / NCHUNK, ch = t - d * NCHUNK;
        st_async16(mapa(dst + 16 * ch, d), mapa(bar, d), src[ch]);
      }
    }
    PROF_MARK(14);
  };
  // this CTA's K best tiles into tk[0..K-1] (all threads; a barrier before, ends with one)
  auto topk = [&](unsigned long long stamp) {
    if constexpr (TOPK == 2) {
      const long long tx0 = prof ? clock64() : 0;
      if (warp == 0) {
        const bool ok = cls->valid && !cls->need && cl_extract<R, K>(trec, cls, clid, inl, tk, lane);
        if (lane == 0) cls->need = ok ? 0 : 1;
        if (ok) form_msg(stamp);
      }
      if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 16, (unsigned long long)(clock64() - tx0));
      __syncthreads();
      // the list cannot give the exact top K: a full scan this round; the list is rebuilt
      // after the publication (rebuild_after), off the path to the message
      if (cls->need) {
        if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 473, 1ull);   // scans (CTA 0)
        cta_topk_scan<R, K>(trec, P.Lc, tk, wk, lane, warp, NW);
        if (warp == 0) form_msg(stamp);
        __syncthreads();
      }
    } else {
      if constexpr (TOPK == 1) cta_topk_scan<R, K>(trec, P.Lc, tk, wk, lane, warp, NW);
      else cta_topk<R, K>(P, lev, trec, tk, lane, warp, NW);
      if (warp == 0) form_msg(stamp);
      __syncthreads();
    }
  };
  // candidate lists: rebuild after the message is out (all threads) when the extraction ran
  // short (need) or left fewer than CL_LOW entries (soon).  A CTA waits for its peers'
  // messages at this point anyway, so the rebuild is hidden unless this CTA is the
  // round's last; before, a rebuild before the publication stalled every peer that round.
  // The list invariant holds across it: the next items add every rewritten tile >= theta.
  auto rebuild_after = [&]() {
    if constexpr (TOPK == 2) {
      const int stg = cls->stage;
      if (cls->need | cls->soon | stg) {   // (uniform: written before the top-K barrier)
        // need: the whole rebuild now; else the staged one, one stage per publication
        const int mode = cls->need ? 0 : stg + 1;
        const long long tr0 = prof ? clock64() : 0;
        if (prof && mode <= 1) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 19, 1ull);
        if (P.prof != nullptr && slot == 0 && tid == 0 && rank < 128 && mode <= 1)   // rebuilds of every CTA
          atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 320 + rank, 1ull);
        cl_rebuild<R, K>(hk, P.Lc, cls, clid, nmx, inl, lane, warp,
                         prof ? reinterpret_cast<unsigned long long*>(P.prof) + 468 : nullptr, !GX, mode);
        if (prof) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 17, (unsigned long long)(clock64() - tr0));
        if (tid == 0) {
          const bool fin = mode == 0 || mode == 3;
          cls->stage = fin ? 0 : mode;
          if (fin) {
            cls->need = 0;
            cls->soon = 0;
          }
        }
        __syncthreads();
      }
    }
  };
  if constexpr (TOPK == 2) {
    if (tid == 0) {
      cls->need = 1;
      cls->valid = 1;
      cls->n = 0;
      cls->soon = 0;
      cls->stage = 0;
    }
    __syncthreads();
  }
  topk(1ull);
  push_msg(0, 1ull);
  rebuild_after();

  long long rounds = 0;
  long long tbusy0 = 0;
  for (int round = 0;; ++round) {
    const int par = round & 1;
    const MsgT* mb = GX ? mail : mail + par * MAX_CLUSTER;
    if constexpr (GX) {
      // every CTA's message of this round (stamp == round + 1): thread c polls CTA c's
      // stamp, then copies its message into shared memory (L2 loads, L1 bypassed)
      const unsigned long long want = (unsigned long long)round + 1;
      constexpr int NCHUNK = (int)(sizeof(MsgT) / 16);
      if constexpr (MPG_GX_COUNTER) {
        if (tid == 0) {
          const long long t0 = clock64();
          while (gx_ld_acquire(P.gx_stamp + 16 * par) != want) spin_check(t0);
        }
        __syncthreads();
      }
      for (int c = tid; c < C; c += blockDim.x) {
        const long long t0 = clock64();
        while (!MPG_GX_COUNTER && gx_ld_acquire(P.gx_stamp + (long long)par * C + c) != want) {
          spin_check(t0);
        }
        const uint4* srcg = reinterpret_cast<const uint4*>(reinterpret_cast<const MsgT*>(P.gx_rec) + (long long)par * C + c);
        uint4* dsts = reinterpret_cast<uint4*>(mail + c);
        uint4 v[NCHUNK];  // all loads in flight before the stores
#pragma unroll
        for (int ch = 0; ch < NCHUNK; ++ch) v[ch] = __ldcg(srcg + ch);
#pragma unroll
        for (int ch = 0; ch < NCHUNK; ++ch) dsts[ch] = v[ch];
      }
      __syncthreads();
    }
    // ---- A0/A1 (warp 0): messages of the previous round; verify its candidates
    if (warp == 0) {
      if constexpr (!GX) mbar_wait(smem_addr(&mbar[par]), (uint32_t)((round >> 1) & 1));
      if (P.prof != nullptr && slot == 0 && tid == 0) tbusy0 = clock64();
      if (prof && round > 0) {  // histogram of the message waits (cycles; 8 buckets: <1k .. >=12k)
        const long long w = clock64() - tprev;
        const int bk = w < 1000 ? 0 : w < 2000 ? 1 : w < 3000 ? 2 : w < 4000 ? 3 : w < 6000 ? 4 : w < 8000 ? 5 : w < 12000 ? 6 : 7;
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 448 + bk, 1ull);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 456 + bk, (unsigned long long)w);
      }
      PROF_MARK(0);
      if (!GX && lane == 0) mbar_arm(smem_addr(&mbar[par]), C * msgbytes);  // slot reused at round + 2
#ifdef MPG_CHECKS
      for (int c = lane; c < C; c += 32)   // every message is the one published for this round
        MPG_CHECK(mb[c].tag == (uint32_t)round + 1u, "mailbox message from another round");
#endif
      const int Gp = st->G;
      int acc = Gp;
      if (Gp >= 2) {
        // V_l = max over CTAs of the candidate-l key; candidate i is accepted iff
        // max_{l<i} V_l < key(c(p_i)) for it and every earlier candidate
        uint32_t vk[BMAX];
#pragma unroll
        for (int l = 0; l < BMAX; ++l) vk[l] = 0;
        for (int c = lane; c < C; c += 32)   // lane: CTAs lane, lane + 32, ... (grid mode)
#pragma unroll
          for (int q = 0; q < BMAX / 4; ++q) {
            const uint4 va = *reinterpret_cast<const uint4*>(&mb[c].vkey[4 * q]);
            vk[4 * q] = max(vk[4 * q], va.x);
            vk[4 * q + 1] = max(vk[4 * q + 1], va.y);
            vk[4 * q + 2] = max(vk[4 * q + 2], va.z);
            vk[4 * q + 3] = max(vk[4 * q + 3], va.w);
          }
        uint32_t run = 0;
#pragma unroll
        for (int l = 0; l < BMAX - 1; ++l) {
          const uint32_t V = __reduce_max_sync(0xffffffffu, vk[l]);
          if (l < lane) run = max(run, V);
        }
        const bool fail = lane >= 1 && lane < Gp && run >= st->ckey[lane < BMAX ? lane : 0];
        const unsigned fm = __ballot_sync(0xffffffffu, fail);
        if (fm) acc = __ffs(fm) - 1;
      }
      if (lane == 0) {
        if (acc > 0) {
          if (rank == 0 && slot == 0 && P.sol)  // c(p) += c~ for the accepted atoms, in order (Alg. 1 step 2a)
            for (int g = 0; g < acc; ++g) {
              const Ent& e = ent[st->pick[g]];
              const DictGeo du = sd[e.u];
              double2* s = P.sol + du.off + (long long)e.j * du.MR + e.k;
              double2 c = *s;
              c.x += e.tre;
              c.y += e.tim;
              *s = c;
            }
          st->it += acc;
          st->E = st->Enext[acc - 1];
        }
        st->mode = acc < Gp ? 1 : 0;
        st->rb_from = acc;
        if (prof && acc < Gp) {  // roll-back statistics: rounds, first rejected candidate
          atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 56, 1ull);
          atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 56 + min(acc, 7), 1ull);
        }
      }
      PROF_MARK(1);
    }
    if (warp != 0 || NW == 1) {
      const bool prof1 = P.prof != nullptr && rank == 0 && tid == 32;
      const long long tw0 = prof1 ? clock64() : 0;
      if (!GX && warp != 0) mbar_wait(smem_addr(&mbar[par]), (uint32_t)((round >> 1) & 1));
      const long long tw1 = prof1 ? clock64() : 0;
      // ---- A2: window ranking, in parallel with the verification: merged position
      //      of every published list entry = the number of entries ahead of it in
      //      the total order (score key desc, index asc; empty records: list order),
      //      4 lanes per entry; the NEc first positions name the walk window
      const int NL = C * K;
      const int rw = NW == 1 ? 0 : warp - 1, nrw = NW == 1 ? 1 : NW - 1;
      if constexpr (GX) {
        // stage 1 (one warp, C <= 128 heads, 4 per lane, sorted, NE pops of the lanes'
        // heads): the lists whose heads are among the NEc best heads hold every entry of
        // the window (an entry below the NEc-th best head has NEc heads ahead of it)
        if (rw == 0) {
          uint64_t hk[4];
          uint32_t hp4[4];
          int hi4[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = lane + 32 * j;
            const bool ok = c < C;
            // an empty list (a CTA owning no frames) keeps its id: its head takes the index
            // NO_INDEX - 1 (no real p reaches it), so the NEc pops always name real lists and
            // stage 2 fills every window slot (lists past C stay NO_INDEX, id -1)
            const uint32_t hpc = ok ? mb[c].list[0].p : NO_INDEX;
            hk[j] = ok ? skey64(mb[c].list[0].s) : 0ull;
            hp4[j] = ok && hpc == NO_INDEX ? NO_INDEX - 1u : hpc;
            hi4[j] = ok ? c : -1;
          }
          warp_topk_nc<NE, 4>(hk, hp4, hi4, hsel, lane);
        }
      }
      for (int grp = rw; !GX && grp * 8 < NL; grp += nrw) {
        const int e = grp * 8 + (lane >> 2), sub = lane & 3;
        int c = 0;
        if (e < NL) {
          const RecT& re = mb[e / K].list[e % K];
          const uint64_t ke = skey64(re.s);
          const uint32_t pe = re.p;
#pragma unroll
          for (int i = 0; i < MAX_CLUSTER * K / 4; ++i) {  // every load issued before the compares
            const int f = sub + 4 * i;   // f < MAX_CLUSTER * K: inside the mail array
            const RecT& rf = mb[f / K].list[f % K];
            const uint64_t kf = skey64(rf.s);
            const uint32_t pf = rf.p;
            // branch-free: (kf, -pf, -f) > (ke, -pe, -e), counted for f < NL only
            const bool ahead = (kf > ke) | ((kf == ke) & ((pf < pe) | ((pf == pe) & (f < e))));
            c += (int)(ahead & (f < NL));
          }
        }
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        if (e < NL && sub == 0 && c < NEc) sorted[c] = e;
      }
      if (prof1) {
        const long long tw2 = clock64();
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 30, (unsigned long long)(tw1 - tw0));
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 31, (unsigned long long)(tw2 - tw1));
      }
    }
    __syncthreads();
    PROF_MARK(2);
    const int mode = st->mode;
    int lo = 0, hi = 0, gvend = 0;  // row-item range of this CTA, number of (g, v) pairs searched
    if (mode == 0) {
      if constexpr (GX) {
        // stage 2 (warp 0): the K entries of each selected list, one per lane, ranked
        // among themselves -- exact, since every entry ahead of one of them is one of them
        constexpr int S2 = (NE * K + 31) / 32;   // stage-2 entries per lane
        static_assert(S2 <= 2, "stage-2 candidates fit one warp, two per lane");
        if (warp == 0) {
          uint64_t ke[S2];
          uint32_t pe[S2];
          int e[S2];
          bool hv[S2];
          int cnt[S2];
#pragma unroll
          for (int s = 0; s < S2; ++s) {
            const int x = lane + 32 * s;
            const int hs = x < NEc * K ? hsel[x / K] : -1;
            hv[s] = hs >= 0;   // (always for x < NEc * K: C >= 32 lists, empty ones included)
            const int cl = hv[s] ? hs : 0, q = x % K;
            e[s] = cl * K + q;
            ke[s] = hv[s] ? skey64(mb[cl].list[q].s) : 0ull;
            pe[s] = hv[s] ? mb[cl].list[q].p : NO_INDEX;
            cnt[s] = 0;
          }
#pragma unroll
          for (int t = 0; t < S2; ++t) {
#pragma unroll 8
            for (int j = 0; j < 32; ++j) {
              const uint64_t kf = __shfl_sync(0xffffffffu, ke[t], j);
              const uint32_t pf = __shfl_sync(0xffffffffu, pe[t], j);
              const int ef = __shfl_sync(0xffffffffu, e[t], j);
              const bool in = j + 32 * t < NEc * K;
#pragma unroll
              for (int s = 0; s < S2; ++s) {
                const bool ahead = (kf > ke[s]) | ((kf == ke[s]) & ((pf < pe[s]) | ((pf == pe[s]) & (ef < e[s]))));
                cnt[s] += (int)(in & ahead);
              }
            }
          }
#pragma unroll
          for (int s = 0; s < S2; ++s)
            if (hv[s] && cnt[s] < NEc) sorted[cnt[s]] = e[s];
        }
        __syncthreads();
      }
      PROF_MARK(3);
      // ---- A2b: update geometry of every window entry in every target dictionary,
      //      seen from this CTA (Alg. 3 index sets), and its packed tile rect; and,
      //      one thread per window entry, its decoded index and scalar step
      //      (c~, E~ of Eqs. (19)-(20): c(p) of an entry that is picked is unchanged
      //      by the round's earlier picks, so they are the sequential ones)
      // the scalar steps run on their own warp (no divergence with the geometry threads)
      const int sbase = (NEc * W + 31) & ~31;
      const int nwork = sbase + NEc <= (int)blockDim.x ? sbase + NEc : NEc * W + NEc;
      for (int t = tid; t < nwork; t += blockDim.x) {
        if (nwork == sbase + NEc && t >= NEc * W && t < sbase) continue;
        if (t < NEc * W) {
          const int e = t / W, v = t - e * W;
          const int src = sorted[e];
          const RecT& r = mb[src / K].list[src % K];
          VGeo gg;
          gg.nr = 0;
          gg.nc = 0;
          gg.cntA = 0;
          gg.cntB = 0;
          gg.Tr = 0;
          gg.t0 = 0;
          gg.n0 = 0;
          if (r.p != NO_INDEX) {
            int u, k, j;
            decode_p(r.p, sd, W, u, k, j);
            vgeo<LGTW>(sp[u * W + v], sd[u], sd[v], k, j, rank, C, lgC, gg);
          }
          const int hp = (gg.Tr + TPI - 1) / TPI;   // items per row; its reciprocal for the items
          MPG_CHECK(hp < RCP_N, "items per row beyond the reciprocal table");
          gg.pad = hp > 1 ? (int)rcp[hp] : 0;
          egeo[t] = gg;
          rect[t] = pack_rect(gg);
          const int rows = gg.nc > 0 ? gg.cntA + gg.cntB : 0;
          ecnt[e * 16 + v] = make_int2(rows * hp, rows * gg.Tr);
        } else {
          const int e = t - (nwork == sbase + NEc ? sbase : NEc * W);
          const int src = sorted[e];
          const RecT rl = mb[src / K].list[src % K];
          Ent en;
          en.u = -1;
          en.k = 0;
          en.j = 0;
          en.tre = 0.0;
          en.tim = 0.0;
          en.Et = 0.0;
          en.selfc = 0;
          en.key = score_key(rl.s);
          en.pos = (rl.p != NO_INDEX && rl.s > R(0)) ? 1 : 0;
          en.last = (src % K) == K - 1 ? 1 : 0;   // the K-th entry of its CTA's list
          if (rl.p != NO_INDEX) {
            decode_p(rl.p, sd, W, en.u, en.k, en.j);
            const int u = en.u, k = en.k;
            const int Mu = sd[u].M;
            const bool selfc = (k == 0) || (2 * k == Mu);
            en.selfc = selfc ? 1 : 0;
            const double cre = (double)rl.re, cim = (double)rl.im;
            if (selfc) {  // Z13
              en.tre = cre;
              en.tim = 0.0;
              en.Et = cre * cre;
            } else {      // Eqs. (19)-(20) with rho = h_uu(-2k, 0) (Z11/Z12)
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
              const double tre = nre * inv, tim = nim * inv;
              const double X2 = tre * tre, Y2 = tim * tim, XY = tre * tim;
              en.tre = tre;
              en.tim = tim;
              en.Et = 2.0 * (X2 + Y2 + rre * (X2 - Y2) - 2.0 * rim * XY);
            }
          }
          ent[e] = en;
        }
      }
      __syncthreads();
      PROF_MARK(4);
      // ---- A3: pairwise relations of the window entries, one (a, v) pair per
      //      warp iteration, lane b:
      //      meet[a] bit b  -- tiles(a) and tiles(b) share a tile of dictionary v
      //      cover[a] bit b -- the tile of entry b lies in tiles(a)
      {
        int bu = -1, bj = 0, bt = 0;
        if (lane < NEc) {
          const Ent& eb = ent[lane];
          bu = eb.u;
          bj = eb.j;
          bt = eb.k >> LGTW;
        }
        const int bN = bu >= 0 ? sd[bu].N : 1;
        const int lb = lane < NEc ? lane : 0;
        for (int a = warp; a < NEc; a += NW) {  // warp: entry a, all target dictionaries
          bool meet = false;
#pragma unroll 4
          for (int v = 0; v < W; ++v) meet |= rects_meet(rect[a * W + v], rect[lb * W + v], sd[v].N);
          // entry b's own tile lies in dictionary bu only
          const bool cover = (lane < NEc) && bu >= 0 && rect_has(rect[a * W + (bu >= 0 ? bu : 0)], bj, bt, bN);
          const unsigned mm = __ballot_sync(0xffffffffu, (lane < NEc) && meet);
          const unsigned cm = __ballot_sync(0xffffffffu, cover);
          if (lane == 0) {
            wmeet[a] = mm;
            wcover[a] = cm;
          }
        }
      }
      PROF_MARK(5);
      __syncthreads();
      PROF_MARK(6);
      // ---- A4: the walk (warp 0, all lanes redundantly, bitmask logic); warps 1..
      //      meanwhile (grids beyond L2, C3/C4) bulk-prefetch this CTA's rows of the first
      //      l2pf window entries -- the hull tiles of every owned grid row and its kernel
      //      row -- HBM -> L2 on the TMA unit, one (entry, dictionary) per warp, one row per
      //      lane, so that the items of the picked entries hit L2
      if (GX && warp != 0 && P.l2pf > 0) {   // (grid kernels only: the cluster's grids fit L2)
        const int npf = min(P.l2pf, NEc) * W;
        for (int t = warp - 1; t < npf; t += NW - 1) {
          const VGeo& gg = egeo[t];
          const int rows = gg.nc > 0 ? gg.cntA + gg.cntB : 0;
          const DictGeo& dv = sd[t % W];
          const C2* gb = grid + dv.grid_off + (long long)gg.t0 * TW;
          for (int i = lane; i < rows; i += 32) {
            const int rw2 = i < gg.cntA ? gg.rhoA + (i << lgC) : gg.rA + gg.rhoB + ((i - gg.cntA) << lgC);
            int nrow = gg.n0 + rw2;
            if (nrow >= dv.N) nrow -= dv.N;
            l2_prefetch_bulk(gb + (long long)nrow * dv.stride, (uint32_t)(gg.Tr * TW * sizeof(C2)));
            l2_prefetch_bulk(kern + gg.kbase + (long long)rw2 * gg.nc, (uint32_t)(gg.nc * sizeof(C2)));
          }
        }
      }
      auto item_scan = [&](int Gsc) {
        // this CTA's items (tile pairs of its rows) and tiles of (g, v), at index
        // t = g * 16 + v (g-major; v >= W contribute nothing): lane handles IPL pairs
        const int GW = Gsc * 16;
        int r4[IPL], t4[IPL], rs = 0, ts = 0;
        // a lane's IPL entries share one candidate g (16 % IPL == 0): its window position
        const int pq = st->pick[((lane * IPL) >> 4) & (BMAX - 1)];
#pragma unroll
        for (int q = 0; q < IPL; ++q) {
          const int t = lane * IPL + q;
          int nrw = 0, ntl = 0;
          const int v = t & 15;
          if (t < GW && v < W && !floorm) {
            const int2 cn2 = ecnt[pq * 16 + v];
            nrw = cn2.x;
            ntl = cn2.y;
          }
          r4[q] = nrw;
          t4[q] = ntl;
          rs += nrw;
          ts += ntl;
        }
        int ri = rs, ti = ts;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y1 = __shfl_up_sync(0xffffffffu, ri, o), y2 = __shfl_up_sync(0xffffffffu, ti, o);
          if (lane >= o) {
            ri += y1;
            ti += y2;
          }
        }
        int rr = ri - rs, tt = ti - ts;
#pragma unroll
        for (int q = 0; q < IPL; ++q) {
          const int t = lane * IPL + q;
          if (t <= GW) {
            st->ibase[t] = rr;
            st->tbase[t] = tt;
          }
          rr += r4[q];
          tt += t4[q];
        }
        if (lane == 31 && GW == BMAX * 16) {
          st->ibase[GW] = ri;
          st->tbase[GW] = ti;
        }
      };
      if (MPG_SCAN_W1 && warp == 1) {   // (NW >= 2) waits for the walk's picks, then the item bases
        bar_sync(1, 64);
        item_scan(st->Gw);
      }
      if (warp == 0) {
        const bool have = lane < NEc;
        const Ent& el = ent[have ? lane : 0];   // decoded in the geometry phase
        const unsigned lastm = __ballot_sync(0xffffffffu, have && el.last != 0);
        const unsigned posm = __ballot_sync(0xffffffffu, have && el.pos != 0);
        const long long it0 = st->it;
        const long long rem = P.maxit - it0;
        const int Bm = rem < (long long)B ? (int)max(rem, 0LL) : B;
        const double Etl = have ? el.Et : 0.0;
        const uint32_t keyl = have ? el.key : 0u;
        uint32_t mtr[NE], cvr[NE];  // every entry's masks in every lane (broadcast loads)
#pragma unroll
        for (int j = 0; j < NE; ++j) {
          mtr[j] = wmeet[j];
          cvr[j] = wcover[j];
        }
        PROF_MARK(29);
        unsigned excl = 0, picked = 0;
        int G = 0;
        int pl = 0;                // lane g: window position of pick g (recorded as the walk takes it)
        int why = 0, lastpos = 0;  // walk statistics (profile mode)
        // the walk in window order, statically unrolled and branch-free (the state is
        // warp-uniform): entry j is skipped if a pick covers its tile; otherwise it
        // is picked or it ends the walk.  Passing a skipped entry that was the last
        // of its CTA's list ends the walk at the next entry that is not skipped.
        bool done = false, passed_last = false, passed_cover = false;
#pragma unroll
        for (int j = 0; j < NE; ++j) {
          const unsigned bit = 1u << j;
          const bool inwin = j < NEc;
          const bool skip = (excl & bit) != 0u;
          const bool cand = inwin & !skip & !done;
          const bool e1 = G >= Bm;                       // B picks
          // a CTA list ran out before j, or an entry before j was covered by a pick: such an
          // entry scored above j before the round and often still does after the pick's
          // update, which would reject j one round later (roll-backs 15 -> 12 % of C2's rounds)
          const bool e3 = passed_last | passed_cover;
          const bool e4 = (posm & bit) == 0u;            // zero score (stop rule 4 at G = 0)
          const bool e5 = (mtr[j] & picked) != 0u;       // tiles(j) meet X
          const int w = e1 ? 1 : (e3 ? 3 : (e4 ? 4 : (e5 ? 5 : 0)));
          const bool take = cand & (w == 0);
          why = (cand & (w != 0)) ? w : why;
          done = done | (cand & (w != 0));
          picked |= take ? bit : 0u;
          excl |= take ? cvr[j] : 0u;
          pl = (take & (lane == G)) ? j : pl;
          G += take ? 1 : 0;
          lastpos = take ? j : lastpos;
          const bool e6 = take & ((lastm & bit) != 0u);  // its CTA list is consumed
          why = e6 ? 6 : why;
          done = done | e6;
          passed_last = passed_last | (inwin & skip & !done & ((lastm & bit) != 0u));
          passed_cover = passed_cover | (inwin & skip & !done);
        }
        why = done ? why : 2;                            // window exhausted
        PROF_MARK(27);
        if (prof) {
          atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 20, (unsigned long long)lastpos);
          atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 20 + why, 1ull);
        }
        if (P.prof != nullptr && slot == 0 && rank == 0) {   // (warp-uniform: the whole warp reduces)
          // deepest CTA-list position among the window entries (0..K-1, capped at 3)
          const unsigned qd = __reduce_max_sync(0xffffffffu, have ? (unsigned)(sorted[lane] % K) : 0u);
          if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 464 + min(qd, 3u), 1ull);
        }
        // candidate g = the g-th picked window entry (lane g records its position);
        // E recurrence and the energy stop rules (Z15) in selection order, every lane
        // redundantly on the shuffled E~ of the picks
        if (lane < G) st->pick[lane] = pl;
        // the item bases depend on the picks only: warp 1 computes them (for the walk's G; a
        // stop rule can only shorten the round, and the bases of a prefix are a prefix)
        // while this warp runs the energy chain
        // (every launch has at least 4 warps: runtime.cu set_launch)
#if MPG_SCAN_W1
        if (lane == 0) st->Gw = G;
        __syncwarp();
        bar_sync(1, 64);
#endif
        // (latency-floor mode: no update, so no energy change either -- E~ taken as 0)
        const double Etg = floorm ? 0.0 : __shfl_sync(0xffffffffu, Etl, pl);
        const uint32_t kmine = __shfl_sync(0xffffffffu, keyl, pl);
#if MPG_ECHAIN_BF
        // E_{k+1} = E_k - E~ in selection order, branch-free: every lane runs the whole chain
        // (the same rounded subtractions), lane g keeps the energy before (Epre) and after
        // (Emine) pick g; the first pick whose Epre meets a stop rule (Z15) ends the round
        const double E0r = st->E;
        double Ecur = E0r, Emine = 0.0, Epre = 0.0;
        double egs[BMAX];
#pragma unroll
        for (int g = 0; g < BMAX; ++g) egs[g] = __shfl_sync(0xffffffffu, Etg, g);
#pragma unroll
        for (int g = 0; g < BMAX; ++g) {
          Epre = lane == g ? Ecur : Epre;
          Ecur = Ecur - egs[g];
          Emine = lane == g ? Ecur : Emine;
        }
        const unsigned fm = __ballot_sync(0xffffffffu, lane < G && (Epre <= Etols || Epre < 0.0));
        int Gs = fm ? __ffs(fm) - 1 : G;
        Ecur = Gs == 0 ? E0r : __shfl_sync(0xffffffffu, Emine, (Gs - 1) & 31);
#else
        double Ecur = st->E, Emine = 0.0;
        int Gs = G;
#pragma unroll
        for (int g = 0; g < BMAX; ++g) {   // E_{k+1} = E_k - E~ in selection order
          const double eg = __shfl_sync(0xffffffffu, Etg, g);
          if (g < Gs) {
            if (Ecur <= Etols || Ecur < 0.0) {
              Gs = g;
            } else {
              Ecur = Ecur - eg;
              if (lane == g) Emine = Ecur;
            }
          }
        }
#endif
        int stopr = 0;
        if (Gs == 0) {
          if (it0 >= P.maxit) stopr = 1;
          else if (Ecur <= Etols) stopr = 2;
          else if (Ecur < 0.0) stopr = 3;
          else stopr = 4;
        }
        if (floorm && Gs > 1) Gs = 1;
        G = Gs;
        if (lane < G) {
          st->Enext[lane] = Emine;
          st->ckey[lane] = kmine;
        }
        if (lane == 0) {
          st->G = G;
          st->stop = stopr;
        }
        __syncwarp();
        if (rank == 0 && lane < G) {  // atoms / energies (final once verified)
          const Ent& e = ent[pl];
          AtomOut a;
          a.w = e.u;
          a.m = e.k;
          a.n = e.j;
          a.flags = e.selfc;
          a.re = e.tre;
          a.im = e.tim;
          atoms_out[it0 + lane] = a;
          energy_out[it0 + lane + 1] = Emine;
        }
        PROF_MARK(28);
#if !MPG_SCAN_W1
        item_scan(G);
#endif
      }
      PROF_MARK(9);
      __syncthreads();
      PROF_MARK(10);
      if (st->stop) {
        ++rounds;
        break;
      }
      lo = 0;
      gvend = st->G * 16;
      hi = st->ibase[gvend];
    } else {
      // roll back the rejected candidates' tiles (their items of the last round)
      lo = st->ibase[st->rb_from * 16];
      gvend = st->G * 16;
      hi = st->ibase[gvend];
      PROF_MARK(10);
    }
    ++rounds;
    // ---- B. residual update (or roll-back) over this CTA's rows ------------
    // tile bookkeeping: record, candidate maximum, dirty level-0 node (stamp + list)
    const int stampv = round + 1;
    const uint64_t theta = TOPK == 2 ? cls->theta : 0ull;
    // (the winning lane of the tile's warp argmax)
    auto finish_lane = [&](int l, int g, R bs, uint32_t bp, R bre, R bim, auto upd) {
      {
        RecT rec;
        rec.s = bs;
        rec.re = bre;
        rec.im = bim;
        rec.p = bp;
        if constexpr (sizeof(R) == 8) rec.pad = 0;
        MPG_CHECK(l >= 0 && l < P.Lc && g >= 0 && g < BMAX, "tile record / candidate index out of range");
        trec[l] = rec;
        if constexpr (decltype(upd)::value) atomicMax(&vkey[g], score_key(bs));
        if constexpr (TOPK == 2) {  // a rewritten tile at or above theta joins the candidate list
          hk[l] = hkey(bs);
          if (skey64(bs) >= theta && !inl[l]) {   // (inl[l] = 1 exactly for stored entries)
            const int idx = atomicAdd(&cls->n, 1);
            if (idx < CL_CAP) {
              clid[idx] = (int)l;
              inl[l] = 1;
            }
          }
        }
        const int node = l >> 5;
        if (!notree && atomicExch(&stamp[node], stampv) != stampv) list[atomicAdd(&cnt[0], 1)] = node;
      }
    };
    auto finish = [&](int l, int g, R bs, uint32_t bp, R bre, R bim, auto upd) {
      if (lane == warp_argmax_lane(bs, bp)) finish_lane(l, g, bs, bp, bre, bim, upd);
    };
    // (g, v) of item gi: count the item bases <= gi (ibase is non-decreasing)
    auto item_gv = [&](int gi) {
      int c = 0;
#pragma unroll
      for (int h4 = 0; h4 < IPL / 4; ++h4) {
        const int i0 = lane * IPL + 4 * h4;
        const int4 b4 = *reinterpret_cast<const int4*>(&st->ibase[i0]);
        c += (i0 + 0 >= 1 && i0 + 0 <= gvend && b4.x <= gi) ? 1 : 0;
        c += (i0 + 1 >= 1 && i0 + 1 <= gvend && b4.y <= gi) ? 1 : 0;
        c += (i0 + 2 <= gvend && b4.z <= gi) ? 1 : 0;
        c += (i0 + 3 <= gvend && b4.w <= gi) ? 1 : 0;
      }
      return (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    };
    // one update item in flight: geometry, then every load issued (setup), then the
    // fold-rule update, stores and tile bookkeeping (process)
    struct ItemS {
      C2* row;
      C2* bkrow;
      uint32_t pbase;
      int l0, t0, tt, Tr, MR, g, v;
      C2 cv[TPI][NCH], hd[TPI][NCH], hc[TPI][NCH], z0;
      bool fd[TPI][NCH], fc[TPI][NCH], cf[TPI][NCH];
    };
    auto setup = [&](int gi, ItemS& S) {
      const int gv = item_gv(gi);
      const int g = gv >> 4, v = gv & 15;
      const int e = st->pick[g];
      const VGeo& gg = egeo[e * W + v];
      const DictGeo& dv = sd[v];
      const int Tr = gg.Tr, t0 = gg.t0, MR = dv.MR;
      const int hp = (Tr + TPI - 1) / TPI;
      const int it = gi - st->ibase[gv];
      // row among this CTA's rows of (g, v): it / hp by the reciprocal (exact: it * hp < 2^32)
      const int i = hp > 1 ? (int)__umulhi((uint32_t)it, (uint32_t)gg.pad) : it;
      const int tt = TPI * (it - i * hp);   // first tile of the item
      const int r = i < gg.cntA ? gg.rhoA + (i << lgC) : gg.rA + gg.rhoB + ((i - gg.cntA) << lgC);
      int nrow = gg.n0 + r;
      if (nrow >= dv.N) nrow -= dv.N;
      MPG_CHECK(nrow >= 0 && nrow < dv.N && r >= 0 && r < gg.nr, "item row outside the target grid");
      MPG_CHECK(((dv.frame_off + nrow) & (C - 1)) == rank, "item row not owned by this CTA");
      S.l0 = sown[v].loc_base + ((nrow - sown[v].n_first) >> lgC) * dv.T;
      MPG_CHECK(S.l0 >= 0 && S.l0 + t0 + Tr <= P.Lc, "tile record index out of range");
      MPG_CHECK(st->tbase[gv] + (long long)(i + 1) * Tr <= P.bk_cap, "backup slot out of range");
      MPG_CHECK(gg.kbase + (long long)(r + 1) * gg.nc <= P.kern_elems, "kernel row out of range");
      S.row = grid + dv.grid_off + (long long)nrow * dv.stride;
      S.bkrow = backup + ((long long)st->tbase[gv] + (long long)i * Tr) * TW;
      S.pbase = (uint32_t)dv.off + (uint32_t)nrow * (uint32_t)MR;
      S.t0 = t0;
      S.tt = tt;
      S.Tr = Tr;
      S.MR = MR;
      S.g = g;
      S.v = v;
      const Ent& en = ent[e];
      const PairGeo& pg = sp[en.u * W + v];
      const bool selfc = en.selfc != 0;
      // modulation omega_R^{(k' nu) mod R} of this row (Eq. (15))
      const int rrx = (gg.rr0 + r * gg.rrstep) & (pg.R - 1);
      S.z0 = row_z0<C2, R>(en.tre, en.tim, roots[rrx * pg.rstep]);
      const C2* hrow = kern + gg.kbase + (long long)r * gg.nc;
      const int q0 = gg.q0, nc = gg.nc, Mv = dv.M;
#pragma unroll
      for (int q = 0; q < TPI; ++q)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {  // issue every load before any store
          const int bin = (t0 + tt + q) * TW + ch * 32 + lane;
          const bool valid = (tt + q < Tr) && bin < MR;
          MPG_CHECK(!valid || bin < dv.stride, "bin outside the row stride");
          const int cd = (bin - q0) & (Mv - 1);   // direct source column  (q = bin)
          const int cc = (-bin - q0) & (Mv - 1);  // conjugate source column (q = M - bin)
          S.fd[q][ch] = valid && cd < nc;
          S.fc[q][ch] = valid && !selfc && cc < nc;
          S.cf[q][ch] = cc < cd;                  // oracle order: ascending source column
          S.cv[q][ch] = valid ? S.row[bin] : C2{0, 0};
          S.hd[q][ch] = S.fd[q][ch] ? hrow[cd] : C2{0, 0};
          S.hc[q][ch] = S.fc[q][ch] ? hrow[cc] : C2{0, 0};
        }
    };
    auto process = [&](ItemS& S) {
      if (S.g > 0) {  // speculative candidate: keep the tiles for a roll-back
#pragma unroll
        for (int q = 0; q < TPI; ++q)
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
            if (S.tt + q < S.Tr && (S.t0 + S.tt + q) * TW + ch * 32 + lane < S.MR)
              S.bkrow[(long long)(S.tt + q) * TW + ch * 32 + lane] = S.cv[q][ch];
      }
      const DictGeo& dv = sd[S.v];
#pragma unroll
      for (int q = 0; q < TPI; ++q) {
        if (S.tt + q >= S.Tr) break;
        const int t = S.t0 + S.tt + q;
        C2 cn[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          const int bin = t * TW + ch * 32 + lane;
          cn[ch] = fold_update<R>(S.cv[q][ch], S.z0, S.hd[q][ch], S.hc[q][ch], S.fd[q][ch], S.fc[q][ch], S.cf[q][ch]);
          if (bin < S.MR && (S.fd[q][ch] || S.fc[q][ch])) S.row[bin] = cn[ch];
        }
        R bs, bre, bim;
        uint32_t bp;
        lane_best<R, C2, NCH>(cn, t * TW + lane, S.MR, dv.M, S.pbase, P.pedantic != 0, srho + rho_off[S.v],
                              rho_lo[S.v], rho_n[S.v], bs, bp, bre, bim);
        finish(S.l0 + t, S.g, bs, bp, bre, bim, std::true_type{});
      }
    };
    if (mode == 0) {
      // MPG_ITEMS_IN_FLIGHT = 2: two items per warp in flight (32-bin tiles only; it spills
      // at 128 registers and was slower: C2 2.24 vs 1.93 us/atom)
      constexpr int IF = NCH == 1 ? MPG_ITEMS_IN_FLIGHT : 1;
      for (int gi = lo + warp; gi < hi; gi += IF * NW) {
        ItemS A[IF];
#pragma unroll
        for (int f = 0; f < IF; ++f)   // every item's loads in flight before the first update
          if (gi + f * NW < hi) setup(gi + f * NW, A[f]);
#pragma unroll
        for (int f = 0; f < IF; ++f)
          if (gi + f * NW < hi) process(A[f]);
      }
    } else {
      // roll back the rejected candidates' tiles from their backups
      for (int gi = lo + warp; gi < hi; gi += NW) {
        const int gv = item_gv(gi);
        const int g = gv >> 4, v = gv & 15;
        const VGeo& gg = egeo[st->pick[g] * W + v];
        const DictGeo& dv = sd[v];
        const int Tr = gg.Tr, t0 = gg.t0, MR = dv.MR;
        const int hp = (Tr + TPI - 1) / TPI;
        const int it = gi - st->ibase[gv];
        const int i = hp > 1 ? (int)__umulhi((uint32_t)it, (uint32_t)gg.pad) : it;
        const int tt = TPI * (it - i * hp);
        const int r = i < gg.cntA ? gg.rhoA + (i << lgC) : gg.rA + gg.rhoB + ((i - gg.cntA) << lgC);
        int nrow = gg.n0 + r;
        if (nrow >= dv.N) nrow -= dv.N;
        const int l0 = sown[v].loc_base + ((nrow - sown[v].n_first) >> lgC) * dv.T;
        C2* row = grid + dv.grid_off + (long long)nrow * dv.stride;
        const C2* bkrow = backup + ((long long)st->tbase[gv] + (long long)i * Tr) * TW;
        const uint32_t pbase = (uint32_t)dv.off + (uint32_t)nrow * (uint32_t)MR;
        for (int q = 0; q < TPI && tt + q < Tr; ++q) {
          const int t = t0 + tt + q;
          const C2* bk = bkrow + (long long)(tt + q) * TW;
          C2 cv[NCH];
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int bin = t * TW + ch * 32 + lane;
            if (bin < MR) cv[ch] = bk[ch * 32 + lane];
          }
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int bin = t * TW + ch * 32 + lane;
            if (bin < MR) row[bin] = cv[ch];
          }
          R bs, bre, bim;
          uint32_t bp;
          lane_best<R, C2, NCH>(cv, t * TW + lane, MR, dv.M, pbase, P.pedantic != 0, srho + rho_off[v], rho_lo[v],
                                rho_n[v], bs, bp, bre, bim);
          finish(l0 + t, g, bs, bp, bre, bim, std::false_type{});
        }
      }
    }
    PROF_MARK(11);
    __syncthreads();
    // ---- C. level-0 refresh of the dirty nodes, then the upper levels, one level
    //      at a time, nodes spread over the warps
    if (!notree) {  // level 0 (children: the tile records)
      const int nl = cnt[0];
      const bool up = P.nlev > 1;
      for (int idx = warp; idx < nl; idx += NW) {
        const int node = list[idx];
        const long long c = (long long)node * 32 + lane;
        const RecT rc = c < P.Lc ? trec[c] : empty_rec(R(0));
        if (lane == warp_argmax_lane(rc.s, rc.p)) {
          lev[node] = rc;
          if (up) {
            const int par2 = node >> 5;
            int* st2 = stamp + P.lev_off[1];
            if (atomicExch(&st2[par2], stampv) != stampv) list[P.lev_off[1] + atomicAdd(&cnt[1], 1)] = par2;
          }
        }
      }
      __syncthreads();
    }
    for (int l = 1; !notree && l < P.nlev; ++l) {
      const int nl = cnt[l];
      const RecT* child = lev + P.lev_off[l - 1];
      const long long nchild = (long long)P.lev_n[l - 1];
      for (int idx = warp; idx < nl; idx += NW) {
        const int node = list[P.lev_off[l] + idx];
        const long long c = (long long)node * 32 + lane;
        const RecT rc = c < nchild ? child[c] : empty_rec(R(0));
        if (lane == warp_argmax_lane(rc.s, rc.p)) {
          lev[P.lev_off[l] + node] = rc;
          if (l + 1 < P.nlev) {
            const int par2 = node >> 5;
            int* st2 = stamp + P.lev_off[l + 1];
            if (atomicExch(&st2[par2], stampv) != stampv) list[P.lev_off[l + 1] + atomicAdd(&cnt[l + 1], 1)] = par2;
          }
        }
      }
      __syncthreads();
    }
    PROF_MARK(12);
    // (no barrier needed: every use of cnt ended at the refresh's last barrier, and
    // st->G is next read by this thread's warp after the message exchange)
    if (tid == 0) {
      for (int l = 0; l < P.nlev; ++l) cnt[l] = 0;
      if (mode == 1) st->G = 0;  // nothing to verify after a roll-back
    }
    topk((unsigned long long)round + 2);
    if (P.prof != nullptr && slot == 0 && tid == 0) {  // per-CTA busy time (receive -> publish) and items
      const unsigned long long busy = (unsigned long long)(clock64() - tbusy0);
      if (rank < 16) atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 40 + rank, busy);
      if (rank < 128) {
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 64 + rank, busy);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 192 + rank, (unsigned long long)(hi - lo));
      }
      // every CTA's rounds by items (8 per bucket) and by busy cycles (4096 per bucket)
      atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 480 + min((hi - lo) >> 3, 15), 1ull);
      atomicAdd(reinterpret_cast<unsigned long long*>(P.prof) + 496 + (int)min(busy >> 12, 15ull), 1ull);
    }
    push_msg(par ^ 1, (unsigned long long)round + 2);
    rebuild_after();
  }
  if (rank == 0 && tid == 0) {
    P.result[slot].n_done = st->it;
    P.result[slot].stop = st->stop;
    P.result[slot].E_final = st->E;
    P.result[slot].rounds = rounds;
    P.result[slot].E0 = E0s;
  }
  if (prof) P.prof[15] = rounds;
#undef PROF_MARK
  if constexpr (!GX) cg::this_cluster().sync();  // keep shared memory alive until all remote stores are done
}

template <typename R, int TW, bool SREC, int K, bool GX, int TOPK = 0>
cudaError_t launch_t(const LoopParams& P, int threads, cudaStream_t st) {
  auto kfn = mp_multi_kernel<R, TW, SREC, K, GX, TOPK>;
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

template <typename R, int TW, bool SREC, int K>
int max_cluster_t(int threads, size_t smem) {
  auto kfn = mp_multi_kernel<R, TW, SREC, K, false>;
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
template <typename R, int TW, bool SREC, int K>
int max_grid_t(int threads, size_t smem) {
  auto kfn = mp_multi_kernel<R, TW, SREC, K, true>;
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
  if (P.topk_scan == 2) switch (P.TW) {  // candidate lists (records in shared or global memory)
      case 32: return launch_t<R, 32, SREC, MULTI_K, GX, 2>(P, threads, st);
      case 64: return launch_t<R, 64, SREC, MULTI_K, GX, 2>(P, threads, st);
      case 128: return launch_t<R, 128, SREC, MULTI_K, GX, 2>(P, threads, st);
    }
  if constexpr (SREC && !GX) {
    if (P.topk_scan == 1) switch (P.TW) {
        case 32: return launch_t<R, 32, true, MULTI_K, false, 1>(P, threads, st);
        case 64: return launch_t<R, 64, true, MULTI_K, false, 1>(P, threads, st);
        case 128: return launch_t<R, 128, true, MULTI_K, false, 1>(P, threads, st);
      }
  }
  switch (P.TW) {
    case 32: return launch_t<R, 32, SREC, MULTI_K, GX>(P, threads, st);
    case 64: return launch_t<R, 64, SREC, MULTI_K, GX>(P, threads, st);
    case 128: return launch_t<R, 128, SREC, MULTI_K, GX>(P, threads, st);
  }
  return cudaErrorInvalidValue;
}
template <typename R, bool GX>
int max_cluster_g(bool srec, int TW, int threads, size_t smem) {
  auto one = [&](auto srec_c) -> int {
    constexpr bool S = decltype(srec_c)::value;
    switch (TW) {
      case 32:
        if constexpr (GX) return max_grid_t<R, 32, S, MULTI_K>(threads, smem);
        else return max_cluster_t<R, 32, S, MULTI_K>(threads, smem);
      case 64:
        if constexpr (GX) return max_grid_t<R, 64, S, MULTI_K>(threads, smem);
        else return max_cluster_t<R, 64, S, MULTI_K>(threads, smem);
      case 128:
        if constexpr (GX) return max_grid_t<R, 128, S, MULTI_K>(threads, smem);
        else return max_cluster_t<R, 128, S, MULTI_K>(threads, smem);
    }
    return 0;
  };
  return srec ? one(std::true_type{}) : one(std::false_type{});
}

}  // namespace

// one translation unit per (precision, exchange mode): its launcher and occupancy query
#define MPG_MULTI_TU(R, GX, NAME)                                                                 \
  cudaError_t launch_multi_##NAME(const LoopParams& P, int threads, cudaStream_t st) {           \
    return P.srec ? launch_r<R, true, GX>(P, threads, st) : launch_r<R, false, GX>(P, threads, st); \
  }                                                                                               \
  int max_multi_##NAME(bool srec, int TW, int threads, size_t smem) {                             \
    return max_cluster_g<R, GX>(srec, TW, threads, smem);                                         \
  }
