/*
 * mploop.c -- oracle coefficient-domain matching pursuit loop (fp64, one thread).
 *
 * TEST INFRASTRUCTURE ONLY: called from oracle/loop.py by tests/, smoke() and
 * bench.py's cpu_baseline leg.  Shares no code with the CUDA path.
 *
 * Follows, step by step (readings Z9..Z15 in DESIGN.md):
 *   Alg. 1 with the approximate recursion Eq. (9) P:424-434,
 *   the real-atom adjustment Eq. (19) P:863-875 and pair energy Eq. (20) P:876-892,
 *   the rho lookup from the auto-kernel P:961-967,
 *   the residual update of Alg. 3 P:978-1029 over the subsampled, modulated
 *   cross-kernels Eq. (15)-(17) P:558-573, with the fold rule Z14.
 * Max tracking is a per-frame max cache plus a 64-frame group level (the
 * paper's tournament trees P:923-958 reduced to two levels, O11); a
 * full-scan mode exists to pin it.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction so that
 * |c|^2 = re*re + im*im is evaluated exactly as written).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t a, M, N, MR;   /* hop, channels, frames N = L/a, reduced bins M/2+1 */
  int64_t off;           /* first global coefficient index p of this dictionary */
} orc_dict;

typedef struct {
  int32_t a_c, M_c;                    /* common grid              */
  int32_t mu_lo, mu_hi, nu_lo, nu_hi;  /* bounding box of kept entries          */
  const double* h;                     /* [nu][mu] complex interleaved, zeros   */
} orc_kernel;

typedef struct {
  int32_t w, m, n, flags;  /* flags bit0: self-conjugate atom (m = 0 or m = M/2) */
  double re, im;           /* adjusted coefficient c~ (Eq. (19))                 */
} orc_atom;

enum { STOP_MAXIT = 1, STOP_ERRTOL = 2, STOP_NEGEST = 3, STOP_ZERO = 4 };

static int64_t floordiv_i(int64_t a, int64_t b) { int64_t q = a / b; if ((a % b) && ((a < 0) != (b < 0))) --q; return q; }
static int64_t floormod_i(int64_t a, int64_t b) { int64_t r = a % b; if (r < 0) r += b; return r; }

typedef struct {
  int32_t W;
  const orc_dict* D;
  const orc_kernel* K;
  double* res;          /* residual c^ : complex interleaved, index p */
  int64_t P, F, G;      /* coefficients, frames, 64-frame groups */
  int64_t* fr_off;      /* first frame id of each dictionary */
  double* fs; int64_t* fi;   /* per-frame best score / index */
  double* gs; int64_t* gi;   /* per-group best score / index */
  int64_t* touched; int64_t ntouched, cap;
  int32_t pedantic;
} st_t;

static void rho_lookup(const st_t* S, int32_t u, int64_t k, double* rre, double* rim);

/* selection score of coefficient p = atom (w, bin k):
 *   non-pedantic (default, Z9): |c^|^2;
 *   pedantic: the energy Eq. (20) removes, with c~ of Eq. (19) (reading Z11)
 *   -- (Re c^)^2 for a self-conjugate atom (Z13), else 2[X^2+Y^2+Re rho(X^2-Y^2)-2 Im rho XY],
 *   c~ = X + iY = (c^ - conj(rho) conj(c^)) * (1/(1-|rho|^2)), rho = h_ww(-2k, 0) (Z12). */
static double score_wk(const st_t* S, int32_t w, int64_t k, int64_t p) {
  double re = S->res[2 * p], im = S->res[2 * p + 1];
  if (!S->pedantic) return re * re + im * im;
  if (k == 0 || 2 * k == S->D[w].M) return re * re;
  double rre, rim; rho_lookup(S, w, k, &rre, &rim);
  double inv = 1.0 / (1.0 - (rre * rre + rim * rim));
  double nre = re - (rre * re - rim * im);
  double nim = im + (rre * im + rim * re);
  double X = nre * inv, Y = nim * inv;
  double X2 = X * X, Y2 = Y * Y, XY = X * Y;
  return 2.0 * (X2 + Y2 + rre * (X2 - Y2) - 2.0 * rim * XY);
}

static double score_at(const st_t* S, int64_t p) {
  int32_t w = 0;
  while (w + 1 < S->W && S->D[w + 1].off <= p) ++w;
  return score_wk(S, w, (p - S->D[w].off) % S->D[w].MR, p);
}

static void frame_wn(const st_t* S, int64_t f, int32_t* w, int64_t* n) {
  int32_t v = 0;
  while (v + 1 < S->W && S->fr_off[v + 1] <= f) ++v;
  *w = v; *n = f - S->fr_off[v];
}

/* frame max: strict '>' over ascending bins keeps the lowest index among ties (Z10) */
static void scan_frame(st_t* S, int64_t f) {
  int32_t w; int64_t n; frame_wn(S, f, &w, &n);
  int64_t p0 = S->D[w].off + n * S->D[w].MR;
  double bs = -1.0; int64_t bi = p0;
  for (int64_t p = p0; p < p0 + S->D[w].MR; ++p) {
    double s = score_wk(S, w, p - p0, p);
    if (s > bs) { bs = s; bi = p; }
  }
  S->fs[f] = bs; S->fi[f] = bi;
}

static void scan_group(st_t* S, int64_t g) {
  int64_t f0 = g * 64, f1 = f0 + 64 < S->F ? f0 + 64 : S->F;
  double bs = -1.0; int64_t bi = 0;
  for (int64_t f = f0; f < f1; ++f)
    if (S->fs[f] > bs) { bs = S->fs[f]; bi = S->fi[f]; }
  S->gs[g] = bs; S->gi[g] = bi;
}

static void touch(st_t* S, int32_t v, int64_t n) {
  if (S->ntouched == S->cap) {
    S->cap *= 2;
    S->touched = (int64_t*)realloc(S->touched, (size_t)S->cap * sizeof(int64_t));
  }
  S->touched[S->ntouched++] = S->fr_off[v] + n;
}

/* second best over all p != pstar (for the near-tie gap report):
 * s2 = max of the score over every coefficient other than p*.  With the max caches
 * (up to date before every selection) the frame of p* is rescanned and every other
 * frame contributes its cached maximum; in full-scan mode the caches are never
 * refreshed, so s2 is a plain scan over all p != p*. */
static double second_best(const st_t* S, int64_t pstar, int64_t fstar, int32_t full_scan) {
  double s2 = 0.0;
  if (full_scan) {
    for (int64_t p = 0; p < S->P; ++p)
      if (p != pstar) { double s = score_at(S, p); if (s > s2) s2 = s; }
    return s2;
  }
  int32_t w; int64_t n; frame_wn(S, fstar, &w, &n);
  int64_t p0 = S->D[w].off + n * S->D[w].MR;
  for (int64_t p = p0; p < p0 + S->D[w].MR; ++p)
    if (p != pstar) { double s = score_at(S, p); if (s > s2) s2 = s; }
  int64_t gstar = fstar / 64;
  for (int64_t g = 0; g < S->G; ++g) {
    if (g != gstar) { if (S->gs[g] > s2) s2 = S->gs[g]; continue; }
    int64_t f1 = g * 64 + 64 < S->F ? g * 64 + 64 : S->F;
    for (int64_t f = g * 64; f < f1; ++f)
      if (f != fstar && S->fs[f] > s2) s2 = S->fs[f];
  }
  return s2;
}

/*
 * Residual update (Alg. 3) for one selected atom (u, k, j) with
 * adjusted coefficient ct, over every dictionary v:
 *   a_c = min(a_u,a_v), M_c = max(M_u,M_v), s_m = M_c/M_v, k' = k M_c/M_u, t_u = j a_u,
 *   for nu in box with (t_u + nu a_c) = 0 mod a_v:  n = (t_u + nu a_c)/a_v mod N_v,
 *     z0 = ct * omega_R^{(k' nu) mod R},  R = M_c/a_c         (Eq. (15))
 *     for mu in box with (k' + mu) = 0 mod s_m:  q = (k'+mu)/s_m mod M_v,  z = z0 h(mu,nu)
 *       direct:  q <= M_v/2            -> c^_v(q,n) -= z
 *       conj (pair atoms only, Z14): q == 0 or q >= M_v/2  -> c^_v((M_v-q) mod M_v, n) -= conj(z)
 */
static void update(st_t* S, int32_t u, int64_t k, int64_t j, double cre, double cim, int selfconj) {
  const orc_dict* du = &S->D[u];
  for (int32_t v = 0; v < S->W; ++v) {
    const orc_dict* dv = &S->D[v];
    const orc_kernel* K = &S->K[u * S->W + v];
    int64_t a_c = K->a_c, M_c = K->M_c, R = M_c / a_c;
    int64_t s_m = M_c / dv->M;
    int64_t kp = k * (M_c / du->M);
    int64_t t_u = j * du->a;
    int64_t nmu = K->mu_hi - K->mu_lo + 1;
    /* first nu >= nu_lo with (t_u + nu a_c) divisible by a_v, then step a_v/a_c */
    int64_t s_n = dv->a / a_c > 0 ? dv->a / a_c : 1;
    int64_t nu = K->nu_lo;
    while (floormod_i(t_u + nu * a_c, dv->a) != 0) ++nu;
    for (; nu <= K->nu_hi; nu += s_n) {
      int64_t n = floormod_i(floordiv_i(t_u + nu * a_c, dv->a), dv->N);
      int64_t r = floormod_i(kp * nu, R);
      double ang = 2.0 * M_PI * (double)r / (double)R;     /* omega_R^r, r reduced first (O5) */
      double wre = cos(ang), wim = sin(ang);
      double z0re = cre * wre - cim * wim, z0im = cre * wim + cim * wre;
      const double* hrow = K->h + 2 * (nu - K->nu_lo) * nmu;
      double* cv = S->res + 2 * (dv->off + n * dv->MR);
      int64_t mu = K->mu_lo;
      while (floormod_i(kp + mu, s_m) != 0) ++mu;
      for (; mu <= K->mu_hi; mu += s_m) {
        int64_t q = floormod_i(floordiv_i(kp + mu, s_m), dv->M);
        double hre = hrow[2 * (mu - K->mu_lo)], him = hrow[2 * (mu - K->mu_lo) + 1];
        double zre = z0re * hre - z0im * him, zim = z0re * him + z0im * hre;
        if (2 * q <= dv->M) { cv[2 * q] -= zre; cv[2 * q + 1] -= zim; }
        if (!selfconj && (q == 0 || 2 * q >= dv->M)) {
          int64_t qc = floormod_i(dv->M - q, dv->M);
          cv[2 * qc] -= zre; cv[2 * qc + 1] += zim;      /* -= conj(z) */
        }
      }
      touch(S, v, n);
    }
  }
}

/* rho = <d, conj d> = h_uu(-2k mod M_u, 0) if kept, else 0 (Z12) */
static void rho_lookup(const st_t* S, int32_t u, int64_t k, double* rre, double* rim) {
  const orc_kernel* K = &S->K[u * S->W + u];
  int64_t M = S->D[u].M;
  int64_t mu = floormod_i(-2 * k, M);
  if (2 * mu > M) mu -= M;
  *rre = 0.0; *rim = 0.0;
  if (mu < K->mu_lo || mu > K->mu_hi || 0 < K->nu_lo || 0 > K->nu_hi) return;
  int64_t nmu = K->mu_hi - K->mu_lo + 1;
  const double* e = K->h + 2 * ((0 - K->nu_lo) * nmu + (mu - K->mu_lo));
  *rre = e[0]; *rim = e[1];
}

int orc_mp_run(int32_t W, const orc_dict* D, const orc_kernel* K, double* res, double* sol,
               int64_t maxit, double Etol, double E0, int32_t full_scan, int32_t pedantic,
               orc_atom* atoms, double* energy, double* gaps, int64_t* n_done, int32_t* stop) {
  st_t S;
  memset(&S, 0, sizeof S);
  S.W = W; S.D = D; S.K = K; S.res = res; S.pedantic = pedantic;
  S.fr_off = (int64_t*)malloc((size_t)(W + 1) * sizeof(int64_t));
  S.P = 0; S.F = 0;
  for (int32_t w = 0; w < W; ++w) { S.fr_off[w] = S.F; S.F += D[w].N; S.P += (int64_t)D[w].N * D[w].MR; }
  S.fr_off[W] = S.F;
  S.G = (S.F + 63) / 64;
  S.fs = (double*)malloc((size_t)S.F * sizeof(double)); S.fi = (int64_t*)malloc((size_t)S.F * sizeof(int64_t));
  S.gs = (double*)malloc((size_t)S.G * sizeof(double)); S.gi = (int64_t*)malloc((size_t)S.G * sizeof(int64_t));
  S.cap = 1024; S.touched = (int64_t*)malloc((size_t)S.cap * sizeof(int64_t));
  for (int64_t f = 0; f < S.F; ++f) scan_frame(&S, f);
  for (int64_t g = 0; g < S.G; ++g) scan_group(&S, g);

  double E = E0;                          /* E_0 = ||x||^2 (Alg. 1 init) */
  int64_t it = 0;
  energy[0] = E;
  *stop = 0;
  for (;;) {
    /* a. stop tests, before selection, on the estimate E_k (Z15) */
    if (it >= maxit) { *stop = STOP_MAXIT; break; }
    if (E <= Etol) { *stop = STOP_ERRTOL; break; }
    if (E < 0.0) { *stop = STOP_NEGEST; break; }
    /* b. selection p* = argmax of the score (|c^|^2, or pedantic), ties -> lowest p (Alg. 1 step 1, Z9/Z10) */
    int64_t ps; double s1;
    if (full_scan) {
      s1 = -1.0; ps = 0;
      for (int64_t p = 0; p < S.P; ++p) { double s = score_at(&S, p); if (s > s1) { s1 = s; ps = p; } }
    } else {
      s1 = -1.0; ps = 0;
      for (int64_t g = 0; g < S.G; ++g) if (S.gs[g] > s1) { s1 = S.gs[g]; ps = S.gi[g]; }
    }
    if (!(s1 > 0.0)) { *stop = STOP_ZERO; break; }
    int32_t u = 0;
    while (u + 1 < W && D[u + 1].off <= ps) ++u;
    int64_t j = (ps - D[u].off) / D[u].MR, k = (ps - D[u].off) % D[u].MR;
    if (gaps) {
      double s2 = second_best(&S, ps, S.fr_off[u] + j, full_scan);
      gaps[it] = (s1 - s2) / s1;
    }
    /* c. scalar step: c~ (Eq. (19), reading Z11 uses conj(rho)) and E~ (Eq. (20)) */
    double cre = res[2 * ps], cim = res[2 * ps + 1], tre, tim, Et;
    int selfconj = (k == 0) || (2 * k == D[u].M);
    if (selfconj) {                      /* real atom, no conjugate partner (Z13) */
      tre = cre; tim = 0.0; Et = tre * tre;
    } else {
      double rre, rim; rho_lookup(&S, u, k, &rre, &rim);
      double den = 1.0 - (rre * rre + rim * rim);
      /* c^ - conj(rho) conj(c^) = (cre + i cim) - (rre - i rim)(cre - i cim) */
      double nre = cre - (rre * cre - rim * cim);
      double nim = cim - (-rre * cim - rim * cre);
      tre = nre / den; tim = nim / den;
      double X2 = tre * tre, Y2 = tim * tim, XY = tre * tim;
      Et = 2.0 * (X2 + Y2 + rre * (X2 - Y2) - 2.0 * rim * XY);
    }
    /* d. record: E_{k+1} = E_k - E~, atom list, solution c(p) += c~ (Z19) */
    double Enext = E - Et;
    atoms[it].w = u; atoms[it].m = (int32_t)k; atoms[it].n = (int32_t)j;
    atoms[it].flags = selfconj ? 1 : 0; atoms[it].re = tre; atoms[it].im = tim;
    energy[it + 1] = Enext;
    if (sol) { sol[2 * ps] += tre; sol[2 * ps + 1] += tim; }
    /* e. residual update (Alg. 3 with fold rule) */
    S.ntouched = 0;
    update(&S, u, k, j, tre, tim, selfconj);
    if (!full_scan) {
      for (int64_t t = 0; t < S.ntouched; ++t) scan_frame(&S, S.touched[t]);
      for (int64_t t = 0; t < S.ntouched; ++t) scan_group(&S, S.touched[t] / 64);
    }
    E = Enext;
    ++it;                                /* f. */
  }
  *n_done = it;
  free(S.fr_off); free(S.fs); free(S.fi); free(S.gs); free(S.gi); free(S.touched);
  return 0;
}
