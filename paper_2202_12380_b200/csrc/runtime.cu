// runtime.cu -- host runtime and C ABI of libmpgabor (include/mpgabor.h).
//
// Owns the handle: dictionary validation, window/twiddle/root tables,
// kernel precompute orchestration (N2), per-length layout (padding Z3, grids,
// tiles, tile-record slices), device buffers, launches of N1/N4/N5/N6 and the
// error strings.  Every arithmetic step of the method runs in the CUDA kernels;
// this file only computes sizes, offsets and launch geometry.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/mpgabor.h"
#include "launch.h"

namespace {

thread_local std::string g_create_error = "no error";

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n ? n : 16);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const { return reinterpret_cast<T*>(p); }
};

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

}  // namespace

struct mpgabor {
  std::vector<mpg_dict> dicts;
  int W = 0;
  int precision = MPG_F64;
  std::string err = "no error";
  int device = -1;

  // tables
  int twres = 0, Rmax = 0, a_min = 0, M_max = 0;
  DevBuf tw, roots, win;
  std::vector<int64_t> win_off;

  // kernels
  bool have_kernels = false;
  double thr = 0.0;
  std::vector<PairGeo> pairs;
  std::vector<int> nu_first, nlag;
  std::vector<double> pair_mx;
  std::vector<int64_t> pair_kept, box_off;
  int64_t kern_elems = 0, box_total = 0, kept_total = 0;
  DevBuf kern, boxcopy, d_pairs, rho, rho_meta, Hscratch, mxbox;
  std::vector<int> rho_lo, rho_n, rho_off;
  int rho_total = 0;

  // launch tuning
  int cluster_req = 0, threads = 512, TW_req = 0, srec_req = 0;  // 0 = automatic
  int TW = 64, srec = 0;
  int run_threads = 512;  // threads of the planned loop launch
  // grid slots [0, pad_clean) of the allocation pad_ptr hold zero row padding for the
  // current layout: their analysis skips the padding stores (a new layout or a new
  // allocation resets it)
  int pad_clean = 0;
  void* pad_ptr = nullptr;
  int batch = 0;          // candidates per round: 0 auto (multi-selection, multi_max_batch()), 1 one selection
  int kind = 2;           // loop kernel: 0 mploop.cu, 2 mpmulti.cu
  bool force_single = false;  // multi-selection impossible for this layout: use mploop.cu
  bool gx = false;            // loop kernel as a cooperative grid (> 16 CTAs, global exchange)
  bool batch_mode = false;    // batched signals: one cluster per signal
  int batch_C = 16;           // batched signals: automatic cluster size per signal
  int pedantic = 0;           // 1: pedantic selection (Eq. (20) energies)
  DevBuf sfirst, sdone;       // synthesis scratch: first atom per coefficient, retired atoms + control words
  DevBuf gxrec, gxstamp;

  // per-length layout
  int64_t L = -1, Ls_cached = -1;
  int lay_TW = 0, lay_C = 0;
  std::vector<DictGeo> geo;
  std::vector<OwnGeo> own;
  DevBuf d_own;
  int64_t grid_elems = 0, total_tiles = 0, Lc = 0, P_R = 0;
  LoopParams lp{};
  DevBuf d_geo, grid, rec, xp, partial, flag, E0, result, backup;

  // synth / host-api scratch
  DevBuf sol, frames, hx, hatoms, henergy, hy;
  DevBuf rr, yy;          // resets: signal-domain residual r_out and the pass synthesis
  int passes = 0;         // passes of the last mpgabor_run_reset

  int prof_mode = 0;
  long long prof_host[MPG_PROF_SLOTS] = {};
  DevBuf prof;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  // DGT fork/join: the W dictionaries' analysis kernels run on side streams so that one
  // kernel's tail waves overlap the next kernel's first (MPGABOR_DGT_STREAMS=0: in line)
  cudaStream_t dgt_st[MPG_MAX_DICTS] = {};
  cudaEvent_t dgt_fork = nullptr, dgt_join[MPG_MAX_DICTS] = {};
  int dgt_streams = -1;   // -1 not decided, 0 off, 1 on
  float t_dgt = 0, t_init = 0, t_loop = 0;
  int64_t launches = 0;  // kernels of this library enqueued through this handle

  int fail(int code, const std::string& msg) {
    err = msg;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* where) {
    err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    cudaGetLastError();
    return e == cudaErrorMemoryAllocation ? MPG_ENOMEM : MPG_ECUDA;
  }
  bool f64() const { return precision == MPG_F64; }
  size_t celem() const { return f64() ? sizeof(double2) : sizeof(float2); }
};

#define TRY_CUDA(h, expr)                                \
  do {                                                   \
    cudaError_t e__ = (expr);                            \
    if (e__ != cudaSuccess) return (h)->cuda_fail(e__, #expr); \
  } while (0)

// a launcher call that enqueues n of this library's kernels (counted for the bench)
#define TRY_LAUNCH(h, n, expr) \
  do {                         \
    TRY_CUDA(h, expr);         \
    (h)->launches += (n);      \
  } while (0)

// side streams for the DGT fork/join, created on first use (after enter_device)
static bool dgt_side_streams(mpgabor* h) {
  if (h->dgt_streams < 0) {
    const char* e = getenv("MPGABOR_DGT_STREAMS");
    h->dgt_streams = (e && e[0] == '0') ? 0 : 1;
    if (h->dgt_streams) {
      bool ok = cudaEventCreateWithFlags(&h->dgt_fork, cudaEventDisableTiming) == cudaSuccess;
      for (int w = 1; ok && w < h->W; ++w)
        ok = cudaStreamCreateWithFlags(&h->dgt_st[w], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&h->dgt_join[w], cudaEventDisableTiming) == cudaSuccess;
      if (!ok) {
        (void)cudaGetLastError();
        h->dgt_streams = 0;
      }
    }
  }
  return h->dgt_streams == 1;
}

static int enter_device(mpgabor* h) {
  if (h->device < 0) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      cudaGetLastError();
      return h->fail(MPG_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    TRY_CUDA(h, cudaGetDevice(&h->device));
    cudaDeviceProp prop;
    TRY_CUDA(h, cudaGetDeviceProperties(&prop, h->device));
    if (prop.major < 10) {
      h->device = -1;
      return h->fail(MPG_ECUDA, "libmpgabor is built for sm_100a (B200); device is sm_" +
                                    std::to_string(prop.major) + std::to_string(prop.minor));
    }
    for (auto& e2 : h->ev) TRY_CUDA(h, cudaEventCreate(&e2));
  } else {
    TRY_CUDA(h, cudaSetDevice(h->device));
  }
  return MPG_OK;
}

// ---------------------------------------------------------------------------
// create / destroy / errors
// ---------------------------------------------------------------------------
extern "C" int mpgabor_create(const mpg_dict* dicts, int32_t W, int32_t precision, mpgabor** out) {
  if (out) *out = nullptr;
  if (!dicts || !out) return g_create_error = "null pointer", MPG_EINVAL;
  if (W < 1 || W > MPG_MAX_DICTS) return g_create_error = "W must be in [1, 16]", MPG_EINVAL;
  if (precision != MPG_F64 && precision != MPG_F32) return g_create_error = "precision must be MPG_F64 or MPG_F32", MPG_EINVAL;
  for (int w = 0; w < W; ++w) {
    const mpg_dict& d = dicts[w];
    if (d.win < MPG_WIN_HANN || d.win > MPG_WIN_GAUSS)
      return g_create_error = "dictionary " + std::to_string(w) + ": unknown window", MPG_EINVAL;
    if (d.gl < 1 || d.a < 1 || d.M < 1 || d.gl > (1 << 20))
      return g_create_error = "dictionary " + std::to_string(w) + ": gl, a, M must be >= 1", MPG_EINVAL;
    if (!is_pow2(d.M) || d.M < 2 || d.M > 16384)
      return g_create_error = "dictionary " + std::to_string(w) + ": M must be a power of two in [2, 16384]", MPG_EINVAL;
    if (d.M % d.a)
      return g_create_error = "dictionary " + std::to_string(w) + ": M/a must be an integer (P:300-301)", MPG_EINCOMPAT;
  }
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const mpg_dict &du = dicts[u], &dv = dicts[v];
      if (std::max(du.a, dv.a) % std::min(du.a, dv.a) || std::max(du.M, dv.M) % std::min(du.M, dv.M))
        return g_create_error = "dictionaries " + std::to_string(u) + "," + std::to_string(v) +
                                " are not compatible (P:296-303)",
               MPG_EINCOMPAT;
    }
  mpgabor* h = new mpgabor();
  h->dicts.assign(dicts, dicts + W);
  h->W = W;
  h->precision = precision;
  h->a_min = dicts[0].a;
  h->M_max = dicts[0].M;
  for (auto& d : h->dicts) {
    h->a_min = std::min(h->a_min, d.a);
    h->M_max = std::max(h->M_max, d.M);
  }
  h->twres = h->M_max;
  h->Rmax = h->M_max / h->a_min;
  *out = h;
  return MPG_OK;
}

extern "C" void mpgabor_destroy(mpgabor* h) {
  if (!h) return;
  if (h->device >= 0) {
    cudaSetDevice(h->device);
    for (DevBuf* b : {&h->tw, &h->roots, &h->win, &h->kern, &h->boxcopy, &h->d_pairs, &h->rho, &h->rho_meta,
                      &h->Hscratch, &h->mxbox, &h->d_geo, &h->grid, &h->rec, &h->xp, &h->partial, &h->flag,
                      &h->E0, &h->result, &h->sol, &h->frames, &h->hx, &h->hatoms, &h->henergy, &h->hy, &h->prof, &h->d_own, &h->backup, &h->gxrec, &h->gxstamp, &h->rr, &h->yy, &h->sfirst, &h->sdone})
      b->release();
    for (auto e : h->ev)
      if (e) cudaEventDestroy(e);
    for (auto e : h->dgt_join)
      if (e) cudaEventDestroy(e);
    if (h->dgt_fork) cudaEventDestroy(h->dgt_fork);
    for (auto s2 : h->dgt_st)
      if (s2) cudaStreamDestroy(s2);
  }
  delete h;
}

extern "C" const char* mpgabor_last_error(const mpgabor* h) {
  return h ? h->err.c_str() : g_create_error.c_str();
}

// ---------------------------------------------------------------------------
// kernels (N2)
// ---------------------------------------------------------------------------
static int overlap_lags(const mpg_dict& du, const mpg_dict& dv, int a_c, int& nu_lo, int& nu_hi) {
  const int ju0 = -(du.gl / 2), ju1 = ju0 + du.gl - 1;
  const int jv0 = -(dv.gl / 2), jv1 = jv0 + dv.gl - 1;
  nu_lo = (int)-fdiv64(jv1 - ju0, a_c);  // ceil((ju0 - jv1)/a_c)
  nu_hi = (int)fdiv64(ju1 - jv0, a_c);
  return nu_hi - nu_lo + 1;
}

extern "C" int mpgabor_kernels(mpgabor* h, double thr, void* stream) {
  if (!h) return MPG_EINVAL;
  if (!(thr >= 0.0 && thr < 1.0)) return h->fail(MPG_EINVAL, "threshold must be in [0, 1)");
  int rc = enter_device(h);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int W = h->W;
  h->have_kernels = false;
  h->thr = thr;
  // tables
  TRY_CUDA(h, h->tw.ensure(sizeof(double2) * (h->twres / 2 + 1)));
  TRY_CUDA(h, h->roots.ensure(sizeof(double2) * h->Rmax));
  TRY_LAUNCH(h, 1, launch_tables(h->tw.as<double2>(), h->twres, h->roots.as<double2>(), h->Rmax, st));
  h->win_off.assign(W + 1, 0);
  for (int w = 0; w < W; ++w) h->win_off[w + 1] = h->win_off[w] + h->dicts[w].gl;
  TRY_CUDA(h, h->win.ensure(sizeof(double) * h->win_off[W]));
  for (int w = 0; w < W; ++w) {
    const mpg_dict& d = h->dicts[w];
    TRY_LAUNCH(h, 1, launch_window(d.win, d.gl, d.a, d.M, h->win.as<double>() + h->win_off[w], st));
  }
  // per pair: common grid, lag range, rows h(m >= 0, nu) into its own scratch slice
  h->pairs.assign(W * W, PairGeo{});
  h->nu_first.assign(W * W, 0);
  h->nlag.assign(W * W, 0);
  h->pair_mx.assign(W * W, 0.0);
  h->pair_kept.assign(W * W, 0);
  std::vector<int64_t> hoff(W * W + 1, 0);
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const int i = u * W + v;
      const mpg_dict &du = h->dicts[u], &dv = h->dicts[v];
      PairGeo& pg = h->pairs[i];
      pg.a_c = std::min(du.a, dv.a);
      pg.M_c = std::max(du.M, dv.M);
      pg.R = pg.M_c / pg.a_c;
      pg.s_m = pg.M_c / dv.M;
      pg.s_n = std::max(1, dv.a / pg.a_c);
      pg.rstep = h->Rmax / pg.R;
      pg.sh = (ilog2(pg.a_c) << PG_SH_AC) | (ilog2(pg.s_m) << PG_SH_SM) | (ilog2(pg.s_n) << PG_SH_SN) |
              ((ilog2(pg.M_c) - ilog2(du.M)) << PG_SH_MCU) | ((ilog2(du.a) - ilog2(pg.a_c)) << PG_SH_AUC) |
              (ilog2(dv.a) << PG_SH_AV);
      int lo, hi;
      h->nlag[i] = overlap_lags(du, dv, pg.a_c, lo, hi);
      h->nu_first[i] = lo;
      hoff[i + 1] = hoff[i] + (int64_t)h->nlag[i] * (pg.M_c / 2 + 1);
    }
  TRY_CUDA(h, h->Hscratch.ensure(sizeof(double2) * hoff[W * W]));
  TRY_CUDA(h, h->mxbox.ensure(64 * W * W));
  std::vector<unsigned char> mb(64 * W * W);
  for (int i = 0; i < W * W; ++i) {
    unsigned long long z = 0;
    int box[5] = {INT32_MAX, INT32_MIN, INT32_MAX, INT32_MIN, 0};
    std::memcpy(&mb[64 * i], &z, 8);
    std::memcpy(&mb[64 * i + 8], box, sizeof box);
  }
  TRY_CUDA(h, cudaMemcpyAsync(h->mxbox.p, mb.data(), mb.size(), cudaMemcpyHostToDevice, st));
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const int i = u * W + v;
      const mpg_dict &du = h->dicts[u], &dv = h->dicts[v];
      const PairGeo& pg = h->pairs[i];
      unsigned char* base = h->mxbox.as<unsigned char>() + 64 * i;
      double2* H = h->Hscratch.as<double2>() + hoff[i];
      TRY_LAUNCH(h, 1, launch_kern_rows(pg.a_c, pg.M_c, h->nu_first[i], h->nlag[i], h->win.as<double>() + h->win_off[u],
                                        du.gl, h->win.as<double>() + h->win_off[v], dv.gl, h->tw.as<double2>(),
                                        h->twres, H, st));
      TRY_LAUNCH(h, 2, launch_kern_max_box(H, h->nlag[i], pg.M_c, h->nu_first[i], thr,
                                           reinterpret_cast<unsigned long long*>(base), reinterpret_cast<int*>(base + 8),
                                           st));
    }
  TRY_CUDA(h, cudaMemcpyAsync(mb.data(), h->mxbox.p, mb.size(), cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));   // the boxes size the kernel storage
  h->kern_elems = 0;
  h->box_total = 0;
  h->kept_total = 0;
  h->box_off.assign(W * W + 1, 0);
  for (int i = 0; i < W * W; ++i) {
    unsigned long long mxbits;
    int box[5];
    std::memcpy(&mxbits, &mb[64 * i], 8);
    std::memcpy(box, &mb[64 * i + 8], sizeof box);
    double mx;
    std::memcpy(&mx, &mxbits, 8);
    if (box[0] > box[1]) return h->fail(MPG_ECUDA, "empty kernel box (all-zero kernel)");
    PairGeo& pg = h->pairs[i];
    pg.mu_lo = box[0];
    pg.mu_hi = box[1];
    pg.nu_lo = box[2];
    pg.nu_hi = box[3];
    pg.nmu = box[1] - box[0] + 1;
    pg.nnu = box[3] - box[2] + 1;
    pg.koff = h->kern_elems;
    h->kern_elems += (int64_t)pg.nmu * pg.nnu;
    h->pair_mx[i] = mx;
    h->pair_kept[i] = box[4];
    h->kept_total += box[4];
    h->box_off[i + 1] = h->box_off[i] + (int64_t)pg.nmu * pg.nnu;
  }
  h->box_total = h->kern_elems;
  // conjugate-pair rows (nu = 0 of h_uu)
  h->rho_lo.assign(W, 0);
  h->rho_n.assign(W, 0);
  h->rho_off.assign(W, 0);
  h->rho_total = 0;
  for (int u = 0; u < W; ++u) {
    const PairGeo& pg = h->pairs[u * W + u];
    h->rho_off[u] = h->rho_total;
    h->rho_lo[u] = pg.mu_lo;
    h->rho_n[u] = (pg.nu_lo <= 0 && pg.nu_hi >= 0) ? pg.nmu : 0;
    h->rho_total += h->rho_n[u];
  }
  TRY_CUDA(h, h->kern.ensure(h->celem() * std::max<int64_t>(1, h->kern_elems)));
  TRY_CUDA(h, h->boxcopy.ensure(sizeof(double2) * std::max<int64_t>(1, h->box_total)));
  TRY_CUDA(h, h->rho.ensure(sizeof(RhoEnt) * std::max(1, h->rho_total)));
  // compact every box into the per-alignment-class layout
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const int i = u * W + v;
      const PairGeo& pg = h->pairs[i];
      unsigned char* base = h->mxbox.as<unsigned char>() + 64 * i;
      const double2* H = h->Hscratch.as<double2>() + hoff[i];
      RhoEnt* rrow = (u == v && h->rho_n[u] > 0) ? h->rho.as<RhoEnt>() + h->rho_off[u] : nullptr;
      if (h->f64())
        TRY_LAUNCH(h, 1, launch_kern_compact<double>(H, pg.M_c, h->nu_first[i], thr,
                                                     reinterpret_cast<const unsigned long long*>(base), pg,
                                                     h->kern.as<double2>(), h->boxcopy.as<double2>() + h->box_off[i],
                                                     rrow, st));
      else
        TRY_LAUNCH(h, 1, launch_kern_compact<float>(H, pg.M_c, h->nu_first[i], thr,
                                                    reinterpret_cast<const unsigned long long*>(base), pg,
                                                    h->kern.as<float2>(), h->boxcopy.as<double2>() + h->box_off[i],
                                                    rrow, st));
    }
  TRY_CUDA(h, h->d_pairs.ensure(sizeof(PairGeo) * W * W));
  TRY_CUDA(h, cudaMemcpyAsync(h->d_pairs.p, h->pairs.data(), sizeof(PairGeo) * W * W, cudaMemcpyHostToDevice, st));
  std::vector<int> meta(3 * W);
  for (int u = 0; u < W; ++u) {
    meta[u] = h->rho_lo[u];
    meta[W + u] = h->rho_n[u];
    meta[2 * W + u] = h->rho_off[u];
  }
  TRY_CUDA(h, h->rho_meta.ensure(sizeof(int) * 3 * W));
  TRY_CUDA(h, cudaMemcpyAsync(h->rho_meta.p, meta.data(), sizeof(int) * 3 * W, cudaMemcpyHostToDevice, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  h->have_kernels = true;
  h->L = -1;  // layout depends on kernel boxes (validation), recompute at next run
  return MPG_OK;
}

extern "C" int mpgabor_kernel_stats(const mpgabor* h, int64_t* box_entries, int64_t* kept_entries, int64_t* bytes) {
  if (!h) return MPG_EINVAL;
  if (!h->have_kernels) return const_cast<mpgabor*>(h)->fail(MPG_ESTATE, "kernels not computed");
  if (box_entries) *box_entries = h->box_total;
  if (kept_entries) *kept_entries = h->kept_total;
  if (bytes) *bytes = h->kern_elems * (int64_t)h->celem();
  return MPG_OK;
}

extern "C" int mpgabor_kernel_box(mpgabor* h, int32_t u, int32_t v, int32_t* box, double* values, double* mx) {
  if (!h || !box) return MPG_EINVAL;
  if (!h->have_kernels) return h->fail(MPG_ESTATE, "kernels not computed");
  if (u < 0 || v < 0 || u >= h->W || v >= h->W) return h->fail(MPG_EINVAL, "pair index out of range");
  const PairGeo& pg = h->pairs[u * h->W + v];
  box[0] = pg.mu_lo;
  box[1] = pg.mu_hi;
  box[2] = pg.nu_lo;
  box[3] = pg.nu_hi;
  if (mx) *mx = h->pair_mx[u * h->W + v];
  if (values) {
    int rc = enter_device(h);
    if (rc) return rc;
    TRY_CUDA(h, cudaMemcpy(values, h->boxcopy.as<double2>() + h->box_off[u * h->W + v],
                           sizeof(double2) * pg.nmu * pg.nnu, cudaMemcpyDeviceToHost));
  }
  return MPG_OK;
}

// ---------------------------------------------------------------------------
// layout
// ---------------------------------------------------------------------------
static int64_t ell_of(const mpgabor* h) {
  int64_t ell = 1;
  for (auto& d : h->dicts) {
    ell = std::lcm(ell, (int64_t)d.a);
    ell = std::lcm(ell, (int64_t)d.M);
  }
  return ell;
}

extern "C" int mpgabor_layout(const mpgabor* h, int64_t Ls, int64_t* L_pad, int64_t* N, int64_t* M_R,
                              int64_t* row_stride, int64_t* coef_offset) {
  if (!h) return MPG_EINVAL;
  if (Ls < 1) return const_cast<mpgabor*>(h)->fail(MPG_EINVAL, "Ls must be >= 1");
  const int64_t ell = ell_of(h);
  if (Ls > (int64_t)1 << 40) return const_cast<mpgabor*>(h)->fail(MPG_ELEN, "Ls too large");
  const int64_t L = (Ls + ell - 1) / ell * ell;
  if (L_pad) *L_pad = L;
  int64_t off = 0;
  for (int w = 0; w < h->W; ++w) {
    const int64_t n = L / h->dicts[w].a, mr = h->dicts[w].M / 2 + 1;
    if (N) N[w] = n;
    if (M_R) M_R[w] = mr;
    if (row_stride) row_stride[w] = mr;  // exchanged coefficient vectors are dense
    if (coef_offset) coef_offset[w] = off;
    off += n * mr;
  }
  if (coef_offset) coef_offset[h->W] = off;
  return MPG_OK;
}

extern "C" int mpgabor_set_launch(mpgabor* h, int32_t cluster, int32_t threads, int32_t tile_width,
                                  int32_t records) {
  if (!h) return MPG_EINVAL;
  if (cluster < 0 || cluster > 128 || (cluster && (cluster & (cluster - 1))))
    return h->fail(MPG_EINVAL, "cluster must be 0, a power of two <= 16 (one cluster) or 32/64/128 (grid)");
  if (threads && (threads < 128 || threads > multi_max_threads() || threads % 32))
    return h->fail(MPG_EINVAL, "threads must be in [128," + std::to_string(multi_max_threads()) + "], multiple of 32");
  if (tile_width && tile_width != 32 && tile_width != 64 && tile_width != 128)
    return h->fail(MPG_EINVAL, "tile width must be 32, 64 or 128");
  if (records < 0 || records > 2) return h->fail(MPG_EINVAL, "records must be 0 (auto), 1 (shared) or 2 (global)");
  h->cluster_req = cluster;
  if (threads) h->threads = threads;
  h->TW_req = tile_width;
  h->srec_req = records;
  h->L = -1;
  return MPG_OK;
}

// grids and tiles of every dictionary for tile width TW (fills h->geo, sizes)
static int plan_grids(mpgabor* h, int64_t L, int TW) {
  const int W = h->W;
  h->pad_clean = 0;
  h->geo.assign(W, DictGeo{});
  int64_t off = 0, goff = 0, toff = 0, foff = 0;
  for (int w = 0; w < W; ++w) {
    DictGeo& d = h->geo[w];
    const mpg_dict& s = h->dicts[w];
    d.win = s.win;
    d.gl = s.gl;
    d.a = s.a;
    d.M = s.M;
    d.N = (int32_t)(L / s.a);
    d.frame_off = (int32_t)foff;
    foff += d.N;
    d.MR = s.M / 2 + 1;
    d.mr_magic = (uint32_t)((0x100000000ull + (uint64_t)d.MR - 1) / (uint64_t)d.MR);
    d.T = (d.MR + TW - 1) / TW;
    d.stride = d.T * TW;
    d.off = off;
    d.grid_off = goff;
    d.tile_off = toff;
    off += (int64_t)d.N * d.MR;
    goff += (int64_t)d.N * d.stride;
    toff += (int64_t)d.N * d.T;
  }
  h->P_R = off;
  h->grid_elems = goff;
  h->total_tiles = toff;
  if (h->P_R >= (int64_t)NO_INDEX || h->total_tiles > INT32_MAX)
    return h->fail(MPG_ELEN, "more than 2^32-1 reduced coefficients");
  return MPG_OK;
}

// Automatic choice between the loop kernels (mpgabor_set_batch 0).  A multi-selection
// round has a fixed cost (list exchange, ranking, walk, candidate lists) and yields
// several atoms; an iteration of the one-selection loop pays the exchange for every atom.
// Measured on B200 (profiles/r01_configs.md, full runs, us/atom one-selection vs multi):
// C0 2.25 vs 2.03, C1 2.52 vs 1.16, C2 2.72 vs 1.79, C3 5.42 vs 2.54 (grid 64), C4 9.63
// vs 5.61 (grid 128): multi-selection wins on every config.  It needs atoms whose
// updates are mostly disjoint, so it is taken while the mean update (kernel boxes,
// subsampled per target, averaged over the selected dictionary) is a small fraction of
// the grid (C0: 2.6 %).
static double mean_update(const mpgabor* h) {
  const int W = h->W;
  double sum = 0.0;
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const PairGeo& pg = h->pairs[u * W + v];
      sum += (double)pg.nnu / pg.s_n * ((double)pg.nmu / pg.s_m);
    }
  return sum / W;
}

static bool auto_multi(const mpgabor* h, int64_t P_R) {
  const double per_atom = mean_update(h);
  // (wide updates run the multi-selection kernel as a grid of 64 / 128 CTAs, below)
  return per_atom < 0.05 * (double)P_R;
}
static bool auto_multi(const mpgabor* h) { return auto_multi(h, h->P_R); }

// loop parameters for (TW, srec, C); returns shared-memory bytes (SIZE_MAX if the tree is too deep)
static size_t plan_loop(mpgabor* h, int TW, int srec, int C) {
  LoopParams& P = h->lp;
  P = LoopParams{};
  P.W = h->W;
  P.TW = TW;
  P.srec = srec;
  P.Rmax = h->Rmax;
  P.rho_total = h->rho_total;
  P.C = C;
  P.gx = h->gx ? 1 : 0;
  // frame ownership: global frame f -> CTA f mod C; per (CTA, dictionary) first owned
  // frame, owned-frame count and the local index of the first tile record
  h->own.assign((size_t)C * h->W, OwnGeo{});
  int64_t Lc = 0;
  for (int c = 0; c < C; ++c) {
    int64_t loc = 0;
    for (int v = 0; v < h->W; ++v) {
      const DictGeo& d = h->geo[v];
      OwnGeo& o = h->own[(size_t)c * h->W + v];
      o.n_first = (int32_t)(((c - d.frame_off) % C + C) % C);
      o.n_own = o.n_first < d.N ? (d.N - 1 - o.n_first) / C + 1 : 0;
      o.loc_base = (int32_t)loc;
      loc += (int64_t)o.n_own * d.T;
    }
    Lc = std::max(Lc, loc);
  }
  P.Lc = Lc;
  int n = (int)((P.Lc + 31) / 32), nl = 0, o = 0;
  for (;;) {
    if (nl >= MAX_LEVELS) return SIZE_MAX;
    P.lev_n[nl] = n;
    P.lev_off[nl] = o;
    o += n;
    ++nl;
    if (n <= TOP_SCAN) break;
    n = (n + 31) / 32;
  }
  P.nlev = nl;
  // loop kernel: 2 = mpmulti.cu, 0 = mploop.cu (batch 1, or the automatic choice)
  const int kind = (h->batch == 1 || h->force_single || (h->batch == 0 && !auto_multi(h))) ? 0 : 2;
  h->kind = kind;
  h->run_threads = h->threads;
  P.spec = h->batch == 0 ? multi_max_batch() : h->batch;
  P.smem_bytes = kind == 2 ? multi_smem_bytes(P, h->f64()) : loop_smem_bytes(P, h->f64());
  return P.smem_bytes;
}

static int ensure_layout(mpgabor* h, int64_t Ls) {
  const int64_t ell = ell_of(h);
  const int64_t L = (Ls + ell - 1) / ell * ell;
  if (L == h->L) return MPG_OK;
  const int W = h->W;
  if (L > ((int64_t)1 << 30)) return h->fail(MPG_ELEN, "L_pad larger than 2^30");
  // aliasing / box checks (circular Gram == direct overlap needs L >= gl_u + gl_v)
  for (int u = 0; u < W; ++u)
    for (int v = 0; v < W; ++v) {
      const PairGeo& pg = h->pairs[u * W + v];
      if (L < (int64_t)h->dicts[u].gl + h->dicts[v].gl)
        return h->fail(MPG_ELEN, "L_pad shorter than gl_u + gl_v (kernel would alias circularly)");
      const int rows = (pg.nnu + pg.s_n - 1) / pg.s_n, cols = (pg.nmu + pg.s_m - 1) / pg.s_m;
      if (rows > L / h->dicts[v].a || cols > h->dicts[v].M)
        return h->fail(MPG_ELEN, "kernel box wider than the target grid");
    }
  // candidate launch plans, first schedulable wins
  struct Cand { int TW, srec; };
  std::vector<Cand> cands;
  // automatic tile width: 64 (then 128) for the one-selection loop; 32 first for the
  // multi-selection loop (its rounds are bound by the per-tile work of several atoms:
  // narrower tiles load and rescan 2x fewer bins, profiles/r01_configs.md)
  {
    const int rc = plan_grids(h, L, 64);  // P_R for the automatic kernel choice
    if (rc) return rc;
  }
  const bool multi_wanted = !(h->batch == 1 || (h->batch == 0 && !auto_multi(h)));
  // multi-selection: narrow tiles matter more than shared-memory records (C3 fp64: 64-bin
  // tiles with global records 4.31 us/atom, 128-bin tiles with shared records 6.66); as a
  // grid of 64 / 128 CTAs (C3 / C4) 64-bin tiles are best
  auto candidates = [&](bool grid) {
    static const Cand multi_grid[6] = {{64, 1}, {64, 0}, {32, 1}, {32, 0}, {128, 1}, {128, 0}};
    static const Cand multi_cluster[6] = {{32, 1}, {64, 1}, {64, 0}, {32, 0}, {128, 1}, {128, 0}};
    static const Cand single[4] = {{64, 1}, {128, 1}, {64, 0}, {128, 0}};
    const Cand req[2] = {{h->TW_req, 1}, {h->TW_req, 0}};
    const Cand* pref = h->TW_req ? req : (multi_wanted ? (grid ? multi_grid : multi_cluster) : single);
    const int n = h->TW_req ? 2 : (multi_wanted ? 6 : 4);
    std::vector<Cand> out;
    for (int i = 0; i < n; ++i)
      if ((pref[i].srec == 1 && h->srec_req != 2) || (pref[i].srec == 0 && h->srec_req != 1)) out.push_back(pref[i]);
    return out;
  };
  std::string why = "no candidate";
  bool ok = false;
  // the multi-selection kernel packs tile rects as (row 20 bits, rows 12 bits) and
  // needs more shared memory: fall back to the one-selection kernel when it cannot run
  h->force_single = false;
  for (int v = 0; v < W; ++v)
    if (L / h->dicts[v].a >= (1 << 20)) h->force_single = true;
  for (int i = 0; i < W * W; ++i)
    if ((h->pairs[i].nnu + h->pairs[i].s_n - 1) / h->pairs[i].s_n >= (1 << 12)) h->force_single = true;
  // automatic grid mode: wide updates spread over 64 / 128 CTAs beat one 16-CTA cluster
  // despite the global-memory exchange: multi-selection rounds from ~10k
  // coefficients per atom (C3: 2.85 vs 4.20 us/atom on 64 CTAs; C4, 54k: 3.93 on 128 CTAs),
  // the one-selection loop (exchange every atom) from ~30k (C4: 7.5 on 64 CTAs)
  const double per_atom = mean_update(h);
  const int grid_C = !multi_wanted ? (per_atom > 30000.0 ? 64 : 0) : (per_atom > 40000.0 ? 128 : (per_atom > 10000.0 ? 64 : 0));
  const bool try_grid = h->cluster_req == 0 && grid_C > 0 && !h->batch_mode;
  const bool force_single0 = h->force_single;
  for (int pass = try_grid ? 0 : 1; pass < 2 && !ok; ++pass) {
  int creq = pass == 0 ? grid_C : (h->batch_mode && h->cluster_req > MAX_CLUSTER ? 0 : h->cluster_req);
  if (pass == 1 && h->batch_mode && h->cluster_req == 0) creq = h->batch_C;
  h->gx = creq > MAX_CLUSTER;
  h->force_single = force_single0;
  cands = candidates(h->gx);
  for (int attempt = 0; attempt < 2 && !ok; ++attempt) {
  if (attempt == 1) {
    if (h->kind != 2) break;
    h->force_single = true;
  }
  for (const Cand& c : cands) {
    int rc = plan_grids(h, L, c.TW);
    if (rc) return rc;
    for (int C = creq ? creq : MAX_CLUSTER; C >= 1; C >>= 1) {
      const size_t smem = plan_loop(h, c.TW, c.srec, C);
      if (smem > 227 * 1024) {
        why = "shared memory " + std::to_string(smem) + " B";
        break;  // smaller clusters need more per-CTA memory
      }
      const int cmax = h->kind == 2 ? multi_max_cluster(h->f64(), c.srec, c.TW, h->run_threads, smem, h->gx)
                                    : loop_max_cluster(h->f64(), c.srec, c.TW, h->run_threads, smem, h->gx);
      if (cmax >= C) {
        ok = true;
        break;
      }
      why = "cluster of " + std::to_string(C) + " not schedulable";
      if (creq) break;
    }
    if (ok) {
      h->TW = c.TW;
      h->srec = c.srec;
      break;
    }
  }
  }
  }
  if (!ok) return h->fail(MPG_ECUDA, "no launch plan for the MP loop: " + why);
  LoopParams& P = h->lp;
  // multi-selection with shared-memory records: each CTA's top K from its candidate list
  // (mpmulti.cu ClState: tiles at or above a threshold, kept across rounds, rebuilt by a
  // radix select when it runs short) instead of the node tree (2) or a scan of every
  // record (1); env MPGABOR_TOPK = 0/1/2 overrides, for measurements
  {
    const char* ev = std::getenv("MPGABOR_TOPK");
    const int want = ev ? std::atoi(ev) : 2;
    P.topk_scan = h->kind == 2 ? std::max(0, std::min(2, want)) : 0;
    if ((h->gx || !h->srec) && P.topk_scan == 1) P.topk_scan = 0;  // (scan: shared records of a cluster)
    if (P.topk_scan) {  // the list's shared memory (membership flags per record) must fit
      P.smem_bytes = multi_smem_bytes(P, h->f64());
      if (P.smem_bytes > 227 * 1024) {
        P.topk_scan = 0;
        P.smem_bytes = multi_smem_bytes(P, h->f64());
      }
    }
  }
  // multi-selection over residual grids and kernels much larger than L2 (C4: 1.07 GB + 0.36 GB):
  // bulk-prefetch the walk window's rows into L2 (mpmulti.cu, after the window geometry);
  // env MPGABOR_L2PF = number of window entries overrides, for measurements
  {
    int dev = 0, l2 = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev) != cudaSuccess) {
      cudaGetLastError();
      l2 = 0;
    }
    const double bytes = (double)h->celem() * ((double)h->grid_elems + (double)h->kern_elems);
    const char* ev = std::getenv("MPGABOR_L2PF");
    // (on when they exceed 4x L2: C4 5.13 -> 5.08 us/atom; C3, 2.3x L2, 2.558 -> 2.577 with it)
    P.l2pf = h->kind == 2 ? (ev ? std::max(0, std::atoi(ev)) : (l2 > 0 && bytes > 4.0 * (double)l2 ? multi_window() : 0)) : 0;
  }
  h->lay_C = P.C;
  // buffers
  TRY_CUDA(h, h->d_geo.ensure(sizeof(DictGeo) * W));
  TRY_CUDA(h, cudaMemcpy(h->d_geo.p, h->geo.data(), sizeof(DictGeo) * W, cudaMemcpyHostToDevice));
  TRY_CUDA(h, h->d_own.ensure(sizeof(OwnGeo) * h->own.size()));
  TRY_CUDA(h, cudaMemcpy(h->d_own.p, h->own.data(), sizeof(OwnGeo) * h->own.size(), cudaMemcpyHostToDevice));
  TRY_CUDA(h, h->grid.ensure(h->celem() * h->grid_elems));
  TRY_CUDA(h, h->rec.ensure((h->f64() ? sizeof(Rec<double>) : sizeof(Rec<float>)) * P.C * P.Lc));
  TRY_CUDA(h, h->xp.ensure(sizeof(double) * L));
  TRY_CUDA(h, h->partial.ensure(sizeof(double) * 256));
  TRY_CUDA(h, h->flag.ensure(sizeof(int)));
  TRY_CUDA(h, h->E0.ensure(sizeof(double)));
  TRY_CUDA(h, h->result.ensure(sizeof(LoopResult)));
  if (h->gx) {
    // one-selection kernel: [2][C] root records; multi-selection kernel: [2][C] messages
    TRY_CUDA(h, h->gxrec.ensure(std::max(h->f64() ? sizeof(Rec<double>) : sizeof(Rec<float>), multi_msg_bytes(h->f64())) *
                                2 * P.C));
    TRY_CUDA(h, h->gxstamp.ensure(sizeof(unsigned long long) * std::max(2 * P.C, 64)));  // (>= 64: mpmulti.cuh GX_COUNTER)
  }
  if (h->kind == 2) {
    // roll-back backups: per CTA and round at most spec x max_u sum_v (rows/C + 1) x (hull tiles)
    // items (rows = alignment-class sub-box rows, hull tiles <= cols/TW + 1)
    int64_t per_atom = 0;
    for (int u = 0; u < W; ++u) {
      int64_t s = 0;
      for (int v = 0; v < W; ++v) {
        const PairGeo& pg = h->pairs[u * W + v];
        const int64_t rows = (pg.nnu + pg.s_n - 1) / pg.s_n, cols = (pg.nmu + pg.s_m - 1) / pg.s_m;
        const int64_t tiles = std::min<int64_t>(h->geo[v].T, (cols + h->TW - 1) / h->TW + 1);
        s += ((rows + P.C - 1) / P.C + 1) * tiles;
      }
      per_atom = std::max(per_atom, s);
    }
    P.bk_cap = per_atom * P.spec;
    TRY_CUDA(h, h->backup.ensure(h->celem() * (size_t)h->TW * P.bk_cap * P.C));
  }
  h->L = L;
  h->lay_TW = h->TW;
  return MPG_OK;
}

extern "C" int mpgabor_launch_info(const mpgabor* h, int32_t* cluster, int32_t* threads, int32_t* tile_width,
                                   int32_t* records, int64_t* smem_bytes) {
  if (!h) return MPG_EINVAL;
  if (h->L < 0) return const_cast<mpgabor*>(h)->fail(MPG_ESTATE, "no run yet");
  if (cluster) *cluster = h->lp.C;
  if (threads) *threads = h->run_threads;
  if (tile_width) *tile_width = h->TW;
  if (records) *records = h->srec ? 1 : 2;
  if (smem_bytes) *smem_bytes = (int64_t)h->lp.smem_bytes;
  return MPG_OK;
}

// ---------------------------------------------------------------------------
// run
// ---------------------------------------------------------------------------
// DGT + loop; etol_abs (nullable) replaces the stop level 10^(errdb/10) E_0 (resets)
// B >= 1 independent signals of Ls samples (x_dev[B][Ls], atoms_dev[B][maxit],
// energy_dev[B][maxit+1], res[B]): B > 1 runs the loop kernel of the automatic choice (or
// mpgabor_set_batch) with one cluster per signal (batched mode, no solution vector).
static int run_impl(mpgabor* h, const double* x_dev, int64_t Ls, int64_t maxit, double errdb, const double* etol_abs,
                    mpg_atom* atoms_dev, double* energy_dev, double* coef_dev, mpg_result* res, void* stream,
                    int B = 1) {
  if (!h) return MPG_EINVAL;
  if (!x_dev || !energy_dev || !res || (maxit > 0 && !atoms_dev)) return h->fail(MPG_EINVAL, "null pointer");
  if (Ls < 1) return h->fail(MPG_EINVAL, "Ls must be >= 1");
  if (maxit < 0) return h->fail(MPG_EINVAL, "maxit must be >= 0");
  if (std::isnan(errdb)) return h->fail(MPG_EINVAL, "errdb is NaN");
  if (!h->have_kernels) return h->fail(MPG_ESTATE, "mpgabor_kernels must run before mpgabor_run");
  if (B < 1 || (B > 1 && coef_dev)) return h->fail(MPG_EINVAL, "batched runs need B >= 1 and no solution vector");
  int rc = enter_device(h);
  if (rc) return rc;
  // batched signals: one cluster per signal; smaller clusters let more signals run at
  // once (measured aggregate it/s on B200, profiles/r01_batch.md)
  int bc = B <= 4 ? 16 : (B <= 12 ? 8 : 4);
  if (bc == 4) {
    // multi-selection kernel: 4-CTA clusters only while the tile records still fit in
    // shared memory (C1: 7.5 M it/s for 36 signals; C2 falls to 1.7 M with global
    // records against 2.9 M on 8-CTA clusters, profiles/r01_batch.md)
    const int64_t L = (Ls + ell_of(h) - 1) / ell_of(h) * ell_of(h);
    int64_t P_R = 0;
    for (int w = 0; w < h->W; ++w) P_R += (L / h->dicts[w].a) * (h->dicts[w].M / 2 + 1);
    const bool multi = h->batch >= 2 || (h->batch == 0 && auto_multi(h, P_R));
    const size_t rec_bytes = (size_t)(P_R / 4 / 32 + 1) * (h->f64() ? sizeof(Rec<double>) : sizeof(Rec<float>));
    if (multi && rec_bytes > 150 * 1024) bc = 8;
  }
  if (h->batch_mode != (B > 1) || (B > 1 && bc != h->batch_C)) {
    h->batch_mode = B > 1;
    h->batch_C = bc;
    h->L = -1;
  }
  rc = ensure_layout(h, Ls);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int W = h->W;
  LoopParams& P = h->lp;
  if (B > 1) {
    TRY_CUDA(h, h->grid.ensure(h->celem() * h->grid_elems * B));
    TRY_CUDA(h, h->rec.ensure((h->f64() ? sizeof(Rec<double>) : sizeof(Rec<float>)) * P.C * P.Lc * B));
    if (h->kind == 2) TRY_CUDA(h, h->backup.ensure(h->celem() * (size_t)h->TW * P.bk_cap * P.C * B));
  }
  TRY_CUDA(h, h->E0.ensure(sizeof(double) * B));
  TRY_CUDA(h, h->result.ensure(sizeof(LoopResult) * B));
  const size_t recsz = h->f64() ? sizeof(Rec<double>) : sizeof(Rec<float>);
  TRY_CUDA(h, cudaEventRecord(h->ev[0], st));
  TRY_CUDA(h, cudaMemsetAsync(h->flag.p, 0, sizeof(int), st));
  if (h->grid.p != h->pad_ptr) {
    h->pad_ptr = h->grid.p;
    h->pad_clean = 0;
  }
  for (int b = 0; b < B; ++b) {
    const int write_pad = b >= h->pad_clean ? 1 : 0;
    TRY_LAUNCH(h, 2, launch_pad_energy(x_dev + (int64_t)b * Ls, Ls, h->xp.as<double>(), h->L, h->partial.as<double>(),
                                       h->flag.as<int>(), h->E0.as<double>() + b, st));
    const bool fork = dgt_side_streams(h) && W > 1;
    if (fork) TRY_CUDA(h, cudaEventRecord(h->dgt_fork, st));
    for (int w = 0; w < W; ++w) {
      const DictGeo& d = h->geo[w];
      const double* g = h->win.as<double>() + h->win_off[w];
      const int64_t goff = d.grid_off + (int64_t)b * h->grid_elems;
      // dictionary 0 stays on the caller's stream; the others fork off it and join back
      // (the next signal's padding rewrites xp, the tile init reads every grid)
      cudaStream_t sw = fork && w > 0 ? h->dgt_st[w] : st;
      if (sw != st) TRY_CUDA(h, cudaStreamWaitEvent(sw, h->dgt_fork, 0));
      if (h->f64())
        TRY_LAUNCH(h, 1, launch_dgt<double>(h->xp.as<double>(), h->L, d, g, h->tw.as<double2>(), h->twres,
                                            h->grid.as<double2>() + goff, sw, write_pad));
      else
        TRY_LAUNCH(h, 1, launch_dgt<float>(h->xp.as<double>(), h->L, d, g, h->tw.as<double2>(), h->twres,
                                           h->grid.as<float2>() + goff, sw, write_pad));
      if (sw != st) TRY_CUDA(h, cudaEventRecord(h->dgt_join[w], sw));
    }
    if (fork)
      for (int w = 1; w < W; ++w) TRY_CUDA(h, cudaStreamWaitEvent(st, h->dgt_join[w], 0));
  }
  h->pad_clean = std::max(h->pad_clean, B);
  TRY_CUDA(h, cudaEventRecord(h->ev[1], st));
  const SelScore sel{h->pedantic, h->rho.as<RhoEnt>(), h->rho_meta.as<int>()};
  for (int b = 0; b < B; ++b) {
    unsigned char* recb = h->rec.as<unsigned char>() + recsz * P.C * P.Lc * b;
    if (h->f64())
      TRY_LAUNCH(h, 2, launch_tile_init<double>(h->grid.as<double2>() + (int64_t)b * h->grid_elems, h->d_geo.as<DictGeo>(),
                                                h->d_own.as<OwnGeo>(), W, h->total_tiles, P.C, P.Lc, h->TW,
                                                reinterpret_cast<Rec<double>*>(recb), sel, st));
    else
      TRY_LAUNCH(h, 2, launch_tile_init<float>(h->grid.as<float2>() + (int64_t)b * h->grid_elems, h->d_geo.as<DictGeo>(),
                                               h->d_own.as<OwnGeo>(), W, h->total_tiles, P.C, P.Lc, h->TW,
                                               reinterpret_cast<Rec<float>*>(recb), sel, st));
    TRY_CUDA(h, cudaMemcpyAsync(energy_dev + (int64_t)b * (maxit + 1), h->E0.as<double>() + b, sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
  }
  if (coef_dev) TRY_CUDA(h, cudaMemsetAsync(coef_dev, 0, sizeof(double2) * h->P_R, st));
  TRY_CUDA(h, cudaEventRecord(h->ev[2], st));
  // no host round trip before the loop: the loop kernel reads E_0 and the non-finite
  // flag from the device and forms the stop level 10^(errdb/10) E_0 itself (P:340-341,
  // P:1153); the one synchronisation is the result read-back after the loop
  P.nslot = B;
  P.E0v = h->E0.as<double>();
  P.nonfinite = h->flag.as<int>();
  if (etol_abs) {
    P.etol_mode = 2;
    P.etol_val = *etol_abs;
  } else if (errdb == -INFINITY) {
    P.etol_mode = 0;
    P.etol_val = 0.0;
  } else {
    P.etol_mode = 1;
    P.etol_val = std::pow(10.0, errdb / 10.0);
  }
  P.slot_grid = h->grid_elems;
  P.slot_atoms = maxit;
  P.dicts = h->d_geo.as<DictGeo>();
  P.own = h->d_own.as<OwnGeo>();
  P.pairs = h->d_pairs.as<PairGeo>();
  P.roots = h->roots.as<double2>();
  P.rho = h->rho.as<RhoEnt>();
  P.rho_lo = h->rho_meta.as<int>();
  P.rho_n = h->rho_meta.as<int>() + W;
  P.rho_off = h->rho_meta.as<int>() + 2 * W;
  P.grid = h->grid.p;
  P.kern = h->kern.p;
  P.kern_elems = h->kern_elems;
  P.rec = h->rec.p;
  P.maxit = maxit;
  P.E0 = 0.0;
  P.atoms = reinterpret_cast<AtomOut*>(atoms_dev);
  P.energy = energy_dev;
  P.sol = reinterpret_cast<double2*>(coef_dev);
  P.result = h->result.as<LoopResult>();
  P.floor_mode = (h->prof_mode & 2) ? 1 : 0;
  P.pedantic = h->pedantic;
  P.prof = nullptr;
  if (h->prof_mode & 1) {
    TRY_CUDA(h, h->prof.ensure(sizeof(long long) * MPG_PROF_SLOTS));
    TRY_CUDA(h, cudaMemsetAsync(h->prof.p, 0, sizeof(long long) * MPG_PROF_SLOTS, st));
    P.prof = h->prof.as<long long>();
  }
  TRY_CUDA(h, cudaEventRecord(h->ev[3], st));
  P.backup = h->backup.p;
  P.gx_rec = nullptr;
  P.gx_stamp = nullptr;
  if (h->gx) {  // stamps start at 0: the first roots carry stamp 1
    TRY_CUDA(h, cudaMemsetAsync(h->gxstamp.p, 0, sizeof(unsigned long long) * std::max(2 * P.C, 64), st));
    P.gx_rec = h->gxrec.p;
    P.gx_stamp = h->gxstamp.as<unsigned long long>();
  }
  if (h->kind == 2)
    TRY_LAUNCH(h, 1, launch_multi_loop(P, h->f64(), h->run_threads, st));
  else
    TRY_LAUNCH(h, 1, launch_mp_loop(P, h->f64(), h->run_threads, st));
  TRY_CUDA(h, cudaEventRecord(h->ev[4], st));
  std::vector<LoopResult> lr(B);
  TRY_CUDA(h, cudaMemcpyAsync(lr.data(), h->result.p, sizeof(LoopResult) * B, cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  TRY_CUDA(h, cudaEventElapsedTime(&h->t_dgt, h->ev[0], h->ev[1]));
  TRY_CUDA(h, cudaEventElapsedTime(&h->t_init, h->ev[1], h->ev[2]));
  TRY_CUDA(h, cudaEventElapsedTime(&h->t_loop, h->ev[3], h->ev[4]));
  if (P.prof) TRY_CUDA(h, cudaMemcpy(h->prof_host, P.prof, sizeof(long long) * MPG_PROF_SLOTS, cudaMemcpyDeviceToHost));
  for (int b = 0; b < B; ++b)
    if (lr[b].stop == STOP_NONFINITE) return h->fail(MPG_ENONFINITE, "x contains NaN or Inf");
  for (int b = 0; b < B; ++b) {
    res[b].n_atoms = lr[b].n_done;
    res[b].L_pad = h->L;
    res[b].stop_reason = lr[b].stop;
    res[b].cluster = h->lay_C;
    res[b].E0 = lr[b].E0;
    res[b].E_final = lr[b].E_final;
    res[b].rounds = h->kind == 2 ? lr[b].rounds : lr[b].n_done + 1;
  }
  return MPG_OK;
}

extern "C" int mpgabor_run_batch(mpgabor* h, const double* x_dev, int32_t B, int64_t Ls, int64_t maxit, double errdb,
                                 mpg_atom* atoms_dev, double* energy_dev, mpg_result* res, void* stream) {
  if (!h) return MPG_EINVAL;
  if (B < 1) return h->fail(MPG_EINVAL, "B must be >= 1");
  return run_impl(h, x_dev, Ls, maxit, errdb, nullptr, atoms_dev, energy_dev, nullptr, res, stream, B);
}

extern "C" int mpgabor_run(mpgabor* h, const double* x_dev, int64_t Ls, int64_t maxit, double errdb,
                           mpg_atom* atoms_dev, double* energy_dev, double* coef_dev, mpg_result* res,
                           void* stream) {
  return run_impl(h, x_dev, Ls, maxit, errdb, nullptr, atoms_dev, energy_dev, coef_dev, res, stream);
}

// Alg. 2: passes of the loop on the signal-domain residual r_out (zero-padded
// to L, reading Z3), each started from c^ = D^* r_out (the DGT of run_impl) and stopped
// after reset_every selections or by the inner stop rules, then r_out -= D c (synthesis
// of the pass's atoms on all L samples).  The stop level stays 10^(errdb/10) ||x||^2.
extern "C" int mpgabor_run_reset(mpgabor* h, const double* x_dev, int64_t Ls, int64_t maxit, double errdb,
                                 int64_t reset_every, mpg_atom* atoms_dev, double* energy_dev, mpg_result* res,
                                 void* stream) {
  if (!h) return MPG_EINVAL;
  if (!x_dev || !energy_dev || !res || (maxit > 0 && !atoms_dev)) return h->fail(MPG_EINVAL, "null pointer");
  if (Ls < 1 || maxit < 0 || reset_every < 1) return h->fail(MPG_EINVAL, "need Ls >= 1, maxit >= 0, reset_every >= 1");
  if (std::isnan(errdb)) return h->fail(MPG_EINVAL, "errdb is NaN");
  if (!h->have_kernels) return h->fail(MPG_ESTATE, "mpgabor_kernels must run before mpgabor_run_reset");
  int rc = enter_device(h);
  if (rc) return rc;
  rc = ensure_layout(h, Ls);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t L = h->L;
  TRY_CUDA(h, h->rr.ensure(sizeof(double) * L));
  TRY_CUDA(h, h->yy.ensure(sizeof(double) * L));
  TRY_CUDA(h, cudaMemsetAsync(h->rr.p, 0, sizeof(double) * L, st));
  TRY_CUDA(h, cudaMemcpyAsync(h->rr.p, x_dev, sizeof(double) * Ls, cudaMemcpyDeviceToDevice, st));
  // ||x||^2 and the absolute stop level
  TRY_CUDA(h, cudaMemsetAsync(h->flag.p, 0, sizeof(int), st));
  TRY_LAUNCH(h, 2, launch_pad_energy(x_dev, Ls, h->xp.as<double>(), L, h->partial.as<double>(), h->flag.as<int>(),
                                     h->E0.as<double>(), st));
  double E0 = 0.0;
  int nonfinite = 0;
  TRY_CUDA(h, cudaMemcpyAsync(&E0, h->E0.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaMemcpyAsync(&nonfinite, h->flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  if (nonfinite) return h->fail(MPG_ENONFINITE, "x contains NaN or Inf");
  const double Etol = (errdb == -INFINITY) ? -INFINITY : std::pow(10.0, errdb / 10.0) * E0;
  int64_t k = 0, rounds = 0;
  int stop = MPG_STOP_MAXIT, passes = 0;
  float t_loop = 0.f, t_dgt = 0.f;
  while (k < maxit) {
    mpg_result r{};
    rc = run_impl(h, h->rr.as<double>(), L, std::min<int64_t>(reset_every, maxit - k), errdb, &Etol,
                  atoms_dev + k, energy_dev + k, nullptr, &r, stream);
    if (rc) return rc;
    ++passes;
    rounds += r.rounds;
    t_loop += h->t_loop;
    t_dgt += h->t_dgt;
    if (r.n_atoms == 0) {  // the true residual energy reached the level, or a zero score
      stop = r.stop_reason;
      break;
    }
    rc = mpgabor_synth(h, atoms_dev + k, r.n_atoms, h->yy.as<double>(), L, stream);   // D c on all L samples
    if (rc) return rc;
    TRY_LAUNCH(h, 1, launch_sub(h->rr.as<double>(), h->yy.as<double>(), L, st));       // r_out -= D c
    k += r.n_atoms;
    if (r.stop_reason == MPG_STOP_ZERO) {
      stop = MPG_STOP_ZERO;
      break;
    }
  }
  double Ek = E0;
  TRY_CUDA(h, cudaMemcpyAsync(&Ek, energy_dev + k, sizeof(double), cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  h->t_loop = t_loop;
  h->t_dgt = t_dgt;
  h->passes = passes;
  res->n_atoms = k;
  res->L_pad = L;
  res->stop_reason = stop;
  res->cluster = h->lay_C;
  res->E0 = E0;
  res->E_final = Ek;
  res->rounds = rounds;
  return MPG_OK;
}

extern "C" int mpgabor_last_passes(const mpgabor* h, int32_t* passes) {
  if (!h || !passes) return MPG_EINVAL;
  *passes = h->passes;
  return MPG_OK;
}

extern "C" int mpgabor_residual(mpgabor* h, double* out_dev, void* stream) {
  if (!h || !out_dev) return MPG_EINVAL;
  if (h->L < 0 || !h->have_kernels) return h->fail(MPG_ESTATE, "no run yet");
  int rc = enter_device(h);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (h->f64())
    TRY_LAUNCH(h, 1, launch_grid_export<double>(h->grid.as<double2>(), h->d_geo.as<DictGeo>(), h->W, h->P_R,
                                           reinterpret_cast<double2*>(out_dev), st));
  else
    TRY_LAUNCH(h, 1, launch_grid_export<float>(h->grid.as<float2>(), h->d_geo.as<DictGeo>(), h->W, h->P_R,
                                          reinterpret_cast<double2*>(out_dev), st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  return MPG_OK;
}

extern "C" int mpgabor_set_pedantic(mpgabor* h, int32_t on) {
  if (!h) return MPG_EINVAL;
  if (on != 0 && on != 1) return h->fail(MPG_EINVAL, "pedantic must be 0 or 1");
  h->pedantic = on;
  return MPG_OK;
}

extern "C" int mpgabor_set_batch(mpgabor* h, int32_t max_batch) {
  if (!h) return MPG_EINVAL;
  if (max_batch < 0 || max_batch > multi_max_batch())
    return h->fail(MPG_EINVAL, "max_batch must be in [0, " + std::to_string(multi_max_batch()) + "]");
  if (max_batch != h->batch) h->L = -1;  // the loop kernel and its buffers are re-planned
  h->batch = max_batch;
  return MPG_OK;
}

extern "C" int mpgabor_set_profile(mpgabor* h, int32_t mode) {
  if (!h) return MPG_EINVAL;
  if (mode < 0 || mode > 3) return h->fail(MPG_EINVAL, "profile mode must be in [0, 3]");
  h->prof_mode = mode;
  return MPG_OK;
}

extern "C" int mpgabor_last_profile(const mpgabor* h, int64_t* cycles) {
  if (!h || !cycles) return MPG_EINVAL;
  for (int i = 0; i < MPG_PROF_SLOTS; ++i) cycles[i] = h->prof_host[i];
  return MPG_OK;
}

extern "C" int mpgabor_launch_count(const mpgabor* h, int64_t* n) {
  if (!h || !n) return MPG_EINVAL;
  *n = h->launches;
  return MPG_OK;
}

extern "C" int mpgabor_last_timing(const mpgabor* h, double* dgt_ms, double* init_ms, double* loop_ms) {
  if (!h) return MPG_EINVAL;
  if (dgt_ms) *dgt_ms = h->t_dgt;
  if (init_ms) *init_ms = h->t_init;
  if (loop_ms) *loop_ms = h->t_loop;
  return MPG_OK;
}

// ---------------------------------------------------------------------------
// synthesis
// ---------------------------------------------------------------------------
extern "C" int mpgabor_synth(mpgabor* h, const mpg_atom* atoms_dev, int64_t n_atoms, double* y_dev, int64_t Ls,
                             void* stream) {
  if (!h) return MPG_EINVAL;
  if (!y_dev || (n_atoms > 0 && !atoms_dev)) return h->fail(MPG_EINVAL, "null pointer");
  if (Ls < 1 || n_atoms < 0) return h->fail(MPG_EINVAL, "Ls must be >= 1 and n_atoms >= 0");
  if (!h->have_kernels) return h->fail(MPG_ESTATE, "mpgabor_kernels must run before mpgabor_synth");
  int rc = enter_device(h);
  if (rc) return rc;
  rc = ensure_layout(h, Ls);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TRY_CUDA(h, h->sol.ensure(sizeof(double2) * h->P_R));
  int64_t fmax = 0;
  for (auto& d : h->geo) fmax = std::max(fmax, (int64_t)d.N * d.M);
  TRY_CUDA(h, h->frames.ensure(sizeof(double) * fmax));
  TRY_CUDA(h, cudaMemsetAsync(h->sol.p, 0, sizeof(double2) * h->P_R, st));
  if (n_atoms > 0) {
    TRY_CUDA(h, h->sfirst.ensure(sizeof(unsigned int) * h->P_R));
    TRY_CUDA(h, h->sdone.ensure((size_t)(n_atoms + 3) / 4 * 4 + 16));
    TRY_CUDA(h, cudaMemsetAsync(h->sfirst.p, 0xff, sizeof(unsigned int) * h->P_R, st));
    TRY_CUDA(h, cudaMemsetAsync(h->sdone.p, 0, (size_t)(n_atoms + 3) / 4 * 4 + 16, st));
  }
  TRY_LAUNCH(h, (n_atoms > 0 ? 1 : 0),
             launch_synth_scatter(reinterpret_cast<const AtomOut*>(atoms_dev), n_atoms, h->d_geo.as<DictGeo>(), h->W,
                                  h->sol.as<double2>(), h->sfirst.as<unsigned int>(), h->sdone.as<unsigned char>(),
                                  reinterpret_cast<unsigned int*>(h->sdone.as<unsigned char>() + (n_atoms + 3) / 4 * 4), st));
  for (int w = 0; w < h->W; ++w) {
    const DictGeo& d = h->geo[w];
    TRY_LAUNCH(h, 1, launch_synth_frames(h->sol.as<double2>(), d, h->tw.as<double2>(), h->twres, h->frames.as<double>(), st));
    TRY_LAUNCH(h, 1, launch_synth_ola(h->frames.as<double>(), d, h->win.as<double>() + h->win_off[w], Ls, y_dev, w > 0, st));
  }
  return MPG_OK;
}

extern "C" int mpgabor_decompose_host(mpgabor* h, const double* x_host, int64_t Ls, int64_t maxit, double errdb,
                                      mpg_atom* atoms_host, double* energy_host, double* y_host, mpg_result* res,
                                      void* stream) {
  if (!h) return MPG_EINVAL;
  if (!x_host || !res) return h->fail(MPG_EINVAL, "null pointer");
  if (Ls < 1 || maxit < 0) return h->fail(MPG_EINVAL, "Ls must be >= 1 and maxit >= 0");
  int rc = enter_device(h);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  TRY_CUDA(h, h->hx.ensure(sizeof(double) * Ls));
  TRY_CUDA(h, h->hatoms.ensure(sizeof(mpg_atom) * std::max<int64_t>(1, maxit)));
  TRY_CUDA(h, h->henergy.ensure(sizeof(double) * (maxit + 1)));
  TRY_CUDA(h, h->hy.ensure(sizeof(double) * Ls));
  TRY_CUDA(h, cudaMemcpyAsync(h->hx.p, x_host, sizeof(double) * Ls, cudaMemcpyHostToDevice, st));
  rc = mpgabor_run(h, h->hx.as<double>(), Ls, maxit, errdb, h->hatoms.as<mpg_atom>(), h->henergy.as<double>(), nullptr,
                   res, stream);
  if (rc) return rc;
  if (y_host) {
    rc = mpgabor_synth(h, h->hatoms.as<mpg_atom>(), res->n_atoms, h->hy.as<double>(), Ls, stream);
    if (rc) return rc;
    TRY_CUDA(h, cudaMemcpyAsync(y_host, h->hy.p, sizeof(double) * Ls, cudaMemcpyDeviceToHost, st));
  }
  if (atoms_host && res->n_atoms > 0)
    TRY_CUDA(h, cudaMemcpyAsync(atoms_host, h->hatoms.p, sizeof(mpg_atom) * res->n_atoms, cudaMemcpyDeviceToHost, st));
  if (energy_host)
    TRY_CUDA(h, cudaMemcpyAsync(energy_host, h->henergy.p, sizeof(double) * (res->n_atoms + 1),
                                cudaMemcpyDeviceToHost, st));
  TRY_CUDA(h, cudaStreamSynchronize(st));
  return MPG_OK;
}
