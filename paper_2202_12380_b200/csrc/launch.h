// launch.h -- internal launcher declarations of libmpgabor (host side of the CUDA path).
#pragma once
#include "common.cuh"

cudaError_t launch_window(int win, int gl, int a, int M, double* g, cudaStream_t st);
cudaError_t launch_tables(double2* tw, int twres, double2* roots, int R, cudaStream_t st);
cudaError_t launch_pad_energy(const double* x, int64_t Ls, double* xp, int64_t L, double* partial, int* nonfinite,
                              double* E0, cudaStream_t st);
// write_pad = 0: leave the row padding (bins M/2+1 .. stride-1) alone -- it is zero from
// an earlier analysis of the same layout and nothing else writes it
template <typename R>
cudaError_t launch_dgt(const double* xp, int64_t L, const DictGeo& d, const double* g, const double2* tw, int twres,
                       typename cplx<R>::t* out, cudaStream_t st, int write_pad = 1);
cudaError_t launch_kern_rows(int a_c, int M_c, int nu_first, int nlag, const double* gu, int glu, const double* gv,
                             int glv, const double2* tw, int twres, double2* H, cudaStream_t st);
cudaError_t launch_kern_max_box(const double2* H, int nlag, int M_c, int nu_first, double thr, unsigned long long* mx,
                                int* box, cudaStream_t st);
template <typename R>
cudaError_t launch_kern_compact(const double2* H, int M_c, int nu_first, double thr, const unsigned long long* mx,
                                const PairGeo& pg, typename cplx<R>::t* kern, double2* boxcopy, RhoEnt* rho_row,
                                cudaStream_t st);
// sel: pedantic selection (rows of rho per dictionary: rho, rho_meta = {lo[W], n[W], off[W]}) or null
struct SelScore {
  int pedantic;
  const RhoEnt* rho;
  const int* rho_meta;
};
template <typename R>
cudaError_t launch_tile_init(const typename cplx<R>::t* grid, const DictGeo* dg, const OwnGeo* own, int W,
                             int64_t total, int C, int64_t Lc, int TW, Rec<R>* rec, SelScore sel, cudaStream_t st);

template <typename R>
cudaError_t launch_grid_export(const typename cplx<R>::t* grid, const DictGeo* dg, int W, int64_t P, double2* out,
                               cudaStream_t st);

// persistent MP loop (mploop.cu)
struct AtomOut {  // identical layout to mpg_atom
  int32_t w, m, n, flags;
  double re, im;
};
struct LoopResult {
  long long n_done;
  int stop;
  int pad;
  double E_final;
  long long rounds;              // loop rounds (multi-selection kernel; = n_done + 1 for the others)
  double E0;                     // E_0 = ||x||^2 of the slot (copied from E0v by the loop kernel)
};
constexpr int STOP_NONFINITE = -1;  // LoopResult.stop: x held NaN/Inf, the loop did not run

constexpr int MAX_LEVELS = 6;
constexpr int MPG_PROF_SLOTS = 512;  // mpgabor_last_profile slots
constexpr int MAX_CLUSTER = 16;
constexpr int TOP_SCAN = 256;   // the top node level (<= TOP_SCAN nodes) is scanned by one warp

struct LoopParams {
  int W, C, TW;
  int Rmax;
  int srec;                      // 1: this CTA's tile records live in shared memory
  int nlev;                      // node levels above the tiles (level l groups 32 of level l-1)
  int lev_n[MAX_LEVELS];         // node count per level; lev_n[nlev-1] <= TOP_SCAN
  int lev_off[MAX_LEVELS];       // node offset of each level in the shared level array
  int rho_total;                 // total entries of the conjugate-pair rows
  long long Lc;                  // tile records per CTA slice
  const DictGeo* dicts;          // [W]
  const OwnGeo* own;             // [C*W] frame ownership of each CTA
  const PairGeo* pairs;          // [W*W], index u*W + v
  const double2* roots;          // [Rmax]  e^{2 pi i r/Rmax}
  const RhoEnt* rho;             // concatenated nu=0 rows of h_uu (fp64) with 1/(1-|rho|^2)
  const int* rho_lo;             // [W] signed mu of rho[rho_off[u]]
  const int* rho_n;              // [W]
  const int* rho_off;            // [W]
  void* grid;                    // residual grids (cplx<R>)
  const void* kern;              // kernels (cplx<R>), per-class layout
  long long kern_elems;          // kernel entries (bounds checks of debug builds)
  void* rec;                     // Rec<R>[C * Lc] (initial records; the live ones when !srec)
  long long maxit;
  double E0;
  AtomOut* atoms;
  double* energy;
  double2* sol;                  // may be null
  LoopResult* result;
  long long* prof;               // optional [8] clock64 phase sums (rank 0, thread 0), [7] = iterations
  int floor_mode;                // 1: skip the update (latency-floor measurement; results invalid)
  int gx;                        // 1: grid mode (cooperative grid of C CTAs, exchange through global memory)
  void* gx_rec;                  // grid mode: one-selection kernel Rec<R>[2][C] roots, multi-selection
                                 //   kernel its [2][C] messages, in global memory (else null)
  unsigned long long* gx_stamp;  // [2][C] round stamps of gx_rec (zeroed before the launch)
  const double* E0v;             // per-slot E_0 (device, written by the energy kernel; null: the scalar E0)
  const int* nonfinite;          // device flag set by the energy kernel when x holds NaN/Inf (null: none)
  int etol_mode;                 // stop level per slot: 0 none (-inf), 1 etol_val * E0v[slot], 2 etol_val
  double etol_val;               //   (10^(errdb/10) for mode 1; an absolute level for mode 2)
  long long slot_grid;           //   grid elements per slot; the records per slot are C * Lc
  long long slot_atoms;          //   atoms per slot (= maxit); energies per slot = slot_atoms + 1
  int nslot;                     //   signals (clusters) of the launch
  int pedantic;                  // 1: select by the Eq. (20) energy (pedantic), else |c|^2
  int spec;                      // multi-selection: candidates per round (1..multi_max_batch())
  int topk_scan;                 // multi-selection: top-K by a scan of the tile records (no node tree upkeep)
  int l2pf;                      // multi-selection: the first l2pf walk-window entries' grid rows and kernel
                                 //   rows are bulk-prefetched into L2 after the window geometry (0: off;
                                 //   set when the grid and kernels do not fit L2)
  void* backup;                  // multi-selection: per-CTA tile backups [C][bk_cap][TW] (cplx<R>)
  long long bk_cap;              // items per CTA per round the backup holds
  size_t smem_bytes;
};

// default loop kernel (mploop.cu)
size_t loop_smem_bytes(const LoopParams& P, bool f64);
cudaError_t launch_mp_loop(const LoopParams& P, bool f64, int threads, cudaStream_t st);
// gx: the global-exchange grid kernel; returns its co-resident CTA count
int loop_max_cluster(bool f64, bool srec, int TW, int threads, size_t smem, bool gx = false);

// exact multi-selection loop kernel (mpmulti.cu, the default): MULTI_K = length of
// every CTA's published top-K tile list
#ifndef MPG_MULTI_K
#define MPG_MULTI_K 4
#endif
constexpr int MULTI_K = MPG_MULTI_K;
size_t multi_smem_bytes(const LoopParams& P, bool f64);
int multi_max_batch();
int multi_window();     // walk-window entries per round (NE)
int multi_max_threads();  // the multi-selection kernel's launch bound (MPG_LB_THREADS)
cudaError_t launch_multi_loop(const LoopParams& P, bool f64, int threads, cudaStream_t st);
// gx: the global-exchange grid kernel; returns its co-resident CTA count
int multi_max_cluster(bool f64, bool srec, int TW, int threads, size_t smem, bool gx = false);
size_t multi_msg_bytes(bool f64);


// synthesis (synth.cu)
// first: uint32[P_R] all 0xff, done: uint8[n_atoms] all 0, ctl: uint32[3] all 0 (scratch)
cudaError_t launch_synth_scatter(const AtomOut* atoms, int64_t n_atoms, const DictGeo* dg_dev, int W, double2* sol,
                                 unsigned int* first, unsigned char* done, unsigned int* ctl, cudaStream_t st);
cudaError_t launch_synth_frames(const double2* sol, const DictGeo& d, const double2* tw, int twres, double* frames,
                                cudaStream_t st);
cudaError_t launch_sub(double* r, const double* y, int64_t n, cudaStream_t st);  // r -= y
cudaError_t launch_synth_ola(const double* frames, const DictGeo& d, const double* g, int64_t L, double* y,
                             int accumulate, cudaStream_t st);
