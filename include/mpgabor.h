/*
 * mpgabor.h -- C ABI of the B200-native coefficient-domain multi-Gabor matching
 * pursuit library (libmpgabor.so), after Prusa, Holighaus, Balazs,
 * "Fast Matching Pursuit with Multi-Gabor Dictionaries" (arXiv 2202.12380).
 *
 * Citations "P:<line>" refer to the paper text.  The call sequence
 * follows the paper's C workflow:
 *   dgtrealmp_parbuf_add_firwin  -> mpgabor_create   (dictionaries)
 *   dgtrealmp_setparbuf_kernrelthr + dgtrealmp_init -> mpgabor_kernels
 *   dgtrealmp_execute            -> mpgabor_run (+ mpgabor_synth for fout)
 *   dgtrealmp_done               -> mpgabor_destroy
 *
 * Conventions for every call
 *   - Return value: 0 (MPG_OK) on success, a negative MPG_E* code on failure; the
 *     handle keeps a human-readable reason, see mpgabor_last_error().
 *   - "dev" pointers are CUDA device pointers (e.g. torch tensors) on the device
 *     that was current when mpgabor_kernels() first ran; "host" pointers are
 *     ordinary host memory.  The caller owns every pointer it passes.
 *   - The handle owns all internal device memory (kernels, residual grids, max
 *     tracking, scratch) and frees it in mpgabor_destroy().
 *   - A handle is single-owner and not thread-safe; distinct handles may be
 *     used concurrently.
 *   - cuda_stream is a cudaStream_t (NULL = legacy default stream).  Work is
 *     ordered on it; calls that return counts synchronise it before returning.
 *   - All input/output signals, energies and atom coefficients are fp64.  The
 *     precision chosen at create time is the storage/arithmetic precision of
 *     the coefficient-domain residual and of the kernels on the GPU (the
 *     scalar step of each iteration is always fp64, reading Z18).
 */
#ifndef MPGABOR_H
#define MPGABOR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mpgabor mpgabor; /* opaque, library-owned */

/* window kinds (Fig. 1; periodic zero-phase forms, Z1/Z2) */
enum { MPG_WIN_HANN = 1, MPG_WIN_BLACKMAN = 2, MPG_WIN_GAUSS = 3 /* tfr = a*M */ };

/* residual/kernel precision on the GPU */
enum { MPG_F64 = 0, MPG_F32 = 1 };

/* one Gabor dictionary: window kind, window length gl, hop a, channels M
 * (dgtrealmp_parbuf_add_firwin(win, gl, a, M)).  Requirements:
 * M a power of two with 2 <= M <= 16384, a >= 1, M % a == 0,
 * gl >= 1.  The paper only needs pairwise divisibility; the power-of-two
 * M is this library's deliberate restriction (Z25): it covers every
 * configuration of the paper's experiments and lets the DGT and
 * synthesis use radix-2 shared-memory FFTs and the loop kernels shift/mask index
 * arithmetic; other M are rejected with MPG_EINVAL. */
typedef struct {
  int32_t win, gl, a, M;
} mpg_dict;

/* one selected atom: dictionary w, frequency bin m in [0, M_w/2], frame n;
 * flags bit0 = self-conjugate (m == 0 or m == M_w/2, Eq. (18));
 * (re, im) = adjusted coefficient c~ of Eq. (19) P:867-873 (im == 0 for
 * self-conjugate atoms).  32 bytes, naturally aligned. */
typedef struct {
  int32_t w, m, n, flags;
  double re, im;
} mpg_atom;

/* run summary (host struct) */
typedef struct {
  int64_t n_atoms;     /* selections performed                                   */
  int64_t L_pad;       /* working length (Ls zero-padded, Z3)          */
  int32_t stop_reason; /* MPG_STOP_*                                             */
  int32_t cluster;     /* CTAs in the thread-block cluster that ran the loop    */
  double E0;           /* ||x||^2                                                */
  double E_final;      /* energy estimate E_k after the last selection (Alg. 1)  */
  int64_t rounds;      /* persistent-loop rounds (multi-selection: several atoms
                          per round, see mpgabor_set_batch; otherwise n_atoms+1) */
} mpg_result;

enum { /* stop reasons, tested in this order before each selection (Z15) */
  MPG_STOP_MAXIT = 1,  /* k >= maxit      */
  MPG_STOP_ERRTOL = 2, /* E_k <= 10^(errdb/10) ||x||^2     */
  MPG_STOP_NEGEST = 3, /* E_k < 0, i.e. sum of removed energy > ||x||^2  */
  MPG_STOP_ZERO = 4    /* the largest |c|^2 is 0  */
};

enum {
  MPG_OK = 0,
  MPG_EINVAL = -1,     /* null pointer, W<1 or W>MPG_MAX_DICTS, bad window/sizes, thr outside [0,1), maxit<0, Ls<1 */
  MPG_EINCOMPAT = -2,  /* M % a != 0, or a pair with min(a) not dividing max(a) or min(M) not dividing max(M) */
  MPG_ESTATE = -3,     /* mpgabor_run/_synth before mpgabor_kernels                                      */
  MPG_ENOMEM = -4,     /* device allocation failed                                                       */
  MPG_ECUDA = -5,      /* CUDA error or no usable device; detail in mpgabor_last_error()                 */
  MPG_ELEN = -6,       /* L_pad too short for the kernels (circular aliasing: L_pad < gl_u+gl_v, or a
                          kernel box wider than a target grid), or length overflow                      */
  MPG_ENONFINITE = -7  /* NaN or Inf in x                                                                */
};

#define MPG_MAX_DICTS 16

/* Validate the multi-Gabor dictionary (§2.1) and create a handle.
 * dicts: host array of W entries (copied).  precision: MPG_F64 or MPG_F32.
 * *out receives the handle (NULL on failure; the error text of a failed create
 * is available via mpgabor_last_error(NULL)).  No GPU work is done here. */
int mpgabor_create(const mpg_dict* dicts, int32_t W, int32_t precision, mpgabor** out);

/* Precompute all W*W truncated (cross-)kernels h_{u,v} on the common grids
 * (a_c = min(a_u,a_v), M_c = max(M_u,M_v)) with relative threshold thr
 * (Eq. (7) P:407-413 read relative to each kernel's own max|h|, strict '>',
 * DESIGN.md Z5-Z7; Eqs. (14)-(17) P:549-660), their modulation roots
 * and the conjugate-pair lookup, entirely on the GPU.
 * 0 <= thr < 1.  Independent of the signal length.  Recomputes
 * and replaces previous kernels.  Synchronises cuda_stream. */
int mpgabor_kernels(mpgabor* h, double thr, void* cuda_stream);

/* Geometry for a signal of Ls samples (host outputs, each may be NULL):
 * L_pad, and per dictionary w: N[w] frames, M_R[w] = M_w/2+1 reduced bins,
 * row_stride[w] = elements between consecutive frames of dictionary w in every
 * coefficient vector this API exchanges (coef_dev of mpgabor_run, the export of
 * mpgabor_residual) -- these are dense, so row_stride[w] = M_R[w]; the library's
 * internal residual grids pad rows to whole tiles and stay private --
 * coef_offset[w] = global index of (w, n=0, m=0) in the coefficient vector
 * (index p = coef_offset[w] + n*row_stride[w] + m, Z10), coef_offset[W] =
 * total number of reduced coefficients P_R.  Pure host computation. */
int mpgabor_layout(const mpgabor* h, int64_t Ls, int64_t* L_pad, int64_t* N, int64_t* M_R,
                   int64_t* row_stride, int64_t* coef_offset);

/* Run coefficient-domain MP (Alg. 1 P:356-387 with Eq. (9) P:424-434 and Alg. 3
 * P:978-1029) on x_dev (device fp64[Ls]):
 *   DGT analysis of every dictionary, max-structure init,
 *   then the persistent selection/update loop until a stop rule fires.
 * maxit >= 0; errdb: target 10log10(E_k/||x||^2) (use -INFINITY to disable).
 * Outputs (device, caller-owned):
 *   atoms_dev   mpg_atom[maxit]    selected atoms in order (first n_atoms valid)
 *   energy_dev  double[maxit+1]    E_0 .. E_{n_atoms} (first n_atoms+1 valid)
 *   coef_dev    complex double[P_R] (interleaved re,im) solution vector c,
 *               zeroed then accumulated (c(p) += c~, Alg. 1 step 2a); may be NULL
 * res (host) receives the summary.  Synchronises cuda_stream. */
int mpgabor_run(mpgabor* h, const double* x_dev, int64_t Ls, int64_t maxit, double errdb,
                mpg_atom* atoms_dev, double* energy_dev, double* coef_dev, mpg_result* res,
                void* cuda_stream);

/* Approximate coefficient-domain MP with reset, Alg. 2: passes of the
 * loop of mpgabor_run on the signal-domain residual r_out (x zero-padded to L_pad,
 * DESIGN.md Z3).  Each pass starts from c^ = D^* r_out with E_k = ||r_out||^2 and runs
 * until reset_every (>= 1) selections or an inner stop rule; then r_out -= D c
 * (synthesis of the pass's atoms).  The run stops after maxit selections in total,
 * when the true residual energy at a pass start is <= 10^(errdb/10) ||x||^2, or at
 * a zero largest score.  Outputs as for mpgabor_run (atoms of all passes in order;
 * energy_dev[k] is the true residual energy ||r_out||^2 at every pass start k and
 * the Eq. (20) estimate inside a pass); res->E_final = energy_dev[n_atoms].  The
 * solution vector is not produced (it is the sum of the atom list).  Synchronises
 * cuda_stream. */
int mpgabor_run_reset(mpgabor* h, const double* x_dev, int64_t Ls, int64_t maxit, double errdb,
                      int64_t reset_every, mpg_atom* atoms_dev, double* energy_dev, mpg_result* res,
                      void* cuda_stream);
/* Number of passes of the last mpgabor_run_reset (host output). */
int mpgabor_last_passes(const mpgabor* h, int32_t* passes);
/* Batched independent signals: B >= 1 signals of Ls
 * samples each, decomposed concurrently with the same dictionaries and kernels,
 * one cluster per signal (automatic cluster size 16 for B <= 4, 8 for B <= 12,
 * else 4 CTAs, so that many signals run at once on the 148 SMs; mpgabor_set_launch
 * overrides it; clusters that do not fit queue).  x_dev: device fp64[B][Ls]; atoms_dev: mpg_atom[B][maxit]; energy_dev:
 * double[B][maxit+1]; res: host mpg_result[B].  Every signal's results equal those
 * of mpgabor_run on it (bit for bit; every loop kernel gives the same atoms).  The
 * loop kernel follows mpgabor_set_batch (0: the automatic choice, 1: one selection
 * per iteration, 2..8: exact multi-selection); grid mode is not used for batches.
 * Synchronises cuda_stream. */
int mpgabor_run_batch(mpgabor* h, const double* x_dev, int32_t B, int64_t Ls, int64_t maxit, double errdb,
                      mpg_atom* atoms_dev, double* energy_dev, mpg_result* res, void* cuda_stream);
/* Synthesis of the approximation from an atom list (Eq. (18)):
 * y = sum_atoms c~ d (self-conjugate) or 2 Re(c~ d) (pairs), on L_pad samples,
 * truncated to Ls and written to y_dev (device fp64[Ls]).  atoms_dev: device
 * mpg_atom[n_atoms] as produced by mpgabor_run for the same Ls.  Asynchronous
 * on cuda_stream. */
int mpgabor_synth(mpgabor* h, const mpg_atom* atoms_dev, int64_t n_atoms, double* y_dev, int64_t Ls,
                  void* cuda_stream);

/* End-to-end convenience on HOST buffers: copies x_host (fp64[Ls]) to the
 * device, runs mpgabor_run + mpgabor_synth, and copies back atoms_host
 * (mpg_atom[maxit]), energy_host (double[maxit+1]) and y_host (double[Ls]);
 * any output pointer may be NULL.  Uses library-owned device buffers.
 * Synchronises cuda_stream. */
int mpgabor_decompose_host(mpgabor* h, const double* x_host, int64_t Ls, int64_t maxit, double errdb,
                           mpg_atom* atoms_host, double* energy_host, double* y_host,
                           mpg_result* res, void* cuda_stream);

/* Launch tuning of the persistent loop: cluster size (1..16 CTAs, one per SM,
 * power of two; or 32, 64, 128: the loop kernel as a cooperative grid of that many
 * CTAs exchanging their roots / messages through global memory), threads per CTA
 * (128..512, multiple of 32), tile width in bins (32, 64 or 128), tile-record
 * placement (1 shared memory, 2 global memory).  0 selects automatically: a 16-CTA
 * cluster, or a grid of 64 / 128 CTAs for wide updates (multi-selection from ~10k /
 * 40k coefficients per atom, one selection from 30k); tile width 32 then 64 for the
 * multi-selection cluster, 64 first for grids and the one-selection loop; shared
 * records where they fit.  Takes effect at the next run. */
int mpgabor_set_launch(mpgabor* h, int32_t cluster, int32_t threads, int32_t tile_width, int32_t records);

/* Selection rule (Alg. 1 step 1).  on = 0 (default): argmax |c^|^2 over the reduced
 * coefficients (non-pedantic, reading Z9).  on = 1 ("pedantic"): argmax of
 * the energy the selection removes, Eq. (20) with the Eq. (19) coefficient (|c~|^2
 * -> (Re c^)^2 for self-conjugate atoms, 2|c^|^2 where <d, conj d> = 0).  Ties go to
 * the lowest index either way.  EINVAL unless 0 or 1.  Takes effect at the next run. */
int mpgabor_set_pedantic(mpgabor* h, int32_t on);
/* Exact multi-selection: max_batch = the
 * most atoms one loop round may select and update at once.  Every round's extra
 * atoms are verified against the sequential argmax rule (Alg. 1, ties
 * Z10) and rolled back bit-exactly when the proof fails, so the atom sequence,
 * coefficients and energies are those of the one-selection loop for every value.
 * 0 = automatic: batch 8 when an atom's update (estimated from the kernel boxes)
 * covers < 0.5 % of the reduced coefficients (C1..C4), else one selection per
 * iteration (C0); DESIGN.md §6b/§6c have the measured crossovers; 1 = one selection
 * per iteration (the plain persistent loop); 2..8 = that batch.  EINVAL outside
 * [0, 8].  Takes effect at the next run. */
int mpgabor_set_batch(mpgabor* h, int32_t max_batch);
/* The launch plan used by the last mpgabor_run (host outputs, may be NULL);
 * records: 1 shared memory, 2 global memory. */
int mpgabor_launch_info(const mpgabor* h, int32_t* cluster, int32_t* threads, int32_t* tile_width,
                        int32_t* records, int64_t* smem_bytes);

/* Kernel statistics after mpgabor_kernels (host outputs, may be NULL):
 * stored box entries summed over all pairs, entries kept by the threshold,
 * and bytes of device kernel storage. */
int mpgabor_kernel_stats(const mpgabor* h, int64_t* box_entries, int64_t* kept_entries,
                         int64_t* bytes);

/* Copy the (u, v) kernel box to host memory, for parity tests:
 * box (host int32[4]) = {mu_lo, mu_hi, nu_lo, nu_hi};
 * values (host complex double[(mu_hi-mu_lo+1)*(nu_hi-nu_lo+1)] or NULL),
 * row-major [nu][mu], zero where below threshold; *mx = max|h| (may be NULL).
 * Pass values = NULL first to query the box size. */
int mpgabor_kernel_box(mpgabor* h, int32_t u, int32_t v, int32_t* box, double* values, double* mx);

/* Timing split of the last mpgabor_run in milliseconds (host outputs, may be
 * NULL): analysis (pad + energy + DGT), max-structure init, iteration loop. */
int mpgabor_last_timing(const mpgabor* h, double* dgt_ms, double* init_ms, double* loop_ms);

/* Number of this library's CUDA kernels enqueued through h so far (host output). */
int mpgabor_launch_count(const mpgabor* h, int64_t* n);

/* Copy the coefficient-domain residual c^ of the last mpgabor_run (after its
 * final selection; after the DGT alone when maxit = 0) to out_dev (device
 * complex double[P_R], interleaved, index p as in mpgabor_layout), converting
 * from the run precision.  For tests and diagnostics.  Synchronises cuda_stream. */
int mpgabor_residual(mpgabor* h, double* out_dev, void* cuda_stream);

/* Instrumentation of the persistent loop (takes effect at the next run):
 * mode bit0 = accumulate per-phase SM clock cycles on CTA 0 / thread 0;
 * mode bit1 = latency-floor mode: the residual update is skipped (selection,
 * scalar step, max refresh and the cluster barrier still run) -- the results
 * of such a run are NOT a decomposition and must only be used for timing
 * (one-selection kernel).  EINVAL outside [0, 3]. */
int mpgabor_set_profile(mpgabor* h, int32_t mode);

/* cycles (host int64[512]) of the last run with mode bit0, summed over the
 * iterations on CTA 0 / thread 0.  One-selection loop (mpgabor_set_batch 1):
 * [0] wait for the C roots (mailbox barrier), [1] selection + scalar step,
 * [2] block barrier after selection, [3] own update work, [4] block barrier
 * after the update, [5] level-1 refresh + barrier, [6] upper levels + root
 * publication; [7] iterations.  Multi-selection loop: [0] wait for the
 * messages, [1] verification, [2] barrier (window ranking on warps 1..), [3]
 * grid mode: stage-2 ranking, [4] window geometry + scalar steps + barrier, [5]
 * pair masks, [6] wait for the pair warps, [29] walk set-up, [27] walk, [28] E
 * chain + atoms, [9] item bases, [10] barrier, [11] own items, [12] barrier +
 * level refresh, [13] top-K, [14] message push; [15] rounds; [16] candidate-list
 * extraction, [17] candidate-list rebuilds (cycles), [19] rebuilds (count);
 * [20] sum of the walk's last window position, [21..26] walk end reasons (batch
 * full, window, list exhausted, zero score, overlap, last list entry); [30],
 * [31] warp 1: wait, ranking; [40..55] CTAs 0..15: busy cycles (messages
 * received -> message published); [56] roll-back rounds, [57..63] first rejected
 * candidate 1..7; [64..191] CTAs 0..127: busy cycles; [192..319] CTAs 0..127:
 * items; [320..447] CTAs 0..127: candidate-list rebuilds; [448..455] message
 * waits of CTA 0 by length (< 1k, 1-2k, 2-3k, 3-4k, 4-6k, 6-8k, 8-12k, >= 12k
 * cycles): counts, [456..463] their cycle sums; [464..467] rounds by the deepest
 * CTA-list position (0..3) among the walk-window entries; [468..472] candidate-list
 * rebuilds of CTA 0: node maxima, rank counts, gathers (cycles), rank-halving retries,
 * rebuilds, [473] record-scan fallbacks; [480..495] all CTAs' rounds by items (8 per
 * bucket), [496..511] by busy cycles (4096 per bucket). */
int mpgabor_last_profile(const mpgabor* h, int64_t* cycles);

void mpgabor_destroy(mpgabor* h);

/* Reason for the last failure on h (or of the last failed mpgabor_create when
 * h is NULL).  Never NULL; valid until the next call on h. */
const char* mpgabor_last_error(const mpgabor* h);

#ifdef __cplusplus
}
#endif
#endif /* MPGABOR_H */
