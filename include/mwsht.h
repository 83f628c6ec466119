/*
 * mwsht.h — C ABI of the B200-native McEwen–Wiaux spin spherical-harmonic
 * transforms (libmwsht.so, built from paper_1110_6298_b200/csrc/).
 *
 * Drop-in boundary.  The reference (torusht, pure Python/numba) has no native
 * ABI; its plugin/operator interface for this path is the Python entry points
 * in pkg/src/torusht/mw.py and the kernel dispatchers in
 * pkg/src/torusht/kernels/__init__.py.  Each entry point below replaces one of
 * those (cited per function).  A host binding (paper_1110_6298_b200/_lib.py,
 * ctypes) mirrors the reference's Python names, argument meaning and
 * exception types on top of these calls; INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Conventions (identical to the reference):
 *   - N = 2L-1.  Complex values are interleaved (re, im) float64 pairs
 *     (numpy complex128 / C double _Complex layout).
 *   - Flat coefficients: length L*L, index l(l+1)+m, 0 <= l < L, |m| <= l.
 *   - Samples: (L, N) row-major, theta_t = pi(2t+1)/N rows, phi_p = 2 pi p/N cols.
 *   - 2-D coefficient tables (kernel hooks): (L, N), column L-1+m.
 *   - gfold (kernel hooks): (N, L), row L-1+m, column m' >= 0.
 *   - All data pointers are DEVICE pointers on the plan's device unless the
 *     name says _host.  Inputs are read-only; outputs are fully overwritten.
 *   - `stream` is a cudaStream_t (0 = legacy default stream).  Calls are
 *     asynchronous with respect to the host except where noted.  A plan owns
 *     scratch buffers; calls on one plan from several threads and streams are
 *     safe (reentrant): the host side is serialised by a mutex and
 *     on the device each call waits for the previous call's work on another
 *     stream (an event hand-off), so concurrent callers never share scratch
 *     in flight.
 *   - Every entry point restores the caller's current CUDA device.
 *   - Band limits: every L >= 1 up to the documented cap L <= 8192 (the FFT
 *     engine keeps one H <= 8192-point part of each convolution in an SM's
 *     shared memory: halves up to L = 4096, quarters above); larger L fails
 *     with MWSHT_E_DEGREE (UnsupportedDegreeError).
 *   - `recursion`: MWSHT_TRAPANI or MWSHT_RISBO.  Both are accepted for
 *     drop-in compatibility (mw.py:43,562-566); both run the same stable GPU
 *     recursions (inverse: l-recursion, forward: exponent-scaled Trapani
 *     columns), so neither reproduces the reference Trapani's l>~1040
 *     divergence.
 *
 * Every function returns an mwsht_status; the host binding maps it 1:1 onto
 * the reference's exception types (errors.py:8-33).
 */
#ifndef MWSHT_H
#define MWSHT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MWSHT_OK = 0,
  MWSHT_E_BAND_LIMIT = 1,   /* InvalidBandLimitError   (grid.py:37-42)            */
  MWSHT_E_SPIN = 2,         /* InvalidSpinError        (mw.py:121-126, 476-479)   */
  MWSHT_E_CONTRACT = 3,     /* ContractViolationError  (mw.py:61-71, 94-98, 429)  */
  MWSHT_E_SYMMETRY = 4,     /* SymmetryError           (mw.py:543-547)            */
  MWSHT_E_VALUE = 5,        /* ValueError: unknown recursion (mw.py:562-566)      */
  MWSHT_E_CUDA = 6,         /* CUDA runtime failure                              */
  MWSHT_E_DEGREE = 7,       /* UnsupportedDegreeError  (errors.py:24-25): L > 8192 */
  MWSHT_E_NOMEM = 8,        /* device or host allocation failure                 */
  MWSHT_E_PLAN = 9          /* null / mismatched plan                            */
} mwsht_status;

typedef enum { MWSHT_TRAPANI = 0, MWSHT_RISBO = 1 } mwsht_recursion;

typedef struct mwsht_plan mwsht_plan;

/* Library / device introspection. */
const char *mwsht_version(void);
const char *mwsht_status_string(int status);
/* Last CUDA error text recorded by this thread (for diagnostics). */
const char *mwsht_last_error(void);

/* Plan for band-limit L on `device` (cudaGetDevice() if < 0).  Owns the FFT
 * engine's tables (chirps, twiddles, the quadrature-weight spectrum: cf. the
 * reference's _CONV_CACHE, mw.py:225-241), the 1-D recursion tables, the l-independent top-row seed
 * table sqrt(C(2n,n+k))/2^n, per-spin spin-column tables (built lazily), and
 * scratch buffers for up to `max_batch` maps.  Creation synchronises. */
int mwsht_plan_create(int L, int device, int max_batch, mwsht_plan **out);
int mwsht_plan_destroy(mwsht_plan *plan);
/* Device bytes currently held by the plan (tables + scratch). */
size_t mwsht_plan_device_bytes(const mwsht_plan *plan);
/* Build the spin-s tables now (otherwise built on first use; synchronises). */
int mwsht_plan_prepare_spin(mwsht_plan *plan, int spin);

/* ---------------------------------------------------------------- transforms */

/* forward(signal, recursion) -> HarmonicCoeffs          (mw.py:365-375)
 * samples: (L, N) complex;  flm: (L*L,) complex. */
int mwsht_forward_z(mwsht_plan *plan, const void *samples, void *flm, int spin,
                    int recursion, void *stream);

/* inverse(coeffs, recursion) -> MwSignal                (mw.py:419-438)
 * flm: (L*L,) complex (entries l < |spin| must be zero: checked by the host
 * binding, mw.py:429-434);  samples: (L, N) complex. */
int mwsht_inverse_z(mwsht_plan *plan, const void *flm, void *samples, int spin,
                    int recursion, void *stream);

/* forward_real(signal, recursion), spin 0                (mw.py:469-501)
 * samples: (L, N) float64;  flm: (L*L,) complex (m < 0 rebuilt from the
 * reality condition, mw.py:514-521). */
int mwsht_forward_real_d(mwsht_plan *plan, const double *samples, void *flm, int recursion,
                         void *stream);

/* inverse_real(coeffs, recursion), spin 0                (mw.py:524-559)
 * flm: (L*L,) complex satisfying conj(f_lm) = (-1)^m f_l,-m (checked by
 * mwsht_reality_residual);  samples: (L, N) float64. */
int mwsht_inverse_real_d(mwsht_plan *plan, const void *flm, double *samples, int recursion,
                         void *stream);

/* Reality check of inverse_real (mw.py:537-547): writes the worst residual
 * max|conj(f) - (-1)^m f_{l,-m}| and the tolerance 1e-12*max(1, max|f|) to
 * host memory.  Synchronises `stream`. */
int mwsht_reality_residual(mwsht_plan *plan, const void *flm, double *worst_host,
                           double *tol_host, void *stream);

/* The same check without a host sync (pipelined callers, which report the
 * violation later): max-reduces the residual and max|f| into
 * dev_worst_peak[0..1] (device memory, float64 bit patterns as uint64,
 * zero-initialised by the caller); tolerance = 1e-12 max(1, peak). */
int mwsht_reality_residual_async(mwsht_plan *plan, const void *flm,
                                 unsigned long long *dev_worst_peak, void *stream);

/* Batched transforms over `nmaps` independent maps laid out back to back
 * (map stride L*L for coefficients, L*N for samples); nmaps <= max_batch.
 * Same per-map semantics as the single-map calls (the callers'
 * cli.py:159-224 loop over maps). */
int mwsht_forward_z_batch(mwsht_plan *plan, int nmaps, const void *samples, void *flm,
                          int spin, int recursion, void *stream);
int mwsht_inverse_z_batch(mwsht_plan *plan, int nmaps, const void *flm, void *samples,
                          int spin, int recursion, void *stream);

/* Multi-spin batches (the paper's footnote PAPER.md:505
 * on transforms sharing one Wigner recursion): map b (b < nmaps <= 16, and
 * <= max_batch) has spin spins[b] (host array).  Every (m', m) chain's
 * recursion is spin-independent, so two maps of any spins share each chain
 * and only their row weights Delta^l_{m',-s} and phases differ.  Same
 * per-map results as mwsht_forward_z / mwsht_inverse_z with that spin. */
int mwsht_forward_z_multi(mwsht_plan *plan, int nmaps, const void *samples, void *flm,
                          const int *spins, int recursion, void *stream);
int mwsht_inverse_z_multi(mwsht_plan *plan, int nmaps, const void *flm, void *samples,
                          const int *spins, int recursion, void *stream);

/* --------------------------------------------------- kernel-level hooks ----
 * Mirrors of torusht.kernels dispatchers (kernels/__init__.py:67-80) on
 * device buffers, for stage-by-stage parity (test_kernels.py:52-92). */

/* fmm_core(flm2d, cl, L, spin, use_trapani) -> T         (_numba.py:74-105)
 * flm2d: (L, N) complex; cl: (L,) float64; T: (L, N) complex. */
int mwsht_fmm_core(mwsht_plan *plan, const void *flm2d, const double *cl, int spin,
                   int use_trapani, void *T, void *stream);
/* flm_core(gfold, L, spin, use_trapani) -> R             (_numba.py:131-166)
 * gfold: (N, L) complex; R: (L, N) complex. */
int mwsht_flm_core(mwsht_plan *plan, const void *gfold, int spin, int use_trapani, void *R,
                   void *stream);
/* fmm_core_real(flm_half, cl, L, use_trapani) -> T       (_numba.py:108-128)
 * flm_half, T: (L, L) complex. */
int mwsht_fmm_core_real(mwsht_plan *plan, const void *flm_half, const double *cl,
                        int use_trapani, void *T, void *stream);
/* flm_core_real(gfold, L, use_trapani) -> R              (_numba.py:169-188)
 * gfold, R: (L, L) complex. */
int mwsht_flm_core_real(mwsht_plan *plan, const void *gfold, int use_trapani, void *R,
                        void *stream);

/* Forward FFT stages only: samples (L, N) complex -> gfold (N, L) complex
 * (phi_fft, periodic_extend, theta_fft, weighted_convolution, _fold_mprime:
 * mw.py:149-285), for stage-level parity. */
int mwsht_forward_stages_z(mwsht_plan *plan, const void *samples, void *gfold, int spin,
                           void *stream);

/* Kernel launches issued by the most recent transform call on this plan (all
 * of them are this library's own kernels: no library FFT/BLAS is called). */
int mwsht_plan_last_launches(const mwsht_plan *plan, int *own);

/* ------------------------------------------------ m-column / ring sharding ----
 * Stage entry points of ONE complex map split over ranks: a
 * rank owns the orders m0 <= |m| < m1 (m0, m1 multiples of 32, or m1 = L) and
 * the rings t0 <= t < t1.  With the l-recursion / Trapani-column cores every
 * chain is independent, so no Delta halo is exchanged; the only
 * exchange is one all-to-all transpose of the ring spectra per transform,
 * plus an all-gather of the forward's coefficient blocks, done by the caller
 * (paper_1110_6298_b200/shard.py, NCCL) on buffers these kernels read and
 * write in place:
 *   forward: shard_forward_phi writes the phi spectra of rings t0..t1 straight
 *            into the all-to-all SEND layout (bin k, ring t at
 *            out[row_off[k] + t - t0]); after the all-to-all,
 *            shard_forward_rest reads the RECEIVE layout (local order row i,
 *            ring t at in[col_off[t] + i * col_stride[t]]), runs the theta
 *            stage and the forward core for its orders and writes either the
 *            flat flm (packed = 0, its orders only) or its packed coefficient
 *            block (packed = 1: l-major, orders -hi..-max(m0,1), m0..hi per
 *            degree); after an all-gather of the blocks shard_unpack_flm
 *            rebuilds the flat flm on every rank.
 *   inverse: shard_inverse_front (prescale + core + theta synthesis of its
 *            orders) writes ring t of local order row i to out[row_off[t] + i]
 *            (the SEND layout); after the all-to-all, shard_inverse_phi reads
 *            ring t, bin n at in[col_off[n] + (t - t0) * col_stride[n]] and
 *            writes its rings of the samples.
 * Local order row i enumerates +m0..+(m1-1), then -m0..-(m1-1) (m = 0 once).
 * The offset tables are device arrays built by the caller (shard.py); passing
 * NULL tables selects the dense single-GPU layouts, which emulate_mcolumn
 * uses: OUT: L x N, column bin(m); AT: (N + 1) L values with the bins in pairs,
 * bin k, ring t at ((k >> 1) L + t) 2 + (k & 1) (what both stages read and
 * write with 32-byte accesses). */
int mwsht_shard_forward_phi(mwsht_plan *plan, const void *samples_rows, int t0, int t1,
                            const long long *row_off, void *out, void *stream);
int mwsht_shard_forward_rest(mwsht_plan *plan, const void *in, int m0, int m1,
                             const long long *col_off, const int *col_stride, int spin, void *flm,
                             int packed, void *stream);
int mwsht_shard_inverse_front(mwsht_plan *plan, const void *flm, int m0, int m1, int spin,
                              const long long *row_off, void *out, void *stream);
int mwsht_shard_inverse_phi(mwsht_plan *plan, const void *in, int t0, int t1,
                            const long long *col_off, const int *col_stride, void *samples_rows,
                            void *stream);
/* gathered: world blocks of maxlen complex values (rank r's packed block at
 * r * maxlen); bounds: device int[world + 1] order boundaries. */
int mwsht_shard_unpack_flm(mwsht_plan *plan, const void *gathered, long long maxlen,
                           const int *bounds, int world, void *flm, void *stream);

/* ------------------------------------------------ Gauss-Legendre comparator ----
 * gl_fm_core(flm_scaled, x, ch, sh, L, spin) -> F     (_numba.py:237-268)
 * gl_flm_core(a, x, ch, sh, L, spin) -> R             (_numba.py:211-234)
 * Device arrays: flm_scaled (L, N) and R (L, N) complex; a and F (N, L)
 * complex (row = order m + L - 1, column = node); x, ch, sh (L,) float64 (nodes,
 * cos(theta/2), sin(theta/2)); per order row mi the seed of _seed_d
 * (_numba.py:191-208): seed_const[mi] = sign sqrt(C(2nn, nn+mm)) and
 * seed_ints[4 mi .. 4 mi + 2] = (ec, es, l0) (the host binding computes them
 * with the reference's lgamma/exp formula).  No plan: stateless kernels on the
 * current device; L <= 4096 (the stability gate L <= 1024 is the host
 * binding's, gl.py:98-104). */
int mwsht_gl_fm_core(const void *flm_scaled, const double *x, const double *ch, const double *sh,
                     const double *seed_const, const int *seed_ints, int L, int spin, void *F,
                     void *stream);
int mwsht_gl_flm_core(const void *a, const double *x, const double *ch, const double *sh,
                      const double *seed_const, const int *seed_ints, int L, int spin, void *R,
                      void *stream);

/* Inverse-core tiling (no reference counterpart; a scheduling choice only).
 * Paired tiles: each (m', m) chain with m' > m also produces the transposed
 * output T[m, m'] (Delta^l_{m m'} = (-1)^(m'-m) Delta^l_{m' m}), so one
 * recursion feeds two contractions.  Spin 0 only.  mode 0: plain tiles
 * everywhere; mode -1 (default): paired tiles for single spin-0 maps (batches share the
 * recursion between maps instead); mode 1: paired for every spin-0 call.  Results
 * agree to rounding (tests/test_gpu_paired.py). */
int mwsht_plan_set_paired(mwsht_plan *plan, int mode);

/* Per-call event timing of the O(L^3) core kernel (bench / roofline).  When
 * enabled, each transform records CUDA events on its stream around the FFT
 * stages and around the core kernel; last_timing synchronises on them. */
int mwsht_plan_set_timing(mwsht_plan *plan, int on);
/* inverse = 0: last forward call (stages_ms = the FFT stages, which run before
 * the core); inverse = 1: last inverse call (stages_ms = the theta and phi
 * synthesis stages, which run after it). */
int mwsht_plan_last_timing(mwsht_plan *plan, int inverse, float *core_ms, float *stages_ms);

/* DFMA throughput probe (FP64 roofline denominator): TFLOP/s reached by a
 * dependency-free FMA kernel on every SM, best of 5 ~10 ms runs. */
int mwsht_fp64_probe(int device, double *tflops, double *ms);

#ifdef __cplusplus
}
#endif
#endif /* MWSHT_H */
