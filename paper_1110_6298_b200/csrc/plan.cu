// Plan, tables and the extern "C" entry points of libmwsht.so (include/mwsht.h).
#include <cufft.h>
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mwsht.h"
#include "common.cuh"

namespace mwsht {
void launch_inverse_core(const InvArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st);
void launch_forward_core(const FwdArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st);
void launch_extend_transpose(bool real, const double2* A, double2* B, int L, int N, int spin,
                             double scale, long long as, long long bs, int nm, cudaStream_t st);
void launch_pad_twist(const double2* B, double2* C, int rows, int L, int N, int P, long long bs,
                      long long cs, int nm, cudaStream_t st);
void launch_mul_spectrum(double2* C, const double2* W, int P, long long nrows, cudaStream_t st);
void launch_fold(bool real, bool from_conv, const double2* src, double2* gfT, int L, int P,
                 int ldw, int spin, long long ss, long long gs, int nm, cudaStream_t st);
void launch_T2_to_fold(bool real, const double2* gfT, double2* gf, int L, int ldw, cudaStream_t st);
void launch_inv_prescale(bool real, const double2* in, int in_mode, const double* cl,
                         const double* A, int L, int ldw, double2* gp, long long is, long long gs,
                         int nm, cudaStream_t st);
void launch_transpose(const double2* in, double2* out, int rows, int cols, cudaStream_t st);
void launch_untranspose(bool real, const double2* S, double2* Out, int L, int N, long long ss,
                        long long os, int nm, cudaStream_t st);
void launch_reality(const double2* f, int L, unsigned long long* worst, unsigned long long* peak,
                    cudaStream_t st);
}  // namespace mwsht

using namespace mwsht;

static thread_local std::string g_last_error;

static int fail(int code, const char* what, const char* detail) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s: %s", what, detail ? detail : "");
  g_last_error = buf;
  return code;
}

#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) return fail(MWSHT_E_CUDA, #call, cudaGetErrorString(e_)); \
  } while (0)
#define FFT(call)                                                                  \
  do {                                                                             \
    cufftResult r_ = (call);                                                       \
    if (r_ != CUFFT_SUCCESS) {                                                     \
      char b_[32];                                                                 \
      snprintf(b_, sizeof b_, "cufftResult %d", (int)r_);                          \
      return fail(MWSHT_E_CUFFT, #call, b_);                                       \
    }                                                                              \
  } while (0)
#define LAUNCHED(p)                                             \
  do {                                                          \
    cudaError_t e_ = cudaGetLastError();                        \
    if (e_ != cudaSuccess) return fail(MWSHT_E_CUDA, "kernel launch", cudaGetErrorString(e_)); \
    (p)->own_launches++;                                        \
  } while (0)

enum FftKind { F_PHI_Z = 0, F_PHI_D2Z, F_PHI_Z2D, F_ROWN, F_ROWP, F_ROWP_HALF, F_WSPEC };

struct SpinTab {
  double2* rowinv = nullptr;  // [l*ldw + m'] = (kap_l C_l(m'), W_l(m'))
  double2* rowfwd = nullptr;  // [m'*ldw + l] = (alpha(l-m'+1) beta(l+m'-1), W'(l, m'))
};

struct mwsht_plan {
  int L = 0, N = 0, P = 0, device = 0, max_batch = 1;
  int ldw = 0;  // DW tables' leading dimension: L rounded up to the 64-wide tile
  DevTables tabs{};
  std::vector<void*> allocs;
  size_t bytes = 0;
  std::map<int, SpinTab> spins;
  int2 *tiles_inv = nullptr, *tiles_fwd = nullptr;
  int ntiles_inv = 0, ntiles_fwd = 0;
  double2* wspec = nullptr;
  double2 *bufA = nullptr, *bufB = nullptr, *bufC = nullptr, *bufG = nullptr;
  long long strideA = 0, strideB = 0, strideC = 0, strideG = 0;
  std::map<std::pair<int, int>, cufftHandle> ffts;
  void* fft_work = nullptr;
  size_t fft_work_size = 0;
  unsigned long long* red = nullptr;  // 2 slots for the reality check
  int own_launches = 0, cufft_launches = 0;
  bool timing = false;
  cudaEvent_t ev[2][3] = {};  // [forward|inverse][start, core start, core end]
  double* colc = nullptr;  // [l*ldw + m] = C_l(m)
  std::vector<long double> hl_A, hl_V, hl_Bt, hl_lam, hl_kap;  // host tables for the spin builds
  std::mutex mu;
};

static int dev_alloc(mwsht_plan* p, void** ptr, size_t bytes) {
  cudaError_t e = cudaMalloc(ptr, bytes ? bytes : 16);
  if (e != cudaSuccess) return fail(MWSHT_E_NOMEM, "cudaMalloc", cudaGetErrorString(e));
  p->allocs.push_back(*ptr);
  p->bytes += bytes;
  return MWSHT_OK;
}

template <typename T>
static int upload(mwsht_plan* p, T** dptr, const std::vector<T>& h) {
  int rc = dev_alloc(p, (void**)dptr, h.size() * sizeof(T));
  if (rc) return rc;
  CU(cudaMemcpy(*dptr, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return MWSHT_OK;
}

// Run f(lo, hi) over [0, n) on the host's cores (plan-time table builds).
template <typename F>
static void host_parallel(int n, F f) {
  int nt = (int)std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (nt > 32) nt = 32;
  if (n < 256) nt = 1;
  std::vector<std::thread> th;
  for (int t = 0; t < nt; t++) {
    // interleaved blocks: triangular work balances across threads
    th.emplace_back([=]() {
      for (int b = t; b * 64 < n; b += nt) f(b * 64, std::min(n, b * 64 + 64));
    });
  }
  for (auto& x : th) x.join();
}

static int smooth_len(int n) {
  // smallest 2^a 3^b 5^c 7^d >= n (cuFFT-friendly)
  for (int m = n;; m++) {
    int x = m;
    for (int q : {2, 3, 5, 7})
      while (x % q == 0) x /= q;
    if (x == 1) return m;
  }
}

// ------------------------------------------------------------- tables
static int build_tables(mwsht_plan* p) {
  typedef long double ld;
  const int L = p->L, K = 2 * L + 4;
  std::vector<ld> A(K), V(K), Bt(K), lam(L + 2), kap(L + 2);
  A[0] = A[1] = 1.0L;
  for (int k = 2; k < K; k++) A[k] = A[k - 2] * sqrtl((ld)(k - 1) / (ld)k);
  for (int k = 0; k + 1 < K; k++) V[k] = A[k] / (sqrtl((ld)(k + 1)) * A[k + 1]);
  V[K - 1] = 0;
  const int Q = 2 * L + 1;
  for (int q = K - 1; q >= Q - 1; q--) Bt[q] = 1.0L;
  for (int q = Q - 2; q >= 0; q--) Bt[q] = Bt[q + 2] * sqrtl((ld)(q + 2) / (ld)(q + 1));
  std::vector<double> hA(K), hV(K), hBt(K), hal(K, 0.0), hbe(K, 0.0), hlam(L + 2), hkap(L + 2),
      hcl(L);
  for (int k = 0; k < K; k++) {
    hA[k] = (double)A[k];
    hV[k] = (double)V[k];
    hBt[k] = (double)Bt[k];
  }
  for (int q = 1; q < K; q++) hal[q] = (double)(2.0L * A[q - 1] / (A[q] * sqrtl((ld)q)));
  for (int q = 0; q + 1 < K; q++) hbe[q] = (double)(Bt[q + 1] / (Bt[q] * sqrtl((ld)(q + 1))));
  lam[0] = lam[1] = 1.0L;
  for (int l = 1; l + 1 < L + 2; l++) lam[l + 1] = lam[l - 1] * (ld)(l + 1) / (ld)l;
  kap[0] = 0.0L;
  for (int l = 1; l + 1 < L + 2; l++) kap[l] = (ld)(2 * l + 1) * lam[l] / ((ld)l * lam[l + 1]);
  kap[L + 1] = 0;
  for (int l = 0; l < L + 2; l++) {
    hlam[l] = (double)lam[l];
    hkap[l] = (double)kap[l];
  }
  for (int l = 0; l < L; l++) hcl[l] = sqrt((2.0 * l + 1.0) / (4.0 * 3.141592653589793));

  // top-row seeds T(n, k) = sqrt(C(2n, n+k)) / 2^n, 0 <= k <= n < L
  const size_t ntri = (size_t)L * (L + 1) / 2;
  std::vector<double> smant(ntri);
  std::vector<int> sexp(ntri);
  std::vector<ld> t0sq(L);
  t0sq[0] = 1.0L;
  for (int j = 1; j < L; j++) t0sq[j] = t0sq[j - 1] * (ld)(2 * j - 1) / (ld)(2 * j);
  host_parallel(L, [&](int lo, int hi) {
    for (int n = lo; n < hi; n++) {
      ld P = t0sq[n];
      const size_t base = (size_t)n * (n + 1) / 2;
      for (int k = 0; k <= n; k++) {
        int e;
        ld f = frexpl(sqrtl(P), &e);
        smant[base + k] = (double)f;
        sexp[base + k] = e;
        if (k < n) P = P * (ld)(n - k) / (ld)(n + k + 1);
      }
    }
  });
  int rc;
  DevTables& T = p->tabs;
  T.L = L;
  T.N = 2 * L - 1;
  double* d;
  if ((rc = upload(p, &d, hA))) return rc;
  T.A = d;
  if ((rc = upload(p, &d, hV))) return rc;
  T.V = d;
  if ((rc = upload(p, &d, hBt))) return rc;
  T.Bt = d;
  if ((rc = upload(p, &d, hal))) return rc;
  T.alpha = d;
  if ((rc = upload(p, &d, hbe))) return rc;
  T.beta = d;
  if ((rc = upload(p, &d, hlam))) return rc;
  T.lam = d;
  if ((rc = upload(p, &d, hkap))) return rc;
  T.kap = d;
  if ((rc = upload(p, &d, hcl))) return rc;
  T.cl = d;
  if ((rc = upload(p, &d, smant))) return rc;
  T.seed_mant = d;
  int* di;
  if ((rc = upload(p, &di, sexp))) return rc;
  T.seed_exp = di;
  p->hl_A = A;
  p->hl_V = V;
  p->hl_Bt = Bt;
  p->hl_lam = lam;
  p->hl_kap = kap;
  // C_l(m) = m V(l-m) V(l+m) for m <= l (column factor of the l-recursion)
  const int Lp = p->ldw;
  std::vector<double> colc((size_t)L * Lp, 0.0);
  host_parallel(L, [&](int lo, int hi) {
    for (int l = lo; l < hi; l++)
      for (int m = 0; m <= l; m++) colc[(size_t)l * Lp + m] = (double)((ld)m * V[l - m] * V[l + m]);
  });
  if ((rc = upload(p, &p->colc, colc))) return rc;
  return MWSHT_OK;
}

// Per-spin plan tables.  The spin column Delta^l_{x,-s}, x <= l, comes from
// the Trapani column recursion (_numba.py:63-71) run in 80-bit long double
// (whose exponent range removes the reference's float64 overflow), and is
// packed with the recursion coefficients each core reads per step:
//   rowinv[l*ldw + x] = (kap_l C_l(x),               (-1)^l lam_l u_l(x) Delta^l_{x,-s})
//   rowfwd[x*ldw + l] = (alpha(l-x+1) beta(l+x-1),   A(l-x) Bt(l+x) Delta^l_{x,-s})
// with C_l(x) = x V(l-x) V(l+x), u_l(x) = A(l-x) A(l+x)  (common.cuh).
static int build_spin(mwsht_plan* p, int spin) {
  if (p->spins.count(spin)) return MWSHT_OK;
  typedef long double ld;
  const int L = p->L, cs = spin < 0 ? -spin : spin;
  const int Lp = p->ldw;
  std::vector<double2> inv((size_t)L * Lp, make_double2(0.0, 0.0)), fwd(inv);
  std::vector<ld> sq(2 * L + 4);
  for (size_t i = 0; i < sq.size(); i++) sq[i] = sqrtl((ld)i);
  std::vector<ld> t0sq(L);
  t0sq[0] = 1.0L;
  for (int j = 1; j < L; j++) t0sq[j] = t0sq[j - 1] * (ld)(2 * j - 1) / (ld)(2 * j);
  const std::vector<ld>&A = p->hl_A, &V = p->hl_V, &Bt = p->hl_Bt, &lam = p->hl_lam,
                      &kap = p->hl_kap;
  host_parallel(L, [&](int lo, int hi) {
    std::vector<ld> col(L + 2);
    for (int l = lo; l < hi; l++) {
      const bool has = l >= cs;
      if (has) {
        // seed Delta^l_{l,cs} = (-1)^(l-cs) sqrt(C(2l, l+cs))/2^l
        ld P = t0sq[l];
        for (int k = 0; k < cs; k++) P = P * (ld)(l - k) / (ld)(l + k + 1);
        col[l + 1] = 0.0L;
        col[l] = ((l - cs) & 1 ? -1.0L : 1.0L) * sqrtl(P);
        for (int mu = l - 1; mu >= 0; mu--) {
          const ld inv_ = 1.0L / (sq[l + mu + 1] * sq[l - mu]);
          const ld c2 = (mu + 2 <= l) ? sq[l - mu - 1] * sq[l + mu + 2] : 0.0L;
          col[mu] = (2.0L * cs * col[mu + 1] - c2 * col[mu + 2]) * inv_;
        }
      }
      for (int x = 0; x <= l; x++) {
        ld dv = has ? col[x] : 0.0L;
        if (spin > 0 && ((l + x) & 1)) dv = -dv;  // Delta_{x,-s} = (-1)^(l+x) Delta_{x,s}
        ld wi = lam[l] * A[l - x] * A[l + x] * dv;
        if (l & 1) wi = -wi;
        const ld cx = kap[l] * (ld)x * V[l - x] * V[l + x];
        inv[(size_t)l * Lp + x] = make_double2((double)cx, (double)wi);
        ld qn = 0.0L;
        if (x >= 1) {
          const int pp = l - x + 1, qq = l + x - 1;
          qn = (2.0L * A[pp - 1] / (A[pp] * sq[pp])) * (Bt[qq + 1] / (Bt[qq] * sq[qq + 1]));
        }
        fwd[(size_t)x * Lp + l] = make_double2((double)qn, (double)(A[l - x] * Bt[l + x] * dv));
      }
    }
  });
  SpinTab st;
  int rc;
  if ((rc = upload(p, &st.rowinv, inv))) return rc;
  if ((rc = upload(p, &st.rowfwd, fwd))) return rc;
  p->spins[spin] = st;
  return MWSHT_OK;
}

static int build_tiles(mwsht_plan* p) {
  const int L = p->L;
  struct Tl {
    int2 t;
    long long w;
  };
  std::vector<Tl> inv, fwd;
  for (int r0 = 0; r0 < L; r0 += kTileRows)
    for (int c0 = 0; c0 < L; c0 += kTileCols)
      inv.push_back({make_int2(r0, c0), (long long)(L - std::max(r0, c0))});
  for (int l0 = 0; l0 < L; l0 += kTileRows) {
    const int top = std::min(l0 + kTileRows - 1, L - 1);
    for (int c0 = 0; c0 <= top; c0 += kTileCols) fwd.push_back({make_int2(l0, c0), (long long)top + 1});
  }
  auto by_work = [](const Tl& a, const Tl& b) { return a.w > b.w; };
  std::stable_sort(inv.begin(), inv.end(), by_work);
  std::stable_sort(fwd.begin(), fwd.end(), by_work);
  std::vector<int2> hi, hf;
  for (auto& x : inv) hi.push_back(x.t);
  for (auto& x : fwd) hf.push_back(x.t);
  int rc;
  if ((rc = upload(p, &p->tiles_inv, hi))) return rc;
  if ((rc = upload(p, &p->tiles_fwd, hf))) return rc;
  p->ntiles_inv = (int)hi.size();
  p->ntiles_fwd = (int)hf.size();
  return MWSHT_OK;
}

// cuFFT plan cache keyed by (kind, nmaps); all plans share one work area.
static int get_fft(mwsht_plan* p, int kind, int nm, cufftHandle* out) {
  auto key = std::make_pair(kind, nm);
  auto it = p->ffts.find(key);
  if (it != p->ffts.end()) {
    *out = it->second;
    return MWSHT_OK;
  }
  const int L = p->L, N = p->N, P = p->P;
  cufftHandle h;
  FFT(cufftCreate(&h));
  FFT(cufftSetAutoAllocation(h, 0));
  size_t ws = 0;
  int n1[1];
  switch (kind) {
    case F_PHI_Z:
      n1[0] = N;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, N, nullptr, 1, N, CUFFT_Z2Z, L * nm, &ws));
      break;
    case F_PHI_D2Z:
      n1[0] = N;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, N, nullptr, 1, L, CUFFT_D2Z, L * nm, &ws));
      break;
    case F_PHI_Z2D:
      n1[0] = N;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, L, nullptr, 1, N, CUFFT_Z2D, L * nm, &ws));
      break;
    case F_ROWN:
      n1[0] = N;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, N, nullptr, 1, N, CUFFT_Z2Z, N * nm, &ws));
      break;
    case F_ROWP:
      n1[0] = P;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, P, nullptr, 1, P, CUFFT_Z2Z, N * nm, &ws));
      break;
    case F_ROWP_HALF:
      n1[0] = P;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, P, nullptr, 1, P, CUFFT_Z2Z, L * nm, &ws));
      break;
    case F_WSPEC:
      n1[0] = P;
      FFT(cufftMakePlanMany(h, 1, n1, nullptr, 1, P, nullptr, 1, P, CUFFT_Z2Z, 1, &ws));
      break;
  }
  if (ws > p->fft_work_size) {
    if (p->fft_work) {
      CU(cudaDeviceSynchronize());
      auto itp = std::find(p->allocs.begin(), p->allocs.end(), p->fft_work);
      if (itp != p->allocs.end()) p->allocs.erase(itp);
      cudaFree(p->fft_work);
      p->bytes -= p->fft_work_size;
      p->fft_work = nullptr;
    }
    int rc = dev_alloc(p, &p->fft_work, ws);
    if (rc) return rc;
    p->fft_work_size = ws;
    for (auto& kv : p->ffts) FFT(cufftSetWorkArea(kv.second, p->fft_work));
  }
  FFT(cufftSetWorkArea(h, p->fft_work));
  p->ffts[key] = h;
  *out = h;
  return MWSHT_OK;
}

static int build_wspec(mwsht_plan* p) {
  const int L = p->L, P = p->P;
  std::vector<double2> w(P, make_double2(0.0, 0.0));
  // w_rev[i] = w(2L-2-i), i < 4L-3 (mw.py:237, quadrature.py:66-74)
  for (int i = 0; i < 4 * L - 3; i++) {
    const long long k = 2LL * L - 2 - i;
    double2 v = make_double2(0.0, 0.0);
    if (k == 1)
      v.y = 0.5 * 3.141592653589793;
    else if (k == -1)
      v.y = -0.5 * 3.141592653589793;
    else if ((k & 1) == 0)
      v.x = 2.0 / (1.0 - (double)k * (double)k);
    w[i] = v;
  }
  int rc;
  if ((rc = upload(p, &p->wspec, w))) return rc;
  cufftHandle h;
  if ((rc = get_fft(p, F_WSPEC, 1, &h))) return rc;
  FFT(cufftExecZ2Z(h, (cufftDoubleComplex*)p->wspec, (cufftDoubleComplex*)p->wspec, CUFFT_FORWARD));
  CU(cudaDeviceSynchronize());
  std::vector<double2> hw(P);
  CU(cudaMemcpy(hw.data(), p->wspec, P * sizeof(double2), cudaMemcpyDeviceToHost));
  const double sc = 2.0 * 3.141592653589793 / (double)P;  // 2pi (mw.py:238) and the 1/P of the inverse FFT
  for (auto& v : hw) v = make_double2(v.x * sc, v.y * sc);
  CU(cudaMemcpy(p->wspec, hw.data(), P * sizeof(double2), cudaMemcpyHostToDevice));
  return MWSHT_OK;
}

static int check_plan(mwsht_plan* p) {
  if (!p) return fail(MWSHT_E_PLAN, "plan", "null plan");
  CU(cudaSetDevice(p->device));
  return MWSHT_OK;
}

static int check_rec(int recursion) {
  if (recursion != MWSHT_TRAPANI && recursion != MWSHT_RISBO)
    return fail(MWSHT_E_VALUE, "recursion", "must be trapani (0) or risbo (1)");
  return MWSHT_OK;
}

static int check_spin(mwsht_plan* p, int spin) {
  if ((spin < 0 ? -spin : spin) >= p->L)
    return fail(MWSHT_E_SPIN, "spin", "|spin| must be below the band limit");
  return MWSHT_OK;
}

// ------------------------------------------------------------ pipelines
static InvArgs inv_args(mwsht_plan* p, int spin) {
  InvArgs a{};
  a.t = p->tabs;
  a.rowtab = p->spins[spin].rowinv;
  a.colc = p->colc;
  a.gp = p->bufG;
  a.g_stride = p->strideG;
  a.tiles = p->tiles_inv;
  a.spin = spin;
  a.ldw = p->ldw;
  return a;
}

static FwdArgs fwd_args(mwsht_plan* p, int spin) {
  FwdArgs a{};
  a.t = p->tabs;
  a.rowtab = p->spins[spin].rowfwd;
  a.gf = p->bufG;
  a.in_stride = p->strideG;
  a.tiles = p->tiles_fwd;
  a.spin = spin;
  a.ldw = p->ldw;
  return a;
}

// samples (L,N) -> folded plane in the forward core's staging layout (bufG)
static int forward_stages(mwsht_plan* p, int nm, const void* samples, bool real, int spin,
                          cudaStream_t st) {
  const int L = p->L, N = p->N, P = p->P;
  cufftHandle hphi, hrow, hconv;
  int rc;
  if ((rc = get_fft(p, real ? F_PHI_D2Z : F_PHI_Z, nm, &hphi))) return rc;
  if ((rc = get_fft(p, real ? F_PHI_Z : F_ROWN, nm, &hrow))) return rc;
  if ((rc = get_fft(p, real ? F_ROWP_HALF : F_ROWP, nm, &hconv))) return rc;
  FFT(cufftSetStream(hphi, st));
  FFT(cufftSetStream(hrow, st));
  FFT(cufftSetStream(hconv, st));
  const int rows = real ? L : N;
  // 1. phi FFT (mw.py:149-158 / :489)
  if (real)
    FFT(cufftExecD2Z(hphi, (cufftDoubleReal*)samples, (cufftDoubleComplex*)p->bufA));
  else
    FFT(cufftExecZ2Z(hphi, (cufftDoubleComplex*)samples, (cufftDoubleComplex*)p->bufA,
                     CUFFT_FORWARD));
  p->cufft_launches++;
  // 2. periodic extension + transpose + 2pi/N (mw.py:161-177)
  const long long sA = real ? (long long)L * L : (long long)L * N;
  launch_extend_transpose(real, p->bufA, p->bufB, L, N, spin, 2.0 * 3.141592653589793 / N, sA,
                          (long long)rows * N, nm, st);
  LAUNCHED(p);
  // 3. theta FFT over t (mw.py:190)
  FFT(cufftExecZ2Z(hrow, (cufftDoubleComplex*)p->bufB, (cufftDoubleComplex*)p->bufB, CUFFT_FORWARD));
  p->cufft_launches++;
  // 4. twist + scale + zero pad to P (mw.py:191, 250)
  launch_pad_twist(p->bufB, p->bufC, rows, L, N, P, (long long)rows * N, (long long)rows * P, nm,
                   st);
  LAUNCHED(p);
  // 5. correlation with w by FFT at P >= 4L-3 (mw.py:244-251)
  FFT(cufftExecZ2Z(hconv, (cufftDoubleComplex*)p->bufC, (cufftDoubleComplex*)p->bufC, CUFFT_FORWARD));
  p->cufft_launches++;
  launch_mul_spectrum(p->bufC, p->wspec, P, (long long)rows * nm, st);
  LAUNCHED(p);
  FFT(cufftExecZ2Z(hconv, (cufftDoubleComplex*)p->bufC, (cufftDoubleComplex*)p->bufC, CUFFT_INVERSE));
  p->cufft_launches++;
  // 6. extract + m' fold into the core's layout (mw.py:251, 273-285)
  launch_fold(real, true, p->bufC, p->bufG, L, P, p->ldw, spin, (long long)rows * P, p->strideG,
              nm, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

static int do_forward(mwsht_plan* p, int nm, const void* samples, void* flm, int spin, bool real,
                      int recursion, void* stream) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  if ((rc = check_rec(recursion))) return rc;
  if ((rc = check_spin(p, spin))) return rc;
  if (real && spin != 0) return fail(MWSHT_E_SPIN, "forward_real", "spin 0 only");
  if (nm < 1 || nm > p->max_batch) return fail(MWSHT_E_CONTRACT, "nmaps", "exceeds plan max_batch");
  std::lock_guard<std::mutex> lk(p->mu);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int L = p->L;
  if (p->timing) CU(cudaEventRecord(p->ev[0][0], st));
  if ((rc = forward_stages(p, nm, samples, real, spin, st))) return rc;
  if (p->timing) CU(cudaEventRecord(p->ev[0][1], st));
  FwdArgs a = fwd_args(p, spin);
  a.out = (double2*)flm;
  a.out_mode = 0;
  a.out_stride = (long long)L * L;
  launch_forward_core(a, p->ntiles_fwd, nm, real, st);
  LAUNCHED(p);
  if (p->timing) CU(cudaEventRecord(p->ev[0][2], st));
  return MWSHT_OK;
}

static int do_inverse(mwsht_plan* p, int nm, const void* flm, void* samples, int spin, bool real,
                      int recursion, void* stream) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  if ((rc = check_rec(recursion))) return rc;
  if ((rc = check_spin(p, spin))) return rc;
  if (real && spin != 0) return fail(MWSHT_E_SPIN, "inverse_real", "spin 0 only");
  if (nm < 1 || nm > p->max_batch) return fail(MWSHT_E_CONTRACT, "nmaps", "exceeds plan max_batch");
  std::lock_guard<std::mutex> lk(p->mu);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int L = p->L, N = p->N;
  const int rows = real ? L : N;
  cufftHandle hrow, hphi;
  if ((rc = get_fft(p, real ? F_PHI_Z : F_ROWN, nm, &hrow))) return rc;
  if ((rc = get_fft(p, real ? F_PHI_Z2D : F_PHI_Z, nm, &hphi))) return rc;
  FFT(cufftSetStream(hrow, st));
  FFT(cufftSetStream(hphi, st));
  if (p->timing) CU(cudaEventRecord(p->ev[1][0], st));
  // 0. unflatten + c_l u_l(m) scaling into the core's staging rows (mw.py:390-392)
  launch_inv_prescale(real, (const double2*)flm, 0, p->tabs.cl, p->tabs.A, L, p->ldw, p->bufG,
                      (long long)L * L, p->strideG, nm, st);
  LAUNCHED(p);
  // 1. core + phases + m' mirror + theta twist (mw.py:378-402, 445)
  if (p->timing) CU(cudaEventRecord(p->ev[1][1], st));
  InvArgs a = inv_args(p, spin);
  a.out = p->bufB;
  a.out_mode = 0;
  a.out_stride = (long long)rows * N;
  launch_inverse_core(a, p->ntiles_inv, nm, real, st);
  LAUNCHED(p);
  if (p->timing) CU(cudaEventRecord(p->ev[1][2], st));
  // 2. theta synthesis (mw.py:446), unnormalised inverse FFT over m'
  FFT(cufftExecZ2Z(hrow, (cufftDoubleComplex*)p->bufB, (cufftDoubleComplex*)p->bufB, CUFFT_INVERSE));
  p->cufft_launches++;
  // 3. keep t < L, transpose to rings, ifftshift over m (mw.py:436-437)
  const long long sA = real ? (long long)L * L : (long long)L * N;
  launch_untranspose(real, p->bufB, p->bufA, L, N, (long long)rows * N, sA, nm, st);
  LAUNCHED(p);
  // 4. phi synthesis (mw.py:437-438 / 558)
  if (real)
    FFT(cufftExecZ2D(hphi, (cufftDoubleComplex*)p->bufA, (cufftDoubleReal*)samples));
  else
    FFT(cufftExecZ2Z(hphi, (cufftDoubleComplex*)p->bufA, (cufftDoubleComplex*)samples,
                     CUFFT_INVERSE));
  p->cufft_launches++;
  return MWSHT_OK;
}

// ================================================================ C ABI
extern "C" {

const char* mwsht_version(void) { return "mwsht-b200 0.1 (sm_100a, fp64)"; }

const char* mwsht_status_string(int s) {
  switch (s) {
    case MWSHT_OK: return "ok";
    case MWSHT_E_BAND_LIMIT: return "invalid band limit";
    case MWSHT_E_SPIN: return "invalid spin";
    case MWSHT_E_CONTRACT: return "contract violation";
    case MWSHT_E_SYMMETRY: return "symmetry violation";
    case MWSHT_E_VALUE: return "invalid value";
    case MWSHT_E_CUDA: return "CUDA error";
    case MWSHT_E_CUFFT: return "cuFFT error";
    case MWSHT_E_NOMEM: return "out of memory";
    case MWSHT_E_PLAN: return "invalid plan";
  }
  return "unknown";
}

const char* mwsht_last_error(void) { return g_last_error.c_str(); }

int mwsht_plan_create(int L, int device, int max_batch, mwsht_plan** out) {
  if (!out) return fail(MWSHT_E_PLAN, "plan_create", "null out");
  *out = nullptr;
  if (L < 1) return fail(MWSHT_E_BAND_LIMIT, "plan_create", "band limit must be >= 1");
  if (max_batch < 1) max_batch = 1;
  if (LDBL_MANT_DIG < 64) return fail(MWSHT_E_VALUE, "plan_create", "needs 80-bit long double");
  mwsht_plan* p = new mwsht_plan();
  int rc;
  if (device < 0) {
    cudaError_t e = cudaGetDevice(&device);
    if (e != cudaSuccess) {
      delete p;
      return fail(MWSHT_E_CUDA, "cudaGetDevice", cudaGetErrorString(e));
    }
  }
  p->L = L;
  p->N = 2 * L - 1;
  p->P = smooth_len(4 * L - 3);
  p->ldw = (L + kTileRows - 1) / kTileRows * kTileRows;
  p->device = device;
  p->max_batch = max_batch;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete p;
    return fail(MWSHT_E_CUDA, "cudaSetDevice", cudaGetErrorString(e));
  }
  const long long L_ = L, N = p->N, P = p->P;
  p->strideA = L_ * N;
  p->strideB = N * N;
  p->strideC = N * P;
  p->strideG = 2 * L_ * p->ldw;
  if ((rc = build_tables(p)) || (rc = build_tiles(p)) ||
      (rc = dev_alloc(p, (void**)&p->bufA, sizeof(double2) * p->strideA * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->bufB, sizeof(double2) * p->strideB * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->bufC, sizeof(double2) * p->strideC * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->bufG, sizeof(double2) * p->strideG * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->red, 2 * sizeof(unsigned long long))) ||
      (rc = build_wspec(p)) || (rc = build_spin(p, 0))) {
    mwsht_plan_destroy(p);
    return rc;
  }
  *out = p;
  return MWSHT_OK;
}

int mwsht_plan_destroy(mwsht_plan* p) {
  if (!p) return MWSHT_OK;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (auto& kv : p->ffts) cufftDestroy(kv.second);
  for (auto& d : p->ev)
    for (auto& e : d)
      if (e) cudaEventDestroy(e);
  for (void* q : p->allocs) cudaFree(q);
  delete p;
  return MWSHT_OK;
}

size_t mwsht_plan_device_bytes(const mwsht_plan* p) { return p ? p->bytes : 0; }

int mwsht_plan_prepare_spin(mwsht_plan* p, int spin) {
  int rc;
  if ((rc = check_plan(p)) || (rc = check_spin(p, spin))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  return build_spin(p, spin);
}

int mwsht_forward_z(mwsht_plan* p, const void* samples, void* flm, int spin, int recursion,
                    void* stream) {
  return do_forward(p, 1, samples, flm, spin, false, recursion, stream);
}

int mwsht_inverse_z(mwsht_plan* p, const void* flm, void* samples, int spin, int recursion,
                    void* stream) {
  return do_inverse(p, 1, flm, samples, spin, false, recursion, stream);
}

int mwsht_forward_real_d(mwsht_plan* p, const double* samples, void* flm, int recursion,
                         void* stream) {
  return do_forward(p, 1, samples, flm, 0, true, recursion, stream);
}

int mwsht_inverse_real_d(mwsht_plan* p, const void* flm, double* samples, int recursion,
                         void* stream) {
  return do_inverse(p, 1, flm, samples, 0, true, recursion, stream);
}

int mwsht_forward_z_batch(mwsht_plan* p, int nmaps, const void* samples, void* flm, int spin,
                          int recursion, void* stream) {
  return do_forward(p, nmaps, samples, flm, spin, false, recursion, stream);
}

int mwsht_inverse_z_batch(mwsht_plan* p, int nmaps, const void* flm, void* samples, int spin,
                          int recursion, void* stream) {
  return do_inverse(p, nmaps, flm, samples, spin, false, recursion, stream);
}

int mwsht_reality_residual(mwsht_plan* p, const void* flm, double* worst_host, double* tol_host,
                           void* stream) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemsetAsync(p->red, 0, 2 * sizeof(unsigned long long), st));
  launch_reality((const double2*)flm, p->L, p->red, p->red + 1, st);
  LAUNCHED(p);
  unsigned long long h[2];
  CU(cudaMemcpyAsync(h, p->red, sizeof h, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  double w, pk;
  memcpy(&w, &h[0], 8);
  memcpy(&pk, &h[1], 8);
  if (worst_host) *worst_host = w;
  if (tol_host) *tol_host = 1e-12 * (pk > 1.0 ? pk : 1.0);
  return MWSHT_OK;
}

int mwsht_fmm_core(mwsht_plan* p, const void* flm2d, const double* cl, int spin, int use_trapani,
                   void* T, void* stream) {
  int rc;
  if ((rc = check_plan(p)) || (rc = check_spin(p, spin))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_inv_prescale(false, (const double2*)flm2d, 1, cl, p->tabs.A, p->L, p->ldw, p->bufG, 0,
                      p->strideG, 1, st);
  LAUNCHED(p);
  InvArgs a = inv_args(p, spin);
  a.out = (double2*)T;
  a.out_mode = 1;
  launch_inverse_core(a, p->ntiles_inv, 1, false, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_fmm_core_real(mwsht_plan* p, const void* flm_half, const double* cl, int use_trapani,
                        void* T, void* stream) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_inv_prescale(true, (const double2*)flm_half, 1, cl, p->tabs.A, p->L, p->ldw, p->bufG, 0,
                      p->strideG, 1, st);
  LAUNCHED(p);
  InvArgs a = inv_args(p, 0);
  a.out = (double2*)T;
  a.out_mode = 1;
  launch_inverse_core(a, p->ntiles_inv, 1, true, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_flm_core(mwsht_plan* p, const void* gfold, int spin, int use_trapani, void* R,
                   void* stream) {
  int rc;
  if ((rc = check_plan(p)) || (rc = check_spin(p, spin))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_fold(false, false, (const double2*)gfold, p->bufG, p->L, p->P, p->ldw, spin, 0,
              p->strideG, 1, st);
  LAUNCHED(p);
  FwdArgs a = fwd_args(p, spin);
  a.out = (double2*)R;
  a.out_mode = 1;
  // entries |m| > l stay zero, as in the reference's np.zeros output
  CU(cudaMemsetAsync(R, 0, sizeof(double2) * (size_t)p->L * p->N, st));
  launch_forward_core(a, p->ntiles_fwd, 1, false, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_flm_core_real(mwsht_plan* p, const void* gfold, int use_trapani, void* R, void* stream) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  p->own_launches = p->cufft_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_fold(true, false, (const double2*)gfold, p->bufG, p->L, p->P, p->ldw, 0, 0, p->strideG,
              1, st);
  LAUNCHED(p);
  FwdArgs a = fwd_args(p, 0);
  a.out = (double2*)R;
  a.out_mode = 1;
  CU(cudaMemsetAsync(R, 0, sizeof(double2) * (size_t)p->L * p->L, st));
  launch_forward_core(a, p->ntiles_fwd, 1, true, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_forward_stages_z(mwsht_plan* p, const void* samples, void* gfold, int spin,
                           void* stream) {
  int rc;
  if ((rc = check_plan(p)) || (rc = check_spin(p, spin))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  p->own_launches = p->cufft_launches = 0;
  if ((rc = forward_stages(p, 1, samples, false, spin, (cudaStream_t)stream))) return rc;
  launch_T2_to_fold(false, p->bufG, (double2*)gfold, p->L, p->ldw, (cudaStream_t)stream);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_plan_set_timing(mwsht_plan* p, int on) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  for (auto& d : p->ev)
    for (auto& e : d)
      if (!e) CU(cudaEventCreate(&e));
  p->timing = on != 0;
  return MWSHT_OK;
}

int mwsht_plan_last_timing(mwsht_plan* p, int inverse, float* core_ms, float* stages_ms) {
  int rc;
  if ((rc = check_plan(p))) return rc;
  if (!p->timing) return fail(MWSHT_E_VALUE, "last_timing", "timing not enabled");
  cudaEvent_t* e = p->ev[inverse ? 1 : 0];
  CU(cudaEventSynchronize(e[2]));
  float c = 0.f, s0 = 0.f;
  CU(cudaEventElapsedTime(&c, e[1], e[2]));
  CU(cudaEventElapsedTime(&s0, e[0], e[1]));
  if (core_ms) *core_ms = c;
  if (stages_ms) *stages_ms = s0;
  return MWSHT_OK;
}

int mwsht_plan_last_launches(const mwsht_plan* p, int* own, int* cufft) {
  if (!p) return MWSHT_E_PLAN;
  if (own) *own = p->own_launches;
  if (cufft) *cufft = p->cufft_launches;
  return MWSHT_OK;
}

}  // extern "C"
