// Plan, tables and the extern "C" entry points of libmwsht.so (include/mwsht.h).
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <functional>
#include <map>
#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mwsht.h"
#include "common.cuh"

namespace mwsht {
void launch_inverse_core(const InvArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st);
void launch_forward_core(const FwdArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st);
int small_inverse_limit();
int small_forward_limit();
void launch_inverse_small(const InvArgs& a, int nmaps, bool real, cudaStream_t st);
void launch_forward_small(const FwdArgs& a, int nmaps, bool real, cudaStream_t st);
void launch_fold(bool real, const double2* gf, double2* gfT, int L, int ldw, cudaStream_t st);
void launch_T2_to_fold(bool real, const double2* gfT, double2* gf, int L, int ldw, cudaStream_t st);
void launch_inv_prescale(bool real, const double2* in, int in_mode, const double* cl,
                         const double* A, int L, int ldw, double2* gp, long long is, long long gs,
                         int nm, cudaStream_t st, int c0 = 0, int c1 = -1);
void launch_flm_unpack(const double2* gathered, long long maxlen, const int* bounds, int world,
                       int L, double2* flm, cudaStream_t st);
void launch_extract_y(const double2* src, double* dst, long long n, cudaStream_t st);
cudaError_t launch_gl(bool forward, const double2* in, const double* x, const double* ch,
              const double* sh, const double* cst, const int4* seed, int L, int spin,
              double2* out, cudaStream_t st);
void launch_reality(const double2* f, int L, unsigned long long* red, unsigned long long* host,
                    cudaStream_t st);
void fft_launch(int which, bool real, const fft::FftArgs& a, int nsm, cudaStream_t st);
void fft_spectrum(const fft::FftArgs& a, const double2* kern, double2* spec, cudaStream_t st);
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
#define LAUNCHED(p)                                             \
  do {                                                          \
    cudaError_t e_ = cudaGetLastError();                        \
    if (e_ != cudaSuccess) return fail(MWSHT_E_CUDA, "kernel launch", cudaGetErrorString(e_)); \
    (p)->own_launches++;                                        \
  } while (0)


struct SpinTab {
  double2* rowinv = nullptr;  // [blk64(l, m')] = (kap_l C_l(m'), W_l(m'))
  double2* rowfwd = nullptr;  // [blk64(m', l)] = (alpha(l-m'+1) beta(l+m'-1), W'(l, m'))
  double* wcol = nullptr;     // [blk32(l, x)] = W_l(x) (paired inverse tiles)
  double* wrow = nullptr;     // [blk64(l, m')] = W_l(m')    (multi-spin batches, built lazily)
  double* wrowf = nullptr;    // [blk64(m', l)] = W'(l, m')  (multi-spin batches, built lazily)
};

struct mwsht_plan {
  int L = 0, N = 0, device = 0, max_batch = 1;
  int ldw = 0;  // DW tables' leading dimension: L rounded up to the 64-wide tile
  DevTables tabs{};
  std::vector<void*> allocs;
  size_t bytes = 0;
  std::map<int, SpinTab> spins;
  int2 *tiles_inv = nullptr, *tiles_fwd = nullptr, *tiles_invp = nullptr;
  int ntiles_inv = 0, ntiles_fwd = 0, ntiles_invp = 0;
  int paired_mode = -1;  // inverse core: -1 auto (paired tiles for spin 0), 0 off, 1 on
  struct TileSet {
    int2 *inv = nullptr, *fwd = nullptr;
    int ninv = 0, nfwd = 0;
  };
  std::map<std::pair<int, int>, TileSet> range_tiles;  // tiles with c0 in [m0, m1)
  // fused FFT engine (fft.cu): M-point FFT-convolutions in H = M/2 smem halves
  int M = 0, H = 0, logH = 0, nsm = 0, Q = 2;  // convolution length M = Q H
  double2* twM = nullptr;                      // Q = 4: quarter table of w_M
  double2 *tw = nullptr, *chirp = nullptr, *specf = nullptr, *speci = nullptr, *specw = nullptr,
          *sep1 = nullptr, *sep2 = nullptr, *sep3 = nullptr, *scratch = nullptr, *cen = nullptr, *wnk = nullptr, *rho2 = nullptr;
  double2 *bufA = nullptr, *bufB = nullptr, *bufG = nullptr;
  long long strideA = 0, strideB = 0, strideG = 0;
  unsigned long long* red = nullptr;       // 2 device slots for the reality check (kept zero)
  unsigned long long* red_host = nullptr;  // host-mapped result of the reality check
  unsigned long long* red_host_dev = nullptr;
  int own_launches = 0;
  bool timing = false;
  cudaEvent_t ev[2][4] = {};  // [forward|inverse][start, core start, core end, end]
  double* colc = nullptr;  // [blk32(l, m)] = C_l(m)
  std::vector<long double> hl_A, hl_V, hl_Bt, hl_lam, hl_kap;  // host tables for the spin builds
  std::mutex mu;
  // Stream hand-off of the plan's scratch (bufA/B/G, FFT scratch, reality
  // slots): every call records `handoff` on its stream when it has enqueued
  // its work, and a call on a different stream first waits on it, so callers
  // on several streams/threads serialise on the device instead of racing on
  // the scratch (reentrancy; cli.py:205-207 thread pool).
  cudaEvent_t handoff = nullptr;
  cudaStream_t last_st = nullptr;
  bool has_last = false;
  bool capturing = false;  // inside an internal graph capture: no hand-off
};

// Restores the caller's current device on return from every entry point.
struct DevGuard {
  int prev = -1;
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Orders this call after the previous user of the plan's scratch (see
// mwsht_plan::handoff).  Caller holds p->mu.
struct StreamUse {
  mwsht_plan* p;
  cudaStream_t st;
  StreamUse(mwsht_plan* p_, cudaStream_t s) : p(p_), st(s) {
    if (p->handoff && !p->capturing && p->has_last && p->last_st != st)
      cudaStreamWaitEvent(st, p->handoff, 0);
  }
  ~StreamUse() {
    if (p->handoff && !p->capturing) {
      cudaEventRecord(p->handoff, st);
      p->last_st = st;
      p->has_last = true;
    }
  }
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

  // chain-seed factors (common.cuh DevTables): values as (long double mantissa,
  // exponent) pairs renormalised every step, rounded once to (double, exponent)
  struct XL {
    ld m;
    long e;
  };
  auto norm = [](XL x) {
    int e;
    x.m = frexpl(x.m, &e);
    x.e += e;
    return x;
  };
  auto mul = [&](XL a, XL b) { return norm(XL{a.m * b.m, a.e + b.e}); };
  auto inv = [&](XL a) { return norm(XL{1.0L / a.m, -a.e}); };
  auto dev = [](XL x) { return make_double2((double)x.m, (double)x.e); };
  const int J = 2 * L + 2;
  std::vector<XL> R(J);
  R[0] = XL{0.5L, 1};
  for (int j = 1; j < J; j++) R[j] = norm(XL{R[j - 1].m / sqrtl((ld)j), R[j - 1].e});
  std::vector<double2> hpi(L), hqi(J), hpf(L), hr(J);
  for (int j = 0; j < J; j++) {
    hr[j] = dev(R[j]);
    hqi[j] = dev(mul(R[j], inv(norm(XL{A[j], 0}))));
  }
  for (int n = 0; n < L; n++) {
    const XL P0 = inv(norm(XL{R[2 * n].m, R[2 * n].e + n}));  // sqrt((2n)!) / 2^n
    hpi[n] = dev(mul(P0, inv(norm(XL{lam[n] * A[2 * n], 0}))));
    hpf[n] = dev(mul(P0, inv(norm(XL{Bt[2 * n], 0}))));
  }
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
  double2* d2;
  if ((rc = upload(p, &d2, hpi))) return rc;
  T.sd_pi = d2;
  if ((rc = upload(p, &d2, hqi))) return rc;
  T.sd_qi = d2;
  if ((rc = upload(p, &d2, hpf))) return rc;
  T.sd_pf = d2;
  if ((rc = upload(p, &d2, hr))) return rc;
  T.sd_r = d2;
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
      for (int m = 0; m <= l; m++)
        colc[blk<kTileCols>(l, m, L)] = (double)((ld)m * V[l - m] * V[l + m]);
  });
  if ((rc = upload(p, &p->colc, colc))) return rc;
  return MWSHT_OK;
}

// Per-spin plan tables.  The spin column Delta^l_{x,-s}, x <= l, comes from
// the Trapani column recursion (_numba.py:63-71) run in 80-bit long double
// (whose exponent range removes the reference's float64 overflow), and is
// packed with the recursion coefficients each core reads per step:
//   rowinv[blk64(l, x)] = (kap_l C_l(x),             (-1)^l lam_l u_l(x) Delta^l_{x,-s})
//   rowfwd[blk64(x, l)] = (alpha(l-x+1) beta(l+x-1), A(l-x) Bt(l+x) Delta^l_{x,-s})
// with C_l(x) = x V(l-x) V(l+x), u_l(x) = A(l-x) A(l+x)  (common.cuh).
static int build_spin(mwsht_plan* p, int spin) {
  if (p->spins.count(spin)) return MWSHT_OK;
  typedef long double ld;
  const int L = p->L, cs = spin < 0 ? -spin : spin;
  const int Lp = p->ldw;
  std::vector<double2> inv((size_t)L * Lp, make_double2(0.0, 0.0)), fwd(inv);
  std::vector<double> wcol((size_t)L * Lp, 0.0);
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
        inv[blk<kTileRows>(l, x, L)] = make_double2((double)cx, (double)wi);
        wcol[blk<kTileCols>(l, x, L)] = (double)wi;
        ld qn = 0.0L;
        if (x >= 1) {
          const int pp = l - x + 1, qq = l + x - 1;
          qn = (2.0L * A[pp - 1] / (A[pp] * sq[pp])) * (Bt[qq + 1] / (Bt[qq] * sq[qq + 1]));
        }
        fwd[blk<kTileRows>(x, l, L)] = make_double2((double)qn, (double)(A[l - x] * Bt[l + x] * dv));
      }
    }
  });
  SpinTab st;
  int rc;
  if ((rc = upload(p, &st.rowinv, inv))) return rc;
  if ((rc = upload(p, &st.rowfwd, fwd))) return rc;
  if ((rc = upload(p, &st.wcol, wcol))) return rc;
  p->spins[spin] = st;
  return MWSHT_OK;
}

// Core tile order: groups of G row blocks walked column-major, so the CTAs in
// flight share each column block of the staged plane while it sits in L2.
// L=4096, G=8 against plain longest-first: forward core 9.76 -> 2.24 GB DRAM
// read (8.137 -> 8.193 ms), paired inverse core 5.64 -> 2.92 GB (7.216 ->
// 7.185 ms).  With few tiles per SM the grouping costs load balance (L=1024
// real inverse: 130 -> 152 us), so it applies from 4 tiles per SM on.
// MWSHT_FWD_GROUP / MWSHT_INV_GROUP override G.
static int tile_group(const char* env, size_t ntiles, int nsm) {
  if (const char* e = getenv(env)) {
    const int g = atoi(e);
    return g < 1 ? 1 : g;
  }
  return ntiles >= (size_t)4 * nsm ? 8 : 1;
}

static int build_tiles(mwsht_plan* p) {
  const int L = p->L;
  struct Tl {
    int2 t;
    long long w;
  };
  std::vector<Tl> inv, fwd, invp;
  for (int r0 = 0; r0 < L; r0 += kTileRows)
    for (int c0 = 0; c0 < L; c0 += kTileCols)
      inv.push_back({make_int2(r0, c0), (long long)(L - std::max(r0, c0))});
  // paired: tiles with c0 <= r0 + 32.  32x32 blocks strictly below the
  // diagonal also produce their transpose (weight ~1.5x: the recursion is
  // shared), diagonal blocks run plain, blocks above the diagonal are idle.
  // Rows below D run as plain tiles instead (tile.x bit 30, with their upper
  // mirror tiles c0 >= r0 + 64, c0 < D): at small L one paired tile of the
  // longest chains outlasts the per-SM share of the work.  D comes from a
  // longest-first schedule of the weights over the SMs: the smallest D whose
  // makespan is within 3% of the best (measured at L=1024 real: D=256 138 us,
  // D=0 150 us; L >= 2048 gives D=0).
  int nsm = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  auto paired_list = [&](int D) {
    std::vector<Tl> v;
    for (int r0 = 0; r0 < L; r0 += kTileRows)
      for (int c0 = 0; c0 < L; c0 += kTileCols) {
        const long long len = L - std::max(r0, c0);
        const bool lower = c0 + kTileCols <= r0;
        if (r0 >= D) {
          if (c0 <= r0 + kTileCols) v.push_back({make_int2(r0, c0), lower ? (len * 3) / 2 : len});
        } else if (c0 <= r0 + kTileCols || c0 < D) {
          v.push_back({make_int2(r0 | (1 << 30), c0), len});
        }
      }
    std::stable_sort(v.begin(), v.end(), [](const Tl& a, const Tl& b) { return a.w > b.w; });
    return v;
  };
  auto makespan = [&](const std::vector<Tl>& v) {
    std::vector<long long> load(nsm, 0);  // min-heap of SM loads
    for (auto& x : v) {
      std::pop_heap(load.begin(), load.end(), std::greater<long long>());
      load.back() += x.w;
      std::push_heap(load.begin(), load.end(), std::greater<long long>());
    }
    return *std::max_element(load.begin(), load.end());
  };
  {
    std::vector<long long> ms;
    for (int D = 0; D < L; D += kTileRows) ms.push_back(makespan(paired_list(D)));
    const long long best = *std::min_element(ms.begin(), ms.end());
    int D = 0;
    while (ms[D / kTileRows] * 100 > best * 103) D += kTileRows;
    invp = paired_list(D);
    // same grouped column-major walk as the forward tiles (fwd_group)
    const int G = tile_group("MWSHT_INV_GROUP", invp.size(), nsm);
    if (G > 1)
      std::stable_sort(invp.begin(), invp.end(), [&](const Tl& a, const Tl& b) {
        const int ra = a.t.x & 0x3fffffff, rb = b.t.x & 0x3fffffff;
        const int ga = ra / (kTileRows * G), gb = rb / (kTileRows * G);
        if (ga != gb) return ga < gb;  // groups of increasing m' (longest chains first)
        if (a.t.y != b.t.y) return a.t.y < b.t.y;
        return ra < rb;
      });
  }
  for (int l0 = 0; l0 < L; l0 += kTileRows) {
    const int top = std::min(l0 + kTileRows - 1, L - 1);
    for (int c0 = 0; c0 <= top; c0 += kTileCols) fwd.push_back({make_int2(l0, c0), (long long)top + 1});
  }
  auto by_work = [](const Tl& a, const Tl& b) { return a.w > b.w; };
  std::stable_sort(inv.begin(), inv.end(), by_work);
  // forward: longest row blocks first, in groups of G row blocks walked
  // column-major, so the CTAs in flight share each column block of the
  // staged plane (4 MB at L=4096) across G row blocks while it is in L2
  {
    const int G = tile_group("MWSHT_FWD_GROUP", fwd.size(), nsm);
    std::stable_sort(fwd.begin(), fwd.end(), [&](const Tl& a, const Tl& b) {
      const int ga = (L - 1 - a.t.x) / (kTileRows * G), gb = (L - 1 - b.t.x) / (kTileRows * G);
      if (ga != gb) return ga < gb;  // groups of decreasing degree (longest first)
      if (a.t.y != b.t.y) return a.t.y < b.t.y;
      return a.t.x > b.t.x;
    });
  }
  std::vector<int2> hi, hf, hp;
  for (auto& x : inv) hi.push_back(x.t);
  for (auto& x : invp) hp.push_back(x.t);
  for (auto& x : fwd) hf.push_back(x.t);
  int rc;
  if ((rc = upload(p, &p->tiles_inv, hi))) return rc;
  if ((rc = upload(p, &p->tiles_invp, hp))) return rc;
  if ((rc = upload(p, &p->tiles_fwd, hf))) return rc;
  p->ntiles_inv = (int)hi.size();
  p->ntiles_invp = (int)hp.size();
  p->ntiles_fwd = (int)hf.size();
  return MWSHT_OK;
}

// Core tile lists restricted to orders m0 <= m < m1 (m-column sharding,
// SURVEY.md §8e); same heavy-first order as build_tiles.
static int range_tiles(mwsht_plan* p, int m0, int m1, mwsht_plan::TileSet** out) {
  auto key = std::make_pair(m0, m1);
  auto it = p->range_tiles.find(key);
  if (it == p->range_tiles.end()) {
    const int L = p->L;
    struct Tl {
      int2 t;
      long long w;
    };
    std::vector<Tl> inv, fwd;
    for (int r0 = 0; r0 < L; r0 += kTileRows)
      for (int c0 = m0; c0 < m1; c0 += kTileCols)
        inv.push_back({make_int2(r0, c0), (long long)(L - std::max(r0, c0))});
    for (int l0 = 0; l0 < L; l0 += kTileRows) {
      const int top = std::min(l0 + kTileRows - 1, L - 1);
      for (int c0 = m0; c0 < m1 && c0 <= top; c0 += kTileCols)
        fwd.push_back({make_int2(l0, c0), (long long)top + 1});
    }
    auto by_work = [](const Tl& a, const Tl& b) { return a.w > b.w; };
    std::stable_sort(inv.begin(), inv.end(), by_work);
    std::stable_sort(fwd.begin(), fwd.end(), by_work);
    std::vector<int2> hi, hf;
    for (auto& x : inv) hi.push_back(x.t);
    for (auto& x : fwd) hf.push_back(x.t);
    mwsht_plan::TileSet ts;
    int rc;
    if (!hi.empty() && (rc = upload(p, &ts.inv, hi))) return rc;
    if (!hf.empty() && (rc = upload(p, &ts.fwd, hf))) return rc;
    ts.ninv = (int)hi.size();
    ts.nfwd = (int)hf.size();
    it = p->range_tiles.emplace(key, ts).first;
  }
  *out = &it->second;
  return MWSHT_OK;
}

// Fused-FFT tables (fft.cu): quarter twiddles w_M^j, chirp c[n] = e^{i pi n^2/N},
// spectra (half-split DIF of the Bluestein kernels c, conj c and of the
// weight-correlation kernel K'[d mod M] = 2 pi w(-d), |d| <= 2L-2,
// quadrature.py:66-74, mw.py:237-238), and the forward theta glue
// (tau(f(k)) = e^{-i f(k) pi/N}, f(k) = k (k < L), k - N),
// and for the paired forward theta rows (fft.cu): cen[k] = (-1)^k e^{i pi k/N},
// wnk[k] = e^{2 pi i k/N}, rho2[k] = e^{-i f(k) pi/N} / (2 pi N M).
static fft::FftArgs fft_args(mwsht_plan* p) {
  fft::FftArgs a{};
  a.L = p->L;
  a.N = p->N;
  a.M = p->M;
  a.H = p->H;
  a.logH = p->logH;
  a.ldw = p->ldw;
  a.tw = p->tw;
  a.chirp = p->chirp;
  a.specf = p->specf;
  a.speci = p->speci;
  a.specw = p->specw;
  a.sep1 = p->sep1;
  a.sep2 = p->sep2;
  a.sep3 = p->sep3;
  a.cen = p->cen;
  a.wnk = p->wnk;
  a.rho2 = p->rho2;
  a.scratch = p->scratch;
  a.Q = p->Q;
  a.twM = p->twM;
  a.nmaps = 1;
  a.m0 = 0;
  a.m1 = p->L;
  a.t0 = 0;
  return a;
}

static int build_fft_tables(mwsht_plan* p) {
  typedef long double ld;
  const int L = p->L, N = p->N;
  int M = 8;
  while (M < 4 * L - 3 || M < 2 * N - 1) M <<= 1;
  p->M = M;
  // the convolutions split into Q parts of H <= 8192 complex values, one
  // team's row in an SM's shared memory: Q = 2 up to L = 4096, Q = 4 up to 8192
  p->Q = M / 2 <= 8192 ? 2 : 4;
  p->H = M / p->Q;
  p->logH = 0;
  while ((1 << p->logH) < p->H) p->logH++;
  if (p->H > 8192)
    return fail(MWSHT_E_DEGREE, "plan_create",
                "band limit above the documented cap L <= 8192 (FFT engine: four quarter-"
                "convolutions of one SM's shared memory each)");
  const ld PI = 3.141592653589793238462643383279502884L;
  // passes: quarter table of w_{2H} (= w_M at Q = 2); Q = 4 also w_M (global)
  const int M2 = 2 * p->H;
  std::vector<double2> tw(M2 / 4 + 1), ch(N), sep1(N), sep2(N), sep3(N), kf(M, make_double2(0, 0)), ki(kf), kw(kf);
  std::vector<double2> cen(N), wnk(N), rho2(N);
  auto quarter_table = [&](int Mt, std::vector<double2>& t) {
    t.assign(Mt / 4 + 1, make_double2(0, 0));
    for (int j = 0; j <= Mt / 4; j++) {
      const ld a = -2.0L * PI * (ld)j / (ld)Mt;
      t[j] = make_double2((double)cosl(a), (double)sinl(a));
    }
    t[0] = make_double2(1.0, 0.0);
    t[Mt / 4] = make_double2(0.0, -1.0);
  };
  quarter_table(M2, tw);
  if (p->Q == 4) {
    std::vector<double2> twm;
    quarter_table(M, twm);
    int rc2;
    if ((rc2 = upload(p, &p->twM, twm))) return rc2;
  }
  std::vector<ld> cr(N), ci(N);
  for (int n = 0; n < N; n++) {
    const long long e = ((long long)n * n) % (2LL * N);  // c[n] = e^{i pi e/N}
    const ld a = PI * (ld)e / (ld)N;
    cr[n] = cosl(a);
    ci[n] = sinl(a);
    ch[n] = make_double2((double)cr[n], (double)ci[n]);
  }
  for (int k = 0; k < N; k++) {
    const int f = k < L ? k : k - N;
    const ld a = -PI * (ld)f / (ld)N;  // tau phase
    const ld sc = 1.0L / (2.0L * PI * (ld)N * (ld)M);
    const ld tr = cosl(a) * sc, ti = sinl(a) * sc;
    // conj(c) * tau
    rho2[k] = make_double2((double)tr, (double)ti);
    const ld b = PI * (ld)k / (ld)N, sg = (k & 1) ? -1.0L : 1.0L;
    cen[k] = make_double2((double)(sg * cosl(b)), (double)(sg * sinl(b)));
    wnk[k] = make_double2((double)cosl(2.0L * b), (double)sinl(2.0L * b));
    // decoupled stage: the chirp and the 1/2 folded into the separation (common.cuh)
    const ld hr = 0.5L * tr, hi = 0.5L * ti;
    sep1[k] = make_double2((double)(cr[k] * hr + ci[k] * hi), (double)(cr[k] * hi - ci[k] * hr));
    const int kn = (N - k) % N;
    const ld wr = cosl(2.0L * b), wi = sinl(2.0L * b);                     // e^{2 pi i k/N}
    const ld ur = wr * cr[kn] + wi * ci[kn], ui = wi * cr[kn] - wr * ci[kn];  // . conj(c[kn])
    sep2[k] = make_double2((double)(hr * ur - hi * ui), (double)(hr * ui + hi * ur));
    const ld er = sg * cosl(b), ei = sg * sinl(b);
    sep3[k] = make_double2((double)(hr * er - hi * ei), (double)(hr * ei + hi * er));
  }
  for (int j = -(N - 1); j <= N - 1; j++) {
    const int n = j < 0 ? -j : j;
    const int idx = (j + M) % M;
    kf[idx] = ch[n];
    ki[idx] = make_double2(ch[n].x, -ch[n].y);
  }
  for (long long d = -(2LL * L - 2); d <= 2LL * L - 2; d++) {
    const long long k = -d;  // K'[d] = 2 pi w(-d)
    double2 v = make_double2(0.0, 0.0);
    if (k == 1)
      v.y = (double)(PI * PI);  // 2 pi * (i pi/2)
    else if (k == -1)
      v.y = (double)(-PI * PI);
    else if ((k & 1) == 0)
      v.x = (double)(2.0L * PI * 2.0L / (1.0L - (ld)k * (ld)k));
    kw[(d + M) % M] = v;
  }
  int rc;
  if ((rc = upload(p, &p->tw, tw)) || (rc = upload(p, &p->chirp, ch)) ||
      (rc = upload(p, &p->sep1, sep1)) || (rc = upload(p, &p->sep2, sep2)) ||
      (rc = upload(p, &p->sep3, sep3)) || (rc = upload(p, &p->cen, cen)) ||
      (rc = upload(p, &p->wnk, wnk)) || (rc = upload(p, &p->rho2, rho2)))
    return rc;
  double2 *dkf, *dki, *dkw;
  if ((rc = upload(p, &dkf, kf)) || (rc = upload(p, &dki, ki)) || (rc = upload(p, &dkw, kw)))
    return rc;
  if ((rc = dev_alloc(p, (void**)&p->specf, sizeof(double2) * M)) ||
      (rc = dev_alloc(p, (void**)&p->speci, sizeof(double2) * M)) ||
      (rc = dev_alloc(p, (void**)&p->specw, sizeof(double2) * M)))
    return rc;
  fft::FftArgs a = fft_args(p);
  fft_spectrum(a, dkf, p->specf, 0);
  fft_spectrum(a, dki, p->speci, 0);
  fft_spectrum(a, dkw, p->specw, 0);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  int dev;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, dev));
  // per CTA: NR teams x (3H at Q = 2, 10H at Q = 4), NR*H <= 8192 (fft_impl.cuh)
  if ((rc = dev_alloc(p, (void**)&p->scratch,
                      sizeof(double2) * (p->Q == 4 ? 10 : 3) * 8192 * (size_t)p->nsm)))
    return rc;
  return MWSHT_OK;
}

static int check_plan(mwsht_plan* p, DevGuard& g) {
  if (!p) return fail(MWSHT_E_PLAN, "plan", "null plan");
  int cur = -1;
  CU(cudaGetDevice(&cur));
  if (cur != p->device) {
    CU(cudaSetDevice(p->device));
    g.prev = cur;
  }
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

// W-only row tables of one spin for multi-spin batches (the cores' second
// operand per map; the recursion coefficients come from the spin-0 tables).
static int build_msp(mwsht_plan* p, int spin) {
  int rc;
  if ((rc = build_spin(p, spin))) return rc;
  SpinTab& st = p->spins[spin];
  if (st.wrow) return MWSHT_OK;
  const long long n = (long long)p->L * p->ldw;
  if ((rc = dev_alloc(p, (void**)&st.wrow, sizeof(double) * n)) ||
      (rc = dev_alloc(p, (void**)&st.wrowf, sizeof(double) * n)))
    return rc;
  launch_extract_y(st.rowinv, st.wrow, n, 0);
  launch_extract_y(st.rowfwd, st.wrowf, n, 0);
  CU(cudaGetLastError());
  CU(cudaDeviceSynchronize());
  return MWSHT_OK;
}

// Validates a multi-spin batch (host spins[nm]) and builds its tables;
// returns the spin-parity mask of the FFT stages.
static int prepare_msp(mwsht_plan* p, int nm, const int* spins, bool real,
                       unsigned long long* par) {
  int rc;
  if (real) return fail(MWSHT_E_SPIN, "multi-spin", "the real path is spin 0 only");
  if (nm < 1 || nm > kMaxMsp || nm > p->max_batch)
    return fail(MWSHT_E_CONTRACT, "multi-spin", "1 <= nmaps <= min(16, plan max_batch)");
  *par = 0;
  for (int b = 0; b < nm; b++) {
    if ((rc = check_spin(p, spins[b]))) return rc;
    if ((rc = build_msp(p, spins[b]))) return rc;
    if (spins[b] & 1) *par |= 1ull << b;
  }
  return build_spin(p, 0);
}

// Core launch for a whole (unsharded) transform: small band limits run the
// one-thread-per-chain cores (core_small.cu), the rest the tiled cores.
static void core_inverse(const mwsht_plan* p, InvArgs a, int ntiles, int nm, bool real,
                         cudaStream_t st) {
  if (!a.msp && a.out_mode != 2 && p->L <= small_inverse_limit()) {
    a.nmaps = nm;
    launch_inverse_small(a, nm, real, st);
  } else {
    launch_inverse_core(a, ntiles, nm, real, st);
  }
}

static void core_forward(const mwsht_plan* p, FwdArgs a, int ntiles, int nm, bool real,
                         cudaStream_t st) {
  if (!a.msp && a.out_mode != 2 && p->L <= small_forward_limit()) {
    a.nmaps = nm;
    launch_forward_small(a, nm, real, st);
  } else {
    launch_forward_core(a, ntiles, nm, real, st);
  }
}

// ------------------------------------------------------------ pipelines
// Paired inverse tiles (core_inverse_paired.cu) cover the lower triangle
// m' > m and emit the transposed outputs from the same chains.  Built for
// spin 0 (complex and real), where they measured 4-11% faster than the plain
// tiles for one map at L = 1024-4096; spin != 0 runs the plain kernel (the
// paired variant's extra shared-memory traffic made it slower there).  Batches
// of two or more maps run the plain kernel two maps per CTA, which shares each
// recursion between maps instead and measured faster (C4: 12.0 vs 13.0 ms per
// inverse of 8 maps).  mode 1 forces pairing for spin 0, mode 0 disables it.
static bool use_paired(const mwsht_plan* p, int spin, int nmaps) {
  if (spin != 0 || p->paired_mode == 0) return false;
  return p->paired_mode == 1 || nmaps == 1;
}

static InvArgs inv_args(mwsht_plan* p, int spin, int nmaps = 1) {
  InvArgs a{};
  a.t = p->tabs;
  a.rowtab = p->spins[spin].rowinv;
  a.wcol = p->spins[spin].wcol;
  a.colc = p->colc;
  a.gp = p->bufG;
  a.g_stride = p->strideG;
  a.paired = use_paired(p, spin, nmaps) ? 1 : 0;
  a.tiles = a.paired ? p->tiles_invp : p->tiles_inv;
  a.spin = spin;
  a.ldw = p->ldw;
  return a;
}

static int inv_ntiles(const mwsht_plan* p, const InvArgs& a) {
  return a.paired ? p->ntiles_invp : p->ntiles_inv;
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

// samples (L,N) -> folded plane in the forward core's staging layout (bufG):
// fused phi DFT (k_phi_fwd: mw.py:149-158 / :489) writing the transposed ring
// spectra AT, then the fused theta stage (k_theta_fwd: extension, DFT + twist,
// weight correlation, m' fold: mw.py:161-285).
static int forward_stages(mwsht_plan* p, int nm, const void* samples, bool real, int spin,
                          cudaStream_t st, int msp = 0, unsigned long long spin_par = 0) {
  const int L = p->L, N = p->N;
  fft::FftArgs a = fft_args(p);
  a.spin = spin;
  a.msp = msp;
  a.spin_par = spin_par;
  a.nmaps = nm;
  a.nrows = L;
  a.in = samples;
  a.in_stride = (long long)L * N;  // elements (double for real, double2 for complex)
  a.out = p->bufA;
  a.out_stride = p->strideA;
  fft_launch(0, real, a, p->nsm, st);
  LAUNCHED(p);
  a.nrows = real ? L : N;
  a.in = p->bufA;
  a.in_stride = p->strideA;
  a.out = p->bufG;
  a.out_stride = p->strideG;
  fft_launch(1, real, a, p->nsm, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

// spins (host, nm entries, or NULL): a multi-spin batch sharing every chain's
// recursion between maps of different spins (kMaxMsp maps at most).
static int do_forward(mwsht_plan* p, int nm, const void* samples, void* flm, int spin, bool real,
                      int recursion, void* stream, const int* spins = nullptr) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if ((rc = check_rec(recursion))) return rc;
  if (!spins && (rc = check_spin(p, spin))) return rc;
  if (real && spin != 0) return fail(MWSHT_E_SPIN, "forward_real", "spin 0 only");
  if (nm < 1 || nm > p->max_batch) return fail(MWSHT_E_CONTRACT, "nmaps", "exceeds plan max_batch");
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  unsigned long long par = 0;
  if (spins) {
    if ((rc = prepare_msp(p, nm, spins, real, &par))) return rc;
    spin = 0;
  } else if ((rc = build_spin(p, spin))) {
    return rc;
  }
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int L = p->L;
  if (p->timing) CU(cudaEventRecord(p->ev[0][0], st));
  if ((rc = forward_stages(p, nm, samples, real, spin, st, spins ? 1 : 0, par))) return rc;
  if (p->timing) CU(cudaEventRecord(p->ev[0][1], st));
  FwdArgs a = fwd_args(p, spin);
  if (spins) {
    a.msp = 1;
    for (int b = 0; b < nm; b++) {
      a.spin_m[b] = spins[b];
      a.wrow_m[b] = p->spins[spins[b]].wrowf;
    }
  }
  a.out = (double2*)flm;
  a.out_mode = 0;
  a.out_stride = (long long)L * L;
  core_forward(p, a, p->ntiles_fwd, nm, real, st);
  LAUNCHED(p);
  if (p->timing) CU(cudaEventRecord(p->ev[0][2], st));
  return MWSHT_OK;
}

static int do_inverse(mwsht_plan* p, int nm, const void* flm, void* samples, int spin, bool real,
                      int recursion, void* stream, const int* spins = nullptr) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if ((rc = check_rec(recursion))) return rc;
  if (!spins && (rc = check_spin(p, spin))) return rc;
  if (real && spin != 0) return fail(MWSHT_E_SPIN, "inverse_real", "spin 0 only");
  if (nm < 1 || nm > p->max_batch) return fail(MWSHT_E_CONTRACT, "nmaps", "exceeds plan max_batch");
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  unsigned long long par = 0;
  if (spins) {
    if ((rc = prepare_msp(p, nm, spins, real, &par))) return rc;
    spin = 0;
  } else if ((rc = build_spin(p, spin))) {
    return rc;
  }
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int L = p->L, N = p->N;
  const int rows = real ? L : N;
  if (p->timing) CU(cudaEventRecord(p->ev[1][0], st));
  // 0. unflatten + c_l u_l(m) scaling into the core's staging rows (mw.py:390-392)
  launch_inv_prescale(real, (const double2*)flm, 0, p->tabs.cl, p->tabs.A, L, p->ldw, p->bufG,
                      (long long)L * L, p->strideG, nm, st);
  LAUNCHED(p);
  // 1. core + phases + m' mirror + theta twist (mw.py:378-402, 445)
  if (p->timing) CU(cudaEventRecord(p->ev[1][1], st));
  InvArgs a = inv_args(p, spin, nm);
  if (spins) {
    a.paired = 0;  // mixed spins share the recursion between maps instead
    a.tiles = p->tiles_inv;
    a.msp = 1;
    for (int b = 0; b < nm; b++) {
      a.spin_m[b] = spins[b];
      a.wrow_m[b] = p->spins[spins[b]].wrow;
    }
  }
  a.out = p->bufB;
  a.out_mode = 3;  // m' >= 0 half of each spectrum row: the theta stage rebuilds the mirror
  a.out_stride = (long long)rows * N;
  core_inverse(p, a, inv_ntiles(p, a), nm, real, st);
  LAUNCHED(p);
  if (p->timing) CU(cudaEventRecord(p->ev[1][2], st));
  // 2. theta synthesis (mw.py:441-446), keep t < L, transposed to rings (:436-437)
  fft::FftArgs f = fft_args(p);
  f.spin = spin;
  f.msp = spins ? 1 : 0;
  f.spin_par = par;
  f.nmaps = nm;
  f.nrows = rows;
  f.in = p->bufB;
  f.half = 1;
  f.in_stride = (long long)rows * N;
  f.out = p->bufA;
  f.out_stride = p->strideA;
  // even row pitch of the ring plane: the paired theta rows store 32 bytes per ring
  f.pitch = real ? (L + (L & 1)) : N + 1;
  fft_launch(2, real, f, p->nsm, st);
  LAUNCHED(p);
  // 3. phi synthesis (mw.py:437-438 / 558)
  f.nrows = L;
  f.in = p->bufA;
  f.in_stride = p->strideA;
  f.out = samples;
  f.out_stride = (long long)L * N;
  fft_launch(3, real, f, p->nsm, st);
  LAUNCHED(p);
  if (p->timing) CU(cudaEventRecord(p->ev[1][3], st));
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
    case MWSHT_E_DEGREE: return "unsupported degree";
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
  DevGuard dg;
  {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess) dg.prev = cur;
  }
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
  p->ldw = (L + kTileRows - 1) / kTileRows * kTileRows;
  p->device = device;
  p->max_batch = max_batch;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete p;
    return fail(MWSHT_E_CUDA, "cudaSetDevice", cudaGetErrorString(e));
  }
  const long long L_ = L, N = p->N;
  p->strideA = L_ * (N + 1);  // (N, L) ring spectra (forward) / (L, N + 1) ring plane (inverse, even pitch)
  p->strideB = N * N;
  p->strideG = 2 * L_ * p->ldw;
  if ((rc = build_tables(p)) || (rc = build_tiles(p)) || (rc = build_fft_tables(p)) ||
      (rc = dev_alloc(p, (void**)&p->bufA, sizeof(double2) * p->strideA * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->bufB, sizeof(double2) * p->strideB * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->bufG, sizeof(double2) * p->strideG * max_batch)) ||
      (rc = dev_alloc(p, (void**)&p->red, 2 * sizeof(unsigned long long))) ||
      (rc = build_spin(p, 0))) {
    mwsht_plan_destroy(p);
    return rc;
  }
  e = cudaEventCreateWithFlags(&p->handoff, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    mwsht_plan_destroy(p);
    return fail(MWSHT_E_CUDA, "cudaEventCreate", cudaGetErrorString(e));
  }
  e = cudaHostAlloc((void**)&p->red_host, 2 * sizeof(unsigned long long), cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostGetDevicePointer((void**)&p->red_host_dev, p->red_host, 0);
  if (e == cudaSuccess) e = cudaMemset(p->red, 0, 2 * sizeof(unsigned long long));
  if (e != cudaSuccess) {
    mwsht_plan_destroy(p);
    return fail(MWSHT_E_CUDA, "reality-check buffers", cudaGetErrorString(e));
  }
  // the staging buffer's pad columns (m >= L) are read but never written: zero them once
  e = cudaMemset(p->bufG, 0, sizeof(double2) * p->strideG * max_batch);
  if (e != cudaSuccess) {
    mwsht_plan_destroy(p);
    return fail(MWSHT_E_CUDA, "cudaMemset", cudaGetErrorString(e));
  }
  *out = p;
  return MWSHT_OK;
}

int mwsht_plan_destroy(mwsht_plan* p) {
  if (!p) return MWSHT_OK;
  DevGuard dg;
  {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != p->device) dg.prev = cur;
  }
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  if (p->handoff) cudaEventDestroy(p->handoff);
  for (auto& d : p->ev)
    for (auto& e : d)
      if (e) cudaEventDestroy(e);
  for (void* q : p->allocs) cudaFree(q);
  if (p->red_host) cudaFreeHost(p->red_host);
  delete p;
  return MWSHT_OK;
}

size_t mwsht_plan_device_bytes(const mwsht_plan* p) { return p ? p->bytes : 0; }

int mwsht_plan_prepare_spin(mwsht_plan* p, int spin) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin))) return rc;
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

int mwsht_forward_z_multi(mwsht_plan* p, int nmaps, const void* samples, void* flm,
                          const int* spins, int recursion, void* stream) {
  if (!spins) return fail(MWSHT_E_CONTRACT, "forward_z_multi", "null spins");
  return do_forward(p, nmaps, samples, flm, 0, false, recursion, stream, spins);
}

int mwsht_inverse_z_multi(mwsht_plan* p, int nmaps, const void* flm, void* samples,
                          const int* spins, int recursion, void* stream) {
  if (!spins) return fail(MWSHT_E_CONTRACT, "inverse_z_multi", "null spins");
  return do_inverse(p, nmaps, flm, samples, 0, false, recursion, stream, spins);
}

int mwsht_reality_residual(mwsht_plan* p, const void* flm, double* worst_host, double* tol_host,
                           void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  cudaStream_t st = (cudaStream_t)stream;
  launch_reality((const double2*)flm, p->L, p->red, p->red_host_dev, st);
  LAUNCHED(p);
  LAUNCHED(p);
  CU(cudaStreamSynchronize(st));
  unsigned long long h[2];
  memcpy(h, (const void*)p->red_host, sizeof h);
  double w, pk;
  memcpy(&w, &h[0], 8);
  memcpy(&pk, &h[1], 8);
  if (worst_host) *worst_host = w;
  if (tol_host) *tol_host = 1e-12 * (pk > 1.0 ? pk : 1.0);
  return MWSHT_OK;
}

int mwsht_reality_residual_async(mwsht_plan* p, const void* flm, unsigned long long* dev_worst_peak,
                                 void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if (!dev_worst_peak) return fail(MWSHT_E_CONTRACT, "reality_residual_async", "null result buffer");
  launch_reality((const double2*)flm, p->L, dev_worst_peak, nullptr, (cudaStream_t)stream);
  CU(cudaGetLastError());
  return MWSHT_OK;
}

int mwsht_fmm_core(mwsht_plan* p, const void* flm2d, const double* cl, int spin, int use_trapani,
                   void* T, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_inv_prescale(false, (const double2*)flm2d, 1, cl, p->tabs.A, p->L, p->ldw, p->bufG, 0,
                      p->strideG, 1, st);
  LAUNCHED(p);
  InvArgs a = inv_args(p, spin);
  a.out = (double2*)T;
  a.out_mode = 1;
  core_inverse(p, a, inv_ntiles(p, a), 1, false, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_fmm_core_real(mwsht_plan* p, const void* flm_half, const double* cl, int use_trapani,
                        void* T, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_inv_prescale(true, (const double2*)flm_half, 1, cl, p->tabs.A, p->L, p->ldw, p->bufG, 0,
                      p->strideG, 1, st);
  LAUNCHED(p);
  InvArgs a = inv_args(p, 0);
  a.out = (double2*)T;
  a.out_mode = 1;
  core_inverse(p, a, inv_ntiles(p, a), 1, true, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_flm_core(mwsht_plan* p, const void* gfold, int spin, int use_trapani, void* R,
                   void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  if ((rc = build_spin(p, spin))) return rc;
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_fold(false, (const double2*)gfold, p->bufG, p->L, p->ldw, st);
  LAUNCHED(p);
  FwdArgs a = fwd_args(p, spin);
  a.out = (double2*)R;
  a.out_mode = 1;
  // entries |m| > l stay zero, as in the reference's np.zeros output
  CU(cudaMemsetAsync(R, 0, sizeof(double2) * (size_t)p->L * p->N, st));
  core_forward(p, a, p->ntiles_fwd, 1, false, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_flm_core_real(mwsht_plan* p, const void* gfold, int use_trapani, void* R, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  (void)use_trapani;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  launch_fold(true, (const double2*)gfold, p->bufG, p->L, p->ldw, st);
  LAUNCHED(p);
  FwdArgs a = fwd_args(p, 0);
  a.out = (double2*)R;
  a.out_mode = 1;
  CU(cudaMemsetAsync(R, 0, sizeof(double2) * (size_t)p->L * p->L, st));
  core_forward(p, a, p->ntiles_fwd, 1, true, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_forward_stages_z(mwsht_plan* p, const void* samples, void* gfold, int spin,
                           void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  p->own_launches = 0;
  if ((rc = forward_stages(p, 1, samples, false, spin, (cudaStream_t)stream))) return rc;
  launch_T2_to_fold(false, p->bufG, (double2*)gfold, p->L, p->ldw, (cudaStream_t)stream);
  LAUNCHED(p);
  return MWSHT_OK;
}

static int check_shard_size(mwsht_plan* p) {
  (void)p;  // every supported band limit (quarter-split FFTs included) shards
  return MWSHT_OK;
}

static int check_range(mwsht_plan* p, int m0, int m1) {
  if (m0 < 0 || m1 > p->L || m0 >= m1 || (m0 % kTileCols) || ((m1 % kTileCols) && m1 != p->L))
    return fail(MWSHT_E_CONTRACT, "shard", "order range must be [m0, m1) with multiples of 32 (or m1 = L)");
  return MWSHT_OK;
}

int mwsht_shard_forward_phi(mwsht_plan* p, const void* samples_rows, int t0, int t1,
                            const long long* row_off, void* out, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_shard_size(p))) return rc;
  if (t0 < 0 || t1 > p->L || t0 >= t1) return fail(MWSHT_E_CONTRACT, "shard", "bad ring range");
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  p->own_launches = 0;
  fft::FftArgs a = fft_args(p);
  a.nrows = t1 - t0;
  a.t0 = t0;
  a.in = samples_rows;
  a.in_stride = 0;
  a.out = out;
  a.out_stride = 0;
  a.row_off = row_off;
  fft_launch(0, false, a, p->nsm, (cudaStream_t)stream);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_shard_forward_rest(mwsht_plan* p, const void* in, int m0, int m1,
                             const long long* col_off, const int* col_stride, int spin, void* flm,
                             int packed, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin)) || (rc = check_range(p, m0, m1))) return rc;
  if ((col_off == nullptr) != (col_stride == nullptr))
    return fail(MWSHT_E_CONTRACT, "shard", "col_off and col_stride go together");
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  if ((rc = build_spin(p, spin))) return rc;
  mwsht_plan::TileSet* ts;
  if ((rc = range_tiles(p, m0, m1, &ts))) return rc;
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  fft::FftArgs a = fft_args(p);
  a.spin = spin;
  a.m0 = m0;
  a.m1 = m1;
  a.nrows = 2 * (m1 - m0) - (m0 == 0 ? 1 : 0);
  a.in = in;
  a.in_stride = 0;
  a.out = p->bufG;
  a.out_stride = p->strideG;
  a.col_off = col_off;
  a.col_stride = col_stride;
  fft_launch(1, false, a, p->nsm, st);
  LAUNCHED(p);
  FwdArgs f = fwd_args(p, spin);
  f.tiles = ts->fwd;
  f.out = (double2*)flm;
  f.out_mode = packed ? 2 : 0;
  f.m0 = m0;
  f.m1 = m1;
  f.out_stride = (long long)p->L * p->L;
  if (ts->nfwd) {
    launch_forward_core(f, ts->nfwd, 1, false, st);
    LAUNCHED(p);
  }
  return MWSHT_OK;
}

int mwsht_shard_inverse_front(mwsht_plan* p, const void* flm, int m0, int m1, int spin,
                              const long long* row_off, void* out, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_spin(p, spin)) || (rc = check_range(p, m0, m1))) return rc;
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  if ((rc = build_spin(p, spin))) return rc;
  mwsht_plan::TileSet* ts;
  if ((rc = range_tiles(p, m0, m1, &ts))) return rc;
  p->own_launches = 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int L = p->L, N = p->N;
  // only the shard's staging columns (its tiles read nothing else)
  launch_inv_prescale(false, (const double2*)flm, 0, p->tabs.cl, p->tabs.A, L, p->ldw, p->bufG,
                      (long long)L * L, p->strideG, 1, st, m0, m1 == L ? p->ldw : m1);
  LAUNCHED(p);
  InvArgs a = inv_args(p, spin);
  a.paired = 0;  // order-restricted tiles: the transpose would leave the shard's orders
  a.tiles = ts->inv;
  a.out = p->bufB;
  a.out_mode = 3;
  a.out_stride = (long long)N * N;
  if (ts->ninv) {
    launch_inverse_core(a, ts->ninv, 1, false, st);
    LAUNCHED(p);
  }
  fft::FftArgs f = fft_args(p);
  f.spin = spin;
  f.m0 = m0;
  f.m1 = m1;
  f.nrows = 2 * (m1 - m0) - (m0 == 0 ? 1 : 0);
  f.in = p->bufB;
  f.half = 1;
  f.in_stride = 0;
  f.out = out;
  f.out_stride = 0;
  f.row_off = row_off;
  fft_launch(2, false, f, p->nsm, st);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_shard_inverse_phi(mwsht_plan* p, const void* in, int t0, int t1,
                            const long long* col_off, const int* col_stride, void* samples_rows,
                            void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg)) || (rc = check_shard_size(p))) return rc;
  if (t0 < 0 || t1 > p->L || t0 >= t1) return fail(MWSHT_E_CONTRACT, "shard", "bad ring range");
  if ((col_off == nullptr) != (col_stride == nullptr))
    return fail(MWSHT_E_CONTRACT, "shard", "col_off and col_stride go together");
  std::lock_guard<std::mutex> lk(p->mu);
  StreamUse su(p, (cudaStream_t)stream);
  p->own_launches = 0;
  fft::FftArgs f = fft_args(p);
  f.nrows = t1 - t0;
  f.t0 = t0;
  f.in = in;
  f.in_stride = 0;
  f.out = samples_rows;
  f.out_stride = 0;
  f.col_off = col_off;
  f.col_stride = col_stride;
  fft_launch(3, false, f, p->nsm, (cudaStream_t)stream);
  LAUNCHED(p);
  return MWSHT_OK;
}

int mwsht_shard_unpack_flm(mwsht_plan* p, const void* gathered, long long maxlen,
                           const int* bounds, int world, void* flm, void* stream) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if (world < 1 || !bounds || !gathered || !flm)
    return fail(MWSHT_E_CONTRACT, "shard_unpack_flm", "null buffer or world < 1");
  std::lock_guard<std::mutex> lk(p->mu);
  p->own_launches = 0;
  launch_flm_unpack((const double2*)gathered, maxlen, bounds, world, p->L, (double2*)flm,
                    (cudaStream_t)stream);
  LAUNCHED(p);
  return MWSHT_OK;
}

static int gl_core(bool forward, const void* in, const double* x, const double* ch,
                   const double* sh, const double* seed_const, const int* seed_ints, int L,
                   int spin, void* out, void* stream) {
  if (L < 1) return fail(MWSHT_E_BAND_LIMIT, "gl", "band limit must be >= 1");
  if ((spin < 0 ? -spin : spin) >= L) return fail(MWSHT_E_SPIN, "gl", "|spin| must be below L");
  if (L > 4096) return fail(MWSHT_E_DEGREE, "gl", "band limit above the kernels' cap L <= 4096");
  if (!in || !x || !ch || !sh || !seed_const || !seed_ints || !out)
    return fail(MWSHT_E_CONTRACT, "gl", "null buffer");
  const cudaError_t e = launch_gl(forward, (const double2*)in, x, ch, sh, seed_const,
                                  (const int4*)seed_ints, L, spin, (double2*)out,
                                  (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(MWSHT_E_CUDA, "gl kernel launch", cudaGetErrorString(e));
  return MWSHT_OK;
}

int mwsht_gl_fm_core(const void* flm_scaled, const double* x, const double* ch, const double* sh,
                     const double* seed_const, const int* seed_ints, int L, int spin, void* F,
                     void* stream) {
  return gl_core(false, flm_scaled, x, ch, sh, seed_const, seed_ints, L, spin, F, stream);
}

int mwsht_gl_flm_core(const void* a, const double* x, const double* ch, const double* sh,
                      const double* seed_const, const int* seed_ints, int L, int spin, void* R,
                      void* stream) {
  return gl_core(true, a, x, ch, sh, seed_const, seed_ints, L, spin, R, stream);
}

int mwsht_plan_set_paired(mwsht_plan* p, int mode) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if (mode < -1 || mode > 1) return fail(MWSHT_E_VALUE, "paired", "mode must be -1, 0 or 1");
  std::lock_guard<std::mutex> lk(p->mu);
  p->paired_mode = mode;
  return MWSHT_OK;
}

int mwsht_plan_set_timing(mwsht_plan* p, int on) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  for (auto& d : p->ev)
    for (auto& e : d)
      if (!e) CU(cudaEventCreate(&e));
  p->timing = on != 0;
  return MWSHT_OK;
}

int mwsht_plan_last_timing(mwsht_plan* p, int inverse, float* core_ms, float* stages_ms) {
  DevGuard dg;
  int rc;
  if ((rc = check_plan(p, dg))) return rc;
  if (!p->timing) return fail(MWSHT_E_VALUE, "last_timing", "timing not enabled");
  cudaEvent_t* e = p->ev[inverse ? 1 : 0];
  CU(cudaEventSynchronize(e[inverse ? 3 : 2]));
  float c = 0.f, s0 = 0.f;
  CU(cudaEventElapsedTime(&c, e[1], e[2]));
  // forward: the FFT stages run before the core; inverse: after it
  if (inverse)
    CU(cudaEventElapsedTime(&s0, e[2], e[3]));
  else
    CU(cudaEventElapsedTime(&s0, e[0], e[1]));
  if (core_ms) *core_ms = c;
  if (stages_ms) *stages_ms = s0;
  return MWSHT_OK;
}

int mwsht_plan_last_launches(const mwsht_plan* p, int* own) {
  if (!p) return MWSHT_E_PLAN;
  if (own) *own = p->own_launches;
  return MWSHT_OK;
}

}  // extern "C"
