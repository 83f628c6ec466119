// Shared definitions for the sm_100a MW transform kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

namespace mwsht {

// ---------------------------------------------------------------------------
// Recursion tables (device pointers), built once per band-limit on the host in
// 80-bit long double and rounded once to float64 (plan.cu).  With
//   A(0)=A(1)=1, A(k+2)=A(k) sqrt((k+1)/(k+2))
//   V(k)=A(k)/(sqrt(k+1) A(k+1))
//   Bt(Q)=Bt(Q-1)=1 (Q=2L+1), Bt(q)=Bt(q+2) sqrt((q+2)/(q+1))
//   alpha(p)=2A(p-1)/(A(p) sqrt p), beta(q)=Bt(q+1)/(Bt(q) sqrt(q+1))
//   lam(0)=lam(1)=1, lam(l+1)=lam(l-1)(l+1)/l, kap(l)=(2l+1)lam(l)/(l lam(l+1))
// the two recursions in DESIGN.md §3 are
//   inverse (l-recursion, chain (m',m)):
//     Delta^l_{m'm} = (-1)^l lam_l u_l(m) u_l(m') z^l,  u_l(x)=A(l-x)A(l+x)
//     z^{l+1} = kap_l C_l(m) C_l(m') z^l - z^{l-1},      C_l(x)=x V(l-x) V(l+x)
//   forward (Trapani column, chain (l,m), walking mu=m' downward):
//     Delta^l_{mu,m} = A(l-mu) Bt(l+mu) y_mu
//     y_{mu-1} = m alpha(l-mu+1) beta(l+mu-1) y_mu - y_{mu+1}
// ---------------------------------------------------------------------------
struct DevTables {
  int L, N;
  const double* A;      // [2L+4]
  const double* V;      // [2L+4]
  const double* Bt;     // [2L+4]
  const double* alpha;  // [2L+4]
  const double* beta;   // [2L+4]
  const double* lam;    // [L+2]
  const double* kap;    // [L+2]
  const double* cl;     // [L]   sqrt((2l+1)/4pi), as numpy computes it (mw.py:144-146)
  // Chain seeds as products of 1-D factors, each (mantissa in [0.5,1), binary
  // exponent) because the factorials leave every floating range:
  //   inverse z^{l0} = +-Pi(l0) Qi(l0+mu) Qi(l0-mu),  l0 = max(m',m), mu = min(m',m)
  //   forward y_l    = +-Pf(l)  R(l+m)   R(l-m)
  // R(j) = 1/sqrt(j!), Qi(j) = R(j)/A(j), P0(n) = sqrt((2n)!)/2^n,
  // Pi(n) = P0(n)/(lam_n A(2n)), Pf(n) = P0(n)/Bt(2n)  (plan.cu build_tables).
  const double2* sd_pi;  // [L]
  const double2* sd_qi;  // [2L]
  const double2* sd_pf;  // [L]
  const double2* sd_r;   // [2L]
};

// Exponent-level machinery.  A chain whose true value is
// below 2^-568 carries a level lev>0 with stored value z = true * 2^(768 lev),
// |z| <= 2^200.  It contributes nothing while lev>0 (|true| < 2^-568) and is
// rescaled by 2^-768 when |z| reaches 2^200.
constexpr int kLevShift = 768;
constexpr int kLevTop = 200;

__device__ __forceinline__ double pow2i(int e) {
  // 2^e for -1022 <= e <= 1023
  return __hiloint2double((e + 1023) << 20, 0);
}

// true value = m * 2^ex (m a double of modest magnitude): returns stored z, lev.
__device__ __forceinline__ double split_level(double m, int ex, int& lev) {
  if (m == 0.0) {
    lev = 0;
    return 0.0;
  }
  int e2;
  double f = frexp(m, &e2);  // m = f * 2^e2, 0.5 <= |f| < 1
  int X = ex + e2;
  int l = (kLevTop - X) / kLevShift;  // X <= 200 always here (values <= ~1)
  if (X > kLevTop) l = 0;
  if (l < 0) l = 0;
  lev = l;
  return ldexp(f, X + kLevShift * l);
}

// |z| >= 2^200 test on the high word (integer pipe, keeps the FP64 pipe free).
__device__ __forceinline__ bool above_top(double z) {
  return (__double2hiint(z) & 0x7ff00000) >= ((1023 + kLevTop) << 20);
}

// product of three (mantissa, exponent) factors: returns the mantissa product, ex = exponent sum
__device__ __forceinline__ double seed3(double2 a, double2 b, double2 c, int& ex) {
  ex = (int)a.y + (int)b.y + (int)c.y;
  return a.x * b.x * c.x;
}

// i^p for p mod 4, as (re, im)
__device__ __forceinline__ double2 ipow(int p) {
  p &= 3;
  return p == 0 ? make_double2(1, 0) : p == 1 ? make_double2(0, 1) : p == 2 ? make_double2(-1, 0)
                                                                            : make_double2(0, -1);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// ---------------------------------------------------------------- core args
constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = 32 * kConsumerWarps;
// Core CTA = 3 warpgroups: warpgroup 0 holds the TMA producer warp (its other
// three warps retire) and gives up registers with setmaxnreg; warpgroups 1-2
// are the 8 consumer warps, which raise their budget to kConsumerRegs (per
// SMSP: 40 + 2 x 232 regs/thread x 32 lanes <= 64 KB).  With a single
// 288-thread layout the consumers were capped at 168 registers.
constexpr int kCoreThreadsWS = 128 + kConsumerThreads;
constexpr int kProducerRegs = 40;
constexpr int kConsumerRegs = 232;
constexpr int kTileRows = 64;  // inverse: m' rows; forward: l rows
constexpr int kTileCols = 32;  // m columns
constexpr int kChunk = 16;     // l (inverse) or m' (forward) steps per pipeline stage
constexpr int kStages = 5;     // depth of the mbarrier ring

// All 2-D plan tables and staged planes have leading dimension ldw = L rounded
// up to kTileRows, zero-padded, so every bulk copy is in bounds and aligned.
// Multi-spin batches: maps of different
// spins share every chain's recursion (kap_l C_l(m') C_l(m), resp. the Trapani
// column coefficients, do not depend on the spin); only the row weight W and
// the phases do.  At most kMaxMsp maps per call; W-only row tables per map.
constexpr int kMaxMsp = 16;

struct InvArgs {
  DevTables t;
  const double2* rowtab;  // [l*ldw + m'] = (kap_l C_l(m'), (-1)^l lam_l u_l(m') Delta^l_{m',-s})
  const double* colc;     // [l*ldw + m]  = C_l(m)
  const double2* gp;      // pre-scaled coefficients: gp[l*ldw+m] = c_l u_l(m) f_{l,m},
                          // gn = gp + L*ldw: c_l u_l(m) (-1)^l f_{l,-m}  (zero for m > l)
  double2* out;           // out_mode 0: theta-synthesis spectrum (N,N) [complex] / (L,N) [real]
                          // out_mode 3: the same, bins m' >= 0 only (the mirrored half is not written)
                          // out_mode 1: raw T (L,N) [complex] / (L,L) [real]
  const double* wcol;     // paired tiles: [blk32(l, m)] = W_l(m) (the row weight at column indices)
  const int2* tiles;
  int out_mode, spin;
  int ldw;
  int paired;                      // tiles cover the lower triangle and also emit the transpose
  int nmaps;                       // maps in the batch (set by launch_inverse_core)
  long long g_stride, out_stride;  // per-map element strides (batch = gridDim.y)
  int msp;                         // multi-spin: map b has spin spin_m[b], weights wrow_m[b]
  int spin_m[kMaxMsp];
  const double* wrow_m[kMaxMsp];   // [blk64(l, m')] = W_l(m'; spin_m[b]) (SpinTab::wrow)
};

struct FwdArgs {
  DevTables t;
  const double2* rowtab;  // [m'*ldw + l] = (alpha(l-m'+1) beta(l+m'-1), A(l-m') Bt(l+m') Delta^l_{m',-s})
  const double2* gf;      // gfT[m'*ldw + m] = gfold[+m][m'];  + L*ldw: (-1)^m' gfold[-m][m']
  double2* out;           // out_mode 0: flat flm (phases, c_l applied) ; 1: raw R (L,N) / (L,L)
  const int2* tiles;
  int out_mode, spin;
  int ldw;
  int nmaps;  // maps in the batch (set by launch_forward_core)
  long long in_stride, out_stride;
  int m0, m1;  // out_mode 2: the shard's order range (packed flm, shard_flm_index)
  int msp;     // multi-spin: map b has spin spin_m[b], weights wrow_m[b]
  int spin_m[kMaxMsp];
  const double* wrow_m[kMaxMsp];  // [blk64(m', l)] = W'(l, m'; spin_m[b]) (SpinTab::wrowf)
};

// Packed coefficient block of an order-range shard m0 <= |m| < m1 (m-column
// sharding, out_mode 2 of the forward core): l-major, and within a degree
// the orders in increasing m (-hi .. -max(m0,1), then m0 .. hi, hi =
// min(l, m1-1)), i.e. the flat l(l+1)+m layout restricted to the shard.
__host__ __device__ __forceinline__ long long shard_flm_base(int l, int m0, int m1) {
  const long long k = l - m0 < 0 ? 0 : (l - m0 > m1 - m0 ? m1 - m0 : l - m0);
  const long long s1 = k * (k + 1) / 2 + (long long)(m1 - m0) * (l > m1 ? l - m1 : 0);
  return 2 * s1 - (m0 == 0 ? l : 0);
}
__host__ __device__ __forceinline__ long long shard_flm_index(int l, int m, int m0, int m1) {
  const int hi = l < m1 - 1 ? l : m1 - 1;
  const int mn = m0 > 0 ? m0 : 1;
  const long long b = shard_flm_base(l, m0, m1);
  return m < 0 ? b + (m + hi) : b + (hi - mn + 1) + (m - m0);
}

namespace fft {
// Arguments of the fused FFT-stage kernels (fft.cu).
struct FftArgs {
  int L, N, M, H, logH, ldw, spin;
  const double2* tw;      // w_M^j = e^{-2 pi i j/M}, j = 0..M/4 (global; staged to smem)
  const double2* chirp;   // c[n] = e^{+i pi n^2 / N}, n < N
  const double2* specf;   // forward Bluestein spectrum, halves [0,H) and [H,2H) (DFT_M of c)
  const double2* speci;   // inverse Bluestein spectrum (DFT_M of conj c)
  const double2* specw;   // weight-correlation spectrum (DFT_M of K'), 2pi included
  // decoupled forward theta stage (two rows per transform), with y the Bluestein
  // output before its chirp: F_1[k] = a + b, F_2[k] = -i (a - b), a = y[k] sep1[k],
  // b = eps_1 (y[N-k] sep2[k] - cc sep3[k]); one row: F[k] = 2 y[k] sep1[k]
  const double2* sep1;    // tau(f(k)) conj(c[k]) / (4 pi N M)
  const double2* sep2;    // tau(f(k)) e^{2 pi i k/N} conj(c[(N-k) mod N]) / (4 pi N M)
  const double2* sep3;    // tau(f(k)) (-1)^k e^{i pi k/N} / (4 pi N M)
  const double2* cen;     // paired forward theta rows: (-1)^k e^{i pi k/N}  (k < N)
  const double2* wnk;     //                            e^{2 pi i k/N}       (k < N)
  const double2* rho2;    //                            tau(f(k)) / (2 pi N M)
  double2* scratch;       // per-CTA L2 scratch: 3H complex per team
  const void* in;         // stage input
  void* out;              // stage output
  long long in_stride, out_stride;  // per-map strides (elements)
  int nrows, nmaps;
  int m0, m1;  // theta kernels: rows are the orders m with m0 <= |m| < m1 (full: 0, L)
  int t0;      // phi kernels: rows are the rings t0 .. t0+nrows-1
  // m-column sharding exchange layouts (shard.py builds the tables; nullptr =
  // dense layouts).  Local row i of an order-range shard is row_order(i).
  //   k_phi_fwd   out: bin k, ring t   -> out[row_off[k] + (t - t0)]
  //   k_theta_fwd in:  row i, ring t   -> in[col_off[t] + i * col_stride[t]]
  //   k_theta_inv out: row i, ring t   -> out[row_off[t] + i]
  //   k_phi_inv   in:  ring t, bin n   -> in[col_off[n] + (t - t0) * col_stride[n]]
  const long long* row_off;
  const long long* col_off;
  const int* col_stride;
  int spread;  // set by the launcher: rows dealt team-major (fft_impl.cuh first_row)
  int pitch;   // inverse stages: row pitch of the ring plane between theta and phi synthesis (0: dense)
  int half;    // inverse theta stage: the spectrum rows hold the m' >= 0 half only (core out_mode 3)
  int msp;                // multi-spin batch: map b's spin parity is bit b of spin_par
  unsigned long long spin_par;
  int Q;                  // convolution split: M = Q H (2, or 4 for 4096 < L <= 8192)
  const double2* twM;     // Q = 4: quarter table of w_M (M/4 + 1 entries, global)
};
// spin of map `map` as far as the FFT stages need it (its parity)
__host__ __device__ __forceinline__ int stage_spin(const FftArgs& a, int map) {
  return a.msp ? (int)((a.spin_par >> map) & 1ull) : a.spin;
}
}  // namespace fft

}  // namespace mwsht

// ------------------------------------------------------- blocked layouts
// The cores' per-degree inputs are stored column-blocked so that one chunk of
// kChunk consecutive steps of a tile is ONE contiguous TMA bulk copy:
//   blk<W>(step, col, L) = (col / W) * (L * W) + step * W + col % W,
// W = kTileCols (32) for column-indexed data (C_l(m), the staging planes)
// and kTileRows (64) for the row tables.  A plane of L steps x ldw columns
// (ldw a multiple of 64) keeps its L * ldw size.
namespace mwsht {
template <int W>
__host__ __device__ __forceinline__ long long blk(int step, int col, int L) {
  return (long long)(col / W) * ((long long)L * W) + (long long)step * W + (col % W);
}
}  // namespace mwsht

// ------------------------------------------------------- register budget
namespace mwsht {
// bit e set when chain e (4-bit level nibble e of lv) is at level 0
template <int NE>
__device__ __forceinline__ unsigned level_zero_mask(unsigned lv) {
  unsigned m = 0;
#pragma unroll
  for (int e = 0; e < NE; e++) m |= (((lv >> (4 * e)) & 15u) == 0) ? (1u << e) : 0u;
  return m;
}

// compile-time bool for generic-lambda dispatch
template <bool B>
struct BoolC {
  static constexpr bool value = B;
};

template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
}  // namespace mwsht

// ------------------------------------------------------- async bulk copies
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) completing on an mbarrier,
// used to stage per-chunk row/column data without occupying registers.
namespace mwsht {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy of `bytes` (multiple of 16, both addresses 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace mwsht

// ------------------------------------------------------- launch helpers
namespace mwsht {
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the call costs microseconds of host time, which dominated small-L transforms.
inline void smem_attr_once(const void* kern, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done.insert(std::make_pair(kern, dev)).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
}  // namespace mwsht

// ------------------------------------------------------- programmatic dependent launch
// The transform kernels can launch with programmatic stream serialisation: each
// kernel triggers its dependents at entry (griddepcontrol.launch_dependents),
// so the next kernel's CTAs start on SMs as this kernel's last wave drains and
// run their prologue (plan tables, twiddles, chain seeds -- constant data)
// before griddepcontrol.wait, which returns once the previous kernel has
// completed and its memory is visible.  Every access to a mutable buffer comes
// after the wait.  The dependents can only launch once every CTA of this grid
// has started, so a waiting dependent never holds an SM this grid still needs.
// Measured (bench.py, B200): C3 0.5485 -> 0.5466 ms per pair, C5 23.69 ->
// 24.08 ms, so it is OFF by default; MWSHT_PDL=1 in the environment turns it
// on (the kernels' griddepcontrol instructions are no-ops without it).
namespace mwsht {
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MWSHT_PDL");
    return e && e[0] == '1';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace mwsht
