// Fused FFT stages (replaces cuFFT on the hot path): Bluestein DFTs of the odd
// lengths N = 2L-1 (8191 is prime) and the quadrature-weight correlation, each
// as an M-point FFT-convolution (M = P = 2^ceil(log2(4L-3))) run in one CTA's
// shared memory.
//
// Engine.  A size-M FFT-convolution y = IDFT_M(DFT_M(x) . S) is split by its
// first radix-2 step into two independent H = M/2 halves:
//   half 0: x0[j] = x[j] + x[j+H],      half 1: x1[j] = (x[j] - x[j+H]) w_M^j
//   z_h = DIT_H( DIF_H(x_h) . S_h )     (S_h = even / odd-index DFT_M(kernel))
//   y[k] = z0[k] + w_M^-k z1[k],  y[k+H] = z0[k] - w_M^-k z1[k]   (unnormalised)
// DIF_H leaves its output in digit-reversed order, the precomputed spectra S_h
// are produced by the same DIF code (same order), and DIT_H consumes that
// order, so no reordering pass exists anywhere.  H complex doubles (128 KB at
// L = 4096) live in padded shared memory next to a quarter twiddle table;
// z1 and intermediate rows spill to a per-CTA L2-resident scratch.
//
// Kernels (persistent: one CTA per SM loops over rows, rows x maps):
//   k_phi_fwd    mw.py:149-158 / :489   samples row t -> AT[k][t] = 2pi/N DFT_N (transposed)
//   k_theta_fwd  mw.py:161-285           AT row -> extension -> DFT_N -> twist -> weight
//                                        correlation -> m' fold -> core staging (gfT)
//   k_theta_fwd2                         the same stage for H >= 2048, decoupled: shared-memory-only
//                                        half-convolutions + element-wise global loops, waiting
//                                        rows parked in tensor memory (see conv_smem)
//   k_theta_inv  mw.py:441-446           spectrum row m -> IDFT_N -> Out[t][bin(m)], t < L
//   k_phi_inv    mw.py:437-438 / :558    Out row t -> IDFT_N -> samples row t
//   k_spectrum   plan time: S_0, S_1 of a length-M kernel
#pragma once
#include "common.cuh"

namespace mwsht {
namespace fft {

#ifndef MWSHT_FFT_THREADS
#define MWSHT_FFT_THREADS 512  // 256 measured 5-35% slower (fewer warps per SM)
#endif
constexpr int kT = MWSHT_FFT_THREADS;  // threads per CTA



// i-th order row of an |m| range [m0, m1): +m0..+(m1-1), then -m0..-(m1-1) (m = 0 once)
__device__ __forceinline__ int row_order(int i, int m0, int m1, bool real) {
  const int n = m1 - m0;
  if (real || i < n) return m0 + i;
  return -(m0 + (i - n) + (m0 == 0 ? 1 : 0));
}

// XOR swizzle of 16-byte elements inside each 128-byte segment: strided and
// contiguous radix-R accesses of a warp land on distinct bank groups.
__device__ __forceinline__ int phys(int i) { return i ^ ((i >> 3) & 7); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

// w_M^e from the quarter table (M a power of two >= 8)
__device__ __forceinline__ double2 omega(const double2* tw, int e, int M) {
  e &= (M - 1);
  const int q = M >> 2;
  const int quad = e / q, r = e - quad * q;
  const double2 v = tw[r];
  switch (quad) {
    case 0: return v;
    case 1: return make_double2(v.y, -v.x);   // -i v
    case 2: return make_double2(-v.x, -v.y);  // -v
    default: return make_double2(-v.y, v.x);  // +i v
  }
}

// x * e^{-2 pi i e/16} (CONJ: e^{+}), e a compile-time constant after unrolling:
// multiples of pi/2 are sign/swap moves, odd multiples of pi/4 cost 2 adds + 2 muls.
template <bool CONJ>
__device__ __forceinline__ double2 rot16(double2 x, int e) {
  constexpr double C1 = 0.92387953251128674, S1 = 0.38268343236508978, H = 0.70710678118654752;
  e &= 15;
  if (CONJ) e = (16 - e) & 15;
  switch (e) {
    case 0: return x;
    case 4: return make_double2(x.y, -x.x);
    case 8: return make_double2(-x.x, -x.y);
    case 12: return make_double2(-x.y, x.x);
    case 2: return make_double2(H * (x.x + x.y), H * (x.y - x.x));
    case 6: return make_double2(H * (x.y - x.x), -H * (x.x + x.y));
    case 10: return make_double2(-H * (x.x + x.y), H * (x.x - x.y));
    case 14: return make_double2(H * (x.x - x.y), H * (x.x + x.y));
    case 1: return cmul(x, make_double2(C1, -S1));
    case 3: return cmul(x, make_double2(S1, -C1));
    case 5: return cmul(x, make_double2(-S1, -C1));
    case 7: return cmul(x, make_double2(-C1, -S1));
    case 9: return cmul(x, make_double2(-C1, S1));
    case 11: return cmul(x, make_double2(-S1, C1));
    case 13: return cmul(x, make_double2(S1, C1));
    default: return cmul(x, make_double2(C1, S1));
  }
}

// In-register radix-2 DIF network (R <= 16): x[bitrev(k)] <- sum_r x_r e^{-2 pi i rk/R}
template <int R>
__device__ __forceinline__ void net_fwd(double2 (&x)[R]) {
#pragma unroll
  for (int span = R / 2; span >= 1; span >>= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * span) {
#pragma unroll
      for (int j = 0; j < span; j++) {
        const double2 u = x[b + j], v = x[b + j + span];
        x[b + j] = cadd(u, v);
        x[b + j + span] = rot16<false>(csub(u, v), j * (8 / span));  // W_{2 span}^j
      }
    }
  }
}
// exact inverse (unnormalised): natural order out of bit-reversed registers
template <int R>
__device__ __forceinline__ void net_inv(double2 (&x)[R]) {
#pragma unroll
  for (int span = 1; span <= R / 2; span <<= 1) {
#pragma unroll
    for (int b = 0; b < R; b += 2 * span) {
#pragma unroll
      for (int j = 0; j < span; j++) {
        const double2 v = rot16<true>(x[b + j + span], j * (8 / span));
        const double2 u = x[b + j];
        x[b + j] = cadd(u, v);
        x[b + j + span] = csub(u, v);
      }
    }
  }
}

template <int R>
__device__ __forceinline__ int brev(int k) {
  int r = 0;
#pragma unroll
  for (int b = 1; b < R; b <<= 1) r = (r << 1) | ((k & b) ? 1 : 0);
  return r;
}

// w[k] = w1^k, k < R, by a product tree (dependency depth log2 R instead of R)
template <int R>
__device__ __forceinline__ void powers(double2 (&w)[R], double2 w1) {
  w[0] = make_double2(1.0, 0.0);
  if (R > 1) w[1] = w1;
#pragma unroll
  for (int k = 2; k < R; k++) w[k] = cmul(w[k / 2], w[k - k / 2]);
}

// ------------------------------------------------------------ schedule
// Compile-time plan for H = 2^LOGH: NP passes of radix <= 16 (outer first),
// TEAM threads per row (one radix-16 butterfly each), NR rows in flight per
// 512-thread CTA, each team with its own buffer and named barrier.
template <int LOGH>
struct Cfg {
  static constexpr int H = 1 << LOGH;
  static constexpr int M = 2 * H;
  static constexpr int NP = (LOGH + 3) / 4;
  // Small rows (H <= 512, L <= 256): one-warp teams, 4 per 128-thread CTA, with
  // the team's L2 scratch (z1, F rows: 3H) in shared memory instead -- these
  // sizes are latency-bound, every global round trip shows
  static constexpr bool SMEM_SCR = LOGH <= 9;
  static constexpr int KT = SMEM_SCR ? 128 : kT;  // threads per CTA
  static constexpr int TEAM = (H / 16) < 32 ? 32 : ((H / 16) > KT ? KT : (H / 16));
  static constexpr int NR = KT / TEAM;
  static constexpr int lr(int p) { return LOGH / NP + (p < LOGH - (LOGH / NP) * NP ? 1 : 0); }
  static constexpr int n_at(int p) {  // sub-length of DIF pass p
    int n = H;
    for (int q = 0; q < p; q++) n >>= lr(q);
    return n;
  }
};

template <int TEAM>
__device__ __forceinline__ void team_sync(int team) {
  if (TEAM <= 32)
    __syncwarp();
  else
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(TEAM) : "memory");
}

// Storage order of the precomputed spectra: the fused innermost pass (radix R,
// butterfly b = lt + q*TEAM reads positions b*R + k) finds its R values at
// (q*R + k)*TEAM + lt, so each warp-wide load is one contiguous 512-byte run
// instead of 32 lines 128 bytes apart.  Natural order when a team has idle
// lanes (H/R < TEAM).
template <int H, int R, int TEAM>
__host__ __device__ constexpr int spec_index(int b, int k, int lt) {
  return ((H / R) % TEAM == 0) ? (b - lt) * R + k * TEAM + lt : b * R + k;
}

// One radix-R pass on sub-length n (stride s = n/R), compile-time shape.  MODE:
//   0 DIF   (load via LD, butterfly, twiddle, store via ST)
//   1 DIT   (load, untwiddle, inverse butterfly, store)
//   2 fused innermost DIF + spectrum multiply + innermost DIT (s = 1, j = 0)
template <int R, int MODE, int H, int M, int n, int TEAM, class LD, class ST>
__device__ __forceinline__ void pass(const double2* tw, const double2* spec, int lt, LD ld, ST st) {
  constexpr int s = n / R, nb = H / R, tstep = M / n;
  // one butterfly per thread when nb == TEAM (H = 8192): no unrolled copy (code size)
  constexpr int UNR = nb > TEAM ? 2 : 1;
#pragma unroll UNR
  for (int b = lt; b < nb; b += TEAM) {
    const int blk = b / s, j = b - blk * s, base = blk * n + j;
    double2 x[R];
    if (MODE == 0) {
#pragma unroll
      for (int r = 0; r < R; r++) x[r] = ld(base + r * s);
      double2 w[R];
      powers<R>(w, omega(tw, j * tstep, M));
      net_fwd<R>(x);
      st(base, x[0]);
#pragma unroll
      for (int k = 1; k < R; k++) st(base + k * s, cmul(x[brev<R>(k)], w[k]));
    } else if (MODE == 1) {
      double2 w[R];
      powers<R>(w, omega(tw, j * tstep, M));
      x[0] = ld(base);
#pragma unroll
      for (int k = 1; k < R; k++) x[brev<R>(k)] = cmulc(ld(base + k * s), w[k]);
      net_inv<R>(x);
#pragma unroll
      for (int r = 0; r < R; r++) st(base + r * s, x[r]);
    } else {
      // spectra are stored thread-major (spec_index): a warp's loads coalesce
      double2 sp[R];
#pragma unroll
      for (int k = 0; k < R; k++) sp[k] = spec[spec_index<H, R, TEAM>(b, k, lt)];
#pragma unroll
      for (int r = 0; r < R; r++) x[r] = ld(base + r);
      net_fwd<R>(x);
#pragma unroll
      for (int k = 0; k < R; k++) x[brev<R>(k)] = cmul(x[brev<R>(k)], sp[k]);
      net_inv<R>(x);
#pragma unroll
      for (int r = 0; r < R; r++) st(base + r, x[r]);
    }
  }
}

template <int LOGH, int P, class IN, class LDS, class STS>
__device__ __forceinline__ void dif_chain(const double2* tw, int lt, int team, IN in, LDS lds,
                                          STS sts) {
  using C = Cfg<LOGH>;
  if constexpr (P < C::NP - 1) {
    constexpr int R = 1 << C::lr(P), n = C::n_at(P);
    if constexpr (P == 0)
      pass<R, 0, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, in, sts);
    else
      pass<R, 0, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, lds, sts);
    team_sync<C::TEAM>(team);
    dif_chain<LOGH, P + 1>(tw, lt, team, in, lds, sts);
  }
}

template <int LOGH, int P, class OUT, class LDS, class STS>
__device__ __forceinline__ void dit_chain(const double2* tw, int lt, int team, OUT out, LDS lds,
                                          STS sts) {
  using C = Cfg<LOGH>;
  if constexpr (P >= 0) {
    constexpr int R = 1 << C::lr(P), n = C::n_at(P);
    if constexpr (P == 0)
      pass<R, 1, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, lds, out);
    else
      pass<R, 1, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, lds, sts);
    team_sync<C::TEAM>(team);
    dit_chain<LOGH, P - 1>(tw, lt, team, out, lds, sts);
  }
}

template <int LOGH, int P, class LDS, class STS>
__device__ __forceinline__ void dit_mid(const double2* tw, int lt, int team, LDS lds, STS sts) {
  using C = Cfg<LOGH>;
  if constexpr (P >= 1) {
    constexpr int R = 1 << C::lr(P), n = C::n_at(P);
    pass<R, 1, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, lds, sts);
    team_sync<C::TEAM>(team);
    dit_mid<LOGH, P - 1>(tw, lt, team, lds, sts);
  }
}

// The passes between the first DIF pass and the last DIT pass touch only the
// shared-memory row, so call sites with OUTLINE share ONE out-of-line copy of
// them: k_theta_fwd (four half-convolutions per task) then fits the
// instruction cache, which its fully inlined form (7 passes per call site,
// ~2.7k instructions each) did not.  Kernels with two call sites keep the
// inlined form (the call costs ~3% there).
template <int LOGH>
__device__ __noinline__ void conv_middle(double2* X, const double2* tw, const double2* S, int lt,
                                         int team) {
  using C = Cfg<LOGH>;
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  constexpr int RL = 1 << C::lr(C::NP - 1), nL = C::n_at(C::NP - 1);
  dif_chain<LOGH, 1>(tw, lt, team, lds, lds, sts);
  pass<RL, 2, C::H, C::M, nL, C::TEAM>(tw, S, lt, lds, sts);
  team_sync<C::TEAM>(team);
  dit_mid<LOGH, C::NP - 2>(tw, lt, team, lds, sts);
}

// z = DIT_H( DIF_H(x) . S ), x from IN(j), z delivered to OUT(k, z_k) (unnormalised).
// The first DIF pass reads IN, the innermost DIF pass + spectrum multiply +
// innermost DIT pass are one register pass, the last DIT pass hands results to OUT.
template <int LOGH, bool OUTLINE = false, class IN, class OUT>
__device__ __forceinline__ void conv_half(double2* X, const double2* tw, const double2* S, int lt,
                                          int team, IN in, OUT out) {
  using C = Cfg<LOGH>;
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  team_sync<C::TEAM>(team);
  constexpr int RL = 1 << C::lr(C::NP - 1), nL = C::n_at(C::NP - 1);
  if constexpr (C::NP == 1) {
    pass<RL, 2, C::H, C::M, nL, C::TEAM>(tw, S, lt, in, out);
    team_sync<C::TEAM>(team);
  } else {
    if constexpr (OUTLINE) {
      constexpr int R0 = 1 << C::lr(0);
      pass<R0, 0, C::H, C::M, C::H, C::TEAM>(tw, nullptr, lt, in, sts);
      team_sync<C::TEAM>(team);
      conv_middle<LOGH>(X, tw, S, lt, team);
      pass<R0, 1, C::H, C::M, C::H, C::TEAM>(tw, nullptr, lt, lds, out);
      team_sync<C::TEAM>(team);
    } else {
      dif_chain<LOGH, 0>(tw, lt, team, in, lds, sts);
      pass<RL, 2, C::H, C::M, nL, C::TEAM>(tw, S, lt, lds, sts);
      team_sync<C::TEAM>(team);
      dit_chain<LOGH, C::NP - 2>(tw, lt, team, out, lds, sts);
    }
  }
}

// First row (task) of a team; rows then advance by gridDim.x * NR.  With
// fewer rows than team slots (small L) rows are dealt team-major, so each row
// gets its own SM instead of NR rows sharing one CTA; otherwise CTA-major.
template <int NR>
__device__ __forceinline__ int first_row(const FftArgs& a, int team) {
  return a.spread ? team * (int)gridDim.x + (int)blockIdx.x : (int)blockIdx.x * NR + team;
}

// the passes' twiddles w_{2H}^e: quarter table of 2H/4 + 1 entries in smem
template <int LOGH>
__device__ __forceinline__ void load_tw(double2* tws, const FftArgs& a) {
  for (int i = threadIdx.x; i <= Cfg<LOGH>::M / 4; i += Cfg<LOGH>::KT) tws[i] = a.tw[i];
  __syncthreads();
}

// Quarter split (Q = 4, band limits 4096 < L <= 8192): the M = 4H-point
// convolution is decimated into four H-point convolutions (radix-4 first
// step: x_q[j] = w_M^{jq} sum_r x[j + rH] (-i)^{rq}, spectra S_q = DIF_H of
// the kernel's q-th component) and merged at the end,
// y[k + pH] = sum_q i^{pq} w_M^{-kq} z_q[k].  w_M^e comes from a global
// quarter table (twM); z_1..z_3 wait in the team's L2 scratch.
__device__ __forceinline__ double2 rot_mi(double2 v, int q) {  // v (-i)^q
  switch (q & 3) {
    case 0: return v;
    case 1: return make_double2(v.y, -v.x);
    case 2: return make_double2(-v.x, -v.y);
    default: return make_double2(-v.y, v.x);
  }
}

__device__ __forceinline__ int fbin(int k, int N) { return k >= 0 ? k : k + N; }

// Dense layout of the ring spectra AT between the forward phi and theta stages
// (complex maps): bins go in pairs, at_idx(k, t) = ((k >> 1) L + t) 2 + (k & 1)
// -- (N + 1) L entries.  The phi stage's transposed stores of neighbouring bins
// (neighbouring lanes) then share a 32-byte sector, and the theta stage, whose
// tasks are exactly these pairs (orders 2k, 2k+1; bins N-2k, N-2k-1), reads both
// rows of a ring as one 32-byte load.  (16-byte stores one row apart cost the
// phi stage 0.25 ms of 1.18 at L = 4096, timing probe.)
__device__ __forceinline__ long long at_idx(int k, int t, int L) {
  return ((long long)(k >> 1) * L + t) * 2 + (k & 1);
}

// Bluestein DFT_N of x (fx(n), n < N): forward (conj chirp, spec f) or inverse
// (chirp, spec i).  Half 1 leaves z1 in scr; half 0 calls fin(k, y_k) with the
// merged y[k] = z0[k] + w^-k z1[k] (unnormalised; DFT = chirp' . y / M).
template <int LOGH, bool INV, bool OUTLINE = false, int Q = 2, class FX, class FIN>
__device__ __forceinline__ void bluestein(double2* X, const double2* tw, double2* scr,
                                          const FftArgs& a, int lt, int team, FX fx, FIN fin) {
  using C = Cfg<LOGH>;
  const double2* spec = INV ? a.speci : a.specf;
  const int N = a.N;
  if constexpr (Q == 4) {
    // N <= 2H: x[j + rH] is nonzero for r = 0, 1 only; fin(n, y_n) for n < 2H
    constexpr int H = C::H, MQ = 4 * C::H;
    auto xv = [&](int n) {
      double2 v = make_double2(0.0, 0.0);
      if (n < N) {
        const double2 c = a.chirp[n];
        v = INV ? cmul(fx(n), c) : cmulc(fx(n), c);
      }
      return v;
    };
#pragma unroll 1
    for (int q = 3; q >= 1; q--) {
      conv_half<LOGH, OUTLINE>(
          X, tw, spec + q * H, lt, team,
          [&](int j) { return cmul(cadd(xv(j), rot_mi(xv(j + H), q)), omega(a.twM, j * q, MQ)); },
          [&](int k, double2 v) { scr[(q - 1) * H + k] = v; });
    }
    conv_half<LOGH, OUTLINE>(
        X, tw, spec, lt, team, [&](int j) { return cadd(xv(j), xv(j + H)); },
        [&](int k, double2 z0) {
          const double2 t1 = cmulc(scr[k], omega(a.twM, k, MQ));
          const double2 t2 = cmulc(scr[H + k], omega(a.twM, 2 * k, MQ));
          const double2 t3 = cmulc(scr[2 * H + k], omega(a.twM, 3 * k, MQ));
          const double2 e = cadd(z0, t2), o = cadd(t1, t3), d = csub(t1, t3);
          fin(k, cadd(e, o));                                                       // p = 0
          const double2 ze = csub(z0, t2);
          fin(k + H, make_double2(ze.x - d.y, ze.y + d.x));                         // p = 1: + i d
        });
    return;
  }
  auto in1 = [&](int j) {
    double2 v = make_double2(0.0, 0.0);
    if (j < N) {
      const double2 c = a.chirp[j];
      v = INV ? cmul(fx(j), c) : cmulc(fx(j), c);
      v = cmul(v, omega(tw, j, C::M));
    }
    return v;
  };
  auto in0 = [&](int j) {
    double2 v = make_double2(0.0, 0.0);
    if (j < N) {
      const double2 c = a.chirp[j];
      v = INV ? cmul(fx(j), c) : cmulc(fx(j), c);
    }
    return v;
  };
  auto out1 = [&](int k, double2 v) { scr[k] = v; };
  auto out0 = [&](int k, double2 v) { fin(k, cadd(v, cmulc(scr[k], omega(tw, k, C::M)))); };
  conv_half<LOGH, OUTLINE>(X, tw, spec + C::H, lt, team, in1, out1);
  conv_half<LOGH, OUTLINE>(X, tw, spec, lt, team, in0, out0);
}

// Per-CTA setup shared by the stage kernels: team split, buffers, twiddles.
#define FFT_PROLOGUE                                                         \
  pdl_trigger();                                                             \
  using C = Cfg<LOGH>;                                                       \
  extern __shared__ __align__(16) double2 sm[];                              \
  const int team = threadIdx.x / C::TEAM, lt = threadIdx.x - team * C::TEAM; \
  double2* X = sm + team * C::H;                                             \
  double2* tws = sm + C::NR * C::H;                                          \
  load_tw<LOGH>(tws, a);                                                     \
  pdl_wait(); /* every access below touches the previous stage's output */   \
  double2* scr = C::SMEM_SCR ? sm + C::NR * C::H + (C::M / 4 + 1) + team * 3 * C::H             \
                             : a.scratch + ((long long)blockIdx.x * C::NR + team) * (Q == 4 ? 10 : 3) * C::H;

// ------------------------------------------------------------------ kernels
// Team scratch (L2): Q = 2: [z1 | F row 0 | F row 1] (3H).  Q = 4: [z1 z2 z3 |
// Bluestein output y (2H, N <= 2H does not fit the team's H-entry shared row)
// | F row 0 (2H) | F row 1 (2H) | correlation outputs y[3H + k] (H)] (10H).
template <int Q, int LOGH>
struct YStage {  // where a Bluestein output of length N waits for its next pass
  double2* X;
  double2* g;
  __device__ __forceinline__ double2& operator()(int k) const {
    if constexpr (Q == 4)
      return g[k];
    else
      return X[phys(k)];
  }
};

// phi DFT of each ring (forward): AT[k][t] = (2 pi/N) sum_p f[t][p] e^{-2 pi i kp/N}
// complex: k < N, AT is (N, L); real: k < L (rfft bins), AT is (L, L).
// Real rings go two per transform: z = f_t + i f_{t+1}, Z = DFT_N(z), then
// F_t[k] = (Z[k] + conj Z[N-k]) / 2 and F_{t+1}[k] = (Z[k] - conj Z[N-k]) / 2i.
template <bool REAL, int LOGH, bool SH = false, int Q = 2>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_phi_fwd(FftArgs a) {
  FFT_PROLOGUE
  const int L = a.L, N = a.N;
  const int kout = REAL ? L : N;
  constexpr int MQ = Q * C::H;  // the convolution length (the DFTs' scale)
  const YStage<Q, LOGH> ys{X, scr + 3 * C::H};
  const double sc = 2.0 * 3.141592653589793 / (double)N / (double)MQ;
  const int per_map = REAL ? (a.nrows + 1) / 2 : a.nrows;  // transforms per map
  for (int row = first_row<C::NR>(a, team); row < per_map * a.nmaps; row += gridDim.x * C::NR) {
    const int map = row / per_map, q = row - map * per_map;
    double2* at = (double2*)a.out + (long long)map * a.out_stride;
    if (REAL) {
      const int tl = 2 * q, t = a.t0 + tl;
      const bool two = tl + 1 < a.nrows;
      const double* f = (const double*)a.in + (long long)map * a.in_stride + (long long)tl * N;
      const double* f2 = two ? f + N : f;
      bluestein<LOGH, false, false, Q>(
          X, tws, scr, a, lt, team,
          [&](int n) { return make_double2(f[n], two ? f2[n] : 0.0); },
          [&](int k, double2 y) {
            if (k < N) ys(k) = cmulc(y, a.chirp[k]);
          });
      team_sync<C::TEAM>(team);
      const double h = 0.5 * sc;
      // the two rings are neighbouring columns of AT: one aligned 32-byte store per bin
      const bool wide = two && !(L & 1) && !(t & 1) && (((unsigned long long)at & 31ull) == 0);
      for (int k = lt; k < L; k += C::TEAM) {
        const double2 zk = ys(k), zn = ys(k ? N - k : 0);
        const double2 v1 = make_double2(h * (zk.x + zn.x), h * (zk.y - zn.y));
        const double2 v2 = make_double2(h * (zk.y + zn.y), h * (zn.x - zk.x));
        if (wide) {
          asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(at + (long long)k * L + t),
                       "d"(v1.x), "d"(v1.y), "d"(v2.x), "d"(v2.y)
                       : "memory");
        } else {
          at[(long long)k * L + t] = v1;
          if (two) at[(long long)k * L + t + 1] = v2;
        }
      }
      team_sync<C::TEAM>(team);
    } else {
      const int tl = q, t = a.t0 + tl;
      auto fin = [&](int k, double2 y) {
        if (k < kout) {
          const double2 v = cscale(cmulc(y, a.chirp[k]), sc);
          if constexpr (SH)
            at[a.row_off[k] + tl] = v;  // shard send layout (per destination rank)
          else
            at[at_idx(k, t, L)] = v;
        }
      };
      const double2* f = (const double2*)a.in + (long long)map * a.in_stride + (long long)tl * N;
      bluestein<LOGH, false, false, Q>(X, tws, scr, a, lt, team, [&](int n) { return f[n]; }, fin);
    }
  }
}

// Inverse theta rows go two per Bluestein transform.  Row m's synthesis
// output is a reflection about t = L-1 with sign eps_m = (-1)^(m+s)
// (F_{m,-m'} = eps_m F_{m,m'}, mw.py:400-401), and consecutive orders m, m+1
// have opposite signs, so the transform of S_1 + i S_2 separates exactly:
// z = y_1 + i y_2 and eps_1 z[N-1-t] = y_1[t] - i y_2[t].
// Tasks pair the orders of magnitude 2k and 2k+1 within the +m block and
// within the -m block, so a sharded order range [m0, m1) with even bounds
// pairs exactly as the whole plane does (bit-identical shards).
__device__ __forceinline__ int pair_count(int lo, int hi) {  // k with [2k, 2k+1] meeting [lo, hi)
  return hi > lo ? (hi - 1) / 2 - lo / 2 + 1 : 0;
}
__device__ __forceinline__ int theta_tasks(int m0, int m1, bool real) {
  return pair_count(m0, m1) + (real ? 0 : pair_count(m0 > 0 ? m0 : 1, m1));
}
// rows of task q: i1 and, when it returns 2, i1 + 1 (row_order indexing)
__device__ __forceinline__ int theta_task(int q, int m0, int m1, bool real, int& i1) {
  const int tp = pair_count(m0, m1);
  int lo = m0, off = 0;
  if (!real && q >= tp) {
    q -= tp;
    lo = m0 > 0 ? m0 : 1;
    off = m1 - m0;
  }
  const int k = lo / 2 + q;
  const int first = max(2 * k, lo), last = min(2 * k + 1, m1 - 1);
  i1 = off + (first - lo);
  return last - first + 1;
}

// theta stage of the forward transform for each order row (m from row_order):
// extension (mw.py:161-177), DFT_N + twist (:180-192), weight correlation
// (:244-251) and m' fold (:273-285, 504-511), written in the forward core's
// staging layout gfT (ldw columns, +m / -m halves).  Two rows per Bluestein
// transform: the extended sequence x of order m satisfies x[N-1-n] = eps_m x[n]
// except at the self-mirrored n = L-1, so its DFT obeys
//   Z[-k] e^{2 pi i k/N} = eps_m Z[k] + (1 - eps_m) x[L-1] (-1)^k e^{i pi k/N},
// and with eps_{m+1} = -eps_m the transform of x_m + i x_{m+1} separates.
template <bool REAL, int LOGH, bool SH = false, int Q = 2>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_theta_fwd(FftArgs a) {
  FFT_PROLOGUE
  // F of the task's rows (N <= H at Q = 2, N <= 2H at Q = 4)
  double2* scrF[2] = {scr + (Q == 4 ? 5 : 1) * C::H, scr + (Q == 4 ? 7 : 2) * C::H};
  double2* y3 = scr + 9 * C::H;  // Q = 4: correlation outputs y[3H + k]
  const YStage<Q, LOGH> ys{X, scr + 3 * C::H};
  const int L = a.L, N = a.N, ldw = a.ldw;
  constexpr int H = C::H, M = Q * C::H;  // M: the convolution length
  // Two rows per transform from H = 2048 (L >= 513) on, where the rows
  // outnumber the teams; below, every row gets its own team in one wave and
  // the shorter unpaired task (4 instead of 6 half-convolutions) wins
  // (L=64: 79 -> 46 us, L=256: 128 -> 74 us per launch).
  // (at Q = 2 the sizes H >= 2048 run k_theta_fwd2, the decoupled form of the
  // paired task; this fused paired form serves the quarter split, Q = 4)
  constexpr bool PAIR = LOGH >= 11;
  const int ntask = PAIR ? theta_tasks(a.m0, a.m1, REAL) : a.nrows;
  for (int task = first_row<C::NR>(a, team); task < ntask * a.nmaps; task += gridDim.x * C::NR) {
    const int map = task / ntask, q = task - map * ntask;
    int i1 = q;
    const bool two = PAIR && theta_task(q, a.m0, a.m1, REAL, i1) == 2;
    int mr[2], il[2];
    double eps[2];
    const double2* g[2];
    for (int u = 0; u < 2; u++) {
      il[u] = two ? i1 + u : i1;
      mr[u] = row_order(il[u], a.m0, a.m1, REAL);
      eps[u] = (((mr[u] + (REAL ? 0 : stage_spin(a, map))) & 1) ? -1.0 : 1.0);
      g[u] = (const double2*)a.in + (long long)map * a.in_stride +
             (REAL ? (long long)mr[u] * L : at_idx(fbin(mr[u], N), 0, L));
    }
    // ring t of row u: dense AT row (real) / bin pair (complex), or the shard's receive layout
    auto gin = [&](int u, int t) -> double2 {
      if constexpr (SH)
        return ((const double2*)a.in)[a.col_off[t] + (long long)il[u] * a.col_stride[t]];
      else
        return g[u][REAL ? t : 2 * t];
    };
    // 1. Bluestein DFT_N of the periodic extension(s): X[k] = M Z[k]
    auto ext = [&](int u, int n) { return n < L ? gin(u, n) : cscale(gin(u, 2 * L - 2 - n), eps[u]); };
    bluestein<LOGH, false, PAIR, Q>(
        X, tws, scr, a, lt, team,
        [&](int n) {
          const double2 x1 = ext(0, n);
          if (!two) return x1;
          const double2 x2 = ext(1, n);
          return make_double2(x1.x - x2.y, x1.y + x2.x);  // x1 + i x2
        },
        [&](int k, double2 y) {
          if (k < N) ys(k) = cmulc(y, a.chirp[k]);
        });
    team_sync<C::TEAM>(team);
    // 2. separate the two rows; F[k] = Z[k] tau(f(k)) / (2 pi N)
    {
      double2 cc = make_double2(0.0, 0.0);  // M (1 - eps_u) x_u[L-1] (i for the second row)
      if (two) {
        const double2 c1 = gin(0, L - 1), c2 = gin(1, L - 1);
        cc = eps[0] < 0 ? make_double2(2.0 * M * c1.x, 2.0 * M * c1.y)
                        : make_double2(-2.0 * M * c2.y, 2.0 * M * c2.x);
      }
      // four elements per thread and pass: the table loads (L2) of a pass are in flight together
      constexpr int U = 4;
      for (int k0 = lt; k0 < N; k0 += U * C::TEAM) {
        double2 r2[U], wk[U], ck[U];
#pragma unroll
        for (int v = 0; v < U; v++) {
          const int k = min(k0 + v * C::TEAM, N - 1);
          r2[v] = __ldg(&a.rho2[k]);
          if (two) {
            wk[v] = __ldg(&a.wnk[k]);
            ck[v] = __ldg(&a.cen[k]);
          }
        }
#pragma unroll
        for (int v = 0; v < U; v++) {
          const int k = k0 + v * C::TEAM;
          if (k >= N) break;
          const double2 zk = ys(k);
          if (!two) {
            scrF[0][k] = cmul(zk, r2[v]);
            continue;
          }
          const double2 zn = ys(k ? N - k : 0);
          const double2 bk = csub(cmul(zn, wk[v]), cmul(cc, ck[v]));
          const double2 eb = cscale(bk, eps[0]);
          const double2 s1 = cadd(zk, eb), s2 = csub(zk, eb);  // 2 Z_1, 2i Z_2
          scrF[0][k] = cscale(cmul(s1, r2[v]), 0.5);
          scrF[1][k] = cscale(cmul(make_double2(s2.y, -s2.x), r2[v]), 0.5);
        }
      }
    }
    team_sync<C::TEAM>(team);
    for (int u = 0; u < (two ? 2 : 1); u++) {
      const double2* F = scrF[u];
      const int m = mr[u];
      const bool neg = !REAL && m < 0;
      const int am = neg ? -m : m;
      // 3. weight correlation on F placed in FFT order (f at f mod M)
      auto Fpl = [&](int p) -> double2 {
        if (p < L) return F[p];
        if (p >= M - L + 1) return F[p - M + N];
        return make_double2(0.0, 0.0);
      };
      if constexpr (Q == 4) {
        // F sits at positions p < L and p > M - L only (L <= H): quarters
        // r = 0 and r = 3 of the input; the fold needs y[j] and y[M - j] =
        // y[3H + (H - j)], i.e. the merge's p = 0 and p = 3 outputs
#pragma unroll 1
        for (int qq = 3; qq >= 1; qq--) {
          conv_half<LOGH, PAIR>(
              X, tws, a.specw + qq * H, lt, team,
              [&](int j) {
                return cmul(cadd(Fpl(j), rot_mi(Fpl(j + 3 * H), 3 * qq)), omega(a.twM, j * qq, M));
              },
              [&](int k, double2 v) { scr[(qq - 1) * H + k] = v; });
        }
        conv_half<LOGH, PAIR>(
            X, tws, a.specw, lt, team, [&](int j) { return cadd(Fpl(j), Fpl(j + 3 * H)); },
            [&](int k, double2 z0) {
              const double2 t1 = cmulc(scr[k], omega(a.twM, k, M));
              const double2 t2 = cmulc(scr[H + k], omega(a.twM, 2 * k, M));
              const double2 t3 = cmulc(scr[2 * H + k], omega(a.twM, 3 * k, M));
              X[phys(k)] = cadd(cadd(z0, t2), cadd(t1, t3));        // y[k]
              const double2 e = csub(z0, t2), d = csub(t1, t3);
              y3[k] = make_double2(e.x + d.y, e.y - d.x);          // y[3H + k] = e - i d
            });
      } else {
        conv_half<LOGH, PAIR>(
            X, tws, a.specw + H, lt, team,
            [&](int j) { return cmul(csub(Fpl(j), Fpl(j + H)), omega(tws, j, M)); },
            [&](int k, double2 v) { scr[k] = v; });
        conv_half<LOGH, PAIR>(
            X, tws, a.specw, lt, team, [&](int j) { return cadd(Fpl(j), Fpl(j + H)); },
            [&](int k, double2 v) { X[phys(k)] = v; });
      }
      team_sync<C::TEAM>(team);
      // 4. G(m') = y[m' mod M]/M; fold gf[j] = G(j) + s G(-j); write staging column
      const double sig = eps[u];  // (-1)^(m+s) (complex) / (-1)^m (real), mw.py:273-285
      const double inv = 1.0 / (double)M;
      double2* gT =
          (double2*)a.out + (long long)map * a.out_stride + (neg ? (long long)L * ldw : 0);
      for (int j = lt; j < L; j += C::TEAM) {
        double2 v;
        if constexpr (Q == 4) {
          v = X[phys(j)];
          if (j > 0) {
            const double2 w = y3[H - j];  // y[M - j]
            v = make_double2(v.x + sig * w.x, v.y + sig * w.y);
          }
        } else {
          v = cadd(X[phys(j)], cmulc(scr[j], omega(tws, j, M)));
          if (j > 0) {
            const int k = H - j;  // position M - j = k + H
            const double2 w = csub(X[phys(k)], cmulc(scr[k], omega(tws, k, M)));
            v = make_double2(v.x + sig * w.x, v.y + sig * w.y);
          }
        }
        v = cscale(v, inv);
        if (neg && (j & 1)) v = make_double2(-v.x, -v.y);
        gT[blk<kTileCols>(j, am, L)] = v;
        if (!REAL && m == 0)
          gT[(long long)L * ldw + blk<kTileCols>(j, 0, L)] = (j & 1) ? make_double2(-v.x, -v.y) : v;
      }
      team_sync<C::TEAM>(team);
    }
  }
}

// ------------------------------------------------------------- tensor memory
// The decoupled kernels park thread-private rows in the SM's 256 KB of tensor
// memory (512 columns x 128 lanes x 32 bit) instead of L2: a warp reaches the
// 32 lanes of its quarter (warp % 4) with tcgen05.ld/st.32x32b, one lane per
// thread, so a thread's 16 complex values of a parked row are 64 consecutive
// columns of its own lane.  The four warps of a lane quarter take 128 columns
// each: two parked rows per team (slots 0 and 1).  No tensor-core instruction
// is involved; this is TMEM as a 12-cycle scratchpad (B300_MICROARCH.md).
struct Tmem {
  uint32_t base;  // this thread's warp: lane quarter + 128-column window
  __device__ __forceinline__ uint32_t at(int slot, int r) const { return base + slot * 64 + r * 4; }
  // four consecutive complex values (16 columns) per instruction
  __device__ __forceinline__ void st4(int slot, int r, const double2 (&v)[4]) const {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(at(slot, r)),
        "r"(__double2loint(v[0].x)), "r"(__double2hiint(v[0].x)), "r"(__double2loint(v[0].y)),
        "r"(__double2hiint(v[0].y)), "r"(__double2loint(v[1].x)), "r"(__double2hiint(v[1].x)),
        "r"(__double2loint(v[1].y)), "r"(__double2hiint(v[1].y)), "r"(__double2loint(v[2].x)),
        "r"(__double2hiint(v[2].x)), "r"(__double2loint(v[2].y)), "r"(__double2hiint(v[2].y)),
        "r"(__double2loint(v[3].x)), "r"(__double2hiint(v[3].x)), "r"(__double2loint(v[3].y)),
        "r"(__double2hiint(v[3].y))
        : "memory");
  }
  __device__ __forceinline__ void ld4(int slot, int r, double2 (&v)[4]) const {
    int w[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
          "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]),
          "=r"(w[14]), "=r"(w[15])
        : "r"(at(slot, r))
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; i++)
      v[i] = make_double2(__hiloint2double(w[4 * i + 1], w[4 * i]),
                          __hiloint2double(w[4 * i + 3], w[4 * i + 2]));
  }
  __device__ __forceinline__ void st_wait() const {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
};
// whole-CTA: warp 0 allocates all 512 columns (one CTA per SM: these kernels
// fill the SM's shared memory), every thread gets its window
__device__ __forceinline__ Tmem tmem_open(uint32_t* slot) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t warp = threadIdx.x >> 5;
  return Tmem{*slot + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 128u};
}
__device__ __forceinline__ void tmem_close(uint32_t* slot) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*slot) : "memory");
}

// ---------------------------------------------------------------------------
// Decoupled form of the stage kernels (H >= 2048): every half-convolution runs
// ALL its passes on the team's shared row through one out-of-line copy
// (conv_smem), and everything that touches global memory is a short
// element-wise loop over the 16 row positions a thread OWNS,
//   pos(r) = lt + r TEAM (r < 8),   H - (lt + (r-8) TEAM) (r >= 8; H/2 for 0),
// so positions j and H - j (the fold's partners) belong to one thread and the
// rows that wait between passes (the half-1 result z1, the first pass's input
// for half 0, the second row's F) are thread-private "parked" arrays in the
// team's L2 scratch, written and read back coalesced by the same thread.
// The loops issue their independent loads in batches, so a global round trip
// is paid once per loop instead of inside a radix-16 butterfly's register
// budget, and the kernel is a third of the fused form's code size.
template <int LOGH>
__device__ __noinline__ void conv_smem(double2* X, const double2* tw, const double2* S, int lt,
                                       int team) {
  using C = Cfg<LOGH>;
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  constexpr int RL = 1 << C::lr(C::NP - 1), nL = C::n_at(C::NP - 1);
  team_sync<C::TEAM>(team);
  dif_chain<LOGH, 0>(tw, lt, team, lds, lds, sts);
  pass<RL, 2, C::H, C::M, nL, C::TEAM>(tw, S, lt, lds, sts);
  team_sync<C::TEAM>(team);
  dit_chain<LOGH, C::NP - 2>(tw, lt, team, sts, lds, sts);
}

template <int LOGH>
struct Own {
  using C = Cfg<LOGH>;
  static constexpr int E = C::H / C::TEAM;  // positions per thread (16)
  static constexpr int B = 4;               // loads in flight per array and batch
  __device__ static __forceinline__ int pos(int r, int lt) {
    if (r < E / 2) return lt + r * C::TEAM;
    const int q = lt + (r - E / 2) * C::TEAM;
    return q ? C::H - q : C::H / 2;
  }
};

template <bool REAL, int LOGH, bool SH = false>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_theta_fwd2(FftArgs a) {
  constexpr int Q = 2;
  __shared__ uint32_t tmem_slot;
  FFT_PROLOGUE
  using O = Own<LOGH>;
  constexpr int H = C::H, M = 2 * C::H, T = C::TEAM, E = O::E, B = O::B;
  static_assert(E == 16 && B == 4, "16 positions per thread, parked four at a time");
  // parked rows: TMEM slot 0 = Bluestein input / F of the running row,
  // slot 1 = z1 of the running convolution; L2 scratch: F of the second row
  const Tmem tm = tmem_open(&tmem_slot);
  double2* const PC = scr;
  const int L = a.L, N = a.N, ldw = a.ldw;
  const int ntask = theta_tasks(a.m0, a.m1, REAL);
  for (int task = first_row<C::NR>(a, team); task < ntask * a.nmaps; task += gridDim.x * C::NR) {
    const int map = task / ntask, q = task - map * ntask;
    int i1 = q;
    const bool two = theta_task(q, a.m0, a.m1, REAL, i1) == 2;
    int mr[2], il[2];
    double eps[2];
    const double2* g[2];
    for (int u = 0; u < 2; u++) {
      il[u] = two ? i1 + u : i1;
      mr[u] = row_order(il[u], a.m0, a.m1, REAL);
      eps[u] = (((mr[u] + (REAL ? 0 : stage_spin(a, map))) & 1) ? -1.0 : 1.0);
      g[u] = (const double2*)a.in + (long long)map * a.in_stride +
             (REAL ? (long long)mr[u] * L : at_idx(fbin(mr[u], N), 0, L));
    }
    // ring t of row u: dense AT row (real) / bin pair (complex), or the shard's receive layout
    auto gin = [&](int u, int t) -> double2 {
      if constexpr (SH)
        return ((const double2*)a.in)[a.col_off[t] + (long long)il[u] * a.col_stride[t]];
      else
        return g[u][REAL ? t : 2 * t];
    };
    // complex dense layout: the task's two bins are one pair, both rows of a ring in 32 bytes
    const bool pair32 = !REAL && !SH && two;
    const double2* gpair = pair32 ? (g[0] < g[1] ? g[0] : g[1]) : nullptr;
    const bool swapped = pair32 && g[1] < g[0];
    // A. Bluestein input xb[n] = (x_1 + i x_2)[n] conj(c[n]) of the extended rows:
    //    parked for half 0, times w^n into the row for half 1
#pragma unroll
    for (int r0 = 0; r0 < E; r0 += B) {
      double2 x1[B], x2[B], ch[B];
#pragma unroll
      for (int v = 0; v < B; v++) {
        const int n = min(O::pos(r0 + v, lt), N - 1), src = n < L ? n : 2 * L - 2 - n;
        if (pair32) {
          double2 lo, hi;
          // (not volatile: the loads may move above the previous batch's stores like plain loads)
          asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
              : "=d"(lo.x), "=d"(lo.y), "=d"(hi.x), "=d"(hi.y)
              : "l"(gpair + 2 * src));
          x1[v] = swapped ? hi : lo;
          x2[v] = swapped ? lo : hi;
        } else {
          x1[v] = gin(0, src);
          x2[v] = two ? gin(1, src) : make_double2(0.0, 0.0);
        }
        ch[v] = a.chirp[n];
      }
#pragma unroll
      for (int v = 0; v < B; v++) {
        const int p = O::pos(r0 + v, lt);
        double2 xb = make_double2(0.0, 0.0);
        if (p < N) {
          const double e0 = p < L ? 1.0 : eps[0], e1 = p < L ? 1.0 : eps[1];
          xb = cmulc(make_double2(e0 * x1[v].x - e1 * x2[v].y, e0 * x1[v].y + e1 * x2[v].x), ch[v]);
        }
        x1[v] = xb;
        X[phys(p)] = cmul(xb, omega(tws, p, M));
      }
      tm.st4(0, r0, x1);
    }
    tm.st_wait();
    conv_smem<LOGH>(X, tws, a.specf + H, lt, team);
    // C. park z1, refill the row with the parked input
#pragma unroll
    for (int r0 = 0; r0 < E; r0 += B) {
      double2 xa[B], z1[B];
      tm.ld4(0, r0, xa);
#pragma unroll
      for (int v = 0; v < B; v++) {
        const int pp = phys(O::pos(r0 + v, lt));
        z1[v] = X[pp];
        X[pp] = xa[v];
      }
      tm.st4(1, r0, z1);
    }
    tm.st_wait();
    conv_smem<LOGH>(X, tws, a.specf, lt, team);
    // E. merge the halves in place: y[k] = z0[k] + conj(w^k) z1[k], k < N (the
    //    output chirp is folded into the separation tables)
#pragma unroll
    for (int r0 = 0; r0 < E; r0 += B) {
      double2 zb[B];
      tm.ld4(1, r0, zb);
#pragma unroll
      for (int v = 0; v < B; v++) {
        const int p = O::pos(r0 + v, lt), pp = phys(p);
        if (p < N) X[pp] = cadd(X[pp], cmulc(zb[v], omega(tws, p, M)));
      }
    }
    team_sync<C::TEAM>(team);
    // F. separate the two rows (common.cuh, sep1..3); F[k] is parked at the
    //    position the weight correlation wants bin k: k (k < L), k + H - N (k >= L)
    {
      double2 cc = make_double2(0.0, 0.0);  // M (1 - eps_u) x_u[L-1] (i for the second row)
      if (two) {
        const double2 c1 = gin(0, L - 1), c2 = gin(1, L - 1);
        cc = eps[0] < 0 ? make_double2(2.0 * M * c1.x, 2.0 * M * c1.y)
                        : make_double2(-2.0 * M * c2.y, 2.0 * M * c2.x);
      }
#pragma unroll
      for (int r0 = 0; r0 < E; r0 += B) {
        double2 t1[B], t2[B], t3[B], f0[B];
        int kk[B];
#pragma unroll
        for (int v = 0; v < B; v++) {
          const int j = O::pos(r0 + v, lt);
          kk[v] = r0 + v < E / 2 ? (j < L ? j : -1) : (j >= H - L + 1 ? j - H + N : -1);
          const int k = max(kk[v], 0);
          t1[v] = __ldg(&a.sep1[k]);
          if (two) {
            t2[v] = __ldg(&a.sep2[k]);
            t3[v] = __ldg(&a.sep3[k]);
          }
        }
#pragma unroll
        for (int v = 0; v < B; v++) {
          const int k = kk[v];
          double2 f1 = make_double2(0.0, 0.0);
          f0[v] = f1;
          if (k >= 0) {
            const double2 av = cmul(X[phys(k)], t1[v]);
            if (!two) {
              f0[v] = make_double2(2.0 * av.x, 2.0 * av.y);
            } else {
              const double2 bv =
                  cscale(csub(cmul(X[phys(k ? N - k : 0)], t2[v]), cmul(cc, t3[v])), eps[0]);
              f0[v] = cadd(av, bv);
              const double2 d = csub(av, bv);
              f1 = make_double2(d.y, -d.x);  // -i (a - b)
            }
          }
          if (two) PC[(r0 + v) * T + lt] = f1;
        }
        tm.st4(0, r0, f0);
      }
      tm.st_wait();
    }
    team_sync<C::TEAM>(team);
    for (int u = 0; u < (two ? 2 : 1); u++) {
      const int m = mr[u];
      const bool neg = !REAL && m < 0;
      const int am = neg ? -m : m;
      // G. half 1 of the weight correlation: (F(j) - F(j + H)) w^j (the two never overlap)
#pragma unroll
      for (int r0 = 0; r0 < E; r0 += B) {
        double2 f[B];
        if (u == 0) {
          tm.ld4(0, r0, f);
        } else {
#pragma unroll
          for (int v = 0; v < B; v++) f[v] = PC[(r0 + v) * T + lt];
          tm.st4(0, r0, f);
        }
#pragma unroll
        for (int v = 0; v < B; v++) {
          const int p = O::pos(r0 + v, lt);
          const double2 w = cmul(f[v], omega(tws, p, M));
          X[phys(p)] = r0 + v < E / 2 ? w : make_double2(-w.x, -w.y);
        }
      }
      tm.st_wait();
      conv_smem<LOGH>(X, tws, a.specw + H, lt, team);
      // I. park z1, refill with F for half 0
#pragma unroll
      for (int r0 = 0; r0 < E; r0 += B) {
        double2 f[B], z1[B];
        tm.ld4(0, r0, f);
#pragma unroll
        for (int v = 0; v < B; v++) {
          const int pp = phys(O::pos(r0 + v, lt));
          z1[v] = X[pp];
          X[pp] = f[v];
        }
        tm.st4(1, r0, z1);
      }
      tm.st_wait();
      conv_smem<LOGH>(X, tws, a.specw, lt, team);
      // K. G(m') = y[m' mod M]/M, y[j] = z0[j] + conj(w^j) z1[j], y[M - j] = z0[H-j] -
      //    conj(w^(H-j)) z1[H-j]; fold gf[j] = G(j) + s G(-j); write the staging column
      const double sig = eps[u], inv = 1.0 / (double)M;
      double2* gT =
          (double2*)a.out + (long long)map * a.out_stride + (neg ? (long long)L * ldw : 0);
#pragma unroll
      for (int r0 = 0; r0 < E / 2; r0 += B) {
        double2 za[B], zp[B];
        tm.ld4(1, r0, za);
        tm.ld4(1, r0 + E / 2, zp);
#pragma unroll
        for (int v = 0; v < B; v++) {
          const int j = lt + (r0 + v) * T;
          if (j >= L) continue;
          double2 y = cadd(X[phys(j)], cmulc(za[v], omega(tws, j, M)));
          if (j > 0) {
            const int k = H - j;
            const double2 w = csub(X[phys(k)], cmulc(zp[v], omega(tws, k, M)));
            y = make_double2(y.x + sig * w.x, y.y + sig * w.y);
          }
          y = cscale(y, inv);
          if (neg && (j & 1)) y = make_double2(-y.x, -y.y);
          gT[blk<kTileCols>(j, am, L)] = y;
          if (!REAL && m == 0)
            gT[(long long)L * ldw + blk<kTileCols>(j, 0, L)] = (j & 1) ? make_double2(-y.x, -y.y) : y;
        }
      }
    }
  }
  tmem_close(&tmem_slot);
}

// inverse theta synthesis per order row: rows[t] = sum_m' S[bin(m')] e^{+2 pi i m' t/N}
// (S already carries the core's twist), keep t < L, write Out[t][col].
template <bool REAL, int LOGH, bool SH = false, int Q = 2>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_theta_inv(FftArgs a) {
  FFT_PROLOGUE
  const int L = a.L, N = a.N;
  const int ocols = a.pitch ? a.pitch : (REAL ? L : N);
  const YStage<Q, LOGH> ys{X, scr + 3 * C::H};
  const double inv = 1.0 / (double)(Q * C::H);
  const int ntask = theta_tasks(a.m0, a.m1, REAL);
  for (int task = first_row<C::NR>(a, team); task < ntask * a.nmaps; task += gridDim.x * C::NR) {
    const int map = task / ntask, q = task - map * ntask;
    int i1;
    const bool two = theta_task(q, a.m0, a.m1, REAL, i1) == 2;
    int mr[2], col[2], il[2];
    const double2* sp[2];
    for (int u = 0; u < 2; u++) {
      il[u] = two ? i1 + u : i1;
      mr[u] = row_order(il[u], a.m0, a.m1, REAL);
      const int r = REAL ? mr[u] : mr[u] + (L - 1);  // plane row of order m
      sp[u] = (const double2*)a.in + (long long)map * a.in_stride + (long long)r * N;
      col[u] = REAL ? mr[u] : fbin(mr[u], N);
    }
    const double e1 = (((mr[0] + (REAL ? 0 : stage_spin(a, map))) & 1) ? -1.0 : 1.0);
    double2* o = (double2*)a.out + (long long)map * a.out_stride;
    bluestein<LOGH, true, false, Q>(
        X, tws, scr, a, lt, team,
        [&](int n) {
          // half rows (core out_mode 3): S[N - x] = eps_m S[x] e^{-2 pi i x/N}; the
          // task's second order has the opposite sign, so S_1 + i S_2 mirrors to
          // eps_1 (S_1 - i S_2)[x] conj(wnk[x])
          const bool mirror = a.half && n >= L;
          const int nn = mirror ? N - n : n;
          const double2 s1 = sp[0][nn];
          double2 v = s1;
          if (two) {
            const double2 s2 = sp[1][nn];
            v = mirror ? make_double2(s1.x + s2.y, s1.y - s2.x)   // S_1 - i S_2
                       : make_double2(s1.x - s2.y, s1.y + s2.x);  // S_1 + i S_2
          }
          if (mirror) v = cscale(cmulc(v, __ldg(&a.wnk[nn])), e1);
          return v;
        },
        [&](int t, double2 y) {
          if (t < N) ys(t) = cscale(cmul(y, a.chirp[t]), inv);
        });
    team_sync<C::TEAM>(team);
    // ring t of order row u: dense (L, N) plane, or the shard's send layout
    auto oat = [&](int t, int u) -> double2& {
      if constexpr (SH)
        return o[a.row_off[t] + il[u]];
      else
        return o[(long long)t * ocols + col[u]];
    };
    // The task's two orders are neighbouring columns of the ring plane: with
    // an even row pitch and the lower column even, both values of a ring go
    // out as ONE aligned 32-byte store (a full sector) instead of two 16-byte
    // halves -- these transposed stores, one 128-byte line per lane, are a
    // fifth of the kernel (ncu: the store data held on the scoreboard).
    const int clo = min(col[0], col[1]);
    const bool wide = !SH && two && !(ocols & 1) && !(clo & 1) && col[0] + col[1] == 2 * clo + 1 &&
                      (((unsigned long long)o & 31ull) == 0);
    for (int t = lt; t < L; t += C::TEAM) {
      const double2 z = ys(t);
      double2 v1 = z, v2 = make_double2(0.0, 0.0);
      if (two) {
        const double2 zr = cscale(ys(N - 1 - t), e1);
        v1 = cscale(cadd(z, zr), 0.5);
        const double2 w = csub(z, zr);  // 2i y_2
        v2 = make_double2(0.5 * w.y, -0.5 * w.x);
      }
      if (REAL && mr[0] == 0) v1.y = 0.0;  // irfft ignores Im of the DC bin
      if (wide) {
        const double2 lo = col[0] < col[1] ? v1 : v2, hi = col[0] < col[1] ? v2 : v1;
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(o + (long long)t * ocols + clo),
                     "d"(lo.x), "d"(lo.y), "d"(hi.x), "d"(hi.y)
                     : "memory");
      } else {
        if (two) oat(t, 1) = v2;
        oat(t, 0) = v1;
      }
    }
    team_sync<C::TEAM>(team);
  }
}

// inverse phi synthesis per ring t: samples[t][p] = sum_m Out[t][bin(m)] e^{+2 pi i m p/N}
// (real: Hermitian completion of the m >= 0 half, real part out; mw.py:558).
// Real rings go two per transform: IDFT(X_t + i X_{t+1}) = x_t + i x_{t+1}.
template <bool REAL, int LOGH, bool SH = false, int Q = 2>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_phi_inv(FftArgs a) {
  FFT_PROLOGUE
  const int L = a.L, N = a.N;
  const double inv = 1.0 / (double)(Q * C::H);
  const int per_map = REAL ? (a.nrows + 1) / 2 : a.nrows;  // transforms per map
  for (int row = first_row<C::NR>(a, team); row < per_map * a.nmaps; row += gridDim.x * C::NR) {
    const int map = row / per_map, q = row - map * per_map;
    if (REAL) {
      const int tl = 2 * q, t = a.t0 + tl;
      const bool two = tl + 1 < a.nrows;
      const int pr = a.pitch ? a.pitch : L;
      const double2* h = (const double2*)a.in + (long long)map * a.in_stride + (long long)t * pr;
      const double2* h2 = h + pr;
      double* o = (double*)a.out + (long long)map * a.out_stride + (long long)tl * N;
      bluestein<LOGH, true, false, Q>(
          X, tws, scr, a, lt, team,
          [&](int n) {
            const double2 x1 = n < L ? h[n] : conjd(h[N - n]);
            if (!two) return x1;
            const double2 x2 = n < L ? h2[n] : conjd(h2[N - n]);
            return make_double2(x1.x - x2.y, x1.y + x2.x);  // x1 + i x2
          },
          [&](int p, double2 y) {
            if (p < N) {
              const double2 v = cmul(y, a.chirp[p]);
              o[p] = v.x * inv;
              if (two) o[N + p] = v.y * inv;
            }
          });
    } else {
      const int tl = q, t = a.t0 + tl;
      const double2* h = (const double2*)a.in + (long long)map * a.in_stride +
                         (long long)t * (a.pitch ? a.pitch : N);
      double2* o = (double2*)a.out + (long long)map * a.out_stride + (long long)tl * N;
      auto hin = [&](int n) -> double2 {  // dense rows, or the shard receive layout
        if constexpr (SH)
          return ((const double2*)a.in)[a.col_off[n] + (long long)tl * a.col_stride[n]];
        else
          return h[n];
      };
      bluestein<LOGH, true, false, Q>(X, tws, scr, a, lt, team, hin,
                            [&](int p, double2 y) {
                              if (p < N) o[p] = cscale(cmul(y, a.chirp[p]), inv);
                            });
    }
  }
}

// plan time: S_0 = DIF_H(k[j] + k[j+H]), S_1 = DIF_H((k[j] - k[j+H]) w^j) of a
// natural-order length-M kernel k, in the digit-reversed layout conv_half uses
// (every DIF pass including the innermost one, no spectrum).  One team.
template <int LOGH, int P, class LDS, class STS>
__device__ __forceinline__ void dif_all(const double2* tw, int lt, LDS lds, STS sts) {
  using C = Cfg<LOGH>;
  if constexpr (P < C::NP) {
    constexpr int R = 1 << C::lr(P), n = C::n_at(P);
    pass<R, 0, C::H, C::M, n, C::TEAM>(tw, nullptr, lt, lds, sts);
    team_sync<C::TEAM>(0);
    dif_all<LOGH, P + 1>(tw, lt, lds, sts);
  }
}

template <int LOGH, int Q = 2>
__global__ void __launch_bounds__(Cfg<LOGH>::KT, 1) k_spectrum(FftArgs a, const double2* kern, double2* spec) {
  FFT_PROLOGUE
  (void)scr;
  if (team != 0) return;
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  constexpr int H = C::H, MQ = Q * C::H;
  for (int part = 0; part < Q; part++) {
    for (int j = lt; j < H; j += C::TEAM) {
      double2 v;
      if constexpr (Q == 4) {  // x_q[j] = w_M^{jq} sum_r kern[j + rH] (-i)^{rq}
        v = make_double2(0.0, 0.0);
        for (int r = 0; r < 4; r++) v = cadd(v, rot_mi(kern[j + r * H], r * part));
        v = cmul(v, omega(a.twM, j * part, MQ));
      } else {
        const double2 u = kern[j], w = kern[j + H];
        v = part ? cmul(csub(u, w), omega(tws, j, C::M)) : cadd(u, w);
      }
      X[phys(j)] = v;
    }
    team_sync<C::TEAM>(0);
    dif_all<LOGH, 0>(tws, lt, lds, sts);
    constexpr int RL = 1 << C::lr(C::NP - 1);
    for (int j = lt; j < H; j += C::TEAM) {
      const int b = j / RL, k = j - b * RL;
      spec[part * H + spec_index<C::H, RL, C::TEAM>(b, k, b % C::TEAM)] = X[phys(j)];
    }
    team_sync<C::TEAM>(0);
  }
}

template <int LOGH>
size_t smem_bytes_t() {
  using C = Cfg<LOGH>;
  return sizeof(double2) * ((size_t)C::NR * C::H + C::M / 4 + 1 +
                            (C::SMEM_SCR ? (size_t)C::NR * 3 * C::H : 0));
}

template <int LOGH, class K>
static void launch_t(K kern, const FftArgs& a, int nsm, cudaStream_t st) {
  using C = Cfg<LOGH>;
  const size_t sm = smem_bytes_t<LOGH>();
  smem_attr_once((const void*)kern, sm);
  long long rows = (long long)a.nrows * a.nmaps;
  // resident CTAs per SM, within the per-SM scratch budget (NR * H * occ <= 8192)
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C::KT, sm);
  if (occ < 1) occ = 1;
  if (!C::SMEM_SCR && occ * C::NR * C::H > 8192) occ = 8192 / (C::NR * C::H);
  // few rows (small L): one CTA per row on as many SMs as there are rows,
  // rows dealt team-major (first_row); else CTA-major on the resident grid
  FftArgs b = a;
  b.spread = rows < (long long)nsm * occ * C::NR ? 1 : 0;
  long long grid = b.spread ? rows : (rows + C::NR - 1) / C::NR;
  if (grid > (long long)nsm * occ) grid = (long long)nsm * occ;
  if (grid < 1) grid = 1;
  launch_pdl(kern, dim3((unsigned)grid), dim3(C::KT), sm, st, b);
}

template <int LOGH>
static void launch_stage(int which, bool real, const FftArgs& a, int nsm, cudaStream_t st) {
  if constexpr (LOGH == 13) {
    if (a.Q == 4) {  // 4096 < L <= 8192: quarter split (and its shard layouts)
      const bool sh4 = !real && (a.row_off || a.col_off);
      switch (which) {
        case 0:
          real ? launch_t<LOGH>(k_phi_fwd<true, LOGH, false, 4>, a, nsm, st)
               : sh4 ? launch_t<LOGH>(k_phi_fwd<false, LOGH, true, 4>, a, nsm, st)
                     : launch_t<LOGH>(k_phi_fwd<false, LOGH, false, 4>, a, nsm, st);
          break;
        case 1:
          real ? launch_t<LOGH>(k_theta_fwd<true, LOGH, false, 4>, a, nsm, st)
               : sh4 ? launch_t<LOGH>(k_theta_fwd<false, LOGH, true, 4>, a, nsm, st)
                     : launch_t<LOGH>(k_theta_fwd<false, LOGH, false, 4>, a, nsm, st);
          break;
        case 2:
          real ? launch_t<LOGH>(k_theta_inv<true, LOGH, false, 4>, a, nsm, st)
               : sh4 ? launch_t<LOGH>(k_theta_inv<false, LOGH, true, 4>, a, nsm, st)
                     : launch_t<LOGH>(k_theta_inv<false, LOGH, false, 4>, a, nsm, st);
          break;
        default:
          real ? launch_t<LOGH>(k_phi_inv<true, LOGH, false, 4>, a, nsm, st)
               : sh4 ? launch_t<LOGH>(k_phi_inv<false, LOGH, true, 4>, a, nsm, st)
                     : launch_t<LOGH>(k_phi_inv<false, LOGH, false, 4>, a, nsm, st);
          break;
      }
      return;
    }
  }
  // SH: the m-column shard exchange layouts (complex maps only)
  const bool sh = !real && (a.row_off || a.col_off);
  switch (which) {
    case 0:
      real ? launch_t<LOGH>(k_phi_fwd<true, LOGH>, a, nsm, st)
           : sh ? launch_t<LOGH>(k_phi_fwd<false, LOGH, true>, a, nsm, st)
                : launch_t<LOGH>(k_phi_fwd<false, LOGH>, a, nsm, st);
      break;
    case 1:
      if constexpr (LOGH >= 11) {  // decoupled form (two rows per transform, TMEM parking)
        real ? launch_t<LOGH>(k_theta_fwd2<true, LOGH>, a, nsm, st)
             : sh ? launch_t<LOGH>(k_theta_fwd2<false, LOGH, true>, a, nsm, st)
                  : launch_t<LOGH>(k_theta_fwd2<false, LOGH>, a, nsm, st);
      } else {
        real ? launch_t<LOGH>(k_theta_fwd<true, LOGH>, a, nsm, st)
             : sh ? launch_t<LOGH>(k_theta_fwd<false, LOGH, true>, a, nsm, st)
                  : launch_t<LOGH>(k_theta_fwd<false, LOGH>, a, nsm, st);
      }
      break;
    case 2:
      real ? launch_t<LOGH>(k_theta_inv<true, LOGH>, a, nsm, st)
           : sh ? launch_t<LOGH>(k_theta_inv<false, LOGH, true>, a, nsm, st)
                : launch_t<LOGH>(k_theta_inv<false, LOGH>, a, nsm, st);
      break;
    default:
      real ? launch_t<LOGH>(k_phi_inv<true, LOGH>, a, nsm, st)
           : sh ? launch_t<LOGH>(k_phi_inv<false, LOGH, true>, a, nsm, st)
                : launch_t<LOGH>(k_phi_inv<false, LOGH>, a, nsm, st);
      break;
  }
}

template <int LOGH>
static void spectrum_t(const FftArgs& a, const double2* kern, double2* spec, cudaStream_t st) {
  const size_t sm = smem_bytes_t<LOGH>();
  if constexpr (LOGH == 13) {
    if (a.Q == 4) {
      smem_attr_once((const void*)k_spectrum<LOGH, 4>, sm);
      k_spectrum<LOGH, 4><<<1, Cfg<LOGH>::KT, sm, st>>>(a, kern, spec);
      return;
    }
  }
  smem_attr_once((const void*)k_spectrum<LOGH>, sm);
  k_spectrum<LOGH><<<1, Cfg<LOGH>::KT, sm, st>>>(a, kern, spec);
}

}  // namespace fft
}  // namespace mwsht

// One translation unit per FFT size (fft_<LOGH>.cu) instantiates these.
#define MWSHT_FFT_INSTANTIATE(K)                                                              \
  namespace mwsht {                                                                        \
  void fft_launch_##K(int which, bool real, const fft::FftArgs& a, int nsm, cudaStream_t st) { \
    fft::launch_stage<K>(which, real, a, nsm, st);                                         \
  }                                                                                        \
  void fft_spectrum_##K(const fft::FftArgs& a, const double2* kern, double2* spec,          \
                        cudaStream_t st) {                                                 \
    fft::spectrum_t<K>(a, kern, spec, st);                                                 \
  }                                                                                        \
  }
