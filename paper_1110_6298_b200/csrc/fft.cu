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
//   k_theta_inv  mw.py:441-446           spectrum row m -> IDFT_N -> Out[t][bin(m)], t < L
//   k_phi_inv    mw.py:437-438 / :558    Out row t -> IDFT_N -> samples row t
//   k_spectrum   plan time: S_0, S_1 of a length-M kernel
#include "common.cuh"

namespace mwsht {
namespace fft {

constexpr int kT = 512;  // threads per CTA



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

// radix schedule: log-radices of the DIF passes (outer first), each <= 4
__device__ __forceinline__ int npass(int logH) { return (logH + 3) / 4; }
__device__ __forceinline__ int nlog(int logH, int p) {
  const int np = npass(logH);
  const int base = logH / np, extra = logH - base * np;
  return base + (p < extra ? 1 : 0);
}

// One radix-R pass on sub-length n (stride s = n/R).  MODE:
//   0 DIF   (load via LD, butterfly, twiddle, store via ST)
//   1 DIT   (load, untwiddle, inverse butterfly, store)
//   2 fused innermost DIF + spectrum multiply + innermost DIT (s = 1, j = 0)
template <int R, int MODE, class LD, class ST>
__device__ __forceinline__ void pass(const double2* tw, const double2* spec, int H, int M, int n,
                                     LD ld, ST st) {
  const int s = n / R, nb = H / R, tstep = M / n;
#pragma unroll 2
  for (int b = threadIdx.x; b < nb; b += kT) {
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
      double2 sp[R];
#pragma unroll
      for (int k = 0; k < R; k++) sp[k] = spec[base + k];  // in flight during the butterfly
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

template <int MODE, class LD, class ST>
__device__ __forceinline__ void pass_r(int lr, const double2* tw, const double2* spec, int H, int M,
                                       int n, LD ld, ST st) {
  switch (lr) {
    case 1: pass<2, MODE>(tw, spec, H, M, n, ld, st); break;
    case 2: pass<4, MODE>(tw, spec, H, M, n, ld, st); break;
    case 3: pass<8, MODE>(tw, spec, H, M, n, ld, st); break;
    default: pass<16, MODE>(tw, spec, H, M, n, ld, st); break;
  }
}

// z = DIT_H( DIF_H(x) . S ), x given by IN(j), z delivered to OUT(k, z_k)
// (unnormalised).  The first DIF pass reads IN directly, the innermost DIF
// pass, the spectrum multiply and the innermost DIT pass are one register
// pass, and the last DIT pass hands results to OUT, so the H-point buffer X
// is touched by 2*(np-1) shared-memory passes instead of 2*np + 2.
#ifndef MWSHT_FFT_FUSE_IO
#define MWSHT_FFT_FUSE_IO 0
#endif
template <class IN, class OUT>
__device__ __forceinline__ void conv_half(double2* X, const double2* tw, const double2* S,
                                          const FftArgs& a, IN in, OUT out) {
  const int H = a.H, M = a.M, logH = a.logH, np = npass(logH);
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  __syncthreads();
  if (!MWSHT_FFT_FUSE_IO) {
    // streaming fill: independent iterations keep many global loads in flight
#pragma unroll 4
    for (int j = threadIdx.x; j < H; j += kT) X[phys(j)] = in(j);
    __syncthreads();
  }
  if (np == 1) {
    if (MWSHT_FFT_FUSE_IO) {
      pass_r<2>(logH, tw, S, H, M, H, in, out);
    } else {
      pass_r<2>(logH, tw, S, H, M, H, lds, sts);
      __syncthreads();
#pragma unroll 4
      for (int k = threadIdx.x; k < H; k += kT) out(k, X[phys(k)]);
    }
    __syncthreads();
    return;
  }
  int n = H;
  for (int p = 0; p < np - 1; p++) {
    const int lr = nlog(logH, p);
    if (p == 0 && MWSHT_FFT_FUSE_IO)
      pass_r<0>(lr, tw, S, H, M, n, in, sts);
    else
      pass_r<0>(lr, tw, S, H, M, n, lds, sts);
    n >>= lr;
    __syncthreads();
  }
  pass_r<2>(nlog(logH, np - 1), tw, S, H, M, n, lds, sts);
  __syncthreads();
  for (int p = np - 2; p >= 0; p--) {
    const int lr = nlog(logH, p);
    n <<= lr;
    if (p == 0 && MWSHT_FFT_FUSE_IO)
      pass_r<1>(lr, tw, S, H, M, n, lds, out);
    else
      pass_r<1>(lr, tw, S, H, M, n, lds, sts);
    __syncthreads();
  }
  if (!MWSHT_FFT_FUSE_IO) {
#pragma unroll 4
    for (int k = threadIdx.x; k < H; k += kT) out(k, X[phys(k)]);
    __syncthreads();
  }
}

__device__ __forceinline__ void load_tw(double2* tws, const FftArgs& a) {
  for (int i = threadIdx.x; i <= a.M / 4; i += kT) tws[i] = a.tw[i];
  __syncthreads();
}

__device__ __forceinline__ int fbin(int k, int N) { return k >= 0 ? k : k + N; }

// Bluestein DFT_N of x (fx(n), n < N): forward (conj chirp, spec f) or inverse
// (chirp, spec i).  Half 1 leaves z1 in scr; half 0 calls fin(k, y_k) with the
// merged y[k] = z0[k] + w^-k z1[k] (unnormalised; DFT = chirp' . y / M).
template <bool INV, class FX, class FIN>
__device__ __forceinline__ void bluestein(double2* X, const double2* tw, double2* scr,
                                          const FftArgs& a, FX fx, FIN fin) {
  const double2* spec = INV ? a.speci : a.specf;
  const int N = a.N, M = a.M;
  auto in1 = [&](int j) {
    double2 v = make_double2(0.0, 0.0);
    if (j < N) {
      const double2 c = a.chirp[j];
      v = INV ? cmul(fx(j), c) : cmulc(fx(j), c);
      v = cmul(v, omega(tw, j, M));
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
  auto out0 = [&](int k, double2 v) { fin(k, cadd(v, cmulc(scr[k], omega(tw, k, M)))); };
  conv_half(X, tw, spec + a.H, a, in1, out1);
  conv_half(X, tw, spec, a, in0, out0);
}

// ------------------------------------------------------------------ kernels

// phi DFT of each ring (forward): AT[k][t] = (2 pi/N) sum_p f[t][p] e^{-2 pi i kp/N}
// complex: k < N, AT is (N, L); real: k < L (rfft bins), AT is (L, L).
template <bool REAL>
__global__ void __launch_bounds__(kT, 1) k_phi_fwd(FftArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  double2* X = sm;
  double2* tws = sm + a.H;
  load_tw(tws, a);
  double2* scr = a.scratch + (long long)blockIdx.x * 2 * a.H;
  const int L = a.L, N = a.N;
  const int kout = REAL ? L : N;
  const double sc = 2.0 * 3.141592653589793 / (double)N / (double)a.M;
  for (int row = blockIdx.x; row < a.nrows * a.nmaps; row += gridDim.x) {
    const int map = row / a.nrows, tl = row - map * a.nrows, t = a.t0 + tl;
    double2* at = (double2*)a.out + (long long)map * a.out_stride;
    auto fin = [&](int k, double2 y) {
      if (k < kout) at[(long long)k * L + t] = cscale(cmulc(y, a.chirp[k]), sc);
    };
    if (REAL) {
      const double* f = (const double*)a.in + (long long)map * a.in_stride + (long long)tl * N;
      bluestein<false>(X, tws, scr, a, [&](int n) { return make_double2(f[n], 0.0); }, fin);
    } else {
      const double2* f = (const double2*)a.in + (long long)map * a.in_stride + (long long)tl * N;
      bluestein<false>(X, tws, scr, a, [&](int n) { return f[n]; }, fin);
    }
  }
}

// theta stage of the forward transform for each order row r (complex: r < N,
// m = r-(L-1); real: r < L, m = r): extension (mw.py:161-177), DFT_N + twist
// (:180-192), weight correlation (:244-251) and m' fold (:273-285, 504-511),
// written in the forward core's staging layout gfT (ldw columns, +m / -m halves).
template <bool REAL>
__global__ void __launch_bounds__(kT, 1) k_theta_fwd(FftArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  double2* X = sm;
  double2* tws = sm + a.H;
  load_tw(tws, a);
  double2* scr = a.scratch + (long long)blockIdx.x * 2 * a.H;  // z1
  double2* scrF = scr + a.H;                                     // F_raw (N)
  const int L = a.L, N = a.N, H = a.H, M = a.M, ldw = a.ldw;
  for (int row = blockIdx.x; row < a.nrows * a.nmaps; row += gridDim.x) {
    const int map = row / a.nrows, r = row - map * a.nrows;
    const int m = row_order(r, a.m0, a.m1, REAL);
    const bool neg = !REAL && m < 0;
    const int am = neg ? -m : m;
    const double eps = (((m + (REAL ? 0 : a.spin)) & 1) ? -1.0 : 1.0);
    const double2* g = (const double2*)a.in + (long long)map * a.in_stride +
                       (long long)(REAL ? m : fbin(m, N)) * L;
    // 1. Bluestein DFT_N of the periodic extension; F_raw[k] = y[k] conj(c[k]) tau(f(k))/M
    bluestein<false>(
        X, tws, scr, a, [&](int n) { return n < L ? g[n] : cscale(g[2 * L - 2 - n], eps); },
        [&](int k, double2 y) {
          if (k < N) scrF[k] = cmul(y, a.rho[k]);
        });
    __syncthreads();
    // 2. weight correlation on F placed in FFT order (f at f mod M)
    auto Fpl = [&](int p) -> double2 {
      if (p < L) return scrF[p];
      if (p >= M - L + 1) return scrF[p - M + N];
      return make_double2(0.0, 0.0);
    };
    conv_half(
        X, tws, a.specw + H, a,
        [&](int j) { return cmul(csub(Fpl(j), Fpl(j + H)), omega(tws, j, M)); },
        [&](int k, double2 v) { scr[k] = v; });
    conv_half(
        X, tws, a.specw, a, [&](int j) { return cadd(Fpl(j), Fpl(j + H)); },
        [&](int k, double2 v) { X[phys(k)] = v; });
    __syncthreads();
    // 3. G(m') = y[m' mod M]/M; fold gf[j] = G(j) + s G(-j); write staging column
    const double sig = eps;  // (-1)^(m+s) (complex) / (-1)^m (real), mw.py:273-285
    const double inv = 1.0 / (double)M;
    double2* gT = (double2*)a.out + (long long)map * a.out_stride + (neg ? (long long)L * ldw : 0);
    for (int j = threadIdx.x; j < L; j += kT) {
      double2 v = cadd(X[phys(j)], cmulc(scr[j], omega(tws, j, M)));
      if (j > 0) {
        const int k = H - j;  // position M - j = k + H
        const double2 u = csub(X[phys(k)], cmulc(scr[k], omega(tws, k, M)));
        v = make_double2(v.x + sig * u.x, v.y + sig * u.y);
      }
      v = cscale(v, inv);
      if (neg && (j & 1)) v = make_double2(-v.x, -v.y);
      gT[(long long)j * ldw + am] = v;
      if (!REAL && m == 0)
        gT[(long long)L * ldw + (long long)j * ldw] = (j & 1) ? make_double2(-v.x, -v.y) : v;
    }
  }
}

// inverse theta synthesis per order row: rows[t] = sum_m' S[bin(m')] e^{+2 pi i m' t/N}
// (S already carries the core's twist), keep t < L, write Out[t][col].
template <bool REAL>
__global__ void __launch_bounds__(kT, 1) k_theta_inv(FftArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  double2* X = sm;
  double2* tws = sm + a.H;
  load_tw(tws, a);
  double2* scr = a.scratch + (long long)blockIdx.x * 2 * a.H;
  const int L = a.L, N = a.N;
  const int ocols = REAL ? L : N;
  const double inv = 1.0 / (double)a.M;
  for (int row = blockIdx.x; row < a.nrows * a.nmaps; row += gridDim.x) {
    const int map = row / a.nrows, i = row - map * a.nrows;
    const int m = row_order(i, a.m0, a.m1, REAL);
    const int r = REAL ? m : m + (L - 1);  // plane row of order m
    const double2* s = (const double2*)a.in + (long long)map * a.in_stride + (long long)r * N;
    double2* o = (double2*)a.out + (long long)map * a.out_stride;
    const int col = REAL ? m : fbin(m, N);
    bluestein<true>(X, tws, scr, a, [&](int n) { return s[n]; }, [&](int t, double2 y) {
      if (t < L) {
        double2 v = cscale(cmul(y, a.chirp[t]), inv);
        if (REAL && r == 0) v.y = 0.0;  // irfft ignores Im of the DC bin
        o[(long long)t * ocols + col] = v;
      }
    });
  }
}

// inverse phi synthesis per ring t: samples[t][p] = sum_m Out[t][bin(m)] e^{+2 pi i m p/N}
// (real: Hermitian completion of the m >= 0 half, real part out; mw.py:558).
template <bool REAL>
__global__ void __launch_bounds__(kT, 1) k_phi_inv(FftArgs a) {
  extern __shared__ __align__(16) double2 sm[];
  double2* X = sm;
  double2* tws = sm + a.H;
  load_tw(tws, a);
  double2* scr = a.scratch + (long long)blockIdx.x * 2 * a.H;
  const int L = a.L, N = a.N;
  const double inv = 1.0 / (double)a.M;
  for (int row = blockIdx.x; row < a.nrows * a.nmaps; row += gridDim.x) {
    const int map = row / a.nrows, tl = row - map * a.nrows, t = a.t0 + tl;
    if (REAL) {
      const double2* h = (const double2*)a.in + (long long)map * a.in_stride + (long long)t * L;
      double* o = (double*)a.out + (long long)map * a.out_stride + (long long)tl * N;
      bluestein<true>(
          X, tws, scr, a, [&](int n) { return n < L ? h[n] : conjd(h[N - n]); },
          [&](int p, double2 y) {
            if (p < N) o[p] = cmul(y, a.chirp[p]).x * inv;
          });
    } else {
      const double2* h = (const double2*)a.in + (long long)map * a.in_stride + (long long)t * N;
      double2* o = (double2*)a.out + (long long)map * a.out_stride + (long long)tl * N;
      bluestein<true>(X, tws, scr, a, [&](int n) { return h[n]; }, [&](int p, double2 y) {
        if (p < N) o[p] = cscale(cmul(y, a.chirp[p]), inv);
      });
    }
  }
}

// plan time: S_0 = DIF_H(k[j] + k[j+H]), S_1 = DIF_H((k[j] - k[j+H]) w^j) of a
// natural-order length-M kernel k, in the digit-reversed layout conv_half uses.
__global__ void __launch_bounds__(kT, 1) k_spectrum(FftArgs a, const double2* kern, double2* spec) {
  extern __shared__ __align__(16) double2 sm[];
  double2* X = sm;
  double2* tws = sm + a.H;
  load_tw(tws, a);
  const int H = a.H, M = a.M, logH = a.logH, np = npass(logH);
  auto lds = [&](int i) { return X[phys(i)]; };
  auto sts = [&](int i, double2 v) { X[phys(i)] = v; };
  for (int half = 0; half < 2; half++) {
    for (int j = threadIdx.x; j < H; j += kT) {
      const double2 u = kern[j], v = kern[j + H];
      X[phys(j)] = half ? cmul(csub(u, v), omega(tws, j, M)) : cadd(u, v);
    }
    __syncthreads();
    int n = H;
    for (int p = 0; p < np; p++) {
      const int lr = nlog(logH, p);
      pass_r<0>(lr, tws, nullptr, H, M, n, lds, sts);
      n >>= lr;
      __syncthreads();
    }
    for (int j = threadIdx.x; j < H; j += kT) spec[half * H + j] = X[phys(j)];
    __syncthreads();
  }
}

size_t smem_bytes(int H, int M) { return sizeof(double2) * ((size_t)H + M / 4 + 1); }

template <class K>
static void launch_persistent(K kern, const FftArgs& a, int nsm, cudaStream_t st) {
  const size_t sm = smem_bytes(a.H, a.M);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  int grid = a.nrows * a.nmaps;
  if (grid > nsm) grid = nsm;
  kern<<<grid, kT, sm, st>>>(a);
}

}  // namespace fft

using fft::FftArgs;

void fft_launch(int which, bool real, const FftArgs& a, int nsm, cudaStream_t st) {
  switch (which) {
    case 0:
      real ? fft::launch_persistent(fft::k_phi_fwd<true>, a, nsm, st)
           : fft::launch_persistent(fft::k_phi_fwd<false>, a, nsm, st);
      break;
    case 1:
      real ? fft::launch_persistent(fft::k_theta_fwd<true>, a, nsm, st)
           : fft::launch_persistent(fft::k_theta_fwd<false>, a, nsm, st);
      break;
    case 2:
      real ? fft::launch_persistent(fft::k_theta_inv<true>, a, nsm, st)
           : fft::launch_persistent(fft::k_theta_inv<false>, a, nsm, st);
      break;
    default:
      real ? fft::launch_persistent(fft::k_phi_inv<true>, a, nsm, st)
           : fft::launch_persistent(fft::k_phi_inv<false>, a, nsm, st);
      break;
  }
}

void fft_spectrum(const FftArgs& a, const double2* kern, double2* spec, cudaStream_t st) {
  const size_t sm = fft::smem_bytes(a.H, a.M);
  cudaFuncSetAttribute(fft::k_spectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  fft::k_spectrum<<<1, fft::kT, sm, st>>>(a, kern, spec);
}

}  // namespace mwsht
