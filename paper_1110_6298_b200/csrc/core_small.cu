// Small band-limit cores: one thread per chain.
//
// The tiled cores (core_forward.cu, core_inverse*.cu) give each CTA a 64 x 32
// block of chains and stream the per-degree tables through a TMA ring.  At
// small L that leaves most of the GPU idle: at L = 64 each core is 2 CTAs on
// 148 SMs (the ncu launch list in profiles/round2/launches_L64.csv shows 36 us
// for a 64-step chain block).  Here every chain is its own thread, so the
// chains spread over the whole GPU and a core costs about one chain's latency:
//   inverse: chain (m', m), degrees l = max(m', m) .. L-1 (the reference's
//            fmm_core, kernels/_numba.py:74-105),
//   forward: chain (l, m), m' = l .. 0 (flm_core, _numba.py:131-166; §3.2),
// with the same scaled recursions, chain seeds, exponent levels (checked every
// step here, per 16-step chunk there: results agree to rounding) and
// epilogues as the tiled kernels.  The tables are read straight from global
// memory (L2-resident at these sizes).
#include "common.cuh"

namespace mwsht {

constexpr int kSmallThreads = 128;
constexpr int kSmallU = 8;  // degrees whose table loads are in flight together

__device__ __forceinline__ void level_step(double& z, double& zp, int& lev) {
  if (lev && above_top(z)) {
    const double sh = pow2i(-kLevShift);
    z *= sh;
    zp *= sh;
    lev--;
  }
}

template <bool REAL>
__global__ void __launch_bounds__(kSmallThreads) k_inverse_small(InvArgs a) {
  pdl_trigger();
  const DevTables& T = a.t;
  const int L = T.L, N = T.N, Lp = a.ldw;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * L) return;
  const int x = idx / L, m = idx - x * L;  // chain (m' = x, m)
  const int map = blockIdx.y;
  const double2* gp = a.gp + (long long)map * a.g_stride;
  const double2* gn = gp + (long long)L * Lp;
  const int l0 = max(x, m), mu = min(x, m);
  int ex, lev;
  double s = seed3(T.sd_pi[l0], T.sd_qi[l0 + mu], T.sd_qi[l0 - mu], ex);
  if (m < x && ((x - m) & 1)) s = -s;
  if (l0 & 1) s = -s;
  double z = split_level(s, ex, lev), zp = 0.0;
  pdl_wait();  // the staged coefficients come from the previous kernel
  double ap0 = 0.0, ap1 = 0.0, an0 = 0.0, an1 = 0.0;
  // kSmallU degrees per round: all their table loads are issued before the
  // round's recursion steps (one memory latency per round, not per degree)
  for (int lb = l0; lb < L; lb += kSmallU) {
    double2 rv[kSmallU], g[kSmallU], h[kSmallU];
    double cc[kSmallU];
#pragma unroll
    for (int u = 0; u < kSmallU; u++) {
      const int l = min(lb + u, L - 1);
      rv[u] = a.rowtab[blk<kTileRows>(l, x, L)];  // (kap_l C_l(m'), W_l(m'))
      cc[u] = a.colc[blk<kTileCols>(l, m, L)];
      g[u] = gp[blk<kTileCols>(l, m, L)];
      if (!REAL) h[u] = gn[blk<kTileCols>(l, m, L)];
    }
#pragma unroll
    for (int u = 0; u < kSmallU; u++) {
      if (lb + u >= L) break;
      if (lev == 0) {
        const double t = z * rv[u].y;
        ap0 = fma(t, g[u].x, ap0);
        ap1 = fma(t, g[u].y, ap1);
        if (!REAL) {
          an0 = fma(t, h[u].x, an0);
          an1 = fma(t, h[u].y, an1);
        }
      }
      const double zn = fma(rv[u].x * cc[u], z, -zp);
      zp = z;
      z = zn;
      level_step(z, zp, lev);
    }
  }
  // epilogue (as k_inverse_core): phases, m' mirror and theta twist
  double2* __restrict__ out = a.out + (long long)map * a.out_stride;
  const double2 Tp = make_double2(ap0, ap1);
  if (a.out_mode == 1) {
    if (REAL) {
      out[(long long)x * L + m] = Tp;
    } else {
      out[(long long)x * N + (L - 1 + m)] = Tp;
      if (m > 0) {
        const double sx = (x & 1) ? -1.0 : 1.0;
        out[(long long)x * N + (L - 1 - m)] = make_double2(sx * an0, sx * an1);
      }
    }
    return;
  }
  double sn, cs;
  sincospi((double)x / (double)N, &sn, &cs);
  const double2 tw = make_double2(cs, sn), twc = make_double2(cs, -sn);
  const int binp = x, binn = x ? N - x : 0;
  // out_mode 3: bins m' >= 0 only (the theta stage rebuilds the mirrored half)
  const bool wmir = x && a.out_mode != 3;
  if (REAL) {
    // fhalf[m, m'] = T[m', m] i^{-m}; mirror (-1)^m (mw.py:550-556)
    const double2 F = cmul(Tp, ipow(-m));
    double2* row = out + (long long)m * N;
    row[binp] = cmul(F, tw);
    if (wmir) row[binn] = cscale(cmul(F, twc), (m & 1) ? -1.0 : 1.0);
  } else {
    // F[m, m'] = (-1)^s i^{-(m+s)} T[m', m]; F[m, -m'] = (-1)^(m+s) F[m, m'] (mw.py:395-401)
    const int spin = a.spin;
    const double sgs = (spin & 1) ? -1.0 : 1.0;
    const double2 Fp = cscale(cmul(Tp, ipow(-(m + spin))), sgs);
    double2* rowp = out + (long long)(L - 1 + m) * N;
    rowp[binp] = cmul(Fp, tw);
    if (wmir) rowp[binn] = cscale(cmul(Fp, twc), ((m + spin) & 1) ? -1.0 : 1.0);
    if (m > 0) {
      const double sx = (x & 1) ? -1.0 : 1.0;
      const double2 Fn = cscale(cmul(make_double2(sx * an0, sx * an1), ipow(m - spin)), sgs);
      double2* rown = out + (long long)(L - 1 - m) * N;
      rown[binp] = cmul(Fn, tw);
      if (wmir) rown[binn] = cscale(cmul(Fn, twc), ((m + spin) & 1) ? -1.0 : 1.0);
    }
  }
}

template <bool REAL>
__global__ void __launch_bounds__(kSmallThreads) k_forward_small(FwdArgs a) {
  pdl_trigger();
  const DevTables& T = a.t;
  const int L = T.L, Lp = a.ldw;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= L * L) return;
  const int l = idx / L, m = idx - l * L;  // chain (l, m), valid for m <= l
  if (m > l) return;
  const int map = blockIdx.y;
  const double2* gp = a.gf + (long long)map * a.in_stride;
  const double2* gn = gp + (long long)L * Lp;
  int ex, lev;
  double s = seed3(T.sd_pf[l], T.sd_r[l + m], T.sd_r[l - m], ex);
  if ((l - m) & 1) s = -s;
  double y = split_level(s, ex, lev), y1 = 0.0;
  const double md = (double)m;
  pdl_wait();
  double ap0 = 0.0, ap1 = 0.0, an0 = 0.0, an1 = 0.0;
  for (int mb = l; mb >= 0; mb -= kSmallU) {
    double2 q[kSmallU], g[kSmallU], h[kSmallU];
#pragma unroll
    for (int u = 0; u < kSmallU; u++) {
      const int mu = max(mb - u, 0);
      q[u] = a.rowtab[blk<kTileRows>(mu, l, L)];  // (coefficient, W'(l, mu))
      g[u] = gp[blk<kTileCols>(mu, m, L)];
      if (!REAL) h[u] = gn[blk<kTileCols>(mu, m, L)];
    }
#pragma unroll
    for (int u = 0; u < kSmallU; u++) {
      if (mb - u < 0) break;
      if (lev == 0) {
        const double t = y * q[u].y;
        ap0 = fma(t, g[u].x, ap0);
        ap1 = fma(t, g[u].y, ap1);
        if (!REAL) {
          an0 = fma(t, h[u].x, an0);
          an1 = fma(t, h[u].y, an1);
        }
      }
      const double yn = fma(md * q[u].x, y, -y1);
      y1 = y;
      y = yn;
      level_step(y, y1, lev);
    }
  }
  // epilogue (as k_forward_core)
  double2* __restrict__ out = a.out + (long long)map * a.out_stride;
  const double2 Rp = make_double2(ap0, ap1);
  if (a.out_mode == 1) {
    if (REAL) {
      out[(long long)l * L + m] = Rp;
    } else {
      const int N = T.N;
      out[(long long)l * N + (L - 1 + m)] = Rp;
      if (m > 0) {
        const double sl = (l & 1) ? -1.0 : 1.0;
        out[(long long)l * N + (L - 1 - m)] = make_double2(sl * an0, sl * an1);
      }
    }
    return;
  }
  const double clv = T.cl[l];
  const long long base = (long long)l * (l + 1);
  if (REAL) {
    // i^m c_l R, mirror f_{l,-m} = (-1)^m conj(f_lm)  (mw.py:499-501, 514-521)
    const double2 f = cscale(cmul(Rp, ipow(m)), clv);
    out[base + m] = f;
    if (m > 0) {
      const double sm_ = (m & 1) ? -1.0 : 1.0;
      out[base - m] = make_double2(sm_ * f.x, -sm_ * f.y);
    }
  } else {
    // (-1)^s i^(m+s) c_l R  (mw.py:317-319)
    const double sgs = (a.spin & 1) ? -1.0 : 1.0;
    out[base + m] = cscale(cmul(Rp, ipow(m + a.spin)), sgs * clv);
    if (m > 0) {
      const double sl = (l & 1) ? -1.0 : 1.0;
      const double2 Rn = make_double2(sl * an0, sl * an1);
      out[base - m] = cscale(cmul(Rn, ipow(a.spin - m)), sgs * clv);
    }
  }
}

// Band limits up to these use the one-thread-per-chain cores (measured
// crossovers, tools/small_sweep.py; MWSHT_SMALL_INV / MWSHT_SMALL_FWD override,
// 0 disables).
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
int small_inverse_limit() {
  static int lim = env_int("MWSHT_SMALL_INV", 160);
  return lim;
}
int small_forward_limit() {
  static int lim = env_int("MWSHT_SMALL_FWD", 320);
  return lim;
}

void launch_inverse_small(const InvArgs& a, int nmaps, bool real, cudaStream_t st) {
  const int L = a.t.L;
  dim3 grid((unsigned)((L * L + kSmallThreads - 1) / kSmallThreads), nmaps);
  if (real)
    launch_pdl(k_inverse_small<true>, grid, dim3(kSmallThreads), 0, st, a);
  else
    launch_pdl(k_inverse_small<false>, grid, dim3(kSmallThreads), 0, st, a);
}

void launch_forward_small(const FwdArgs& a, int nmaps, bool real, cudaStream_t st) {
  const int L = a.t.L;
  dim3 grid((unsigned)((L * L + kSmallThreads - 1) / kSmallThreads), nmaps);
  if (real)
    launch_pdl(k_forward_small<true>, grid, dim3(kSmallThreads), 0, st, a);
  else
    launch_pdl(k_forward_small<false>, grid, dim3(kSmallThreads), 0, st, a);
}

}  // namespace mwsht
