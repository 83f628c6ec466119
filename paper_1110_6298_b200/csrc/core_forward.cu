// Forward core: R[l, m] = sum_{m'=0}^{l} Delta^l_{m'm} Delta^l_{m',-s} gfold[m, m']  (both signs of m).
//
// Replaces the reference's flm_core (pkg/src/torusht/kernels/_numba.py:131-166)
// and flm_core_real (:169-188).  The reduction runs over m', so every output
// (l, m) owns one Trapani column chain that walks m' = l .. 0
// (trapani_step's downward three-term rule, _numba.py:63-71) and accumulates
// its dot product in registers -- no cross-thread reduction at all.  The
// chain is carried in the scaled variable y (Delta = A(l-m') Bt(l+m') y) whose
// recursion y_{m'-1} = m alpha(l-m'+1) beta(l+m'-1) y_{m'} - y_{m'+1} costs one
// DMUL + one DFMA, and in exponent levels while its value is below 2^-568,
// which is what keeps it stable where the reference's float64 Trapani
// overflows.
//
// CTA tile: 64 degrees l x 32 orders m, 256 threads, 4x2 entries per thread;
// a warp's 16 degrees share one parity (spin 0: Delta^l_{m',0} = 0 when l-m'
// is odd, so whole warps skip alternate contraction steps).
#include "common.cuh"

namespace mwsht {

template <bool REAL, bool SPIN0>
__global__ void __launch_bounds__(kThreads, 1) k_forward_core(FwdArgs a) {
  constexpr int NI = 4, NJ = 2, NE = NI * NJ;
  constexpr int NG = REAL ? 1 : 2;
  __shared__ double2 s_q[kChunk][kTileRows];          // (coefficient to step to m'-1, W'(l, m'))
  __shared__ double2 s_g[kChunk][kTileCols][NG];      // gfold[+m][m'], (-1)^m' gfold[-m][m']

  const DevTables& T = a.t;
  const int L = T.L;
  const int2 tile = a.tiles[blockIdx.x];
  const int l0b = tile.x, c0 = tile.y;
  const double2* __restrict__ gf = a.gf + (long long)blockIdx.y * a.in_stride;
  double2* __restrict__ out = a.out + (long long)blockIdx.y * a.out_stride;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = w & 3, wc = w >> 2, r = lane & 3, c = lane >> 2, par = wr & 1;
  int rl[NI], cl[NJ], ll[NI], mm[NJ];
  double md[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    rl[i] = par + 2 * (16 * (wr >> 1) + 4 * i + r);
    ll[i] = l0b + rl[i];
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    cl[j] = 16 * wc + 2 * c + j;
    mm[j] = c0 + cl[j];
    md[j] = (double)mm[j];
  }

  double y[NE], y1[NE], acc[NE][2 * NG];
  int lev[NE];
#pragma unroll
  for (int e = 0; e < NE; e++) {
    y[e] = 0.0;
    y1[e] = 0.0;
    lev[e] = 0;
#pragma unroll
    for (int k = 0; k < 2 * NG; k++) acc[e][k] = 0.0;
  }

  // warp extents.  Valid entries: m <= l < L.  A chain (l, m) starts at mu = l.
  const int wrow_lo = l0b + par + 32 * (wr >> 1);
  const int wrow_hi = min(wrow_lo + 30, L - 1);
  const int wcol_lo = c0 + 16 * wc;
  const bool warp_has = wrow_lo < L && wcol_lo <= wrow_hi;
  // every valid entry has started once mu <= (smallest l with a valid column)
  const int wl_min = max(wrow_lo, wcol_lo);
  bool fast = false;

  const int mu_top = min(l0b + kTileRows - 1, L - 1);
  for (int mc = mu_top; mc >= 0; mc -= kChunk) {
    const int ns = min(kChunk, mc + 1);
    __syncthreads();
    for (int idx = tid; idx < kChunk * kTileRows; idx += kThreads) {
      const int s = idx / kTileRows, q = idx % kTileRows;
      const int mu = mc - s, l = l0b + q;
      double2 v = make_double2(0.0, 0.0);
      if (s < ns && l < L && mu <= l) {
        v.x = mu >= 1 ? T.alpha[l - mu + 1] * T.beta[l + mu - 1] : 0.0;
        v.y = a.DW[(long long)mu * L + l];
      }
      s_q[s][q] = v;
    }
    for (int idx = tid; idx < kChunk * kTileCols; idx += kThreads) {
      const int q = idx / kChunk, s = idx % kChunk;  // s fastest: contiguous gfold reads
      const int mu = mc - s, m = c0 + q;
      double2 gp = make_double2(0.0, 0.0), gn = gp;
      if (s < ns && m < L) {
        if (REAL) {
          gp = gf[(long long)m * L + mu];
        } else {
          gp = gf[(long long)(L - 1 + m) * L + mu];
          gn = gf[(long long)(L - 1 - m) * L + mu];
          if (mu & 1) gn = make_double2(-gn.x, -gn.y);
        }
      }
      s_g[s][q][0] = gp;
      if (!REAL) s_g[s][q][NG - 1] = gn;
    }
    __syncthreads();
    if (!warp_has || wrow_hi < mc - ns + 1) continue;  // no chain of this warp started yet

    if (!fast) {
      int anylev = 0;
#pragma unroll
      for (int e = 0; e < NE; e++) anylev |= lev[e];
      fast = (mc < wl_min) && __all_sync(0xffffffffu, anylev == 0);
    }

    if (fast) {
#pragma unroll 2
      for (int s = 0; s < ns; s++) {
        const int mu = mc - s;
        double2 qp[NI], g[NJ][NG];
#pragma unroll
        for (int i = 0; i < NI; i++) qp[i] = s_q[s][rl[i]];
#pragma unroll
        for (int j = 0; j < NJ; j++)
#pragma unroll
          for (int k = 0; k < NG; k++) g[j][k] = s_g[s][cl[j]][k];
        if (!SPIN0 || ((mu & 1) == par)) {
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double t = y[e] * qp[i].y;
#pragma unroll
              for (int k = 0; k < NG; k++) {
                acc[e][2 * k] = fma(t, g[j][k].x, acc[e][2 * k]);
                acc[e][2 * k + 1] = fma(t, g[j][k].y, acc[e][2 * k + 1]);
              }
            }
        }
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const double yn = fma(md[j] * qp[i].x, y[e], -y1[e]);
            y1[e] = y[e];
            y[e] = yn;
          }
      }
    } else {
      for (int s = 0; s < ns; s++) {
        const int mu = mc - s;
        double2 qp[NI], g[NJ][NG];
#pragma unroll
        for (int i = 0; i < NI; i++) qp[i] = s_q[s][rl[i]];
#pragma unroll
        for (int j = 0; j < NJ; j++)
#pragma unroll
          for (int k = 0; k < NG; k++) g[j][k] = s_g[s][cl[j]][k];
        bool anylive = false;
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const bool valid = mm[j] <= ll[i] && ll[i] < L;
            if (mu == ll[i] && valid) {
              // seed y_l = Delta^l_{l,m} / (A(0) Bt(2l)),  Delta^l_{l,m} = (-1)^(l-m) T(l, m)
              int ex;
              double sm = seed_value(T, ll[i], mm[j], ex);
              if ((ll[i] - mm[j]) & 1) sm = -sm;
              y[e] = split_level(sm / T.Bt[2 * ll[i]], ex, lev[e]);
              y1[e] = 0.0;
            }
            anylive |= valid && mu <= ll[i] && lev[e] == 0;
          }
        if ((!SPIN0 || ((mu & 1) == par)) && __any_sync(0xffffffffu, anylive)) {
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const bool live = mu <= ll[i] && lev[e] == 0;
              const double t = live ? y[e] * qp[i].y : 0.0;
#pragma unroll
              for (int k = 0; k < NG; k++) {
                acc[e][2 * k] = fma(t, g[j][k].x, acc[e][2 * k]);
                acc[e][2 * k + 1] = fma(t, g[j][k].y, acc[e][2 * k + 1]);
              }
            }
        }
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            double yn = fma(md[j] * qp[i].x, y[e], -y1[e]);
            double yo = y[e];
            if (lev[e] > 0 && above_top(yn)) {
              const double sh = pow2i(-kLevShift);
              yn *= sh;
              yo *= sh;
              lev[e] -= 1;
            }
            y1[e] = yo;
            y[e] = yn;
          }
      }
    }
  }

  // ---------------------------------------------------------------- epilogue
  const double sgs = (a.spin & 1) ? -1.0 : 1.0;
#pragma unroll
  for (int i = 0; i < NI; i++) {
    const int l = ll[i];
    if (l >= L) continue;
    const double clv = T.cl[l];
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int m = mm[j];
      if (m > l) continue;
      const int e = i * NJ + j;
      const double2 Rp = make_double2(acc[e][0], acc[e][1]);
      if (a.out_mode == 1) {
        if (REAL) {
          out[(long long)l * L + m] = Rp;
        } else {
          const int N = T.N;
          out[(long long)l * N + (L - 1 + m)] = Rp;
          if (m > 0) {
            const double sl = (l & 1) ? -1.0 : 1.0;
            out[(long long)l * N + (L - 1 - m)] = make_double2(sl * acc[e][2], sl * acc[e][3]);
          }
        }
        continue;
      }
      const long long base = (long long)l * (l + 1);
      if (REAL) {
        // i^m c_l R, mirror f_{l,-m} = (-1)^m conj(f_lm)  (mw.py:499-501, 514-521)
        const double2 f = cscale(cmul(Rp, ipow(m)), clv);
        out[base + m] = f;
        if (m > 0) {
          const double sm = (m & 1) ? -1.0 : 1.0;
          out[base - m] = make_double2(sm * f.x, -sm * f.y);
        }
      } else {
        // (-1)^s i^(m+s) c_l R  (mw.py:317-319)
        out[base + m] = cscale(cmul(Rp, ipow(m + a.spin)), sgs * clv);
        if (m > 0) {
          const double sl = (l & 1) ? -1.0 : 1.0;
          const double2 Rn = make_double2(sl * acc[e][2], sl * acc[e][3]);
          out[base - m] = cscale(cmul(Rn, ipow(a.spin - m)), sgs * clv);
        }
      }
    }
  }
}

void launch_forward_core(const FwdArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st) {
  dim3 grid(ntiles, nmaps);
  if (real)
    k_forward_core<true, true><<<grid, kThreads, 0, st>>>(a);
  else if (a.spin == 0)
    k_forward_core<false, true><<<grid, kThreads, 0, st>>>(a);
  else
    k_forward_core<false, false><<<grid, kThreads, 0, st>>>(a);
}

}  // namespace mwsht
