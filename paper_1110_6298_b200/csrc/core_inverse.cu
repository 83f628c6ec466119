// Inverse core: T[m', m] = sum_l c_l Delta^l_{m'm} Delta^l_{m',-s} f_lm  (both signs of m).
//
// Replaces the reference's fmm_core (pkg/src/torusht/kernels/_numba.py:74-105)
// and fmm_core_real (:108-128).  The reference walks l serially, regenerating
// the whole pi/2 quadrant per degree with Trapani (or Risbo) and scattering
// into T.  Here every (m', m) pair is an independent three-term chain in l
// (DESIGN.md §3.1): no plane is ever materialised, T accumulates in registers
// for the whole l range, and the only per-step inputs are O(L) row/column
// parameters staged through shared memory.
//
// CTA tile: 64 rows m' x 32 columns m, 256 threads, 4x2 entries per thread.
// Warp w covers 16 rows of ONE parity (so for spin 0, where
// Delta^l_{m',0} = 0 whenever l+m' is odd, a whole warp skips the
// contraction on alternate degrees) by 16 columns.
#include "common.cuh"

namespace mwsht {

template <bool REAL, bool SPIN0>
__global__ void __launch_bounds__(kThreads, 1) k_inverse_core(InvArgs a) {
  constexpr int NI = 4, NJ = 2, NE = NI * NJ;
  constexpr int NG = REAL ? 1 : 2;  // complex values of g per column: f_{l,m} (+ f_{l,-m})
  __shared__ double2 s_row[kChunk][kTileRows];       // (kap_l C_l(m'), W_l(m'))
  __shared__ double s_colc[kChunk][kTileCols];       // C_l(m)
  __shared__ double2 s_colg[kChunk][kTileCols][NG];  // c_l u_l(m) f_{l,m}, c_l u_l(m) (-1)^l f_{l,-m}

  const DevTables& T = a.t;
  const int L = T.L, N = T.N;
  const int2 tile = a.tiles[blockIdx.x];
  const int r0 = tile.x, c0 = tile.y;
  const double2* __restrict__ in = a.in + (long long)blockIdx.y * a.in_stride;
  double2* __restrict__ out = a.out + (long long)blockIdx.y * a.out_stride;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wr = w & 3, wc = w >> 2, r = lane & 3, c = lane >> 2, par = wr & 1;
  int rl[NI], cl[NJ], mp[NI], mm[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    rl[i] = par + 2 * (16 * (wr >> 1) + 4 * i + r);
    mp[i] = r0 + rl[i];
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    cl[j] = 16 * wc + 2 * c + j;
    mm[j] = c0 + cl[j];
  }

  double z[NE], zp[NE], acc[NE][2 * NG];
  int lev[NE];
#pragma unroll
  for (int e = 0; e < NE; e++) {
    z[e] = 0.0;
    zp[e] = 0.0;
    lev[e] = 0;
#pragma unroll
    for (int k = 0; k < 2 * NG; k++) acc[e][k] = 0.0;
  }

  // warp extents (rows step 2 within a warp)
  const int wrow_lo = r0 + par + 32 * (wr >> 1);
  const int wrow_hi = min(wrow_lo + 30, L - 1);
  const int wcol_lo = c0 + 16 * wc;
  const int wcol_hi = min(wcol_lo + 15, L - 1);
  const bool warp_has = wrow_lo < L && wcol_lo < L;
  const int wl0_min = max(wrow_lo, wcol_lo);
  const int wl0_max = max(wrow_hi, wcol_hi);
  bool fast = false;

  const int lstart = max(r0, c0);
  for (int lc = lstart; lc < L; lc += kChunk) {
    const int ns = min(kChunk, L - lc);
    __syncthreads();
    // ---- stage row parameters
    for (int idx = tid; idx < kChunk * kTileRows; idx += kThreads) {
      const int s = idx / kTileRows, q = idx % kTileRows;
      const int l = lc + s, x = r0 + q;
      double2 v = make_double2(0.0, 0.0);
      if (s < ns && x <= l) {
        v.x = T.kap[l] * (double)x * T.V[l - x] * T.V[l + x];
        v.y = a.DW[(long long)l * L + x];
      }
      s_row[s][q] = v;
    }
    // ---- stage column parameters
    for (int idx = tid; idx < kChunk * kTileCols; idx += kThreads) {
      const int s = idx / kTileCols, q = idx % kTileCols;
      const int l = lc + s, m = c0 + q;
      double cc = 0.0;
      double2 gp = make_double2(0.0, 0.0), gn = gp;
      if (s < ns && m <= l) {
        cc = (double)m * T.V[l - m] * T.V[l + m];
        const double u = a.cl[l] * T.A[l - m] * T.A[l + m];
        double2 fp, fn;
        if (REAL) {
          fp = a.in_mode == 0 ? in[(long long)l * (l + 1) + m] : in[(long long)l * L + m];
          fn = fp;
        } else if (a.in_mode == 0) {
          fp = in[(long long)l * (l + 1) + m];
          fn = in[(long long)l * (l + 1) - m];
        } else {
          fp = in[(long long)l * N + (L - 1 + m)];
          fn = in[(long long)l * N + (L - 1 - m)];
        }
        gp = cscale(fp, u);
        gn = cscale(fn, (l & 1) ? -u : u);
      }
      s_colc[s][q] = cc;
      s_colg[s][q][0] = gp;
      if (!REAL) s_colg[s][q][NG - 1] = gn;
    }
    __syncthreads();
    if (!warp_has || wl0_min >= lc + ns) continue;  // no chain of this warp has started yet

    if (!fast) {
      int anylev = 0;
#pragma unroll
      for (int e = 0; e < NE; e++) anylev |= lev[e];
      fast = (wl0_max < lc) && __all_sync(0xffffffffu, anylev == 0);
    }

    if (fast) {
      // ------------------------------------------------------- steady state
#pragma unroll 2
      for (int s = 0; s < ns; s++) {
        const int l = lc + s;
        double2 rp[NI];
        double cc[NJ];
        double2 g[NJ][NG];
#pragma unroll
        for (int i = 0; i < NI; i++) rp[i] = s_row[s][rl[i]];
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          cc[j] = s_colc[s][cl[j]];
#pragma unroll
          for (int k = 0; k < NG; k++) g[j][k] = s_colg[s][cl[j]][k];
        }
        if (!SPIN0 || ((l & 1) == par)) {
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double t = z[e] * rp[i].y;
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
            const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
            zp[e] = z[e];
            z[e] = zn;
          }
      }
    } else {
      // ------------------------------------- ramp: seeds, levels, masking
      for (int s = 0; s < ns; s++) {
        const int l = lc + s;
        double2 rp[NI];
        double cc[NJ];
        double2 g[NJ][NG];
#pragma unroll
        for (int i = 0; i < NI; i++) rp[i] = s_row[s][rl[i]];
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          cc[j] = s_colc[s][cl[j]];
#pragma unroll
          for (int k = 0; k < NG; k++) g[j][k] = s_colg[s][cl[j]][k];
        }
        bool anylive = false;
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const int l0 = max(mp[i], mm[j]);
            if (l == l0 && mp[i] < L && mm[j] < L) {
              // seed Delta^{l0}_{m'm} = sign sqrt(C(2 l0, l0 + min))/2^l0
              int ex;
              double sm = seed_value(T, l0, min(mp[i], mm[j]), ex);
              if (mm[j] < mp[i] && ((mp[i] - mm[j]) & 1)) sm = -sm;
              double den = T.lam[l0] * (T.A[l0 - mm[j]] * T.A[l0 + mm[j]]) *
                           (T.A[l0 - mp[i]] * T.A[l0 + mp[i]]);
              if (l0 & 1) den = -den;
              z[e] = split_level(sm / den, ex, lev[e]);
              zp[e] = 0.0;
            }
            anylive |= (l >= l0) && (lev[e] == 0) && mp[i] < L && mm[j] < L;
          }
        if ((!SPIN0 || ((l & 1) == par)) && __any_sync(0xffffffffu, anylive)) {
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const bool live = (l >= max(mp[i], mm[j])) && (lev[e] == 0);
              const double t = live ? z[e] * rp[i].y : 0.0;
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
            double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
            double zo = z[e];
            if (lev[e] > 0 && above_top(zn)) {
              const double sh = pow2i(-kLevShift);
              zn *= sh;
              zo *= sh;
              lev[e] -= 1;
            }
            zp[e] = zo;
            z[e] = zn;
          }
      }
    }
  }

  // ---------------------------------------------------------------- epilogue
  const int sgs = (a.spin & 1) ? -1 : 1;  // (-1)^s
#pragma unroll
  for (int i = 0; i < NI; i++) {
    const int x = mp[i];
    if (x >= L) continue;
    double sn, cs;
    sincospi((double)x / (double)N, &sn, &cs);
    const double2 tw = make_double2(cs, sn);       // e^{+i m' theta0}
    const double2 twc = make_double2(cs, -sn);     // e^{-i m' theta0}
    const int binp = x, binn = x ? N - x : 0;
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int m = mm[j];
      if (m >= L) continue;
      const int e = i * NJ + j;
      const double2 Tp = make_double2(acc[e][0], acc[e][1]);
      if (a.out_mode == 1) {
        if (REAL) {
          out[(long long)x * L + m] = Tp;
        } else {
          out[(long long)x * N + (L - 1 + m)] = Tp;
          if (m > 0) {
            const double sx = (x & 1) ? -1.0 : 1.0;
            out[(long long)x * N + (L - 1 - m)] = make_double2(sx * acc[e][2], sx * acc[e][3]);
          }
        }
        continue;
      }
      if (REAL) {
        // fhalf[m, m'] = T[m', m] i^{-m}; mirror (-1)^m (mw.py:550-556)
        const double2 F = cmul(Tp, ipow(-m));
        double2* row = out + (long long)m * N;
        row[binp] = cmul(F, tw);
        if (x) row[binn] = cscale(cmul(F, twc), (m & 1) ? -1.0 : 1.0);
      } else {
        // F[m, m'] = (-1)^s i^{-(m+s)} T[m', m]; F[m, -m'] = (-1)^(m+s) F[m, m'] (mw.py:395-401)
        const double2 Fp = cscale(cmul(Tp, ipow(-(m + a.spin))), (double)sgs);
        double2* rowp = out + (long long)(L - 1 + m) * N;
        rowp[binp] = cmul(Fp, tw);
        if (x) rowp[binn] = cscale(cmul(Fp, twc), ((m + a.spin) & 1) ? -1.0 : 1.0);
        if (m > 0) {
          const double sx = (x & 1) ? -1.0 : 1.0;
          const double2 Tn = make_double2(sx * acc[e][2], sx * acc[e][3]);
          const double2 Fn = cscale(cmul(Tn, ipow(m - a.spin)), (double)sgs);
          double2* rown = out + (long long)(L - 1 - m) * N;
          rown[binp] = cmul(Fn, tw);
          if (x) rown[binn] = cscale(cmul(Fn, twc), ((m + a.spin) & 1) ? -1.0 : 1.0);
        }
      }
    }
  }
}

void launch_inverse_core(const InvArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st) {
  dim3 grid(ntiles, nmaps);
  const bool s0 = a.spin == 0;
  if (real)
    k_inverse_core<true, true><<<grid, kThreads, 0, st>>>(a);
  else if (s0)
    k_inverse_core<false, true><<<grid, kThreads, 0, st>>>(a);
  else
    k_inverse_core<false, false><<<grid, kThreads, 0, st>>>(a);
}

}  // namespace mwsht
