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
//
// Staging pipeline (per chunk of 16 degrees): warp 0 issues TMA bulk copies
// (cp.async.bulk) of the chunk's raw inputs -- 16 rows of the spin-column
// table and the chunk's +m / -m coefficient runs -- two chunks ahead into a
// double-buffered raw tile; after computing chunk k every thread derives its
// share of chunk k+1's parameters (recursion coefficients from the 1-D tables,
// c_l u_l(m) f scaling, masking) into a double-buffered parameter tile; one
// __syncthreads per chunk.
#include "common.cuh"

namespace mwsht {

namespace inv {
constexpr int R = kTileRows, C = kTileCols, CH = kChunk;
struct Raw {
  double dw[CH][R];     // spin-column table rows (padded table, always in bounds)
  double2 fp[CH][C];    // f_{l, c0 .. c0+cnt-1}
  double2 fn[CH][C];    // f_{l, -(c0+cnt-1) .. -c0} (ascending address)
};
struct Par {
  double2 row[CH][R];   // (kap_l C_l(m'), W_l(m'))
  double colc[CH][C];   // C_l(m)
  double2 gp[CH][C];    // c_l u_l(m) f_{l,m}
  double2 gn[CH][C];    // c_l u_l(m) (-1)^l f_{l,-m}
};
struct Smem {
  Raw raw[2];
  Par par[2];
  uint64_t bar[2];
};
}  // namespace inv

template <bool REAL>
__device__ __forceinline__ int inv_cnt(int l, int c0) {
  return min(c0 + inv::C - 1, l) - c0 + 1;  // valid columns m in [c0, c0+cnt) at degree l
}

// warp 0: issue the bulk copies of chunk starting at degree lc into raw buffer rb
template <bool REAL>
__device__ __forceinline__ void inv_issue(const InvArgs& a, const double2* in, inv::Raw& rb,
                                          uint64_t* bar, int lc, int r0, int c0, int lane) {
  const int L = a.t.L, N = a.t.N, Lp = a.ldw;
  const int ns = min(inv::CH, L - lc);
  // total bytes (every lane computes it; lane 0 arms the barrier first)
  uint32_t bytes = 0;
  for (int s = 0; s < ns; s++) {
    const int l = lc + s, cnt = inv_cnt<REAL>(l, c0);
    bytes += inv::R * 8;
    if (cnt > 0) bytes += (REAL ? 1u : 2u) * cnt * 16u;
  }
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane < inv::CH) {
    const int s = lane, l = lc + s;
    if (s < ns) bulk_g2s(&rb.dw[s][0], a.DW + (long long)l * Lp + r0, inv::R * 8, bar);
  } else {
    const int s = lane - inv::CH, l = lc + s;
    if (s < ns) {
      const int cnt = inv_cnt<REAL>(l, c0);
      if (cnt > 0) {
        const double2* srcp;
        const double2* srcn = nullptr;
        if (REAL) {
          srcp = a.in_mode == 0 ? in + (long long)l * (l + 1) + c0 : in + (long long)l * L + c0;
        } else if (a.in_mode == 0) {
          srcp = in + (long long)l * (l + 1) + c0;
          srcn = in + (long long)l * (l + 1) - (c0 + cnt - 1);
        } else {
          srcp = in + (long long)l * N + (L - 1 + c0);
          srcn = in + (long long)l * N + (L - 1 - (c0 + cnt - 1));
        }
        bulk_g2s(&rb.fp[s][0], srcp, cnt * 16, bar);
        if (!REAL) bulk_g2s(&rb.fn[s][0], srcn, cnt * 16, bar);
      }
    }
  }
}

// all threads: raw chunk -> parameters
template <bool REAL>
__device__ __forceinline__ void inv_derive(const InvArgs& a, const inv::Raw& rb, inv::Par& pb,
                                           int lc, int r0, int c0, int tid) {
  const DevTables& T = a.t;
  const int L = T.L;
  const int ns = min(inv::CH, L - lc);
  for (int idx = tid; idx < inv::CH * inv::R; idx += kThreads) {
    const int s = idx / inv::R, q = idx % inv::R;
    const int l = lc + s, x = r0 + q;
    double2 v = make_double2(0.0, 0.0);
    if (s < ns && x <= l) v = make_double2(T.kap[l] * (double)x * T.V[l - x] * T.V[l + x], rb.dw[s][q]);
    pb.row[s][q] = v;
  }
  for (int idx = tid; idx < inv::CH * inv::C; idx += kThreads) {
    const int s = idx / inv::C, q = idx % inv::C;
    const int l = lc + s, m = c0 + q;
    double cc = 0.0;
    double2 gp = make_double2(0.0, 0.0), gn = gp;
    if (s < ns && m <= l) {
      cc = (double)m * T.V[l - m] * T.V[l + m];
      const double u = a.cl[l] * T.A[l - m] * T.A[l + m];
      gp = cscale(rb.fp[s][q], u);
      if (!REAL) gn = cscale(rb.fn[s][inv_cnt<REAL>(l, c0) - 1 - q], (l & 1) ? -u : u);
    }
    pb.colc[s][q] = cc;
    pb.gp[s][q] = gp;
    if (!REAL) pb.gn[s][q] = gn;
  }
}

template <bool REAL, bool SPIN0>
__global__ void __launch_bounds__(kThreads, 1) k_inverse_core(InvArgs a) {
  constexpr int NI = 4, NJ = 2, NE = NI * NJ;
  constexpr int NG = REAL ? 1 : 2;  // complex values of g per column: f_{l,m} (+ f_{l,-m})
  extern __shared__ __align__(128) unsigned char smem_raw[];
  inv::Smem& sm = *reinterpret_cast<inv::Smem*>(smem_raw);

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
    cl[j] = 16 * wc + c + 8 * j;
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
  const int nchunks = (L - lstart + kChunk - 1) / kChunk;

  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (w == 0) {
    inv_issue<REAL>(a, in, sm.raw[0], &sm.bar[0], lstart, r0, c0, lane);
    if (nchunks > 1) inv_issue<REAL>(a, in, sm.raw[1], &sm.bar[1], lstart + kChunk, r0, c0, lane);
  }
  mbar_wait(&sm.bar[0], 0);
  inv_derive<REAL>(a, sm.raw[0], sm.par[0], lstart, r0, c0, tid);
  __syncthreads();

  for (int k = 0; k < nchunks; k++) {
    const int lc = lstart + k * kChunk;
    const int ns = min(kChunk, L - lc);
    if (w == 0 && k + 2 < nchunks) {
      fence_proxy_async();
      inv_issue<REAL>(a, in, sm.raw[k & 1], &sm.bar[k & 1], lc + 2 * kChunk, r0, c0, lane);
    }
    const inv::Par& P = sm.par[k & 1];

    if (warp_has && wl0_min < lc + ns) {
      if (!fast) {
        int anylev = 0;
#pragma unroll
        for (int e = 0; e < NE; e++) anylev |= lev[e];
        fast = (wl0_max < lc) && __all_sync(0xffffffffu, anylev == 0);
      }
      if (fast) {
        // ----------------------------------------------------- steady state
        auto rec_step = [&](int s) {
          double2 rp[NI];
          double cc[NJ];
#pragma unroll
          for (int i = 0; i < NI; i++) rp[i] = P.row[s][rl[i]];
#pragma unroll
          for (int j = 0; j < NJ; j++) cc[j] = P.colc[s][cl[j]];
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
              zp[e] = z[e];
              z[e] = zn;
            }
        };
        auto full_step = [&](int s) {
          double2 rp[NI];
          double cc[NJ];
          double2 g[NJ][NG];
#pragma unroll
          for (int i = 0; i < NI; i++) rp[i] = P.row[s][rl[i]];
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            cc[j] = P.colc[s][cl[j]];
            g[j][0] = P.gp[s][cl[j]];
            if (!REAL) g[j][NG - 1] = P.gn[s][cl[j]];
          }
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double t = z[e] * rp[i].y;
#pragma unroll
              for (int k2 = 0; k2 < NG; k2++) {
                acc[e][2 * k2] = fma(t, g[j][k2].x, acc[e][2 * k2]);
                acc[e][2 * k2 + 1] = fma(t, g[j][k2].y, acc[e][2 * k2 + 1]);
              }
              const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
              zp[e] = z[e];
              z[e] = zn;
            }
        };
        if (SPIN0) {
          // lc is even: step pairs (even l, odd l); rows of parity par contract
          int s = 0;
          for (; s + 1 < ns; s += 2) {
            if (par == 0) {
              full_step(s);
              rec_step(s + 1);
            } else {
              rec_step(s);
              full_step(s + 1);
            }
          }
          if (s < ns) {
            if (par == 0)
              full_step(s);
            else
              rec_step(s);
          }
        } else {
#pragma unroll 2
          for (int s = 0; s < ns; s++) full_step(s);
        }
      } else {
        // --------------------------------- ramp: seeds, levels, masking
        for (int s = 0; s < ns; s++) {
          const int l = lc + s;
          double2 rp[NI];
          double cc[NJ];
          double2 g[NJ][NG];
#pragma unroll
          for (int i = 0; i < NI; i++) rp[i] = P.row[s][rl[i]];
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            cc[j] = P.colc[s][cl[j]];
            g[j][0] = P.gp[s][cl[j]];
            if (!REAL) g[j][NG - 1] = P.gn[s][cl[j]];
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
                double sm_ = seed_value(T, l0, min(mp[i], mm[j]), ex);
                if (mm[j] < mp[i] && ((mp[i] - mm[j]) & 1)) sm_ = -sm_;
                double den = T.lam[l0] * (T.A[l0 - mm[j]] * T.A[l0 + mm[j]]) *
                             (T.A[l0 - mp[i]] * T.A[l0 + mp[i]]);
                if (l0 & 1) den = -den;
                z[e] = split_level(sm_ / den, ex, lev[e]);
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
                for (int k2 = 0; k2 < NG; k2++) {
                  acc[e][2 * k2] = fma(t, g[j][k2].x, acc[e][2 * k2]);
                  acc[e][2 * k2 + 1] = fma(t, g[j][k2].y, acc[e][2 * k2 + 1]);
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
    if (k + 1 < nchunks) {
      mbar_wait(&sm.bar[(k + 1) & 1], ((k + 1) >> 1) & 1);
      inv_derive<REAL>(a, sm.raw[(k + 1) & 1], sm.par[(k + 1) & 1], lc + kChunk, r0, c0, tid);
    }
    __syncthreads();
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

template <bool REAL, bool SPIN0>
static void launch_inv(const InvArgs& a, dim3 grid, cudaStream_t st) {
  const size_t smem = sizeof(inv::Smem);
  cudaFuncSetAttribute(k_inverse_core<REAL, SPIN0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  k_inverse_core<REAL, SPIN0><<<grid, kThreads, smem, st>>>(a);
}

void launch_inverse_core(const InvArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st) {
  dim3 grid(ntiles, nmaps);
  if (real)
    launch_inv<true, true>(a, grid, st);
  else if (a.spin == 0)
    launch_inv<false, true>(a, grid, st);
  else
    launch_inv<false, false>(a, grid, st);
}

}  // namespace mwsht
