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
//
// Staging (per chunk of 16 m' values, walking down): warp 0 issues TMA bulk
// copies two chunks ahead -- 16 rows of the (m', l) spin-column table and the
// 16 m'-rows of the transposed folded plane gfT[m'][row] restricted to the
// tile's +m and -m runs -- into a double-buffered raw tile; after each chunk
// every thread derives its share of the next chunk's parameters.
#include "common.cuh"

namespace mwsht {

namespace fwd {
constexpr int R = kTileRows, C = kTileCols, CH = kChunk;
struct Raw {
  double dw[CH][R];     // DWfwd[mu][l0b .. l0b+63]
  double2 gp[CH][C];    // gfT[mu][row(+m)], m = c0 .. c0+cnt-1
  double2 gn[CH][C];    // gfT[mu][row(-m)], ascending address = descending m
};
struct Par {
  double2 q[CH][R];     // (coefficient producing y_{mu-1}, W'(l, mu))
  double2 gp[CH][C];    // gfold[+m][mu]
  double2 gn[CH][C];    // (-1)^mu gfold[-m][mu]
};
struct Smem {
  Raw raw[2];
  Par par[2];
  uint64_t bar[2];
};
}  // namespace fwd

template <bool REAL>
__device__ __forceinline__ void fwd_issue(const FwdArgs& a, const double2* gfT, fwd::Raw& rb,
                                          uint64_t* bar, int mc, int l0b, int c0, int lane) {
  const int L = a.t.L, N = a.t.N, Lp = a.ldw;
  const int ns = min(fwd::CH, mc + 1);
  const int cnt = min(fwd::C, L - c0);
  const int rowlen = REAL ? L : N;
  const uint32_t bytes = ns * (fwd::R * 8u + (REAL ? 1u : 2u) * cnt * 16u);
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (lane < fwd::CH) {
    const int s = lane, mu = mc - s;
    if (s < ns) bulk_g2s(&rb.dw[s][0], a.DW + (long long)mu * Lp + l0b, fwd::R * 8, bar);
  } else {
    const int s = lane - fwd::CH, mu = mc - s;
    if (s < ns) {
      const double2* row = gfT + (long long)mu * rowlen;
      if (REAL) {
        bulk_g2s(&rb.gp[s][0], row + c0, cnt * 16, bar);
      } else {
        bulk_g2s(&rb.gp[s][0], row + (L - 1 + c0), cnt * 16, bar);
        bulk_g2s(&rb.gn[s][0], row + (L - 1 - (c0 + cnt - 1)), cnt * 16, bar);
      }
    }
  }
}

template <bool REAL>
__device__ __forceinline__ void fwd_derive(const FwdArgs& a, const fwd::Raw& rb, fwd::Par& pb,
                                           int mc, int l0b, int c0, int tid) {
  const DevTables& T = a.t;
  const int L = T.L;
  const int ns = min(fwd::CH, mc + 1);
  const int cnt = min(fwd::C, L - c0);
  for (int idx = tid; idx < fwd::CH * fwd::R; idx += kThreads) {
    const int s = idx / fwd::R, q = idx % fwd::R;
    const int mu = mc - s, l = l0b + q;
    double2 v = make_double2(0.0, 0.0);
    if (s < ns && l < L && mu <= l)
      v = make_double2(mu >= 1 ? T.alpha[l - mu + 1] * T.beta[l + mu - 1] : 0.0, rb.dw[s][q]);
    pb.q[s][q] = v;
  }
  for (int idx = tid; idx < fwd::CH * fwd::C; idx += kThreads) {
    const int s = idx / fwd::C, q = idx % fwd::C;
    const int mu = mc - s;
    double2 gp = make_double2(0.0, 0.0), gn = gp;
    if (s < ns && q < cnt) {
      gp = rb.gp[s][q];
      if (!REAL) {
        gn = rb.gn[s][cnt - 1 - q];
        if (mu & 1) gn = make_double2(-gn.x, -gn.y);
      }
    }
    pb.gp[s][q] = gp;
    if (!REAL) pb.gn[s][q] = gn;
  }
}

template <bool REAL, bool SPIN0>
__global__ void __launch_bounds__(kThreads, 1) k_forward_core(FwdArgs a) {
  constexpr int NI = 4, NJ = 2, NE = NI * NJ;
  constexpr int NG = REAL ? 1 : 2;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  fwd::Smem& sm = *reinterpret_cast<fwd::Smem*>(smem_raw);

  const DevTables& T = a.t;
  const int L = T.L;
  const int2 tile = a.tiles[blockIdx.x];
  const int l0b = tile.x, c0 = tile.y;
  const double2* __restrict__ gfT = a.gf + (long long)blockIdx.y * a.in_stride;
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
    cl[j] = 16 * wc + c + 8 * j;
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
  const int wl_min = max(wrow_lo, wcol_lo);  // every valid chain started once mu < wl_min
  bool fast = false;

  const int mu_top = min(l0b + kTileRows - 1, L - 1);
  const int nchunks = (mu_top + kChunk) / kChunk;

  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (w == 0) {
    fwd_issue<REAL>(a, gfT, sm.raw[0], &sm.bar[0], mu_top, l0b, c0, lane);
    if (nchunks > 1) fwd_issue<REAL>(a, gfT, sm.raw[1], &sm.bar[1], mu_top - kChunk, l0b, c0, lane);
  }
  mbar_wait(&sm.bar[0], 0);
  fwd_derive<REAL>(a, sm.raw[0], sm.par[0], mu_top, l0b, c0, tid);
  __syncthreads();

  for (int k = 0; k < nchunks; k++) {
    const int mc = mu_top - k * kChunk;
    const int ns = min(kChunk, mc + 1);
    if (w == 0 && k + 2 < nchunks) {
      fence_proxy_async();
      fwd_issue<REAL>(a, gfT, sm.raw[k & 1], &sm.bar[k & 1], mc - 2 * kChunk, l0b, c0, lane);
    }
    const fwd::Par& P = sm.par[k & 1];

    if (warp_has && wrow_hi >= mc - ns + 1) {
      if (!fast) {
        int anylev = 0;
#pragma unroll
        for (int e = 0; e < NE; e++) anylev |= lev[e];
        fast = (mc < wl_min) && __all_sync(0xffffffffu, anylev == 0);
      }
      if (fast) {
        auto rec_step = [&](int s) {
          double2 qp[NI];
#pragma unroll
          for (int i = 0; i < NI; i++) qp[i] = P.q[s][rl[i]];
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double yn = fma(md[j] * qp[i].x, y[e], -y1[e]);
              y1[e] = y[e];
              y[e] = yn;
            }
        };
        auto full_step = [&](int s) {
          double2 qp[NI], g[NJ][NG];
#pragma unroll
          for (int i = 0; i < NI; i++) qp[i] = P.q[s][rl[i]];
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            g[j][0] = P.gp[s][cl[j]];
            if (!REAL) g[j][NG - 1] = P.gn[s][cl[j]];
          }
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              const double t = y[e] * qp[i].y;
#pragma unroll
              for (int k2 = 0; k2 < NG; k2++) {
                acc[e][2 * k2] = fma(t, g[j][k2].x, acc[e][2 * k2]);
                acc[e][2 * k2 + 1] = fma(t, g[j][k2].y, acc[e][2 * k2 + 1]);
              }
              const double yn = fma(md[j] * qp[i].x, y[e], -y1[e]);
              y1[e] = y[e];
              y[e] = yn;
            }
        };
        if (SPIN0) {
          // contraction when mu has the warp's degree parity; mc parity alternates per chunk
          int s = 0;
          const bool first_full = ((mc & 1) == par);
          for (; s + 1 < ns; s += 2) {
            if (first_full) {
              full_step(s);
              rec_step(s + 1);
            } else {
              rec_step(s);
              full_step(s + 1);
            }
          }
          if (s < ns) {
            if (first_full)
              full_step(s);
            else
              rec_step(s);
          }
        } else {
#pragma unroll 2
          for (int s = 0; s < ns; s++) full_step(s);
        }
      } else {
        for (int s = 0; s < ns; s++) {
          const int mu = mc - s;
          double2 qp[NI], g[NJ][NG];
#pragma unroll
          for (int i = 0; i < NI; i++) qp[i] = P.q[s][rl[i]];
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            g[j][0] = P.gp[s][cl[j]];
            if (!REAL) g[j][NG - 1] = P.gn[s][cl[j]];
          }
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
                double sm_ = seed_value(T, ll[i], mm[j], ex);
                if ((ll[i] - mm[j]) & 1) sm_ = -sm_;
                y[e] = split_level(sm_ / T.Bt[2 * ll[i]], ex, lev[e]);
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
    if (k + 1 < nchunks) {
      mbar_wait(&sm.bar[(k + 1) & 1], ((k + 1) >> 1) & 1);
      fwd_derive<REAL>(a, sm.raw[(k + 1) & 1], sm.par[(k + 1) & 1], mc - kChunk, l0b, c0, tid);
    }
    __syncthreads();
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
          const double sm_ = (m & 1) ? -1.0 : 1.0;
          out[base - m] = make_double2(sm_ * f.x, -sm_ * f.y);
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

template <bool REAL, bool SPIN0>
static void launch_fwd(const FwdArgs& a, dim3 grid, cudaStream_t st) {
  const size_t smem = sizeof(fwd::Smem);
  cudaFuncSetAttribute(k_forward_core<REAL, SPIN0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  k_forward_core<REAL, SPIN0><<<grid, kThreads, smem, st>>>(a);
}

void launch_forward_core(const FwdArgs& a, int ntiles, int nmaps, bool real, cudaStream_t st) {
  dim3 grid(ntiles, nmaps);
  if (real)
    launch_fwd<true, true>(a, grid, st);
  else if (a.spin == 0)
    launch_fwd<false, true>(a, grid, st);
  else
    launch_fwd<false, false>(a, grid, st);
}

}  // namespace mwsht
