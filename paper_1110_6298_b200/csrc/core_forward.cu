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
// CTA: 8 consumer warps own 64 degrees l x 32 orders m, 4x2 chains per thread;
// a warp's 16 degrees share one parity (spin 0: Delta^l_{m',0} = 0 when l-m'
// is odd, so whole warps skip alternate contraction steps).  A producer warp
// (warpgroup 0, registers handed to the consumers with setmaxnreg) streams,
// per 16-value chunk of m' (walking down), the plan-table rows (coefficient,
// W'(l, m')) and the folded staging rows gfT[m'][+m] and (-1)^m' gfT[m'][-m]
// with one TMA bulk copy per array into a kStages-deep mbarrier ring (the
// tables and staging planes are column-blocked, common.cuh).
#include "common.cuh"

#ifndef MWSHT_FWD_UNROLL
#define MWSHT_FWD_UNROLL 4  // degree pairs per loop iteration: 4 measured 3% faster than 8 (full)
#endif
namespace mwsht {
#ifndef MWSHT_FNS_UNROLL
#define MWSHT_FNS_UNROLL 16  // degrees per loop iteration (spin != 0): full chunk measured best
#endif
constexpr int FWD_UNR = MWSHT_FWD_UNROLL, FNS_UNR = MWSHT_FNS_UNROLL;

namespace fwd {
constexpr int R = kTileRows, C = kTileCols, CH = kChunk;
// MB maps of a batch share every chain (one recursion, MB contractions);
// their staging rows double the stage size, so the ring is one stage shorter.
// MSP (multi-spin): each map also gets its own weights W'(l, m'; s_map).
template <int MB, bool MSP>
struct Stage {
  double2 q[CH][R];        // (coefficient producing y_{m'-1}, W'(l, m'))
  double2 gp[MB][CH][C];   // gfold[+m][m']
  double2 gn[MB][CH][C];   // (-1)^m' gfold[-m][m']
};
// multi-spin stages also carry each map's W'(l, m'; s_map) (no member otherwise:
// the plain stages keep their 128-byte-multiple size)
template <int MB>
struct Stage<MB, true> {
  double2 q[CH][R];
  double2 gp[MB][CH][C];
  double2 gn[MB][CH][C];
  double w[MB][CH][R];
};
template <int MB, bool MSP = false, int FW = kConsumerWarps>
struct Smem {
  static constexpr int NB = MSP ? kStages - 2 : (MB == 1 ? kStages : kStages - 1);
  Stage<MB, MSP> st[NB];
  double seedy[2048 / (32 * FW)][32 * FW];  // one seed per chain of the 64 x 32 tile
  uint64_t full[NB], empty[NB];
};
}  // namespace fwd

// one level step down (x 2^-768) for every chain whose stored value reached 2^200
template <int NE>
__device__ __forceinline__ void rescale(double (&y)[NE], double (&y1)[NE], unsigned& lv) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (((lv >> (4 * e)) & 15u) && above_top(y[e])) {
      const double sh = pow2i(-kLevShift);
      y[e] *= sh;
      y1[e] *= sh;
      lv -= 1u << (4 * e);
    }
  }
}

// Warp-specialised 384-thread CTA (common.cuh): warpgroup 0 = TMA producer,
// warpgroups 1-2 = 8 consumer warps with a raised register budget.
// FW consumer warps: 8 (4 x 2 chains per thread, registers raised to 232 with
// setmaxnreg) or 16 (2 x 2 chains per thread: twice the warps per scheduler
// to hide the FP64 latency; 96 registers, no register hand-off needed).
template <bool REAL, bool SPIN0, int MB, bool MSP = false, int FW = kConsumerWarps>
__global__ void __launch_bounds__(128 + 32 * FW, 1) k_forward_core(FwdArgs a) {
  constexpr int NI = 32 / FW, NJ = 2, NE = NI * NJ;
  constexpr int PB = 4 * NI;  // row pairs per warp (a warp's rows share one parity)
  constexpr int NG = REAL ? 1 : 2;
  using Sm = fwd::Smem<MB, MSP, FW>;
  constexpr int NB = Sm::NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  pdl_trigger();  // dependents may start their prologue once every tile has started
  // maps of this CTA: MB * blockIdx.y + mb (the last pair of an odd batch repeats
  // its map; that copy's results are not written)
  auto map_of = [&](int mb) { return min(MB * (int)blockIdx.y + mb, a.nmaps - 1); };

  const DevTables& T = a.t;
  const int L = T.L, Lp = a.ldw;
  const int2 tile = a.tiles[blockIdx.x];
  const int l0b = tile.x, c0 = tile.y;
  const int mu_top = min(l0b + kTileRows - 1, L - 1);
  const int nchunks = (mu_top + kChunk) / kChunk;
  const int lane = threadIdx.x & 31, wall = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; b++) {
      mbar_init(&sm.full[b], 1);
      mbar_init(&sm.empty[b], FW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (wall < 4) {
    // warpgroup 0: warp 0 streams the stages, warps 1-3 retire
    if constexpr (FW == 8) setmaxnreg_dec<kProducerRegs>();
    if (wall != 0) return;
    pdl_wait();  // staged inputs come from the previous kernel
    // ------------------------------------------------------------ producer
    const double2* gpm[MB];
#pragma unroll
    for (int mb = 0; mb < MB; mb++) gpm[mb] = a.gf + (long long)map_of(mb) * a.in_stride;
    // blocked layouts (common.cuh): the chunk's steps mu = mc .. mc-ns+1 are one
    // contiguous block (ascending mu), placed in stage rows CH-ns .. CH-1 so
    // that step s (mu = mc - s) always sits in row CH-1-s
    if (lane == 0) {
      for (int k = 0; k < nchunks; k++) {
        const int b = k % NB, mc = mu_top - k * kChunk, ns = min(kChunk, mc + 1);
        if (k >= NB) mbar_wait(&sm.empty[b], ((k / NB) - 1) & 1);
        fence_proxy_async();
        mbar_arrive_expect_tx(&sm.full[b], ns * (fwd::R * 16u + MB * NG * fwd::C * 16u +
                                                 (MSP ? MB * fwd::R * 8u : 0u)));
        auto& S = sm.st[b];
        const int mlo = mc - ns + 1;
        const long long oc = blk<fwd::C>(mlo, c0, L);
        bulk_g2s(&S.q[fwd::CH - ns][0], a.rowtab + blk<fwd::R>(mlo, l0b, L), ns * fwd::R * 16,
                 &sm.full[b]);
        if constexpr (MSP) {
#pragma unroll
          for (int mb = 0; mb < MB; mb++)
            bulk_g2s(&S.w[mb][fwd::CH - ns][0], a.wrow_m[map_of(mb)] + blk<fwd::R>(mlo, l0b, L),
                     ns * fwd::R * 8, &sm.full[b]);
        }
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          bulk_g2s(&S.gp[mb][fwd::CH - ns][0], gpm[mb] + oc, ns * fwd::C * 16, &sm.full[b]);
          if (!REAL)
            bulk_g2s(&S.gn[mb][fwd::CH - ns][0], gpm[mb] + (long long)L * Lp + oc,
                     ns * fwd::C * 16, &sm.full[b]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if constexpr (FW == 8) setmaxnreg_inc<kConsumerRegs>();
  const int w = wall - 4, tid = threadIdx.x - 128;
  const int wr = w % (FW / 2), wc = w / (FW / 2), r = lane & 3, c = lane >> 2, par = wr & 1;
  int rl[NI], cl[NJ], ll[NI], mm[NJ];
  double md[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    rl[i] = par + 2 * (PB * (wr >> 1) + 4 * i + r);
    ll[i] = l0b + rl[i];
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    cl[j] = 16 * wc + c + 8 * j;
    mm[j] = c0 + cl[j];
    md[j] = (double)mm[j];
  }

  int rl0 = rl[0], cl0 = cl[0];
  asm volatile("" : "+r"(rl0), "+r"(cl0));

  // seeds: y_l = Delta^l_{l,m} / (A(0) Bt(2l)), Delta^l_{l,m} = (-1)^(l-m) sqrt(C(2l,l+m))/2^l
  unsigned slv = 0;
#pragma unroll
  for (int i = 0; i < NI; i++)
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int e = i * NJ + j;
      double ys = 0.0;
      int lev = 0;
      if (mm[j] <= ll[i] && ll[i] < L) {
        int ex;
        double s_ = seed3(T.sd_pf[ll[i]], T.sd_r[ll[i] + mm[j]], T.sd_r[ll[i] - mm[j]], ex);
        if ((ll[i] - mm[j]) & 1) s_ = -s_;
        ys = split_level(s_, ex, lev);
      }
      sm.seedy[e][tid] = ys;
      slv |= (unsigned)lev << (4 * e);
    }
  pdl_wait();  // the epilogue overwrites outputs the previous kernel may read

  double y[NE], y1[NE], acc[MB][NE][2 * NG];
#pragma unroll
  for (int e = 0; e < NE; e++) {
    y[e] = 0.0;
    y1[e] = 0.0;
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int k = 0; k < 2 * NG; k++) acc[mb][e][k] = 0.0;
  }
  unsigned lv = 0;

  // warp extents.  Valid chains: m <= l < L; chain (l, m) starts at m' = l.
  const int wrow_lo = l0b + par + 2 * PB * (wr >> 1);
  const int wrow_hi = min(wrow_lo + 2 * PB - 2, L - 1);
  const int wcol_lo = c0 + 16 * wc;
  const bool warp_has = wrow_lo < L && wcol_lo <= wrow_hi;
  bool fast = false, started = false;

  for (int k = 0; k < nchunks; k++) {
    const int b = k % NB, mc = mu_top - k * kChunk, ns = min(kChunk, mc + 1);
    mbar_wait(&sm.full[b], (k / NB) & 1);
    // rl[i] = rl0 + 8 i, cl[j] = cl0 + 8 j: one base pointer per array and chunk
    const auto& S = sm.st[b];
    const double2* rowp = &S.q[fwd::CH - 1][0] + rl0;  // step s at row CH-1-s
    const double2* gpp = &S.gp[0][fwd::CH - 1][0] + cl0;
    const double2* gnp = &S.gn[0][fwd::CH - 1][0] + cl0;
    const double* wpp = nullptr;
    if constexpr (MSP) wpp = &S.w[0][fwd::CH - 1][0] + rl0;
    constexpr int MS = fwd::CH * fwd::C;  // distance between maps' staging rows
    constexpr int MW = fwd::CH * fwd::R;  // distance between maps' weight rows (MSP)

    if (warp_has && wrow_hi >= mc - ns + 1) {
      if (!started) {
        // Ghost start: above its first value m' = l the
        // chain's coefficient m alpha(l-m'+1) beta(l+m'-1) is exactly 0 (the
        // tables are zero for m' > l), so (y_l, y_{l+1}) = (seed, 0) has the
        // exact continuation y_mu = (-1)^((mu-l)/2) seed for mu = l mod 2,
        // else 0.  Starting every chain there at this chunk's top value needs
        // no per-step injection; the ghost terms meet W'(l, mu) = 0.
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const int d = mc - ll[i];  // >= 0: the first chunk holds the warp's top degree
            const double sd = sm.seedy[e][tid];
            const double g0 = ((d >> 1) & 1) ? -sd : sd;        // y_{mc}   (d even)
            const double g1 = (((d + 1) >> 1) & 1) ? -sd : sd;  // y_{mc+1} (d odd)
            y[e] = (d & 1) ? 0.0 : g0;
            y1[e] = (d & 1) ? g1 : 0.0;
          }
        lv = slv;
        started = true;
      }
      if (!fast) fast = __all_sync(0xffffffffu, lv == 0);
      {
        // ------------------------------------------------------- steady state
        // Every chain runs (ghost or live).  Chains still carrying exponent levels are
        // masked out of the contraction for the whole chunk and checked for a
        // rescale once at its end (no overflow: stored values stay far below
        // 2^1023 within 16 steps of 2^200; a chain reaching level 0 inside the
        // chunk is below 2^-464 there and contributes from the next chunk).
        unsigned live = 0xffffffffu;
        if (!fast) {
          live = 0;
#pragma unroll
          for (int e = 0; e < NE; e++) live |= (((lv >> (4 * e)) & 15u) == 0) ? (1u << e) : 0u;
        }
        const bool contract = fast || __any_sync(0xffffffffu, live != 0);
        auto rec_step = [&](int s) {
          double2 qp[NI];
#pragma unroll
          for (int i = 0; i < NI; i++) qp[i] = rowp[-s * fwd::R + 8 * i];
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
        auto full_step = [&](auto masked, int s) {
          double2 qp[NI], g[MB][NJ][NG];
          double wv[MSP ? MB : 1][NI];
#pragma unroll
          for (int i = 0; i < NI; i++) qp[i] = rowp[-s * fwd::R + 8 * i];
          if constexpr (MSP) {
#pragma unroll
            for (int mb = 0; mb < MB; mb++)
#pragma unroll
              for (int i = 0; i < NI; i++) wv[mb][i] = wpp[mb * MW - s * fwd::R + 8 * i];
          }
#pragma unroll
          for (int mb = 0; mb < MB; mb++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              g[mb][j][0] = gpp[mb * MS - s * fwd::C + 8 * j];
              if (!REAL) g[mb][j][NG - 1] = gnp[mb * MS - s * fwd::C + 8 * j];
            }
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              double t = y[e] * qp[i].y;
              if (decltype(masked)::value) t = ((live >> e) & 1u) ? t : 0.0;
#pragma unroll
              for (int mb = 0; mb < MB; mb++) {
                double tm = t;
                if constexpr (MSP) {
                  tm = y[e] * wv[mb][i];
                  if (decltype(masked)::value) tm = ((live >> e) & 1u) ? tm : 0.0;
                }
#pragma unroll
                for (int k2 = 0; k2 < NG; k2++) {
                  acc[mb][e][2 * k2] = fma(tm, g[mb][j][k2].x, acc[mb][e][2 * k2]);
                  acc[mb][e][2 * k2 + 1] = fma(tm, g[mb][j][k2].y, acc[mb][e][2 * k2 + 1]);
                }
              }
              const double yn = fma(md[j] * qp[i].x, y[e], -y1[e]);
              y1[e] = y[e];
              y[e] = yn;
            }
        };
        auto run = [&](auto masked) {
          // contraction when m' has the warp's degree parity (spin 0)
          const bool first_full = ((mc & 1) == par);
          if (ns == kChunk) {
            // full chunk: straight-line code, compile-time smem offsets
            if (SPIN0) {
              if (first_full) {
#pragma unroll FWD_UNR
                for (int s = 0; s < kChunk; s += 2) {
                  full_step(masked, s);
                  rec_step(s + 1);
                }
              } else {
#pragma unroll FWD_UNR
                for (int s = 0; s < kChunk; s += 2) {
                  rec_step(s);
                  full_step(masked, s + 1);
                }
              }
            } else {
#pragma unroll FNS_UNR
              for (int s = 0; s < kChunk; s++) full_step(masked, s);
            }
          } else if (SPIN0) {
            int s = 0;
            for (; s + 1 < ns; s += 2) {
              if (first_full) {
                full_step(masked, s);
                rec_step(s + 1);
              } else {
                rec_step(s);
                full_step(masked, s + 1);
              }
            }
            if (s < ns) {
              if (first_full)
                full_step(masked, s);
              else
                rec_step(s);
            }
          } else {
            for (int s = 0; s < ns; s++) full_step(masked, s);
          }
        };
        if (fast) {
          run(BoolC<false>());
        } else {
          if (contract)
            run(BoolC<true>());
          else
            for (int s = 0; s < ns; s++) rec_step(s);
          rescale(y, y1, lv);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[b]);
  }

  // ---------------------------------------------------------------- epilogue
#pragma unroll
  for (int mb = 0; mb < MB; mb++) {
  if (MB * (int)blockIdx.y + mb >= a.nmaps) break;
  const int spin = MSP ? a.spin_m[map_of(mb)] : a.spin;
  const double sgs = (spin & 1) ? -1.0 : 1.0;
  double2* __restrict__ out = a.out + (long long)map_of(mb) * a.out_stride;
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
      const double2 Rp = make_double2(acc[mb][e][0], acc[mb][e][1]);
      if (a.out_mode == 2) {  // shard's packed block (m-column sharding, common.cuh)
        const double2 f = cscale(cmul(Rp, ipow(m + spin)), sgs * clv);
        out[shard_flm_index(l, m, a.m0, a.m1)] = f;
        if (m > 0) {
          const double sl = (l & 1) ? -1.0 : 1.0;
          const double2 Rn = make_double2(sl * acc[mb][e][2], sl * acc[mb][e][3]);
          out[shard_flm_index(l, -m, a.m0, a.m1)] = cscale(cmul(Rn, ipow(spin - m)), sgs * clv);
        }
        continue;
      }
      if (a.out_mode == 1) {
        if (REAL) {
          out[(long long)l * L + m] = Rp;
        } else {
          const int N = T.N;
          out[(long long)l * N + (L - 1 + m)] = Rp;
          if (m > 0) {
            const double sl = (l & 1) ? -1.0 : 1.0;
            out[(long long)l * N + (L - 1 - m)] = make_double2(sl * acc[mb][e][2], sl * acc[mb][e][3]);
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
        out[base + m] = cscale(cmul(Rp, ipow(m + spin)), sgs * clv);
        if (m > 0) {
          const double sl = (l & 1) ? -1.0 : 1.0;
          const double2 Rn = make_double2(sl * acc[mb][e][2], sl * acc[mb][e][3]);
          out[base - m] = cscale(cmul(Rn, ipow(spin - m)), sgs * clv);
        }
      }
    }
  }
}
}

template <bool REAL, bool SPIN0, int MB, bool MSP = false, int FW = kConsumerWarps>
static void launch_fwd(const FwdArgs& a, int ntiles, cudaStream_t st) {
  const size_t smem = sizeof(fwd::Smem<MB, MSP, FW>);
  smem_attr_once((const void*)k_forward_core<REAL, SPIN0, MB, MSP, FW>, smem);
  dim3 grid(ntiles, (a.nmaps + MB - 1) / MB);
  launch_pdl(k_forward_core<REAL, SPIN0, MB, MSP, FW>, grid, dim3(128 + 32 * FW), smem, st, a);
}

// Consumer warps of the single-map forward core: 16 up to L = 1024 (C3 forward
// core 0.147 -> 0.128 ms: shorter tiles per warp balance better), 8 above
// (C5: 7.87 ms vs 8.53 ms with 16).  MWSHT_FWD_CW=8|16 overrides.
static int fwd_warps(int L) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MWSHT_FWD_CW");
    env = e ? atoi(e) : 0;
  }
  if (env == 8 || env == 16) return env;
  return L <= 1024 ? 16 : 8;
}

template <int MB>
static void launch_fwd_mb(const FwdArgs& a, int ntiles, bool real, cudaStream_t st) {
  if (a.msp) {  // mixed spins: every m' contracts (no spin-0 parity skip)
    launch_fwd<false, false, 2, true>(a, ntiles, st);
  } else if (MB == 1 && fwd_warps(a.t.L) == 16) {
    if (real)
      launch_fwd<true, true, 1, false, 16>(a, ntiles, st);
    else if (a.spin == 0)
      launch_fwd<false, true, 1, false, 16>(a, ntiles, st);
    else
      launch_fwd<false, false, 1, false, 16>(a, ntiles, st);
  } else if (real)
    launch_fwd<true, true, MB>(a, ntiles, st);
  else if (a.spin == 0)
    launch_fwd<false, true, MB>(a, ntiles, st);
  else
    launch_fwd<false, false, MB>(a, ntiles, st);
}

// Batches of two or more maps run two maps per CTA: each chain's recursion
// then feeds both maps' contractions.
void launch_forward_core(const FwdArgs& a0, int ntiles, int nmaps, bool real, cudaStream_t st) {
  FwdArgs a = a0;
  a.nmaps = nmaps;
  if (nmaps >= 2)
    launch_fwd_mb<2>(a, ntiles, real, st);
  else
    launch_fwd_mb<1>(a, ntiles, real, st);
}

}  // namespace mwsht
