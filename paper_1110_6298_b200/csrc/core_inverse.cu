// Inverse core: T[m', m] = sum_l c_l Delta^l_{m'm} Delta^l_{m',-s} f_lm  (both signs of m).
//
// Replaces the reference's fmm_core (pkg/src/torusht/kernels/_numba.py:74-105)
// and fmm_core_real (:108-128).  The reference walks l serially, regenerating
// the whole pi/2 quadrant per degree with Trapani (or Risbo) and scattering
// into T.  Here every (m', m) pair is an independent three-term chain in l
// (DESIGN.md §3.1): no plane is ever materialised, T accumulates in registers
// for the whole l range, and the only per-step inputs are O(L) row/column
// parameters.
//
// CTA: 8 consumer warps own a 64 (m') x 32 (m) tile, 4x2 chains per thread;
// a warp's 16 rows share one parity (spin 0: Delta^l_{m',0} = 0 when l+m' is
// odd, so a whole warp skips the contraction on alternate degrees).  A
// producer warp (warpgroup 0, registers handed to the consumers with
// setmaxnreg) streams the per-degree parameters -- rows of the plan table
// (kap_l C_l(m'), W_l(m')), rows of C_l(m), and rows of the pre-scaled
// coefficients c_l u_l(m) f_{l,+-m} -- with TMA bulk copies (cp.async.bulk ->
// UBLKCP) into a kStages-deep ring of 16-degree stages guarded by full/empty
// mbarriers, one bulk copy per array and stage (the tables and staging planes
// are column-blocked, common.cuh).  Consumer warps never meet at a CTA barrier;
// full 16-degree chunks run as straight-line code.
//
// Spin 0 uses the paired variant of this kernel (core_inverse_paired.cu),
// which feeds two contractions from one recursion via the transpose symmetry.
#include "common.cuh"

#ifndef MWSHT_INV_UNROLL
// degree pairs per loop iteration (spin 0) for two-map CTAs; one-map CTAs
// unroll the whole chunk.  C4 (8 maps, L=2048): 2 -> 11.36 ms per inverse
// batch, 4 -> 12.15, 8 -> 12.08.
#define MWSHT_INV_UNROLL 2
#endif
#ifndef MWSHT_NS_UNROLL
#define MWSHT_NS_UNROLL 16  // degrees per loop iteration (spin != 0): full chunk measured best
#endif
namespace mwsht {
constexpr int INV_UNR = MWSHT_INV_UNROLL, NS_UNR = MWSHT_NS_UNROLL;


namespace inv {
constexpr int R = kTileRows, C = kTileCols, CH = kChunk;
// MB maps of a batch share every chain (one recursion, MB contractions);
// their staging rows enlarge the stage, so the ring is one stage shorter.
// MSP (multi-spin): each map also gets its own row weights W_l(m'; s_map).
template <int MB, bool MSP>
struct Stage {
  double2 row[CH][R];      // (kap_l C_l(m'), W_l(m'))
  double colc[CH][C];      // C_l(m)
  double2 gp[MB][CH][C];   // c_l u_l(m) f_{l,m}
  double2 gn[MB][CH][C];   // c_l u_l(m) (-1)^l f_{l,-m}
};
// multi-spin stages also carry each map's W_l(m'; s_map) (no member otherwise:
// the plain stages keep their 128-byte-multiple size)
template <int MB>
struct Stage<MB, true> {
  double2 row[CH][R];
  double colc[CH][C];
  double2 gp[MB][CH][C];
  double2 gn[MB][CH][C];
  double w[MB][CH][R];
};
template <int MB, bool MSP = false, int FW = kConsumerWarps>
struct Smem {
  static constexpr int NB = MSP ? kStages - 2 : (MB == 1 ? kStages : kStages - 1);
  Stage<MB, MSP> st[NB];
  double seedz[2048 / (32 * FW)][32 * FW];  // one seed per chain of the 64 x 32 tile
  uint64_t full[NB], empty[NB];
};
}  // namespace inv

// one level step down (x 2^-768) for every chain whose stored value reached 2^200
template <int NE>
__device__ __forceinline__ void rescale(double (&z)[NE], double (&zp)[NE], unsigned& lv) {
#pragma unroll
  for (int e = 0; e < NE; e++) {
    if (((lv >> (4 * e)) & 15u) && above_top(z[e])) {
      const double sh = pow2i(-kLevShift);
      z[e] *= sh;
      zp[e] *= sh;
      lv -= 1u << (4 * e);
    }
  }
}

// FW consumer warps: 8 (4 x 2 chains per thread, registers raised with
// setmaxnreg) or 16 (2 x 2 chains per thread, no register hand-off; one map,
// L <= 1024, as the forward core).
template <bool REAL, bool SPIN0, int MB, bool MSP = false, int FW = kConsumerWarps>
__global__ void __launch_bounds__(128 + 32 * FW, 1) k_inverse_core(InvArgs a) {
  constexpr int NI = 32 / FW, NJ = 2, NE = NI * NJ;
  constexpr int PB = 4 * NI;  // row pairs per warp (a warp's rows share one parity)
  constexpr int NG = REAL ? 1 : 2;  // complex g values per column: f_{l,m} (+ f_{l,-m})
  using Sm = inv::Smem<MB, MSP, FW>;
  constexpr int NB = Sm::NB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  pdl_trigger();  // dependents may start their prologue once every tile has started
  // maps of this CTA: MB * blockIdx.y + mb (the last pair of an odd batch repeats
  // its map; that copy's results are not written)
  auto map_of = [&](int mb) { return min(MB * (int)blockIdx.y + mb, a.nmaps - 1); };

  const DevTables& T = a.t;
  const int L = T.L, N = T.N, Lp = a.ldw;
  const int2 tile = a.tiles[blockIdx.x];
  const int r0 = tile.x, c0 = tile.y;
  const int lstart = max(r0, c0);
  const int nchunks = (L - lstart + kChunk - 1) / kChunk;
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
    // warpgroup 0: warp 0 streams the stages, warps 1-3 retire; registers go to the consumers
    if constexpr (FW == 8) setmaxnreg_dec<kProducerRegs>();
    if (wall != 0) return;
    pdl_wait();  // staged inputs come from the previous kernel
    // ------------------------------------------------------------ producer
    const double2* rowtab = a.rowtab;
    const double2* gpm[MB];
#pragma unroll
    for (int mb = 0; mb < MB; mb++) gpm[mb] = a.gp + (long long)map_of(mb) * a.g_stride;
    // blocked layouts (common.cuh): a chunk is one contiguous copy per array
    if (lane == 0) {
      for (int k = 0; k < nchunks; k++) {
        const int b = k % NB, lc = lstart + k * kChunk, ns = min(kChunk, L - lc);
        if (k >= NB) mbar_wait(&sm.empty[b], ((k / NB) - 1) & 1);
        fence_proxy_async();
        mbar_arrive_expect_tx(&sm.full[b],
                              ns * (inv::R * 16u + inv::C * 8u + MB * NG * inv::C * 16u +
                                    (MSP ? MB * inv::R * 8u : 0u)));
        auto& S = sm.st[b];
        const long long oc = blk<inv::C>(lc, c0, L);
        bulk_g2s(&S.row[0][0], rowtab + blk<inv::R>(lc, r0, L), ns * inv::R * 16, &sm.full[b]);
        if constexpr (MSP) {
#pragma unroll
          for (int mb = 0; mb < MB; mb++)
            bulk_g2s(&S.w[mb][0][0], a.wrow_m[map_of(mb)] + blk<inv::R>(lc, r0, L),
                     ns * inv::R * 8, &sm.full[b]);
        }
        bulk_g2s(&S.colc[0][0], a.colc + oc, ns * inv::C * 8, &sm.full[b]);
#pragma unroll
        for (int mb = 0; mb < MB; mb++) {
          bulk_g2s(&S.gp[mb][0][0], gpm[mb] + oc, ns * inv::C * 16, &sm.full[b]);
          if (!REAL)
            bulk_g2s(&S.gn[mb][0][0], gpm[mb] + (long long)L * Lp + oc, ns * inv::C * 16,
                     &sm.full[b]);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  if constexpr (FW == 8) setmaxnreg_inc<kConsumerRegs>();
  const int w = wall - 4, tid = threadIdx.x - 128;
  const int wr = w % (FW / 2), wc = w / (FW / 2), r = lane & 3, c = lane >> 2, par = wr & 1;
  int rl[NI], cl[NJ], mp[NI], mm[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    rl[i] = par + 2 * (PB * (wr >> 1) + 4 * i + r);
    mp[i] = r0 + rl[i];
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    cl[j] = 16 * wc + c + 8 * j;
    mm[j] = c0 + cl[j];
  }

  int rl0 = rl[0], cl0 = cl[0];
  asm volatile("" : "+r"(rl0), "+r"(cl0));

  // seeds: z^{l0} = Delta^{l0}_{m'm} / ((-1)^l0 lam_l0 u_l0(m) u_l0(m')), l0 = max(m', m),
  // Delta^{l0}_{m'm} = sign sqrt(C(2 l0, l0 + min))/2^l0 = sign P0(l0) R(l0+mu) R(l0-mu)
  // (common.cuh seed factors), carried in exponent levels
  unsigned slv = 0;  // seed levels, 4 bits per chain
#pragma unroll
  for (int i = 0; i < NI; i++)
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int e = i * NJ + j;
      double zs = 0.0;
      int lev = 0;
      if (mp[i] < L && mm[j] < L) {
        const int l0 = max(mp[i], mm[j]), mu = min(mp[i], mm[j]);
        int ex;
        double s_ = seed3(T.sd_pi[l0], T.sd_qi[l0 + mu], T.sd_qi[l0 - mu], ex);
        if (mm[j] < mp[i] && ((mp[i] - mm[j]) & 1)) s_ = -s_;
        if (l0 & 1) s_ = -s_;
        zs = split_level(s_, ex, lev);
      }
      sm.seedz[e][tid] = zs;
      slv |= (unsigned)lev << (4 * e);
    }
  pdl_wait();  // the epilogue overwrites outputs the previous kernel may read

  double z[NE], zp[NE], acc[MB][NE][2 * NG];
#pragma unroll
  for (int e = 0; e < NE; e++) {
    z[e] = 0.0;
    zp[e] = 0.0;
#pragma unroll
    for (int mb = 0; mb < MB; mb++)
#pragma unroll
      for (int k = 0; k < 2 * NG; k++) acc[mb][e][k] = 0.0;
  }
  unsigned lv = 0;  // current levels, 4 bits per chain (0 = true scale)

  const int wrow_lo = r0 + par + 2 * PB * (wr >> 1);
  const int wcol_lo = c0 + 16 * wc;
  const bool warp_has = wrow_lo < L && wcol_lo < L;
  const int wl0_min = max(wrow_lo, wcol_lo);
  bool fast = false, started = false;

  for (int k = 0; k < nchunks; k++) {
    const int b = k % NB, lc = lstart + k * kChunk, ns = min(kChunk, L - lc);
    mbar_wait(&sm.full[b], (k / NB) & 1);
    // rl[i] = rl0 + 8 i, cl[j] = cl0 + 8 j: one base pointer per array and chunk,
    // constant offsets per entry (rl0/cl0 opaque: never rematerialised from %tid)
    const auto& S = sm.st[b];
    const double2* rowp = &S.row[0][0] + rl0;
    const double* colp = &S.colc[0][0] + cl0;
    const double2* gpp = &S.gp[0][0][0] + cl0;
    const double2* gnp = &S.gn[0][0][0] + cl0;
    const double* wpp = nullptr;
    if constexpr (MSP) wpp = &S.w[0][0][0] + rl0;
    constexpr int MS = inv::CH * inv::C;  // distance between maps' staging rows
    constexpr int MW = inv::CH * inv::R;  // distance between maps' weight rows (MSP)

    if (warp_has && wl0_min < lc + ns) {
      if (!started) {
        // Ghost start: below its first degree l0 a chain's
        // recursion coefficient kap_l C_l(m') C_l(m) is exactly 0 (the tables
        // are zero for x > l), so the recursion maps (z^l, z^{l-1}) to
        // (-z^{l-1}, z^l) and the pair (seed, 0) at l0 has the exact
        // continuation z^l = (-1)^((l0-l)/2) seed for l = l0 mod 2, else 0.
        // Starting every chain there at this chunk's first degree needs no
        // per-degree injection; its ghost terms contract against W_l(m') or
        // g_l(m), which are exactly 0 below l0.
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const int d = max(mp[i], mm[j]) - lc;  // >= 0: lc <= wl0_min <= l0
            const double sd = (mp[i] < L && mm[j] < L) ? sm.seedz[e][tid] : 0.0;
            const double g0 = ((d >> 1) & 1) ? -sd : sd;  // z^{lc}   (d even)
            const double g1 = (((d + 1) >> 1) & 1) ? -sd : sd;  // z^{lc-1} (d odd)
            z[e] = (d & 1) ? 0.0 : g0;
            zp[e] = (d & 1) ? g1 : 0.0;
          }
        lv = slv;
        started = true;
      }
      if (!fast) fast = __all_sync(0xffffffffu, lv == 0);
      {
        // ------------------------------------------------------- steady state
        // Every chain runs (ghost or live).  Chains still carrying exponent levels
        // (lv != 0: true value below 2^-568) are masked out of the contraction
        // for the whole chunk; one rescale check at the chunk end suffices
        // (a chain grows at most 4x per degree: 2^32 per chunk from <= 2^200),
        // and a chain that reaches level 0 inside a chunk contributes from the
        // next one without loss.  fast: no chain in the warp carries a level.
        unsigned live = 0xffffffffu;
        if (!fast) {
          live = 0;
#pragma unroll
          for (int e = 0; e < NE; e++) live |= (((lv >> (4 * e)) & 15u) == 0) ? (1u << e) : 0u;
        }
        const bool contract = fast || __any_sync(0xffffffffu, live != 0);
        auto rec_step = [&](int s) {
          double2 rp[NI];
          double cc[NJ];
#pragma unroll
          for (int i = 0; i < NI; i++) rp[i] = rowp[s * inv::R + 8 * i];
#pragma unroll
          for (int j = 0; j < NJ; j++) cc[j] = colp[s * inv::C + 8 * j];
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
        auto full_step = [&](auto masked, int s) {
          double2 rp[NI];
          double cc[NJ];
          double2 g[MB][NJ][NG];
          double wv[MSP ? MB : 1][NI];
#pragma unroll
          for (int i = 0; i < NI; i++) rp[i] = rowp[s * inv::R + 8 * i];
          if constexpr (MSP) {
#pragma unroll
            for (int mb = 0; mb < MB; mb++)
#pragma unroll
              for (int i = 0; i < NI; i++) wv[mb][i] = wpp[mb * MW + s * inv::R + 8 * i];
          }
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            cc[j] = colp[s * inv::C + 8 * j];
#pragma unroll
            for (int mb = 0; mb < MB; mb++) {
              g[mb][j][0] = gpp[mb * MS + s * inv::C + 8 * j];
              if (!REAL) g[mb][j][NG - 1] = gnp[mb * MS + s * inv::C + 8 * j];
            }
          }
#pragma unroll
          for (int i = 0; i < NI; i++)
#pragma unroll
            for (int j = 0; j < NJ; j++) {
              const int e = i * NJ + j;
              double t = z[e] * rp[i].y;
              if (decltype(masked)::value) t = ((live >> e) & 1u) ? t : 0.0;
#pragma unroll
              for (int mb = 0; mb < MB; mb++) {
                double tm = t;
                if constexpr (MSP) {
                  tm = z[e] * wv[mb][i];
                  if (decltype(masked)::value) tm = ((live >> e) & 1u) ? tm : 0.0;
                }
#pragma unroll
                for (int k2 = 0; k2 < NG; k2++) {
                  acc[mb][e][2 * k2] = fma(tm, g[mb][j][k2].x, acc[mb][e][2 * k2]);
                  acc[mb][e][2 * k2 + 1] = fma(tm, g[mb][j][k2].y, acc[mb][e][2 * k2 + 1]);
                }
              }
              const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
              zp[e] = z[e];
              z[e] = zn;
            }
        };
        auto run = [&](auto masked) {
          if (ns == kChunk) {
            // full chunk: straight-line code, compile-time smem offsets
            if (SPIN0) {
              // lc is even (tile corners are multiples of 32): pairs (even l, odd l)
              if (par == 0) {
#pragma unroll(MB == 2 ? INV_UNR : kChunk / 2)
                for (int s = 0; s < kChunk; s += 2) {
                  full_step(masked, s);
                  rec_step(s + 1);
                }
              } else {
#pragma unroll(MB == 2 ? INV_UNR : kChunk / 2)
                for (int s = 0; s < kChunk; s += 2) {
                  rec_step(s);
                  full_step(masked, s + 1);
                }
              }
            } else {
#pragma unroll NS_UNR
              for (int s = 0; s < kChunk; s++) full_step(masked, s);
            }
          } else if (SPIN0) {
            int s = 0;
            for (; s + 1 < ns; s += 2) {
              if (par == 0) {
                full_step(masked, s);
                rec_step(s + 1);
              } else {
                rec_step(s);
                full_step(masked, s + 1);
              }
            }
            if (s < ns) {
              if (par == 0)
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
          rescale(z, zp, lv);
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
  const int sgs = (spin & 1) ? -1 : 1;  // (-1)^s
  double2* __restrict__ out = a.out + (long long)map_of(mb) * a.out_stride;
#pragma unroll
  for (int i = 0; i < NI; i++) {
    const int x = mp[i];
    if (x >= L) continue;
    double sn, cs;
    sincospi((double)x / (double)N, &sn, &cs);
    const double2 tw = make_double2(cs, sn);       // e^{+i m' theta0}
    const double2 twc = make_double2(cs, -sn);     // e^{-i m' theta0}
    const int binp = x, binn = x ? N - x : 0;
    // out_mode 3: the m' >= 0 half only (the theta stage rebuilds F[m, -m'] = +-F[m, m'] e^{-2 pi i m'/N})
    const bool wmir = x && a.out_mode != 3;
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int m = mm[j];
      if (m >= L) continue;
      const int e = i * NJ + j;
      const double2 Tp = make_double2(acc[mb][e][0], acc[mb][e][1]);
      if (a.out_mode == 1) {
        if (REAL) {
          out[(long long)x * L + m] = Tp;
        } else {
          out[(long long)x * N + (L - 1 + m)] = Tp;
          if (m > 0) {
            const double sx = (x & 1) ? -1.0 : 1.0;
            out[(long long)x * N + (L - 1 - m)] = make_double2(sx * acc[mb][e][2], sx * acc[mb][e][3]);
          }
        }
        continue;
      }
      if (REAL) {
        // fhalf[m, m'] = T[m', m] i^{-m}; mirror (-1)^m (mw.py:550-556)
        const double2 F = cmul(Tp, ipow(-m));
        double2* row = out + (long long)m * N;
        row[binp] = cmul(F, tw);
        if (wmir) row[binn] = cscale(cmul(F, twc), (m & 1) ? -1.0 : 1.0);
      } else {
        // F[m, m'] = (-1)^s i^{-(m+s)} T[m', m]; F[m, -m'] = (-1)^(m+s) F[m, m'] (mw.py:395-401)
        const double2 Fp = cscale(cmul(Tp, ipow(-(m + spin))), (double)sgs);
        double2* rowp = out + (long long)(L - 1 + m) * N;
        rowp[binp] = cmul(Fp, tw);
        if (wmir) rowp[binn] = cscale(cmul(Fp, twc), ((m + spin) & 1) ? -1.0 : 1.0);
        if (m > 0) {
          const double sx = (x & 1) ? -1.0 : 1.0;
          const double2 Tn = make_double2(sx * acc[mb][e][2], sx * acc[mb][e][3]);
          const double2 Fn = cscale(cmul(Tn, ipow(m - spin)), (double)sgs);
          double2* rown = out + (long long)(L - 1 - m) * N;
          rown[binp] = cmul(Fn, tw);
          if (wmir) rown[binn] = cscale(cmul(Fn, twc), ((m + spin) & 1) ? -1.0 : 1.0);
        }
      }
    }
  }
}
}

template <bool REAL, bool SPIN0, int MB, bool MSP = false, int FW = kConsumerWarps>
static void launch_inv(const InvArgs& a, int ntiles, cudaStream_t st) {
  const size_t smem = sizeof(inv::Smem<MB, MSP, FW>);
  smem_attr_once((const void*)k_inverse_core<REAL, SPIN0, MB, MSP, FW>, smem);
  dim3 grid(ntiles, (a.nmaps + MB - 1) / MB);
  launch_pdl(k_inverse_core<REAL, SPIN0, MB, MSP, FW>, grid, dim3(128 + 32 * FW), smem, st, a);
}

// Consumer warps of the single-map plain inverse core (MWSHT_INV_CW=8|16
// overrides): 16 up to L = 320 (C2 inverse core 55.5 -> 53.1 us), 8 above
// (L = 512 / 1024: 1-3% slower with 16; tools/inv_ab.sh).
static int inv_warps(int L) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("MWSHT_INV_CW");
    env = e ? atoi(e) : 0;
  }
  if (env == 8 || env == 16) return env;
  return L <= 320 ? 16 : 8;
}

template <int MB>
static void launch_inv_mb(const InvArgs& a, int ntiles, bool real, cudaStream_t st) {
  if (a.msp) {  // mixed spins: every degree contracts (no spin-0 parity skip)
    launch_inv<false, false, 2, true>(a, ntiles, st);
  } else if (MB == 1 && inv_warps(a.t.L) == 16) {
    if (real)
      launch_inv<true, true, 1, false, 16>(a, ntiles, st);
    else if (a.spin == 0)
      launch_inv<false, true, 1, false, 16>(a, ntiles, st);
    else
      launch_inv<false, false, 1, false, 16>(a, ntiles, st);
  } else if (real)
    launch_inv<true, true, MB>(a, ntiles, st);
  else if (a.spin == 0)
    launch_inv<false, true, MB>(a, ntiles, st);
  else
    launch_inv<false, false, MB>(a, ntiles, st);
}

void launch_inverse_core_paired(const InvArgs& a, int ntiles, int nmaps, bool real,
                                cudaStream_t st);  // core_inverse_paired.cu

// Batches of two or more maps run two maps per CTA: each chain's recursion
// then feeds both maps' contractions.
void launch_inverse_core(const InvArgs& a0, int ntiles, int nmaps, bool real, cudaStream_t st) {
  if (a0.paired) {
    launch_inverse_core_paired(a0, ntiles, nmaps, real, st);
    return;
  }
  InvArgs a = a0;
  a.nmaps = nmaps;
  if (nmaps >= 2)
    launch_inv_mb<2>(a, ntiles, real, st);
  else
    launch_inv_mb<1>(a, ntiles, real, st);
}


}  // namespace mwsht
