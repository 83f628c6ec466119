// Inverse core, paired tiles (spin 0): T[m', m] = sum_l c_l Delta^l_{m'm} Delta^l_{m',0} f_lm.
//
// Same computation and chain recursion as core_inverse.cu (which replaces the
// reference's fmm_core / fmm_core_real, pkg/src/torusht/kernels/_numba.py:74-128;
// read that file's header first).  The transpose symmetry
// Delta^l_{m m'} = (-1)^(m'-m) Delta^l_{m' m} lets the
// chain of (m', m) with m' > m also produce T[m, m'] = (-1)^(m'-m) sum_l z
// W_l(m) g_l(m'): one recursion feeds two contractions, 7 instead of 9 FP64
// instructions per output and degree pair at spin 0.
//
// Tiles cover c0 <= r0 + 32 only.  A warp's 32x32 block strictly below the
// diagonal runs both contractions, a diagonal block runs plain, a block above
// the diagonal idles.  A warp's rows share one parity and so do its columns
// (spin 0: the direct contraction runs on degrees l = m' mod 2, the transposed
// one on l = m mod 2).  The two warps on an SMSP run the same (row, column)
// parity code path, and full chunks run as a rolled loop over degree pairs:
// four such bodies are live per CTA and an unrolled chunk per body overflowed
// the instruction cache (ncu: no_instruction stalls, 2x slower).  Stages hold
// 16 degrees (3 x 72 KB); the chain seeds are recomputed at the ghost start
// instead of parked in shared memory (8 -> 16 degrees per stage: 7.64 ->
// 7.22 ms at L=4096).
#include "common.cuh"

#ifndef MWSHT_PAIR_UNROLL
#define MWSHT_PAIR_UNROLL 1
#endif
namespace mwsht {
constexpr int kPairUnroll = MWSHT_PAIR_UNROLL;  // degree pairs per rolled-loop iteration
}

namespace mwsht {

namespace invp {
constexpr int R = kTileRows, C = kTileCols;
template <int CH, bool P>
struct Stage {
  double2 row[CH][R];  // (kap_l C_l(m'), W_l(m'))
  double colc[CH][C];  // C_l(m)
  double2 gp[CH][C];   // c_l u_l(m) f_{l,m}
  double2 gn[CH][C];   // c_l u_l(m) (-1)^l f_{l,-m}
  // paired tiles only: W_l(m) at the tile's columns; g at the tile's rows (two 32-blocks)
  double wc[P ? CH : 1][C];
  double2 gpr[P ? 2 : 1][P ? CH : 1][C];
  double2 gnr[P ? 2 : 1][P ? CH : 1][C];
};
template <int CH, bool P>
struct Smem {
  static constexpr int NB = 3;  // 3 x 72 KB stages of 16 degrees (no seed buffer: see ghost start)
  Stage<CH, P> st[NB];
  uint64_t full[NB], empty[NB];
};
}  // namespace invp

// one level step down (x 2^-768) for every chain whose stored value reached 2^200
template <int NE>
__device__ __forceinline__ void rescale_p(double (&z)[NE], double (&zp)[NE], unsigned& lv) {
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

template <bool REAL, bool SPIN0, bool PAIRED>
__global__ void __launch_bounds__(kCoreThreadsWS, 1) k_inverse_core_paired(InvArgs a) {
  // Built for spin 0 only (plan.cu use_paired); the SPIN0 / PAIRED template
  // parameters keep the general control flow readable next to core_inverse.cu.
  static_assert(SPIN0 && PAIRED, "paired tiles are instantiated for spin 0 only");
  constexpr int CH = kChunk;  // degrees per stage
  constexpr int NB = invp::Smem<CH, PAIRED>::NB;
  constexpr int NI = 4, NJ = 2, NE = NI * NJ;
  constexpr int NG = REAL ? 1 : 2;     // complex g values per column: f_{l,m} (+ f_{l,-m})
  constexpr int CJ = PAIRED ? 16 : 8;  // column distance between a thread's chains
  constexpr int NA = PAIRED ? NE : 1;  // transposed accumulators
  using Sm = invp::Smem<CH, PAIRED>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Sm& sm = *reinterpret_cast<Sm*>(smem_raw);
  pdl_trigger();  // dependents may start their prologue once every tile has started

  const DevTables& T = a.t;
  const int L = T.L, N = T.N, Lp = a.ldw;
  const int2 tile = a.tiles[blockIdx.x];
  // bit 30 of tile.x: a plain tile (no transpose, every block direct) -- the
  // longest chains at small L, where paired tiles would set the critical path
  const bool plain_tile = (tile.x >> 30) & 1;
  const int r0 = tile.x & 0x3fffffff, c0 = tile.y;
  const int lstart = max(r0, c0);
  const int nchunks = (L - lstart + CH - 1) / CH;
  const int lane = threadIdx.x & 31, wall = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int b = 0; b < NB; b++) {
      mbar_init(&sm.full[b], 1);
      mbar_init(&sm.empty[b], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (wall < 4) {
    // warpgroup 0: warp 0 streams the stages, warps 1-3 retire; registers go to the consumers
    setmaxnreg_dec<kProducerRegs>();
    if (wall != 0) return;
    pdl_wait();  // staged inputs come from the previous kernel
    // ------------------------------------------------------------ producer
    const double2* rowtab = a.rowtab;
    const double2* gp = a.gp + (long long)blockIdx.y * a.g_stride;
    const double2* gn = gp + (long long)L * Lp;
    // blocked layouts (common.cuh): a chunk is one contiguous copy per array
    if (lane == 0) {
      for (int k = 0; k < nchunks; k++) {
        const int b = k % NB, lc = lstart + k * CH, ns = min(CH, L - lc);
        if (k >= NB) mbar_wait(&sm.empty[b], ((k / NB) - 1) & 1);
        fence_proxy_async();
        uint32_t bytes = ns * (invp::R * 16u + invp::C * 8u + NG * invp::C * 16u);
        if (PAIRED && !plain_tile) bytes += ns * (invp::C * 8u + NG * 2u * invp::C * 16u);
        mbar_arrive_expect_tx(&sm.full[b], bytes);
        auto& S = sm.st[b];
        const long long oc = blk<invp::C>(lc, c0, L);
        bulk_g2s(&S.row[0][0], rowtab + blk<invp::R>(lc, r0, L), ns * invp::R * 16, &sm.full[b]);
        bulk_g2s(&S.colc[0][0], a.colc + oc, ns * invp::C * 8, &sm.full[b]);
        bulk_g2s(&S.gp[0][0], gp + oc, ns * invp::C * 16, &sm.full[b]);
        if (!REAL) bulk_g2s(&S.gn[0][0], gn + oc, ns * invp::C * 16, &sm.full[b]);
        if (PAIRED && !plain_tile) {
          bulk_g2s(&S.wc[0][0], a.wcol + oc, ns * invp::C * 8, &sm.full[b]);
#pragma unroll
          for (int hh = 0; hh < 2; hh++) {
            const long long orr = blk<invp::C>(lc, r0 + hh * invp::C, L);
            bulk_g2s(&S.gpr[hh][0][0], gp + orr, ns * invp::C * 16, &sm.full[b]);
            if (!REAL) bulk_g2s(&S.gnr[hh][0][0], gn + orr, ns * invp::C * 16, &sm.full[b]);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  setmaxnreg_inc<kConsumerRegs>();
  const int w = wall - 4;
  double2* __restrict__ out = a.out + (long long)blockIdx.y * a.out_stride;
  // Warps w and w+4 share an SMSP (warp id mod 4).  Plain: (par, h) = bits of w & 3,
  // wc = w >> 2.  Paired: the SMSP's two warps run the same (par, pc) code path
  // (one unrolled body per SMSP in the instruction cache) and differ in h.
  const int wr = w & 3, wc = w >> 2, r = lane & 3, c = lane >> 2;
  const int par = w & 1;
  const int h = PAIRED ? (w >> 2) : (wr >> 1);
  const int pc = PAIRED ? ((w >> 1) & 1) : 0;  // paired: the warp's column parity
  int rl[NI], cl[NJ], mp[NI], mm[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    rl[i] = par + 32 * h + 8 * i + 2 * r;
    mp[i] = r0 + rl[i];
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    cl[j] = PAIRED ? (pc + 2 * c + CJ * j) : (16 * wc + c + CJ * j);
    mm[j] = c0 + cl[j];
  }

  int rl0 = rl[0], cl0 = cl[0], hr0 = par + 2 * r;
  asm volatile("" : "+r"(rl0), "+r"(cl0), "+r"(hr0));

  // seeds: z^{l0} = Delta^{l0}_{m'm} / ((-1)^l0 lam_l0 u_l0(m) u_l0(m')), l0 = max(m', m),
  // Delta^{l0}_{m'm} = sign sqrt(C(2 l0, l0 + min))/2^l0 = sign P0(l0) R(l0+mu) R(l0-mu)
  // (common.cuh seed factors), carried in exponent levels; computed at the
  // ghost start from the constant factor tables (no shared-memory buffer)
  auto seed_of = [&](int i, int j, int& lev) {
    lev = 0;
    if (mp[i] >= L || mm[j] >= L) return 0.0;
    const int l0 = max(mp[i], mm[j]), mu = min(mp[i], mm[j]);
    int ex;
    double s_ = seed3(T.sd_pi[l0], T.sd_qi[l0 + mu], T.sd_qi[l0 - mu], ex);
    if (mm[j] < mp[i] && ((mp[i] - mm[j]) & 1)) s_ = -s_;
    if (l0 & 1) s_ = -s_;
    return split_level(s_, ex, lev);
  };
  pdl_wait();  // the epilogue overwrites outputs the previous kernel may read

  double z[NE], zp[NE], acc[NE][2 * NG], acm[NA][2 * NG];
#pragma unroll
  for (int e = 0; e < NE; e++) {
    z[e] = 0.0;
    zp[e] = 0.0;
#pragma unroll
    for (int k = 0; k < 2 * NG; k++) acc[e][k] = 0.0;
  }
#pragma unroll
  for (int e = 0; e < NA; e++)
#pragma unroll
    for (int k = 0; k < 2 * NG; k++) acm[e][k] = 0.0;
  unsigned lv = 0;  // current levels, 4 bits per chain (0 = true scale)

  const int wrow_lo = r0 + par + 32 * h;
  const int wcol_lo = PAIRED ? c0 + pc : c0 + 16 * wc;
  bool warp_has = wrow_lo < L && wcol_lo < L;
  bool mir = false;  // warp-uniform: this warp's block also emits the transpose
  if (PAIRED && !plain_tile) {
    const int rb = r0 + 32 * h;
    if (rb < c0) warp_has = false;  // above the diagonal: produced by the mirror block
    mir = rb >= c0 + 32;
  }
  const int wl0_min = max(wrow_lo, wcol_lo);
  bool fast = false, started = false;

  for (int k = 0; k < nchunks; k++) {
    const int b = k % NB, lc = lstart + k * CH, ns = min(CH, L - lc);
    mbar_wait(&sm.full[b], (k / NB) & 1);
    // rl[i] = rl0 + 8 i, cl[j] = cl0 + CJ j: one base pointer per array and chunk,
    // constant offsets per entry (rl0/cl0 opaque: never rematerialised from %tid)
    const auto& S = sm.st[b];
    const double2* rowp = &S.row[0][0] + rl0;
    const double* colp = &S.colc[0][0] + cl0;
    const double2* gpp = &S.gp[0][0] + cl0;
    const double2* gnp = &S.gn[0][0] + cl0;
    const double* wcp = &S.wc[0][0] + cl0;
    const double2* gprp = &S.gpr[PAIRED ? h : 0][0][0] + hr0;
    const double2* gnrp = &S.gnr[PAIRED ? h : 0][0][0] + hr0;

    // one degree: loads, the contraction(s) enabled by DIR / MIR, the recursion.
    // live: chains at level 0 (only consulted when MASKED).
    auto step = [&](auto masked, auto dir, auto mr, int s, unsigned live) {
      constexpr bool MASKED = decltype(masked)::value;
      constexpr bool DIR = decltype(dir)::value;
      constexpr bool MIR = PAIRED && decltype(mr)::value;
      double2 rp[NI];
      double cc[NJ];
      double2 g[NJ][NG];
      double wv[NJ];
      double2 gr[NI][NG];
#pragma unroll
      for (int i = 0; i < NI; i++) rp[i] = rowp[s * invp::R + 8 * i];
#pragma unroll
      for (int j = 0; j < NJ; j++) {
        cc[j] = colp[s * invp::C + CJ * j];
        if (DIR) {
          g[j][0] = gpp[s * invp::C + CJ * j];
          if (!REAL) g[j][NG - 1] = gnp[s * invp::C + CJ * j];
        }
        if (MIR) wv[j] = wcp[s * invp::C + CJ * j];
      }
      if (MIR) {
#pragma unroll
        for (int i = 0; i < NI; i++) {
          gr[i][0] = gprp[s * invp::C + 8 * i];
          if (!REAL) gr[i][NG - 1] = gnrp[s * invp::C + 8 * i];
        }
      }
#pragma unroll
      for (int i = 0; i < NI; i++)
#pragma unroll
        for (int j = 0; j < NJ; j++) {
          const int e = i * NJ + j;
          if (DIR) {
            double t = z[e] * rp[i].y;
            if (MASKED) t = ((live >> e) & 1u) ? t : 0.0;
#pragma unroll
            for (int k2 = 0; k2 < NG; k2++) {
              acc[e][2 * k2] = fma(t, g[j][k2].x, acc[e][2 * k2]);
              acc[e][2 * k2 + 1] = fma(t, g[j][k2].y, acc[e][2 * k2 + 1]);
            }
          }
          if (MIR) {
            double t = z[e] * wv[j];
            if (MASKED) t = ((live >> e) & 1u) ? t : 0.0;
#pragma unroll
            for (int k2 = 0; k2 < NG; k2++) {
              acm[e % NA][2 * k2] = fma(t, gr[i][k2].x, acm[e % NA][2 * k2]);
              acm[e % NA][2 * k2 + 1] = fma(t, gr[i][k2].y, acm[e % NA][2 * k2 + 1]);
            }
          }
          const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
          zp[e] = z[e];
          z[e] = zn;
        }
    };

    if (warp_has && wl0_min < lc + ns) {
      if (!started) {
        // Ghost start: see core_inverse.cu.  The transposed contraction's
        // ghost terms meet W_l(m) or g_l(m'), likewise exactly 0 below l0.
        unsigned slv = 0;  // seed levels, 4 bits per chain
#pragma unroll
        for (int i = 0; i < NI; i++)
#pragma unroll
          for (int j = 0; j < NJ; j++) {
            const int e = i * NJ + j;
            const int d = max(mp[i], mm[j]) - lc;  // >= 0: lc <= wl0_min <= l0
            int lev;
            const double sd = seed_of(i, j, lev);
            slv |= (unsigned)lev << (4 * e);
            const double g0 = ((d >> 1) & 1) ? -sd : sd;        // z^{lc}   (d even)
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
        // (a chain grows at most 4x per degree: 2^32 per 16-degree chunk from <= 2^200),
        // and a chain that reaches level 0 inside a chunk contributes from the
        // next one without loss.  fast: no chain in the warp carries a level.
        unsigned live = 0xffffffffu;
        if (!fast) live = level_zero_mask<NE>(lv);
        const bool contract = fast || __any_sync(0xffffffffu, live != 0);
        // (dE, mE): contractions on even degrees, (dO, mO): on odd degrees (spin 0);
        // without spin 0 every degree runs (dE, mE).
        auto body = [&](auto masked, auto dE, auto mE, auto dO, auto mO) {
          if (SPIN0) {
            // lc is even (tile corners are multiples of 32, CH even): pairs (even l, odd l)
            if (ns == CH && !PAIRED) {
#pragma unroll
              for (int s = 0; s < CH; s += 2) {
                step(masked, dE, mE, s, live);
                step(masked, dO, mO, s + 1, live);
              }
            } else if (ns == CH) {
              // paired: four (par, pc) bodies are live per CTA; a rolled loop keeps
              // them inside the instruction cache
#pragma unroll kPairUnroll
              for (int s = 0; s < CH; s += 2) {
                step(masked, dE, mE, s, live);
                step(masked, dO, mO, s + 1, live);
              }
            } else {
              int s = 0;
#pragma unroll 1
              for (; s + 1 < ns; s += 2) {
                step(masked, dE, mE, s, live);
                step(masked, dO, mO, s + 1, live);
              }
              if (s < ns) step(masked, dE, mE, s, live);
            }
          } else if (ns == CH && !PAIRED) {
#pragma unroll
            for (int s = 0; s < CH; s++) step(masked, dE, mE, s, live);
          } else if (ns == CH) {
#pragma unroll kPairUnroll
            for (int s = 0; s < CH; s++) step(masked, dE, mE, s, live);
          } else {
#pragma unroll 1
            for (int s = 0; s < ns; s++) step(masked, dE, mE, s, live);
          }
        };
        auto run = [&](auto masked) {
          using T_ = BoolC<true>;
          using F_ = BoolC<false>;
          if (!SPIN0) {
            if (PAIRED && mir)
              body(masked, T_(), T_(), T_(), T_());
            else
              body(masked, T_(), F_(), T_(), F_());
          } else if (!PAIRED || !mir) {
            if (par == 0)
              body(masked, T_(), F_(), F_(), F_());
            else
              body(masked, F_(), F_(), T_(), F_());
          } else if (par == 0) {
            if (pc == 0)
              body(masked, T_(), T_(), F_(), F_());
            else
              body(masked, T_(), F_(), F_(), T_());
          } else {
            if (pc == 0)
              body(masked, F_(), T_(), T_(), F_());
            else
              body(masked, F_(), F_(), T_(), T_());
          }
        };
        if (fast) {
          run(BoolC<false>());
        } else {
          if (contract)
            run(BoolC<true>());
          else
#pragma unroll 1
            for (int s = 0; s < ns; s++)
              step(BoolC<false>(), BoolC<false>(), BoolC<false>(), s, live);
          rescale_p(z, zp, lv);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[b]);
  }

  // ---------------------------------------------------------------- epilogue
  // emit T[x, +m] = (pr, pi) and T[x, -m] = (-1)^x (nr, ni) (the (-1)^l of
  // Delta_{x,-m} = (-1)^(l+x) Delta_{x,m} is folded into gn)
  const int sgs = (a.spin & 1) ? -1 : 1;  // (-1)^s
  auto emit = [&](int x, int m, double pr, double pi, double nr, double ni) {
    double sn, cs;
    sincospi((double)x / (double)N, &sn, &cs);
    const double2 tw = make_double2(cs, sn);    // e^{+i m' theta0}
    const double2 twc = make_double2(cs, -sn);  // e^{-i m' theta0}
    const int binp = x, binn = x ? N - x : 0;
    // out_mode 3: the m' >= 0 half only (the theta stage rebuilds F[m, -m'] = +-F[m, m'] e^{-2 pi i m'/N})
    const bool wmir = x && a.out_mode != 3;
    const double sx = (x & 1) ? -1.0 : 1.0;
    const double2 Tp = make_double2(pr, pi);
    if (a.out_mode == 1) {
      if (REAL) {
        out[(long long)x * L + m] = Tp;
      } else {
        out[(long long)x * N + (L - 1 + m)] = Tp;
        if (m > 0) out[(long long)x * N + (L - 1 - m)] = make_double2(sx * nr, sx * ni);
      }
      return;
    }
    if (REAL) {
      // fhalf[m, m'] = T[m', m] i^{-m}; mirror (-1)^m (mw.py:550-556)
      const double2 F = cmul(Tp, ipow(-m));
      double2* row = out + (long long)m * N;
      row[binp] = cmul(F, tw);
      if (wmir) row[binn] = cscale(cmul(F, twc), (m & 1) ? -1.0 : 1.0);
    } else {
      // F[m, m'] = (-1)^s i^{-(m+s)} T[m', m]; F[m, -m'] = (-1)^(m+s) F[m, m'] (mw.py:395-401)
      const double2 Fp = cscale(cmul(Tp, ipow(-(m + a.spin))), (double)sgs);
      double2* rowp = out + (long long)(L - 1 + m) * N;
      rowp[binp] = cmul(Fp, tw);
      if (wmir) rowp[binn] = cscale(cmul(Fp, twc), ((m + a.spin) & 1) ? -1.0 : 1.0);
      if (m > 0) {
        const double2 Tn = make_double2(sx * nr, sx * ni);
        const double2 Fn = cscale(cmul(Tn, ipow(m - a.spin)), (double)sgs);
        double2* rown = out + (long long)(L - 1 - m) * N;
        rown[binp] = cmul(Fn, tw);
        if (wmir) rown[binn] = cscale(cmul(Fn, twc), ((m + a.spin) & 1) ? -1.0 : 1.0);
      }
    }
  };
  if (!warp_has) return;
#pragma unroll
  for (int i = 0; i < NI; i++) {
    if (mp[i] >= L) continue;
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      if (mm[j] >= L) continue;
      const int e = i * NJ + j;
      emit(mp[i], mm[j], acc[e][0], acc[e][1], acc[e][NG == 2 ? 2 : 0], acc[e][NG == 2 ? 3 : 1]);
      if (PAIRED && mir) {
        // T[m, m'] = (-1)^(m'-m) x the transposed accumulators
        const double sg = ((mp[i] - mm[j]) & 1) ? -1.0 : 1.0;
        const int q = e % NA;
        emit(mm[j], mp[i], sg * acm[q][0], sg * acm[q][1], sg * acm[q][NG == 2 ? 2 : 0],
             sg * acm[q][NG == 2 ? 3 : 1]);
      }
    }
  }
}

template <bool REAL, bool SPIN0, bool PAIRED>
static void launch_inv_paired(const InvArgs& a, dim3 grid, cudaStream_t st) {
  const size_t smem = sizeof(invp::Smem<kChunk, PAIRED>);
  smem_attr_once((const void*)k_inverse_core_paired<REAL, SPIN0, PAIRED>, smem);
  launch_pdl(k_inverse_core_paired<REAL, SPIN0, PAIRED>, grid, dim3(kCoreThreadsWS), smem, st, a);
}

void launch_inverse_core_paired(const InvArgs& a, int ntiles, int nmaps, bool real,
                                cudaStream_t st) {
  // spin 0 only (plan.cu use_paired): the plain kernel (core_inverse.cu) runs spin != 0
  dim3 grid(ntiles, nmaps);
  if (real)
    launch_inv_paired<true, true, true>(a, grid, st);
  else
    launch_inv_paired<false, true, true>(a, grid, st);
}

}  // namespace mwsht
