// FFT-stage kernels around cuFFT (mw.py:149-285 forward, :395-446 inverse).
//
// Each kernel is one coalesced, HBM-bound pass that fuses the reference's
// numpy bookkeeping (fftshift/ifftshift index maps, the (-1)^(m+s)
// periodic-extension sign, the 2pi/N and 1/(2 pi N) scales, the half-sample
// theta twist e^{-+i m' pi/N}, zero padding, the m' fold) into the data
// movement that the FFT layout needs anyway (row <-> column transposes).
#include "common.cuh"

namespace mwsht {

__device__ __forceinline__ int fbin(int k, int N) { return k >= 0 ? k : k + N; }

// Forward: rows t of phi-FFT output A (L x N, unshifted bins) -> extended,
// transposed B (N x N): B[mi][t] = scale * s(t) * A[t'][bin(m)], m = mi-(L-1),
// t' = t (t < L) or 2L-2-t with s = (-1)^(m+s) (mw.py:161-177).
// Real variant: A is (L x L) (rfft bins m = 0..L-1), B is (L x N), sign (-1)^m.
template <bool REAL>
__global__ void k_extend_transpose(const double2* __restrict__ A, double2* __restrict__ B, int L,
                                   int N, int spin, double scale, long long a_stride,
                                   long long b_stride) {
  __shared__ double2 tile[32][33];
  const int rows = REAL ? L : N;   // rows of B (orders)
  const int acols = REAL ? L : N;  // columns of A
  const int tb = blockIdx.x * 32, mb = blockIdx.y * 32;
  const double2* a = A + (long long)blockIdx.z * a_stride;
  double2* b = B + (long long)blockIdx.z * b_stride;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // load: tile[t - tb][mi - mb]
  for (int k = ty; k < 32; k += 8) {
    const int t = tb + k, mi = mb + tx;
    double2 v = make_double2(0.0, 0.0);
    if (t < N && mi < rows) {
      const int m = REAL ? mi : mi - (L - 1);
      const int col = REAL ? mi : fbin(m, N);
      const int ts = t < L ? t : 2 * L - 2 - t;
      v = a[(long long)ts * acols + col];
      double sc = scale;
      if (t >= L && ((m + (REAL ? 0 : spin)) & 1)) sc = -sc;
      v = cscale(v, sc);
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int mi = mb + k, t = tb + tx;
    if (mi < rows && t < N) b[(long long)mi * N + t] = tile[tx][k];
  }
}

// Forward: raw theta-FFT rows (unshifted bins) -> zero-padded correlation rows
// of length P: C[r][j] = B[r][bin(k)] e^{-i k pi/N} / (2 pi N), k = j-(L-1) for
// j < N, else 0 (mw.py:180-192 twist and scale, :249-250 padding).
__global__ void k_pad_twist(const double2* __restrict__ B, double2* __restrict__ C, int rows, int L,
                            int N, int P, long long b_stride, long long c_stride) {
  const int r = blockIdx.y;
  const double2* b = B + (long long)blockIdx.z * b_stride + (long long)r * N;
  double2* c = C + (long long)blockIdx.z * c_stride + (long long)r * P;
  const double inv = 1.0 / (2.0 * 3.141592653589793 * N);
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < P; j += gridDim.x * blockDim.x) {
    double2 v = make_double2(0.0, 0.0);
    if (j < N) {
      const int k = j - (L - 1);
      double sn, cs;
      sincospi(-(double)k / (double)N, &sn, &cs);
      v = cscale(cmul(b[fbin(k, N)], make_double2(cs, sn)), inv);
    }
    c[j] = v;
  }
  (void)rows;
}

// Pointwise multiply by the weight spectrum (already scaled by 2pi/P).
__global__ void k_mul_spectrum(double2* __restrict__ C, const double2* __restrict__ W, int P,
                               long long nrows) {
  const long long total = nrows * P;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx % P);
    C[idx] = cmul(C[idx], W[j]);
  }
}

// Forward: folded plane in the core's staging layout (mw.py:251, 273-285, 504-511):
//   gf[r][j] = G_r(j) + s_r G_r(-j)  (j = m' >= 0; gf[r][0] = G_r(0)), G_r(m') = C[r][3L-3+m'],
//   s_r = (-1)^(m+s) (complex, m = r-(L-1)) or (-1)^r (real),
// written transposed and split by the sign of m, zero-padded to ldw columns:
//   gfT[blk32(j, m)] = gf[row(+m)][j],  gfT[L*ldw + blk32(j, m)] = (-1)^j gf[row(-m)][j].
// SRC_CONV: read G from the correlation rows C (length P); else read an
// already folded (rows x L) plane (kernel-level hook input).
template <bool REAL, bool SRC_CONV>
__global__ void k_fold_T2(const double2* __restrict__ src, double2* __restrict__ gfT, int L, int P,
                          int ldw, int spin, long long s_stride, long long g_stride) {
  __shared__ double2 tile[32][33];
  const int jb = blockIdx.x * 32, mb = blockIdx.y * 32;
  const int map = REAL ? blockIdx.z : (blockIdx.z >> 1);
  const int neg = REAL ? 0 : (blockIdx.z & 1);
  const double2* c = src + (long long)map * s_stride;
  double2* g = gfT + (long long)map * g_stride + (neg ? (long long)L * ldw : 0);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int o = 3 * L - 3;
  for (int k = ty; k < 32; k += 8) {
    const int m = mb + k, j = jb + tx;
    double2 v = make_double2(0.0, 0.0);
    if (m < L && j < L) {
      const int r = REAL ? m : (neg ? L - 1 - m : L - 1 + m);
      if (SRC_CONV) {
        const double2* row = c + (long long)r * P;
        v = row[o + j];
        if (j > 0) {
          const int mm = REAL ? r : r - (L - 1);
          const double sr = ((mm + (REAL ? 0 : spin)) & 1) ? -1.0 : 1.0;
          const double2 u = row[o - j];
          v = make_double2(v.x + sr * u.x, v.y + sr * u.y);
        }
      } else {
        v = c[(long long)r * L + j];
      }
      if (neg && (j & 1)) v = make_double2(-v.x, -v.y);
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int j = jb + k, m = mb + tx;
    if (j < L && m < ldw) g[blk<kTileCols>(j, m, L)] = tile[tx][k];
  }
}

// Hook output: staging layout -> folded plane (N x L) (complex) / (L x L) (real).
template <bool REAL>
__global__ void k_T2_to_fold(const double2* __restrict__ gfT, double2* __restrict__ gf, int L,
                             int ldw) {
  __shared__ double2 tile[32][33];
  const int mb = blockIdx.x * 32, jb = blockIdx.y * 32;
  const int neg = REAL ? 0 : blockIdx.z;
  const double2* g = gfT + (neg ? (long long)L * ldw : 0);
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int j = jb + k, m = mb + tx;
    double2 v = make_double2(0.0, 0.0);
    if (j < L && m < L) {
      v = g[blk<kTileCols>(j, m, L)];
      if (neg && (j & 1)) v = make_double2(-v.x, -v.y);
    }
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int m = mb + k, j = jb + tx;
    if (m < L && j < L && !(neg && m == 0)) {
      const int r = REAL ? m : (neg ? L - 1 - m : L - 1 + m);
      gf[(long long)r * L + j] = tile[tx][k];
    }
  }
}

// Inverse: coefficients -> the core's pre-scaled staging rows (mw.py:390-392
// unflatten + the c_l u_l(m) column factor of the l-recursion):
//   gp[blk32(l, m)] = c_l u_l(m) f_{l,m},  gn[blk32(l, m)] = (-1)^l c_l u_l(m) f_{l,-m},
//   u_l(m) = A(l-m) A(l+m), zero for m > l.
// in_mode 0: flat l(l+1)+m; 1: table (L, N) column L-1+m (real: (L, L) column m).
template <bool REAL>
__global__ void k_inv_prescale(const double2* __restrict__ in, int in_mode,
                               const double* __restrict__ cl, const double* __restrict__ A, int L,
                               int ldw, double2* __restrict__ gp, long long in_stride,
                               long long g_stride) {
  pdl_trigger();
  pdl_wait();  // reads the caller's coefficients, overwrites the core staging
  const int l = blockIdx.y;
  const int N = 2 * L - 1;
  const double2* f = in + (long long)blockIdx.z * in_stride;
  double2* p = gp + (long long)blockIdx.z * g_stride;
  double2* n = p + (long long)L * ldw;
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < ldw; m += gridDim.x * blockDim.x) {
    double2 vp = make_double2(0.0, 0.0), vn = vp;
    if (m <= l) {
      const double u = cl[l] * A[l - m] * A[l + m];
      double2 fp, fn;
      if (REAL) {
        fp = in_mode == 0 ? f[(long long)l * (l + 1) + m] : f[(long long)l * L + m];
        fn = fp;
      } else if (in_mode == 0) {
        fp = f[(long long)l * (l + 1) + m];
        fn = f[(long long)l * (l + 1) - m];
      } else {
        fp = f[(long long)l * N + (L - 1 + m)];
        fn = f[(long long)l * N + (L - 1 - m)];
      }
      vp = cscale(fp, u);
      vn = cscale(fn, (l & 1) ? -u : u);
    }
    p[blk<kTileCols>(l, m, L)] = vp;
    if (!REAL) n[blk<kTileCols>(l, m, L)] = vn;
  }
}

// out[c][r] = in[r][c] for a (rows x cols) complex matrix.
__global__ void k_transpose(const double2* __restrict__ in, double2* __restrict__ out, int rows,
                            int cols) {
  __shared__ double2 tile[32][33];
  const int cb = blockIdx.x * 32, rb = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int r = rb + k, c = cb + tx;
    tile[k][tx] = (r < rows && c < cols) ? in[(long long)r * cols + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int c = cb + k, r = rb + tx;
    if (c < cols && r < rows) out[(long long)c * rows + r] = tile[tx][k];
  }
}

// Inverse: theta-synthesis rows S (orders x N, columns t) -> phi-synthesis
// input Out (L x ...): complex Out[t][bin(m)] = S[L-1+m][t] (mw.py:436-437
// ifftshift), real Out[t][m] = S[m][t] with Im = 0 at m = 0 (irfft ignores it).
template <bool REAL>
__global__ void k_untranspose(const double2* __restrict__ S, double2* __restrict__ Out, int L,
                              int N, long long s_stride, long long o_stride) {
  __shared__ double2 tile[32][33];
  const int rows = REAL ? L : N;
  const int ocols = REAL ? L : N;
  const int mb = blockIdx.x * 32, tb = blockIdx.y * 32;
  const double2* s = S + (long long)blockIdx.z * s_stride;
  double2* o = Out + (long long)blockIdx.z * o_stride;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int mi = mb + k, t = tb + tx;
    double2 v = make_double2(0.0, 0.0);
    if (mi < rows && t < L) v = s[(long long)mi * N + t];
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int t = tb + k, mi = mb + tx;
    if (t < L && mi < rows) {
      double2 v = tile[tx][k];
      int col;
      if (REAL) {
        col = mi;
        if (mi == 0) v.y = 0.0;
      } else {
        col = fbin(mi - (L - 1), N);
      }
      o[(long long)t * ocols + col] = v;
    }
  }
}

// Reality check of inverse_real (mw.py:537-547): max |conj(f_lm) - (-1)^m f_l,-m|
// and max |f| over the flat array, as ordered-bit atomics on nonnegative doubles.
__global__ void k_reality(const double2* __restrict__ f, int L, unsigned long long* worst,
                          unsigned long long* peak) {
  const long long n = (long long)L * L;
  double w = 0.0, p = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    const int l = (int)floor(sqrt((double)idx));
    int ll = l;
    while ((long long)ll * ll > idx) ll--;
    while ((long long)(ll + 1) * (ll + 1) <= idx) ll++;
    const int m = (int)(idx - (long long)ll * (ll + 1));
    const double2 a = f[idx];
    const double2 b = f[(long long)ll * (ll + 1) - m];
    const double sg = (m & 1) ? -1.0 : 1.0;
    const double dx = a.x - sg * b.x, dy = -a.y - sg * b.y;
    w = fmax(w, hypot(dx, dy));
    p = fmax(p, hypot(a.x, a.y));
  }
  for (int off = 16; off; off >>= 1) {
    w = fmax(w, __shfl_xor_sync(0xffffffffu, w, off));
    p = fmax(p, __shfl_xor_sync(0xffffffffu, p, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(worst, __double_as_longlong(w));
    atomicMax(peak, __double_as_longlong(p));
  }
}

// ------------------------------------------------------------- launchers
void launch_extend_transpose(bool real, const double2* A, double2* B, int L, int N, int spin,
                             double scale, long long as, long long bs, int nm, cudaStream_t st) {
  const int rows = real ? L : N;
  dim3 grid((N + 31) / 32, (rows + 31) / 32, nm), block(32, 8);
  if (real)
    k_extend_transpose<true><<<grid, block, 0, st>>>(A, B, L, N, spin, scale, as, bs);
  else
    k_extend_transpose<false><<<grid, block, 0, st>>>(A, B, L, N, spin, scale, as, bs);
}

void launch_pad_twist(const double2* B, double2* C, int rows, int L, int N, int P, long long bs,
                      long long cs, int nm, cudaStream_t st) {
  const int threads = 256;
  dim3 grid((P + threads - 1) / threads, rows, nm);
  k_pad_twist<<<grid, threads, 0, st>>>(B, C, rows, L, N, P, bs, cs);
}

void launch_mul_spectrum(double2* C, const double2* W, int P, long long nrows, cudaStream_t st) {
  const long long total = nrows * P;
  long long blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_mul_spectrum<<<(unsigned)blocks, 256, 0, st>>>(C, W, P, nrows);
}

void launch_fold(bool real, bool from_conv, const double2* src, double2* gfT, int L, int P,
                 int ldw, int spin, long long ss, long long gs, int nm, cudaStream_t st) {
  dim3 grid((L + 31) / 32, ldw / 32, real ? nm : 2 * nm), block(32, 8);
  if (real) {
    if (from_conv)
      k_fold_T2<true, true><<<grid, block, 0, st>>>(src, gfT, L, P, ldw, spin, ss, gs);
    else
      k_fold_T2<true, false><<<grid, block, 0, st>>>(src, gfT, L, P, ldw, spin, ss, gs);
  } else {
    if (from_conv)
      k_fold_T2<false, true><<<grid, block, 0, st>>>(src, gfT, L, P, ldw, spin, ss, gs);
    else
      k_fold_T2<false, false><<<grid, block, 0, st>>>(src, gfT, L, P, ldw, spin, ss, gs);
  }
}

void launch_T2_to_fold(bool real, const double2* gfT, double2* gf, int L, int ldw,
                       cudaStream_t st) {
  dim3 grid((L + 31) / 32, (L + 31) / 32, real ? 1 : 2), block(32, 8);
  if (real)
    k_T2_to_fold<true><<<grid, block, 0, st>>>(gfT, gf, L, ldw);
  else
    k_T2_to_fold<false><<<grid, block, 0, st>>>(gfT, gf, L, ldw);
}

void launch_inv_prescale(bool real, const double2* in, int in_mode, const double* cl,
                         const double* A, int L, int ldw, double2* gp, long long is, long long gs,
                         int nm, cudaStream_t st) {
  const int threads = 128;
  dim3 grid((ldw + threads - 1) / threads, L, nm);
  if (real)
    launch_pdl(k_inv_prescale<true>, grid, threads, 0, st, in, in_mode, cl, A, L, ldw, gp, is, gs);
  else
    launch_pdl(k_inv_prescale<false>, grid, threads, 0, st, in, in_mode, cl, A, L, ldw, gp, is, gs);
}

void launch_transpose(const double2* in, double2* out, int rows, int cols, cudaStream_t st) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32), block(32, 8);
  k_transpose<<<grid, block, 0, st>>>(in, out, rows, cols);
}

void launch_untranspose(bool real, const double2* S, double2* Out, int L, int N, long long ss,
                        long long os, int nm, cudaStream_t st) {
  const int rows = real ? L : N;
  dim3 grid((rows + 31) / 32, (L + 31) / 32, nm), block(32, 8);
  if (real)
    k_untranspose<true><<<grid, block, 0, st>>>(S, Out, L, N, ss, os);
  else
    k_untranspose<false><<<grid, block, 0, st>>>(S, Out, L, N, ss, os);
}

// Hands the two maxima to host-mapped memory with plain stores and re-zeroes the
// device slots: the caller reads the result after a stream sync without a
// copy-engine transfer (which would queue behind large D2H copies of other
// streams, e.g. HostPipeline's).
__global__ void k_reality_publish(unsigned long long* red, unsigned long long* host) {
  host[0] = red[0];
  host[1] = red[1];
  red[0] = 0ull;
  red[1] = 0ull;
}

void launch_reality(const double2* f, int L, unsigned long long* red, unsigned long long* host,
                    cudaStream_t st) {
  long long n = (long long)L * L;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  k_reality<<<(unsigned)blocks, 256, 0, st>>>(f, L, red, red + 1);
  if (host) k_reality_publish<<<1, 1, 0, st>>>(red, host);
}

}  // namespace mwsht
