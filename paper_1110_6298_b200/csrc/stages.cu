// Small glue kernels around the fused FFT engine (fft.cu) and the cores:
// the kernel-level hooks' layout conversions (k_fold_T2, k_T2_to_fold), the
// inverse's coefficient pre-scaling into the core staging (k_inv_prescale,
// mw.py:390-392) and inverse_real's reality check (k_reality, mw.py:537-547).
#include "common.cuh"

namespace mwsht {

// Hook input: an already folded plane gf (N x L complex, row L-1+m; real:
// L x L, row m) -> the forward core's staging layout, transposed, split by
// the sign of m and zero-padded to ldw columns (flm_core hooks,
// _numba.py:132-188):
//   gfT[blk32(j, m)] = gf[row(+m)][j],  gfT[L*ldw + blk32(j, m)] = (-1)^j gf[row(-m)][j].
template <bool REAL>
__global__ void k_fold_T2(const double2* __restrict__ src, double2* __restrict__ gfT, int L,
                          int ldw) {
  __shared__ double2 tile[32][33];
  const int jb = blockIdx.x * 32, mb = blockIdx.y * 32;
  const int neg = REAL ? 0 : (blockIdx.z & 1);
  double2* g = gfT + (neg ? (long long)L * ldw : 0);
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int m = mb + k, j = jb + tx;
    double2 v = make_double2(0.0, 0.0);
    if (m < L && j < L) {
      const int r = REAL ? m : (neg ? L - 1 - m : L - 1 + m);
      v = src[(long long)r * L + j];
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
// Columns c0 <= m < c1 only (an order-range shard's columns; full: 0, ldw).
template <bool REAL>
__global__ void k_inv_prescale(const double2* __restrict__ in, int in_mode,
                               const double* __restrict__ cl, const double* __restrict__ A, int L,
                               int ldw, double2* __restrict__ gp, long long in_stride,
                               long long g_stride, int c0, int c1) {
  pdl_trigger();
  pdl_wait();  // reads the caller's coefficients, overwrites the core staging
  const int l = blockIdx.y;
  const int N = 2 * L - 1;
  const double2* f = in + (long long)blockIdx.z * in_stride;
  double2* p = gp + (long long)blockIdx.z * g_stride;
  double2* n = p + (long long)L * ldw;
  for (int m = c0 + blockIdx.x * blockDim.x + threadIdx.x; m < c1; m += gridDim.x * blockDim.x) {
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

// m-column sharding: the all-gathered packed coefficient blocks (one block of
// `maxlen` entries per rank, shard_flm_index layout) -> flat flm.
__global__ void k_flm_unpack(const double2* __restrict__ gathered, long long maxlen,
                             const int* __restrict__ bounds, int world, int L,
                             double2* __restrict__ flm) {
  const long long n = (long long)L * L;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
       idx += (long long)gridDim.x * blockDim.x) {
    int l = (int)sqrt((double)idx);
    while ((long long)l * l > idx) l--;
    while ((long long)(l + 1) * (l + 1) <= idx) l++;
    const int m = (int)(idx - (long long)l * (l + 1));
    const int am = m < 0 ? -m : m;
    int r = 0;
    while (r + 1 < world && bounds[r + 1] <= am) r++;
    flm[idx] = gathered[(long long)r * maxlen + shard_flm_index(l, m, bounds[r], bounds[r + 1])];
  }
}

// dst[i] = src[i].y (plan time: W-only row tables for multi-spin batches)
__global__ void k_extract_y(const double2* __restrict__ src, double* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i].y;
}

// ------------------------------------------------------------- launchers
void launch_extract_y(const double2* src, double* dst, long long n, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_extract_y<<<(unsigned)blocks, 256, 0, st>>>(src, dst, n);
}

void launch_flm_unpack(const double2* gathered, long long maxlen, const int* bounds, int world,
                       int L, double2* flm, cudaStream_t st) {
  long long n = (long long)L * L;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_flm_unpack<<<(unsigned)blocks, 256, 0, st>>>(gathered, maxlen, bounds, world, L, flm);
}

void launch_fold(bool real, const double2* gf, double2* gfT, int L, int ldw, cudaStream_t st) {
  dim3 grid((L + 31) / 32, ldw / 32, real ? 1 : 2), block(32, 8);
  if (real)
    k_fold_T2<true><<<grid, block, 0, st>>>(gf, gfT, L, ldw);
  else
    k_fold_T2<false><<<grid, block, 0, st>>>(gf, gfT, L, ldw);
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
                         int nm, cudaStream_t st, int c0, int c1) {
  if (c1 < 0) c1 = ldw;
  const int threads = 128;
  dim3 grid((c1 - c0 + threads - 1) / threads, L, nm);
  if (real)
    launch_pdl(k_inv_prescale<true>, grid, threads, 0, st, in, in_mode, cl, A, L, ldw, gp, is, gs,
               c0, c1);
  else
    launch_pdl(k_inv_prescale<false>, grid, threads, 0, st, in, in_mode, cl, A, L, ldw, gp, is, gs,
               c0, c1);
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
