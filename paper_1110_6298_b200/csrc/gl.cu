// Gauss-Legendre comparator cores: the reference's
// gl_fm_core / gl_flm_core (pkg/src/torusht/kernels/_numba.py:211-268), the
// O(L^3) colatitude stages of gl_inverse / gl_forward (gl.py:114-178).
//
// Both run, for every order row mi (m = mi - (L-1), n = -spin) and every
// Gauss-Legendre node x_i, the pointwise three-term degree recursion of
// d^l_{m,n}(theta_i) from its seed at l0 = max(|m|, |n|) (_seed_d,
// _numba.py:191-208; the seeds' sign * sqrt(C(2nn, nn+mm)) constants are
// computed on the host with the reference's own lgamma/exp formula and passed
// in, the node powers ch^ec sh^es are taken here):
//   d^{l+1} = ((2l+1)(l(l+1) x - m n) d^l - (l+1) sqrt((l^2-m^2)(l^2-n^2)) d^{l-1}) / den_l,
//   den_l = l sqrt(((l+1)^2-m^2)((l+1)^2-n^2)),   d^1 = x d^0 at l = 0.
// The per-degree factors depend on (m, n, l) only and are tabulated per CTA
// in shared memory (1/den_l instead of the reference's per-node division).
//
//   k_gl_fm  (inverse): F[mi, i] = sum_l flm_scaled[l, mi] d^l(x_i).  One CTA
//            per order row, one chain per (row, node): no reduction.
//   k_gl_flm (forward): R[l, mi] = sum_i a[mi, i] d^l(x_i).  One CTA per order
//            row, threads over nodes; every 16-degree chunk each thread keeps
//            its partial sums in registers and the CTA reduces them through a
//            shared-memory transpose (deterministic order).
#include "common.cuh"

namespace mwsht {

constexpr int kGlThreads = 256;
constexpr int kGlChunk = 16;
constexpr int kGlMaxNodes = 16;  // nodes per thread: L <= 4096

// per-degree factors of order row (m, n): coefficient of the d^l term is
// (A_l x - B_l), of the d^{l-1} term C_l (all pre-divided by den_l)
__device__ __forceinline__ void gl_tables(int L, int m, int n, double* A, double* B, double* Cc) {
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    double a = 0.0, b = 0.0, c = 0.0;
    if (l >= 1) {
      const double el = (double)l, mm = (double)m * m, nn = (double)n * n;
      const double den = el * sqrt(((el + 1.0) * (el + 1.0) - mm) * ((el + 1.0) * (el + 1.0) - nn));
      const double r = 1.0 / den;
      a = (2.0 * el + 1.0) * (el * (el + 1.0)) * r;
      b = (2.0 * el + 1.0) * ((double)m * (double)n) * r;
      c = (el + 1.0) * sqrt((el * el - mm) * (el * el - nn)) * r;
    }
    A[l] = a;
    B[l] = b;
    Cc[l] = c;
  }
}

// base^e for integer e >= 0 by squaring from r = 1: how the reference's numba
// code evaluates ch[i] ** ec (integer exponent), so the seeds match its bits
__device__ __forceinline__ double int_power(double base, int e) {
  double r = 1.0;
  while (e) {
    if (e & 1) r *= base;
    e >>= 1;
    base *= base;
  }
  return r;
}

__device__ __forceinline__ double gl_seed(double cst, int ec, int es, double ch, double sh) {
  return cst * int_power(ch, ec) * int_power(sh, es);
}

// one recursion step l -> l+1 of (dl, dlm1) at node x
__device__ __forceinline__ void gl_step(int l, double x, const double* A, const double* B,
                                        const double* Cc, double& dl, double& dlm1) {
  if (l == 0) {
    dlm1 = dl;
    dl = x * dl;
  } else {
    const double t = fma(fma(A[l], x, -B[l]), dl, -Cc[l] * dlm1);
    dlm1 = dl;
    dl = t;
  }
}

__global__ void __launch_bounds__(kGlThreads) k_gl_fm(const double2* __restrict__ flm, const double* __restrict__ x,
                                 const double* __restrict__ ch, const double* __restrict__ sh,
                                 const double* __restrict__ cst, const int4* __restrict__ seed,
                                 int L, int spin, double2* __restrict__ F) {
  extern __shared__ __align__(16) double gsm[];
  const int N = 2 * L - 1, mi = blockIdx.x, m = mi - (L - 1), n = -spin;
  double2* f = reinterpret_cast<double2*>(gsm);  // 16-byte aligned first
  double* A = gsm + 2 * L;
  double* B = A + L;
  double* Cc = B + L;
  const int4 sd = seed[mi];  // (ec, es, l0, -)
  const int l0 = sd.z;
  gl_tables(L, m, n, A, B, Cc);
  for (int l = threadIdx.x; l < L; l += blockDim.x) f[l] = flm[(long long)l * N + mi];
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    if (l0 < L) {
      const double xi = x[i];
      double dl = gl_seed(cst[mi], sd.x, sd.y, ch[i], sh[i]), dlm1 = 0.0;
      for (int l = l0; l < L; l++) {
        acc.x = fma(f[l].x, dl, acc.x);
        acc.y = fma(f[l].y, dl, acc.y);
        if (l == L - 1) break;
        gl_step(l, xi, A, B, Cc, dl, dlm1);
      }
    }
    F[(long long)mi * L + i] = acc;
  }
}

__global__ void __launch_bounds__(kGlThreads) k_gl_flm(const double2* __restrict__ a, const double* __restrict__ x,
                                  const double* __restrict__ ch, const double* __restrict__ sh,
                                  const double* __restrict__ cst, const int4* __restrict__ seed,
                                  int L, int spin, double2* __restrict__ R) {
  extern __shared__ __align__(16) double gsm[];
  const int N = 2 * L - 1, mi = blockIdx.x, m = mi - (L - 1), n = -spin;
  double2* red = reinterpret_cast<double2*>(gsm);  // [kGlChunk][kGlThreads], aligned first
  double* A = gsm + 2 * kGlChunk * kGlThreads;
  double* B = A + L;
  double* Cc = B + L;
  const int4 sd = seed[mi];
  const int l0 = sd.z;
  const int tid = threadIdx.x;
  if (l0 >= L) {  // the reference leaves the whole column zero
    for (int l = tid; l < L; l += blockDim.x) R[(long long)l * N + mi] = make_double2(0.0, 0.0);
    return;
  }
  gl_tables(L, m, n, A, B, Cc);
  for (int l = tid; l < l0; l += blockDim.x) R[(long long)l * N + mi] = make_double2(0.0, 0.0);
  // this thread's nodes i = tid + k * blockDim.x and their chain states
  const int nk = (L - tid + kGlThreads - 1) / kGlThreads;
  double dl[kGlMaxNodes], dlm1[kGlMaxNodes];
  __syncthreads();
  const double cs = cst[mi];
#pragma unroll
  for (int k = 0; k < kGlMaxNodes; k++) {
    dl[k] = 0.0;
    dlm1[k] = 0.0;
    if (k < nk) {
      const int i = tid + k * kGlThreads;
      dl[k] = gl_seed(cs, sd.x, sd.y, ch[i], sh[i]);
    }
  }
  for (int lc = l0; lc < L; lc += kGlChunk) {
    const int ns = min(kGlChunk, L - lc);
    double2 p[kGlChunk];
#pragma unroll
    for (int s = 0; s < kGlChunk; s++) p[s] = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kGlMaxNodes; k++) {
      if (k < nk) {
        const int i = tid + k * kGlThreads;
        const double xi = x[i];
        const double2 av = a[(long long)mi * L + i];
        double d = dl[k], dm = dlm1[k];
#pragma unroll
        for (int s = 0; s < kGlChunk; s++) {
          if (s < ns) {
            p[s].x = fma(d, av.x, p[s].x);
            p[s].y = fma(d, av.y, p[s].y);
            if (lc + s < L - 1) gl_step(lc + s, xi, A, B, Cc, d, dm);
          }
        }
        dl[k] = d;
        dlm1[k] = dm;
      }
    }
    // CTA reduction over nodes: transpose through shared memory
#pragma unroll
    for (int s = 0; s < kGlChunk; s++) red[s * kGlThreads + tid] = p[s];
    __syncthreads();
    {
      constexpr int TPD = kGlThreads / kGlChunk;  // threads per degree
      constexpr int SEG = kGlThreads / TPD;       // partials per thread
      const int s = tid / TPD, q = tid % TPD;
      double2 sum = make_double2(0.0, 0.0);
      for (int j = 0; j < SEG; j++) {
        const double2 v = red[s * kGlThreads + q * SEG + j];
        sum.x += v.x;
        sum.y += v.y;
      }
#pragma unroll
      for (int off = TPD / 2; off; off >>= 1) {
        sum.x += __shfl_down_sync(0xffffffffu, sum.x, off, TPD);
        sum.y += __shfl_down_sync(0xffffffffu, sum.y, off, TPD);
      }
      if (q == 0 && s < ns) R[(long long)(lc + s) * N + mi] = sum;
    }
    __syncthreads();
  }
}

cudaError_t launch_gl(bool forward, const double2* in, const double* x, const double* ch,
              const double* sh, const double* cst, const int4* seed, int L, int spin,
              double2* out, cudaStream_t st) {
  const int N = 2 * L - 1;
  // the attribute is set once per kernel: the largest size any L <= 4096 needs
  constexpr int kLmax = 4096;
  if (forward) {
    const size_t smem = sizeof(double) * 3 * L + sizeof(double2) * kGlChunk * kGlThreads;
    smem_attr_once((const void*)k_gl_flm,
                   sizeof(double) * 3 * kLmax + sizeof(double2) * kGlChunk * kGlThreads);
    k_gl_flm<<<N, kGlThreads, smem, st>>>(in, x, ch, sh, cst, seed, L, spin, out);
  } else {
    const size_t smem = sizeof(double) * 3 * L + sizeof(double2) * L;
    smem_attr_once((const void*)k_gl_fm, sizeof(double) * 3 * kLmax + sizeof(double2) * kLmax);
    k_gl_fm<<<N, kGlThreads, smem, st>>>(in, x, ch, sh, cst, seed, L, spin, out);
  }
  return cudaGetLastError();
}

}  // namespace mwsht
