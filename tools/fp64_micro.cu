// FP64 pipe micro-benchmarks for the core kernels' instruction mix (not part of
// the library).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_micro fp64_micro.cu
//
// k_indep<K>:  K independent DFMA chains per thread (pipe peak vs warps/SMSP).
// k_pair:      the inverse core's spin-0 pair step (full + rec) on 8 chains per
//              thread, operands from shared memory like the real kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void k_indep(double* out, int iters, double a) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; k++) x[k] = threadIdx.x + k;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = fma(x[k], a, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; k++) s += x[k];
  if (s == 12345.0) out[0] = s;
}

// K independent chains, every DFMA with three distinct register operands
template <int K>
__global__ void k_indep3(double* out, int iters, double a) {
  double x[K], b[K], c[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    x[k] = threadIdx.x + k;
    b[k] = a + 1e-7 * k;
    c[k] = 1e-9 * (k + threadIdx.x);
  }
  asm volatile("" ::: "memory");
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = fma(x[k], b[k], c[k]);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; k++) s += x[k] + b[k] + c[k];
  if (s == 12345.0) out[0] = s;
}

// K independent DMUL chains
template <int K>
__global__ void k_dmul(double* out, int iters, double a) {
  double x[K], b[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    x[k] = threadIdx.x + k;
    b[k] = a + 1e-7 * k;
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = x[k] * b[k];
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; k++) s += x[k];
  if (s == 12345.0) out[0] = s;
}

// pair step emulation: 4 rows x 2 cols per thread, complex +-m accumulators
__global__ void k_pair(double* out, int iters) {
  __shared__ double2 row[2][64];
  __shared__ double colc[2][32];
  __shared__ double2 g[2][2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    row[i / 64][i % 64] = make_double2(1.0 + 1e-3 * i, 0.5);
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    colc[i / 32][i % 32] = 0.999 + 1e-5 * i;
    g[0][i / 32][i % 32] = make_double2(0.1, 0.2);
    g[1][i / 32][i % 32] = make_double2(0.3, 0.4);
  }
  __syncthreads();
  int rl0 = (w & 1) + 2 * (lane & 3), cl0 = lane >> 2;
  asm volatile("" : "+r"(rl0), "+r"(cl0));
  double z[8], zp[8], acc[8][4];
#pragma unroll
  for (int e = 0; e < 8; e++) {
    z[e] = 1e-3 * (e + 1);
    zp[e] = 0.0;
#pragma unroll
    for (int k = 0; k < 4; k++) acc[e][k] = 0.0;
  }
  for (int it = 0; it < iters; it++) {
    const int s = it & 1;
    // full step
    {
      double2 rp[4];
      double cc[2];
      double2 gg[2][2];
#pragma unroll
      for (int i = 0; i < 4; i++) rp[i] = row[s][rl0 + 8 * i];
#pragma unroll
      for (int j = 0; j < 2; j++) {
        cc[j] = colc[s][cl0 + 8 * j];
        gg[j][0] = g[s][0][cl0 + 8 * j];
        gg[j][1] = g[s][1][cl0 + 8 * j];
      }
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
          const int e = i * 2 + j;
          const double t = z[e] * rp[i].y;
#pragma unroll
          for (int k2 = 0; k2 < 2; k2++) {
            acc[e][2 * k2] = fma(t, gg[j][k2].x, acc[e][2 * k2]);
            acc[e][2 * k2 + 1] = fma(t, gg[j][k2].y, acc[e][2 * k2 + 1]);
          }
          const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
          zp[e] = z[e];
          z[e] = zn;
        }
    }
    // rec step
    {
      double2 rp[4];
      double cc[2];
#pragma unroll
      for (int i = 0; i < 4; i++) rp[i] = row[s ^ 1][rl0 + 8 * i];
#pragma unroll
      for (int j = 0; j < 2; j++) cc[j] = colc[s ^ 1][cl0 + 8 * j];
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 2; j++) {
          const int e = i * 2 + j;
          const double zn = fma(rp[i].x * cc[j], z[e], -zp[e]);
          zp[e] = z[e];
          z[e] = zn;
        }
    }
  }
  double sum = 0;
#pragma unroll
  for (int e = 0; e < 8; e++) sum += z[e] + acc[e][0] + acc[e][1] + acc[e][2] + acc[e][3];
  if (sum == 12345.0) out[0] = sum;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps : {4, 8, 12, 16, 32}) {
    const int th = warps * 32;
    float ms = timeit([&] { k_indep<8><<<nsm, th>>>(out, iters, 0.999999); });
    double fl = 2.0 * 8 * iters * (double)th * nsm;
    printf("indep K=8  warps/SM=%2d: %.2f TF/s\n", warps, fl / ms / 1e9);
  }
  for (int warps : {4, 8, 12, 16}) {
    const int th = warps * 32;
    float ms = timeit([&] { k_indep<16><<<nsm, th>>>(out, iters, 0.999999); });
    double fl = 2.0 * 16 * iters * (double)th * nsm;
    printf("indep K=16 warps/SM=%2d: %.2f TF/s\n", warps, fl / ms / 1e9);
  }
  for (int warps : {8, 16}) {
    const int th = warps * 32;
    float ms = timeit([&] { k_indep3<16><<<nsm, th>>>(out, iters, 0.999999); });
    double fl = 2.0 * 16 * iters * (double)th * nsm;
    printf("indep3 K=16 warps/SM=%2d: %.2f TF/s\n", warps, fl / ms / 1e9);
    ms = timeit([&] { k_dmul<16><<<nsm, th>>>(out, iters, 0.999999); });
    printf("dmul   K=16 warps/SM=%2d: %.2f T DMUL lane-ops/s\n", warps, 16.0 * iters * th * nsm / ms / 1e9);
  }
  for (int warps : {4, 8, 12}) {
    const int th = warps * 32;
    float ms = timeit([&] { k_pair<<<nsm, th>>>(out, iters); });
    // per pair per chain: 9 FP64 instructions (3 DMUL + 6 DFMA)
    double inst = 9.0 * 8 * iters * (double)th * nsm;
    double peak_inst = 64.0 * nsm * 1.965e9 * ms * 1e-3;  // 64 DFMA lanes/clk/SM nominal
    printf("pair       warps/SM=%2d: %.3f ms, FP64 lane-ops/s %.2f T (%.0f%% of 64/clk/SM at 1965 MHz)\n",
           warps, ms, inst / ms / 1e9, 100.0 * inst / peak_inst);
  }
  return 0;
}
